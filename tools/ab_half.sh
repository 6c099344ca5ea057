set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_filter.py tests/test_gpu_real.py tests/test_gpu_multirank.py -m gpu -q -x > gpurun_out/half_tests.log 2>&1; echo "rc=$?" >> gpurun_out/half_tests.log
timeout 300 python tools/width_table.py 13000 4 200,207,208 > gpurun_out/half_wt_c2.jsonl 2>&1
timeout 300 python tools/width_table.py 4096 4 200,207,208 > gpurun_out/half_wt_c1.jsonl 2>&1
CHFSI_K1_LOG=1 timeout 500 python bench.py --no-cpu-baseline --no-e2e --no-sequence > gpurun_out/half_c2.json 2> gpurun_out/half_c2.err; python tools/k1_log_summary.py gpurun_out/half_c2.err 13000 > gpurun_out/half_k1w_c2.txt
CHFSI_K1_LOG=1 timeout 300 python bench.py --config c1 --no-cpu-baseline --no-e2e --no-sequence > gpurun_out/half_c1.json 2> gpurun_out/half_c1.err; python tools/k1_log_summary.py gpurun_out/half_c1.err 4096 > gpurun_out/half_k1w_c1.txt
