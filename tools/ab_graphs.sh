set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_steps.py tests/test_gpu_real.py tests/test_gpu_multirank.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/gr_tests.log 2>&1; echo rc=$? >> gpurun_out/gr_tests.log
for r in 1 2; do
  for g in 1 0; do
    CHFSI_GRAPHS=$g timeout 300 python bench.py --config c1 --no-cpu-baseline --no-e2e --no-sequence > gpurun_out/gr_c1_${g}_$r.json 2>/dev/null
  done
done
for g in 1 0; do CHFSI_GRAPHS=$g timeout 500 python bench.py --no-cpu-baseline --no-e2e --no-sequence > gpurun_out/gr_c2_$g.json 2>/dev/null; done
