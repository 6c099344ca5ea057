#!/bin/bash
# New-feature GPU tests, the NEXT-2 ablation on c1, the real-symmetric filter throughput, and the c3
# (n = 30000) bench line on one GPU.
TAG=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_generalized.py tests/test_gpu_real.py tests/test_gpu_steps.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
python tools/filter_perf.py 13000 624,256,104 4 100,101,102,auto real > gpurun_out/${TAG}_real_perf.log 2>&1
cat gpurun_out/${TAG}_real_perf.log
python tools/ablation.py c1 5 16 > gpurun_out/${TAG}_ablation_c1.jsonl 2>&1
cat gpurun_out/${TAG}_ablation_c1.jsonl
python bench.py --config c3 --steps 1 --warmup 3 > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err; echo "c3 rc=$?"
cat gpurun_out/${TAG}_bench_c3.json; tail -3 gpurun_out/${TAG}_bench_c3.err
