#!/bin/bash
# 3M bring-up: GPU tests, then 3M vs 4M throughput of K1 at the c2 full-width / narrow shapes, then bench.
TAG=${1:-z3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -15 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python tools/filter_perf.py 13000 624,256,104,48 4 auto3,200,201,202,203,204,auto4 > gpurun_out/${TAG}_perf.log 2>&1; echo "perf rc=$?"
cat gpurun_out/${TAG}_perf.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
