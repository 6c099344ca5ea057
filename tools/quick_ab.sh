#!/bin/bash
# A/B of K1 options: stage-refill protocol (CHFSI_K1_REFILL 0/1) on the 3M and 4M paths, the 3M/4M
# switch in the narrow regime, then the GPU tests and the bench line under the chosen defaults.
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for R in 0 1; do
  CHFSI_K1_REFILL=$R timeout 600 python tools/filter_perf.py 13000 624,256,104 4 200,201,auto4 > gpurun_out/${TAG}_refill$R.log 2>&1
  echo "refill=$R"; cat gpurun_out/${TAG}_refill$R.log
done
timeout 600 python tools/filter_perf.py 16384 4,8,12,16,20,24,32 10 auto3,auto4 > gpurun_out/${TAG}_narrow.log 2>&1
echo narrow; cat gpurun_out/${TAG}_narrow.log
