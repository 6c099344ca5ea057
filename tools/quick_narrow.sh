#!/bin/bash
TAG=${1:-nw}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python tools/filter_perf.py 16384 4,8,12,16,20,24,32 10 auto3,5,6,10,11,12 > gpurun_out/${TAG}_narrow.log 2>&1
cat gpurun_out/${TAG}_narrow.log
timeout 900 python tools/c4_sweep.py 16384 64,256 > gpurun_out/${TAG}_c4.jsonl 2>&1
cat gpurun_out/${TAG}_c4.jsonl
