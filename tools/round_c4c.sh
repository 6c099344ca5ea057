#!/bin/bash
TAG=${1:-c4c}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 1500 python tools/c4_sweep.py 8192,16384,32768 64,256,1024,2048 --parity > gpurun_out/${TAG}_sweep.jsonl 2> gpurun_out/${TAG}_sweep.err; echo "sweep rc=$?"
PERF="python tools/filter_perf.py 16384 8 10 auto3"
$PERF > gpurun_out/${TAG}_perf_k8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:filter_step -s 10 -c 1 -o gpurun_out/${TAG}_k1_n16384_k8 -f $PERF > gpurun_out/${TAG}_ncu_k8.log 2>&1
echo "ncu k=8 rc=$?"
