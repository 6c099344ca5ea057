#!/bin/bash
# c4 (BASELINE.json configs[4]) filter-only sweep with oracle parity on sampled columns, the emulated-
# rank pipeline tests, and ncu --set full captures of one compute-bound c4 step (n=16384, k=1024) and
# one narrow HBM-bound step (n=16384, k=8). Outputs in gpurun_out/ (scratch).
set -u
TAG=${1:-c4}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/${TAG}_pytest_multirank.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_multirank.log
tail -2 gpurun_out/${TAG}_pytest_multirank.log
timeout 1500 python tools/c4_sweep.py 8192,16384,32768 64,256,1024,2048 --parity > gpurun_out/${TAG}_sweep.jsonl 2> gpurun_out/${TAG}_sweep.err; echo "sweep rc=$?"
cat gpurun_out/${TAG}_sweep.jsonl
for NK in "16384 1024" "16384 8" "13000 624"; do
  set -- $NK
  PERF="python tools/filter_perf.py $1 $2 4 auto3"
  $PERF > gpurun_out/${TAG}_perf_n$1_k$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:filter_step -s 4 -c 1 -o gpurun_out/${TAG}_k1_n$1_k$2 -f $PERF > gpurun_out/${TAG}_ncu_n$1_k$2.log 2>&1
  echo "ncu n=$1 k=$2 rc=$?"
done
