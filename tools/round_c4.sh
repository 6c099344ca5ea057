#!/bin/bash
# One gpurun call: the BASELINE configs[4] filter-only sweep (oracle parity on sampled columns, cuBLAS ZGEMM
# yardstick, per-step roofline fraction) and ncu --set full captures of a narrow HBM-bound step (k_a = 8)
# and a compute-bound c4 step (n = 16384, k = 1024). Outputs in gpurun_out/ (scratch).
set -u
TAG=${1:-c4}
mkdir -p gpurun_out
timeout 1500 python tools/c4_sweep.py 8192,16384,32768 64,256,1024,2048 --parity > gpurun_out/${TAG}_sweep.jsonl 2> gpurun_out/${TAG}_sweep.err; echo "sweep rc=$?"
for NK in "16384 8 10" "16384 4 10" "16384 1024 4"; do
  set -- $NK
  PERF="python tools/filter_perf.py $1 $2 $3 auto3"
  $PERF > gpurun_out/${TAG}_perf_n$1_k$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:filter_step -s $3 -c 1 -o gpurun_out/${TAG}_k1_n$1_k$2 -f $PERF > gpurun_out/${TAG}_ncu_n$1_k$2.log 2>&1
  echo "ncu n=$1 k=$2 rc=$?"
done
