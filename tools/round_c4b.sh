#!/bin/bash
# c4 sweep with the final chooser (+ cuBLAS ZGEMM yardstick), and ncu --set full captures of narrow steps.
TAG=${1:-c4b}
mkdir -p gpurun_out
timeout 1500 python tools/c4_sweep.py 8192,16384,32768 64,256,1024,2048 --parity > gpurun_out/${TAG}_sweep.jsonl 2> gpurun_out/${TAG}_sweep.err; echo "sweep rc=$?"
for K in 4 8; do
  PERF="python tools/filter_perf.py 16384 $K 10 auto3"
  $PERF > gpurun_out/${TAG}_perf_k$K.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:filter_step -s 10 -c 1 -o gpurun_out/${TAG}_k1_n16384_k$K -f $PERF > gpurun_out/${TAG}_ncu_k$K.log 2>&1
  echo "ncu k=$K rc=$?"
done
