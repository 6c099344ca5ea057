# Re-measure the FP64 roofline denominator (register-only DMMA / DFMA loops) and the same-box library
# yardsticks (cuBLAS ZGEMM / DGEMM, HBM copy), sampling SM clocks during the DMMA probe
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_probe tools/fp64_probe.cu
( for i in $(seq 1 40); do nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw --format=csv,noheader; sleep 0.25; done ) > gpurun_out/peaks_clocks.txt &
timeout 300 /tmp/fp64_probe > gpurun_out/peaks_fp64.jsonl 2>&1
wait
timeout 300 python tools/probe_libs.py > gpurun_out/peaks_libs.jsonl 2>&1
