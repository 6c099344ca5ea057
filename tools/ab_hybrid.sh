# A/B of the DP + stream-K hybrid fold (CHFSI_SK_HYBRID=1, default) vs the plain DP + stream-K tail
# (CHFSI_SK_HYBRID=0) at shapes where the fold applies, spanning the plain split's tail iterations per CTA
set -u
mkdir -p gpurun_out
rm -f gpurun_out/ab_hy.jsonl
for r in 1 2; do
for h in 1 0; do
  CHFSI_SK_HYBRID=$h timeout 300 python tools/filter_perf.py 4096 208,240,456 16 200 | sed "s/^{/{\"hy\": $h, /" >> gpurun_out/ab_hy.jsonl
  CHFSI_SK_HYBRID=$h timeout 300 python tools/filter_perf.py 8192 312,552,112,144,440 8 200 | sed "s/^{/{\"hy\": $h, /" >> gpurun_out/ab_hy.jsonl
  CHFSI_SK_HYBRID=$h timeout 300 python tools/filter_perf.py 13000 120,400,200,96 4 200 | sed "s/^{/{\"hy\": $h, /" >> gpurun_out/ab_hy.jsonl
  CHFSI_SK_HYBRID=$h timeout 300 python tools/filter_perf.py 16384 632,592,544,152 4 200 | sed "s/^{/{\"hy\": $h, /" >> gpurun_out/ab_hy.jsonl
done
done
