# A/B of the stream-K cost model for tiles one warp column short of full: CHFSI_SK_C2 (their per-unit
# speed relative to a full tile) x CHFSI_SK_WOFF, interleaved, forced z200 at n = 13000 (m = 8 steps)
# usage: [K=widths] [CFGS="woff_c2 ..."] bash tools/ab_cover.sh
set -u
mkdir -p gpurun_out
K=${K:-623,578,536,504,466,435,405,374,351,327,304,285,264,246,229,215,201,186,173,159,145,132,118,105}
for r in 1 2; do
  for cfg in ${CFGS:-0.75_1.0 0.75_1.05 0.75_1.1 0.75_1.15 0.6_1.1}; do
    w=${cfg%_*}; c=${cfg#*_}
    CHFSI_SK_WOFF=$w CHFSI_SK_C2=$c timeout 300 python tools/filter_perf.py 13000 $K 8 200 | sed "s/^{/{\"woff\": $w, \"c2\": $c, /" >> gpurun_out/ab_cover.jsonl
  done
done
