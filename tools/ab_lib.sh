# A/B of two builds of libchfsi.so (ab/libchfsi_base.so vs the in-tree one, or $NEW_LIB), interleaved runs of
# tools/filter_perf.py at the given widths: bash tools/ab_lib.sh <n> <k list> <m> <variant> <tag> [reps]
set -u
n=$1; ks=$2; m=$3; v=$4; tag=$5; reps=${6:-3}
mkdir -p gpurun_out
for r in $(seq $reps); do
  CHFSI_LIB=$PWD/ab/libchfsi_base.so timeout 300 python tools/filter_perf.py $n $ks $m $v | sed 's/^{/{"lib": "base", /' >> gpurun_out/${tag}.jsonl
  CHFSI_LIB=${NEW_LIB:-} timeout 300 python tools/filter_perf.py $n $ks $m $v | sed 's/^{/{"lib": "new", /' >> gpurun_out/${tag}.jsonl
done
