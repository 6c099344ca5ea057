# The stream-K hybrid fold on whole benches (sustained, power-capped at mid widths): c2 and c1 bench lines
# with CHFSI_SK_HYBRID=1 (default) and 0, interleaved
set -u
mkdir -p gpurun_out
rm -f gpurun_out/hyb_*.json
for r in 1 2; do
  for h in 1 0; do
    CHFSI_SK_HYBRID=$h timeout 500 python bench.py --no-cpu-baseline --no-e2e --no-sequence > gpurun_out/hyb_c2_${h}_$r.json 2>/dev/null
    CHFSI_SK_HYBRID=$h timeout 300 python bench.py --config c1 --no-cpu-baseline --no-e2e --no-sequence > gpurun_out/hyb_c1_${h}_$r.json 2>/dev/null
  done
done
