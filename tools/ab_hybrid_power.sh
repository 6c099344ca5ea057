# Sustained (power-capped) A/B of the stream-K hybrid fold: tools/power_probe.py at mid widths with
# CHFSI_SK_HYBRID=1 (default) and 0, 8 s each
set -u
mkdir -p gpurun_out
rm -f gpurun_out/hyp.log
for k in 110 150 200 300; do
  for h in 1 0; do
    CHFSI_SK_HYBRID=$h timeout 60 python tools/power_probe.py $k 8 | sed "s/^{/{\"hy\": $h, /" >> gpurun_out/hyp.log
  done
done
