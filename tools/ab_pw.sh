# A/B of the real-symmetric K1 tiles with and without a producer warpgroup (r02): full-width perf and
# the width table at n = 13000
set -u
mkdir -p gpurun_out
timeout 300 python tools/filter_perf.py 13000 624,208,96,40 4 102,132,103,133,105,135 real > gpurun_out/ab_pw_real.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pw_real.log
timeout 600 python tools/width_table.py 13000 8 102,132,103,133,104,105,135 real > gpurun_out/width_table_real.jsonl 2>&1; echo "rc=$?" >> gpurun_out/width_table_real.jsonl
