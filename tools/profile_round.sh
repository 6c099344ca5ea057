#!/bin/bash
# One gpurun call: GPU tests, smoke, the bench line, the ncu launch list of a short bench, one full ncu
# capture of K1 (c2 full-width step), the c1 / c3 bench lines, the 8-emulated-rank bench and the c1
# ablations. Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/ by hand.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
SHORT="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sequence"
$SHORT > gpurun_out/${TAG}_short_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $SHORT > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/${TAG}_ncu_launches.log
PERF="python tools/filter_perf.py 13000 624 4 auto3"
$PERF > gpurun_out/${TAG}_perf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:filter_step -s 4 -c 1 -o gpurun_out/${TAG}_k1 -f $PERF > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${TAG}_ncu_full.log
python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-sequence > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err; echo "c3 rc=$?" >> gpurun_out/${TAG}_bench_c3.err
python bench.py --config c1 --no-cpu-baseline > gpurun_out/${TAG}_bench_c1.json 2> gpurun_out/${TAG}_bench_c1.err; echo "c1 rc=$?" >> gpurun_out/${TAG}_bench_c1.err
python bench.py --emulate-ranks 8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sequence > gpurun_out/${TAG}_bench_emu8.json 2> gpurun_out/${TAG}_bench_emu8.err; echo "emu8 rc=$?" >> gpurun_out/${TAG}_bench_emu8.err
python tools/ablation.py c1 5 16 > gpurun_out/${TAG}_ablation_c1.jsonl 2>&1; echo "ablation rc=$?" >> gpurun_out/${TAG}_ablation_c1.jsonl
