#!/bin/bash
# GPU tests + one bench line (no profilers). Usage: tools/quick_round.sh TAG [pytest-args]
TAG=${1:-q}; shift
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x "$@" > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json
