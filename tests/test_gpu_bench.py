"""bench.py end to end on the GPU: the single-GPU line on the small c0 workload, and the N > 1 path of
the script (row panels, packed operands, collectives, max-over-ranks reductions) run as emulated ranks
on one GPU (--emulate-ranks), which is what a torchrun launch on 2/4 GPUs executes apart from NCCL."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(*args):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c0", "--steps", "1", "--warmup", "3",
                        "--no-cpu-baseline", *args], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    d = bench()
    assert d["converged"] and d["max_resid_over_tol"] <= 1.0
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["bound"] == "tensor" and 0 < d["roofline"]["frac"] < 1.2
    assert "sm_mhz" in d["clocks"]
    assert d["sequence"]["problems"] == 1 and d["sequence"]["converged"]


@pytest.mark.parametrize("P", [2, 4])
def test_bench_emulated_ranks(P):
    d = bench("--emulate-ranks", str(P), "--no-e2e")
    assert d["emulated_ranks"] == P
    assert d["converged"] and d["max_resid_over_tol"] <= 1.0


def test_bench_emulated_ranks_allgather():
    d = bench("--emulate-ranks", "2", "--no-e2e", "--exchange", "allgather")
    assert d["config"]["exchange"] == "allgather"
    assert d["converged"] and d["max_resid_over_tol"] <= 1.0
