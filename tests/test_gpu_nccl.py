"""The NCCL path with real ranks on separate GPUs (tools/nccl_check.py under torchrun): runs only on a box
with at least two GPUs (every box of round 1 has one; the same path is covered on one GPU by the
emulated ranks of test_gpu_multirank.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_gpus() < 2, reason="needs two or more GPUs (one rank per GPU; NCCL refuses two ranks per GPU)")
def test_nccl_filter_and_solve_two_gpus():
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tools", "nccl_check.py")],
                       capture_output=True, text=True, timeout=900, env=dict(os.environ, PYTHONPATH=ROOT))
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
