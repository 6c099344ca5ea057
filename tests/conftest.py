import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # build the native pieces (no-op when up to date); the CUDA library cross-compiles without a GPU
    subprocess.run(["make", "-s", "-C", ROOT, "gen/libgen.so", "oracle/liboracle.so"], check=True)


@pytest.fixture(scope="session")
def gpu_lib():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_4161_b200 as chfsi

    return chfsi
