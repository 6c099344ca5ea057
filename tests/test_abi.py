"""CPU checks of the boundary: libchfsi.so loads, exports every entry point include/chfsi.h declares,
and fails loudly (no CPU fallback) without a CUDA device. The product package never touches oracle/."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "chfsi.h")
PKG = os.path.join(ROOT, "paper_1404_4161_b200")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:chfsi_status|void|const char\s*\*|int64_t)\s*(chfsi_[a-z_]+)\s*\(", src,
                                 flags=re.M)))


@pytest.fixture(scope="module")
def libpath():
    subprocess.run(["make", "-s", "-C", ROOT, "paper_1404_4161_b200/libchfsi.so"], check=True)
    return os.path.join(PKG, "libchfsi.so")


def test_exports_every_declared_symbol(libpath):
    names = declared()
    assert "chfsi_filter" in names and "chfsi_solve_sequence" in names and len(names) >= 10
    L = ctypes.CDLL(libpath)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    dyn = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", dyn), n


def test_binding_names_match_header():
    import paper_1404_4161_b200 as chfsi

    assert sorted(chfsi.EXPORTS) == declared()


def test_built_for_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass and "UTMALDG" in sass  # FP64 tensor-core MMA fed by TMA


def test_no_cpu_fallback_without_gpu(libpath):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = ctypes.CDLL(libpath)
    h = ctypes.c_void_p()
    st = L.chfsi_ctx_create(ctypes.byref(h), 0, None, None, 0, 1)
    assert st == 5  # CHFSI_ERR_CUDA
    import paper_1404_4161_b200 as chfsi

    with pytest.raises(Exception):
        chfsi.Context(0)


def test_product_path_does_not_use_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f
