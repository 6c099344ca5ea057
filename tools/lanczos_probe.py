"""Lanczos bounds timing (CUDA events) at a few sizes, for the CUDA-graph A/B (CHFSI_GRAPHS=0/1).
usage: python tools/lanczos_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4161_b200 as chfsi  # noqa: E402


def main():
    ctx = chfsi.Context(0)
    for n in (512, 1024, 4096, 13000):
        H = chfsi.colmajor(n, n)
        A = torch.randn(n, n, dtype=torch.complex128, device="cuda")
        H.copy_((A + A.conj().t()) / 2)
        del A
        ctx.lanczos_bounds(H, 25, 7)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            ctx.lanczos_bounds(H, 25, 7)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(json.dumps({"n": n, "graphs": os.environ.get("CHFSI_GRAPHS", "1"), "ms": best}), flush=True)
    ctx.close()


main()
