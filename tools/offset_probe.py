"""Does the active block's column offset change K1's speed? Filter a k-column block whose first k - ka
columns finish after 2 steps (so ka columns stay active from column k - ka on) against a ka-column block
(active from column 0), same degree for the active columns; per-launch K1 times from CHFSI_K1_LOG.
usage: CHFSI_K1_LOG=1 python tools/offset_probe.py 2> log"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4161_b200 as chfsi  # noqa: E402


def main():
    n, k, ka, m = 13000, 624, 110, 12
    torch.manual_seed(0)
    H = chfsi.colmajor(n, n)
    H.copy_(torch.randn(n, n, dtype=torch.complex128, device="cuda") / (2 * n) ** 0.5)
    ctx = chfsi.Context(0)
    for label, kk, deg in (("offset", k, [2] * (k - ka) + [m] * ka), ("plain", ka, [m] * ka)):
        Y0 = chfsi.colmajor(n, kk)
        Y0.copy_(torch.randn(n, kk, dtype=torch.complex128, device="cuda"))
        Y = chfsi.colmajor(n, kk)
        for rep in range(3):
            Y.copy_(Y0)
            torch.cuda.synchronize()
            print(f"# {label} rep {rep}", file=sys.stderr, flush=True)
            ctx.filter(H, Y, deg, -2.2, 0.6, 1.6)
            torch.cuda.synchronize()
    ctx.close()


main()
