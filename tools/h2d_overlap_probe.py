"""Does a concurrent pinned H2D upload (the e2e leg's double-buffered H copy) slow K1? Times a c2
full-width filter call (n = 13000, k = 624, 8 steps) alone and with a 2.7 GB host->device copy running on
another stream. usage: python tools/h2d_overlap_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4161_b200 as chfsi  # noqa: E402


def main():
    n, k, m = 13000, 624, 8
    torch.manual_seed(0)
    H = chfsi.colmajor(n, n)
    H.copy_(torch.randn(n, n, dtype=torch.complex128, device="cuda") / (2 * n) ** 0.5)
    Y0 = chfsi.colmajor(n, k)
    Y0.copy_(torch.randn(n, k, dtype=torch.complex128, device="cuda"))
    Y = chfsi.colmajor(n, k)
    host = torch.empty(n * n * 2, dtype=torch.float64, pin_memory=True)
    host.fill_(1.0)
    dev = torch.empty_like(host, device="cuda")
    ctx = chfsi.Context(0)
    side = torch.cuda.Stream()
    deg = [m] * k

    def run(with_copy):
        Y.copy_(Y0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        c0, c1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        if with_copy:
            with torch.cuda.stream(side):
                c0.record(side)
                dev.copy_(host, non_blocking=True)
                c1.record(side)
        ctx.filter(H, Y, deg, -2.2, 0.6, 1.6)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), (c0.elapsed_time(c1) if with_copy else None)

    run(False)
    res = {"alone": [], "with_copy": [], "copy_ms": []}
    for _ in range(4):
        res["alone"].append(run(False)[0])
        t, c = run(True)
        res["with_copy"].append(t)
        res["copy_ms"].append(c)
    print(json.dumps(res))
    print(json.dumps({"alone_min": min(res["alone"]), "with_copy_min": min(res["with_copy"]),
                      "delta_ms": min(res["with_copy"]) - min(res["alone"]), "copy_ms_min": min(res["copy_ms"])}))
    ctx.close()


main()
