"""Where the QR step's time goes at the c2 shape: chfsi_qr on n = 13000 blocks of k = 624 columns with
nlocked = 0 / 100 / 250 / 400 / 520 (X_L orthonormal, the active block a perturbation of random data),
CUDA-event time per call and the CUPTI kernel breakdown. usage: python tools/qr_probe.py"""
import collections
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4161_b200 as chfsi  # noqa: E402


def main():
    n, k = 13000, 624
    torch.manual_seed(0)
    ctx = chfsi.Context(0)
    base = chfsi.colmajor(n, k)
    base.copy_(torch.randn(n, k, dtype=torch.complex128, device="cuda"))
    ctx.qr(base)  # an orthonormal block: its first nl columns serve as X_L
    for nl in (0, 100, 250, 400, 520):
        Y = chfsi.colmajor(n, k)
        Y.copy_(base)
        Y[:, nl:].copy_(torch.randn(n, k - nl, dtype=torch.complex128, device="cuda"))
        Y0 = Y.clone()
        ctx.qr(Y, nlocked=nl)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            Y.copy_(Y0)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            ctx.qr(Y, nlocked=nl)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        Y.copy_(Y0)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            ctx.qr(Y, nlocked=nl)
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
        by = collections.Counter()
        for e in ev:
            by[e.name[:50]] += e.time_range.elapsed_us()
        ka = k - nl
        flops = 32.0 * n * nl * ka + 16.0 * n * ka * ka
        print(json.dumps({"nlocked": nl, "ka": ka, "ms": best, "model_gflop": flops / 1e9,
                          "tflops": flops / best / 1e9, "kernels_ms": {kname: round(t / 1e3, 3) for kname, t in by.most_common(8)},
                          "kernel_sum_ms": round(sum(by.values()) / 1e3, 3)}), flush=True)
    ctx.close()


main()
