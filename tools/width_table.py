"""Measure every 3M tile variant of K1 over the active widths a ChFSI solve visits (n = 13000, widths
28..640, step 4 or argv[2], 2 filter steps each) and print, per width, the time of every built variant
and of the step model's own choice ("auto"). The result calibrates pick_tile for large panels
(profiles/r01_width_table.jsonl, r02_width_table.jsonl). argv[4] = "real": the real-symmetric variants
(profiles/r02_width_table_real.jsonl).
usage: width_table.py [n] [step] [variants] [real]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4161_b200 as chfsi  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 13000
    variants = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "200,207,208").split(",")]
    step = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    real = len(sys.argv) > 4 and sys.argv[4] == "real"
    dt = torch.float64 if real else torch.complex128
    env = "CHFSI_FILTER_VARIANT_REAL" if real else "CHFSI_FILTER_VARIANT_Z3"
    torch.manual_seed(0)
    H = chfsi.colmajor(n, n, dtype=dt)
    H.copy_(torch.randn(n, n, dtype=dt, device="cuda") / (2 * n) ** 0.5)
    ctx = chfsi.Context(0)
    filt = ctx.filter_real if real else ctx.filter
    Y0 = torch.randn(n, 640, dtype=dt, device="cuda")
    for k in range(28, 641, step):
        Yk = chfsi.colmajor(n, k, dtype=dt)
        row = {"n": n, "k": k}
        for v in variants:
            os.environ[env] = str(v)
            best = 1e30
            for _ in range(3):
                Yk.copy_(Y0[:, :k])
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                filt(H, Yk, [2] * k, -2.2, 0.6, 1.6)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            row[str(v)] = best
        os.environ.pop(env, None)
        best = 1e30  # the step model's own choice
        for _ in range(3):
            Yk.copy_(Y0[:, :k])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            filt(H, Yk, [2] * k, -2.2, 0.6, 1.6)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        row["auto"] = best
        print(json.dumps(row), flush=True)
    ctx.close()


main()
