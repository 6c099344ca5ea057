"""Quick K1 throughput probe: chfsi_filter at a fixed shape for each tile variant (CUDA events).
usage: filter_perf.py n k1,k2 m variants [real]
variants: comma list of 4M ids (0..9), 3M ids (200..204), 'auto3' / 'auto4' (the chooser under 3M / 4M),
'auto' (= auto3); real: the real-symmetric ids (104, 132, 133, 135; 100-105 with -DCHFSI_K1_AB) / 'auto'. Flops are 8 n^2 k m (complex,
the 4M convention of SURVEY 8(d)) or 2 n^2 k m (real)."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4161_b200 as chfsi

ENVS = ("CHFSI_FILTER_VARIANT", "CHFSI_FILTER_VARIANT_Z3", "CHFSI_FILTER_VARIANT_REAL")


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 13000
    ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "624").split(",")]
    m = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    variants = (sys.argv[4] if len(sys.argv) > 4 else "auto3,auto4").split(",")
    real = len(sys.argv) > 5 and sys.argv[5] == "real"
    dt = torch.float64 if real else torch.complex128
    torch.manual_seed(0)
    H = chfsi.colmajor(n, n, dtype=dt)
    H.copy_(torch.randn(n, n, dtype=dt, device="cuda") / (2 * n) ** 0.5)
    ctx = chfsi.Context(0)
    filt = ctx.filter_real if real else ctx.filter
    for k in ks:
        Y0 = chfsi.colmajor(n, k, dtype=dt); Y0.copy_(torch.randn(n, k, dtype=dt, device="cuda"))
        Y = chfsi.colmajor(n, k, dtype=dt)
        deg = [m] * k
        Yref = None
        for v in variants:
            for e in ENVS:
                os.environ.pop(e, None)
            mults = 3
            if real:
                if v != "auto":
                    os.environ["CHFSI_FILTER_VARIANT_REAL"] = v
            elif v in ("auto", "auto3"):
                mults = 3
            elif v == "auto4":
                mults = 4
            elif int(v) >= 200:
                os.environ["CHFSI_FILTER_VARIANT_Z3"] = v
            else:
                mults = 4
                os.environ["CHFSI_FILTER_VARIANT"] = v
            ctx.set_complex_mult(mults)
            Y.copy_(Y0); filt(H, Y, deg, -2.2, 0.6, 1.6)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            best = 1e30
            for _ in range(3):
                Y.copy_(Y0)
                e0.record(); filt(H, Y, deg, -2.2, 0.6, 1.6); e1.record(); torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            fl = (2.0 if real else 8.0) * n * n * k * m
            if Yref is None:
                Yref = Y.clone()
            diff = float((Y - Yref).abs().max() / Yref.abs().max())
            print(json.dumps({"rel_diff_vs_first": diff, "n": n, "k": k, "m": m, "variant": v, "real": real,
                              "mults": None if real else mults, "ms": best, "tflops": fl / best / 1e9,
                              "tensor_tflops": (fl if real or mults == 4 else 0.75 * fl) / best / 1e9}), flush=True)

main()
