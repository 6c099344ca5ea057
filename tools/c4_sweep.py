"""BASELINE.json configs[4]: filter-only throughput sweep. H = GUE (stream (5, n)), fixed interval
lambda1 = -2.2, [alpha, beta] = [-1, 2.2]; n in {8192, 16384, 32768}, block width k in {64, 256, 1024, 2048};
degrees uniform 20 or the sorted ramp 8..40. Reports TFLOP/s (ZGEMM convention 8 n^2 sum(deg)) and the
fraction of the FP64 DMMA roofline (37.07 TF/s) in executed tensor flops (3M: 6 n^2 sum(deg)) and,
for narrow blocks (k <= 12, HBM-bound), the H-stream bandwidth vs the measured HBM peak. Parity: the
oracle (Alg 2, naive C) on sampled columns for n <= 16384. JSON lines. The GUE matrix is built on the GPU
with torch for n > 8192 (input construction only; parity runs use the host generator)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen as G  # noqa: E402
import paper_1404_4161_b200 as chfsi  # noqa: E402
from gen.configs import C4_INTERVAL, C4_KS, C4_NS, c4_ramp  # noqa: E402

PEAK = 37.07
HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def roofline_time_ms(n, deg):
    """T* = sum over steps of max(tensor time, H-stream time) for the arithmetic the
    library picks per step: 3M (6 n^2 k_a tensor flops, 24 B of H per entry) at >= 28 active columns,
    4M (8 n^2 k_a, 16 B) below; peaks: the measured FP64 DMMA rate and HBM copy bandwidth."""
    deg = sorted(deg)
    t = 0.0
    for i in range(max(deg)):
        ka = sum(1 for m in deg if m > i)
        fl, by = (6.0 * n * n * ka, 24.0 * n * n) if ka >= 28 else (8.0 * n * n * ka, 16.0 * n * n)
        t += max(fl / (PEAK * 1e12), by / (HBM * 1e9))
    return 1e3 * t


def timed(ctx, H, Y0, deg, l1, c, e, reps=2):
    Y = chfsi.colmajor(*Y0.shape)
    best = 1e30
    for _ in range(reps + 1):
        Y.copy_(Y0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        ctx.filter(H, Y, deg, l1, c, e)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, Y


def main():
    ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(C4_NS)
    ks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(C4_KS)
    parity = "--parity" in sys.argv
    iv = C4_INTERVAL
    c, e = (iv["alpha"] + iv["beta"]) / 2, (iv["beta"] - iv["alpha"]) / 2
    ctx = chfsi.Context(0)
    for n in ns:
        t0 = time.time()
        Hh = None
        if parity and n <= 16384:
            Hh = G.gue(n, 5, G.stream(5, n))
            H = chfsi.to_colmajor(Hh)
        else:
            g = torch.Generator(device="cuda").manual_seed(n)
            A = torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g) / (2 * n) ** 0.5
            H = chfsi.colmajor(n, n)
            H.copy_((A + A.conj().t()) / 2 ** 0.5)
            del A
        gen_s = time.time() - t0
        for k in ks + [4, 8, 12]:
            if k > 12 and "--no-zgemm" not in sys.argv:  # same-box yardstick: cuBLAS ZGEMM H Y
                Yz = torch.randn(n, k, dtype=torch.complex128, device="cuda")
                Hz = H if H.is_contiguous() else None
                A = H.t() if Hz is None else H  # a plain n x n operand (H is Hermitian; layout only)
                torch.matmul(A, Yz)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for _ in range(3):
                    torch.matmul(A, Yz)
                e1.record()
                torch.cuda.synchronize()
                zms = e0.elapsed_time(e1) / 3
                print(json.dumps({"n": n, "k": k, "yardstick": "cuBLAS ZGEMM (torch.matmul complex128)",
                                  "ms": zms, "tflops": 8.0 * n * n * k / zms / 1e9}), flush=True)
                del Yz
            Y0h = G.start_basis(n, k, 5)
            Y0 = chfsi.to_colmajor(Y0h)
            modes = [("uniform20", [20] * k), ("ramp8-40", c4_ramp(k))] if k > 12 else [("narrow10", [10] * k)]
            for label, deg in modes:
                ms, Y = timed(ctx, H, Y0, deg, iv["lambda1"], c, e)
                flops = 8.0 * n * n * sum(deg)
                # tflops: 8 n^2 sum(deg) (ZGEMM convention); the 3M kernel executes 6 n^2 sum(deg) tensor flops
                # (narrow steps, k < 28, run the 4M kernel: 8 n^2 tensor flops per column-step)
                tfac = 1.0 if k < 28 else 0.75
                row = {"n": n, "k": k, "degrees": label, "ms": ms, "tflops": flops / ms / 1e9,
                       "tensor_tflops": tfac * flops / ms / 1e9,
                       "frac_of_fp64_peak": tfac * flops / ms / 1e9 / PEAK,
                       "roofline_ms": roofline_time_ms(n, deg), "frac_of_roofline": roofline_time_ms(n, deg) / ms,
                       "gen_s": gen_s}
                if k <= 12:  # HBM-bound: H streamed once per step
                    steps = max(deg)
                    row["hbm_gbs_H_stream"] = 16.0 * n * n * steps / ms / 1e6
                    row["frac_of_hbm_peak"] = row["hbm_gbs_H_stream"] / HBM
                if Hh is not None and label != "narrow10":
                    cols = [0, k - 1]
                    Yo, _ = __import__("oracle").chebyshev_filter(Hh, Y0h[:, cols], [deg[j] for j in cols],
                                                                  iv["lambda1"], c, e)
                    Yg = Y.cpu().numpy()[:, cols]
                    row["max_rel_err_vs_oracle"] = float(np.max(np.linalg.norm(Yg - Yo, axis=0) /
                                                                np.linalg.norm(Yo, axis=0)))
                print(json.dumps(row), flush=True)
        del H
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
