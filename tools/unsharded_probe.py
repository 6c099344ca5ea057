"""Device times of the k x k pieces of one ChFSI loop that do not shard over row panels (DESIGN.md 9 eta
model): the Cholesky factorisation of CholeskyQR2 (cuSOLVER ZPOTRF, twice per loop, every rank), the dense
Rayleigh-Ritz eigensolve (ZHEEVD via torch.linalg.eigh, the refinement's fallback) and a k x k ZGEMM, at
the active widths a c2 / c3 problem visits. CUDA events, median of 5 after 2 warm-ups."""
import json
import statistics

import torch


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    torch.manual_seed(0)
    for k in (109, 151, 230, 394, 624, 960, 1440):
        A = torch.randn(k, k, dtype=torch.complex128, device="cuda")
        S = A.mH @ A + k * torch.eye(k, dtype=torch.complex128, device="cuda")
        Hm = (A + A.mH) / 2
        rec = {"k": k, "zpotrf_ms": timed(lambda: torch.linalg.cholesky(S)),
               "zheevd_ms": timed(lambda: torch.linalg.eigh(Hm)),
               "zgemm_kkk_ms": timed(lambda: A @ A)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
