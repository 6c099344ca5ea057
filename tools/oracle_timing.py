"""the CPU oracle (oracle/, plain C + OpenMP, as it stands) timed on the host cores of the
GPU box -- the full ChFSI solve of c0 (n = 512) on 1 thread and on all threads, and the filter sample of
c2 the bench uses -- next to the GPU time of the same c0 solve through the C-ABI. Each size runs in a
fresh process because OMP_NUM_THREADS is read when the OpenMP runtime starts. JSON lines.
Usage: python tools/oracle_timing.py"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(mode):
    sys.path.insert(0, ROOT)
    import numpy as np

    import gen as G
    import oracle as O
    from gen.configs import CONFIGS

    cf = CONFIGS["c0"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    X0 = G.start_basis(n, nev + nex, cf["seed"])
    if mode == "gpu":
        import torch

        import paper_1404_4161_b200 as chfsi

        ctx = chfsi.Context(0)
        Hd = chfsi.to_colmajor(H)
        ctx.solve_sequence(lambda ell: Hd, 1, chfsi.to_colmajor(X0), nev, nex, cf["tol"], deg_cap=cf["cap"],
                           seed=cf["seed"])  # warm-up
        Xd = chfsi.to_colmajor(X0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], seed=cf["seed"])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        lam = out["lam"][0]
        print(json.dumps({"what": "c0 full ChFSI solve, GPU (C-ABI)", "s": dt, "loops": out["reports"][0]["loops"],
                          "max_rel_eig_err_vs_exact": float(np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev])))}))
        return
    t0 = time.perf_counter()
    r = O.chfsi_solve(H, X0, nev, nex, cf["tol"], cf["cap"], seed=cf["seed"])
    dt = time.perf_counter() - t0
    lam = r["lam"]
    print(json.dumps({"what": "c0 full ChFSI solve, CPU oracle", "threads": int(os.environ["OMP_NUM_THREADS"]), "s": dt,
                      "max_rel_eig_err_vs_exact": float(np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev])))}))


def main():
    if len(sys.argv) > 1:
        child(sys.argv[1])
        return
    ncores = len(os.sched_getaffinity(0))
    for thr in sorted({1, ncores}):
        env = dict(os.environ, OMP_NUM_THREADS=str(thr), OMP_PROC_BIND="close", OMP_PLACES="cores")
        subprocess.run([sys.executable, __file__, "cpu"], env=env, check=True)
    subprocess.run([sys.executable, __file__, "gpu"], check=True)


if __name__ == "__main__":
    main()
