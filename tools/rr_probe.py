"""Probe of the k x k Rayleigh-Ritz eigenproblems a ChFSI sequence produces (the unsharded term of the
8-GPU model): solve the first problems of a sequence with CHFSI_RR_DUMP set, then run the
Jacobi-type simultaneous refinement on every dumped G (torch, complex128, on the GPU) against
torch.linalg.eigh and report how far G is from diagonal, how often the refinement must fall back to a
dense eigensolve, its iterations, accuracy and time.

usage: python tools/rr_probe.py [config] [nprob] [theta]
"""
import glob
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def refine(G, theta, maxit=6, stop=1e-9):
    """Ogita-Aishima-style refinement from X = I (see supporting.cu: eig_refine)."""
    import torch

    k = G.shape[0]
    eye = torch.eye(k, dtype=G.dtype, device=G.device)
    offd = ~torch.eye(k, dtype=torch.bool, device=G.device)
    X = eye.clone()
    S, R = G, torch.zeros_like(G)
    hist = []
    lam = G.diagonal().real.clone()
    for it in range(maxit):
        if it:
            S = X.mH @ (G @ X)
            R = eye - X.mH @ X
            lam = S.diagonal().real / (1 - R.diagonal().real)
        D = lam[None, :] - lam[:, None]
        num = S + R * lam[None, :]
        E = torch.where(offd, num / torch.where(offd, D, torch.ones_like(D)), torch.zeros_like(num))
        emax = float(E.abs()[offd].max()) if k > 1 else 0.0
        E.diagonal().copy_(R.diagonal() / 2)
        hist.append(emax)
        if emax > theta:
            return None, None, hist
        X = X + X @ E
        if emax <= stop:
            break
    else:
        return None, None, hist
    return lam, X, hist


def main():
    import numpy as np
    import torch

    import gen as G
    import paper_1404_4161_b200 as chfsi
    from gen.configs import CONFIGS, DEG0, HNORM, LANCZOS_STEPS, MAX_LOOPS

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    nprob = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    theta = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
    cf = CONFIGS[cfg]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    d = "/tmp/rrdump"
    os.makedirs(d, exist_ok=True)
    for f in glob.glob(d + "/*.bin"):
        os.remove(f)
    os.environ["CHFSI_RR_DUMP"] = d
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    Hs = [chfsi.to_colmajor(H)]
    for ell in range(1, nprob):
        G.perturb(H, cf["seed"], ell, cf["delta"] * HNORM)
        Hs.append(chfsi.to_colmajor(H))
    del H
    ctx = chfsi.Context(0)
    Xd = chfsi.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
    out = ctx.solve_sequence(lambda ell: Hs[ell], nprob, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], deg0=DEG0,
                             max_loops=MAX_LOOPS, lanczos_steps=LANCZOS_STEPS, seed=cf["seed"])
    ctx.close()
    print(json.dumps({"loops": [r["loops"] for r in out["reports"]]}), flush=True)
    files = sorted(glob.glob(d + "/g_*.bin"), key=lambda f: int(os.path.basename(f).split("_")[1]))
    for f in files:
        k = int(f.rsplit("_k", 1)[1].split(".")[0])
        Gm = torch.from_numpy(np.fromfile(f, dtype=np.complex128).reshape(k, k).T.copy()).cuda()
        Gm = (Gm + Gm.mH) / 2
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        wr, Vr = torch.linalg.eigh(Gm)
        torch.cuda.synchronize()
        t_eigh = time.perf_counter() - t0
        dg = Gm.diagonal().real
        off = Gm - torch.diag(Gm.diagonal())
        Dm = (dg[None, :] - dg[:, None]).abs()
        offd = ~torch.eye(k, dtype=torch.bool, device=Gm.device)
        ratio = (off.abs() / torch.where(offd, Dm, torch.ones_like(Dm)))[offd]
        rec = {"file": os.path.basename(f), "k": k, "offdiag_max": float(off.abs().max()),
               "ratio_max": float(ratio.max()),
               "pairs_over": {str(t): int((ratio > t).sum()) // 2 for t in (0.01, 0.05, 0.1, 0.3, 1.0)},
               "t_eigh_ms": 1e3 * t_eigh}
        for th in (theta, 0.3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lam, X, hist = refine(Gm, th)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            r = {"hist": [float("%.2e" % h) for h in hist], "ms": 1e3 * dt}
            if lam is not None:
                ls, order = torch.sort(lam)
                Xs = X[:, order]
                r["eig_err"] = float((ls - wr).abs().max())
                r["orth"] = float((Xs.mH @ Xs - torch.eye(k, dtype=Xs.dtype, device=Xs.device)).abs().max())
                r["resid"] = float((Gm @ Xs - Xs * ls[None, :]).abs().max())
            rec[f"theta{th}"] = r
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
