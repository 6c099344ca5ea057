"""Measurements of the SURVEY 8(f) "next" rows at the c2 scale, each with its parity check (JSON lines):

  NEXT-1 generalised eigenproblem A x = lambda B x: reduction to standard form (ZPOTRF of B,
         two ZTRSM, hermitise), ChFSI on H = L^{-1} A L^{-H}, back-transform x = L^{-H} y. A = M H1 M^H and
         B = M M^H with the generator's lower factor M, so the generalised eigenvalues are exactly the
         spectrum of H1 (R20); reports the time of each stage and the eigenvalue error.
  NEXT-3 real-symmetric sequence: H1 = Q diag(lambda) Q^T (Q = 8 real Householder reflectors), then
         H_{l+1} = H_l + delta * 40 * G_l (G_l symmetric Gaussian / sqrt(2n)); per-eigenproblem time and the
         real K1 rate (2 n^2 sum(deg) real flops), eigenvalues of problem 1 vs the exact spectrum.
  NEXT-4 independent sequences (k-points): S sequences of the c1 shape solved one after another
         vs concurrently by chfsi_solve_batch with W worker contexts on one GPU; aggregate throughput.

Inputs are built on the GPU with torch where the product is large (input construction only; the solves
go through the C-ABI). Usage: python tools/bench_next.py [next1] [next1p] [next3] [next4] (default: all)."""
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
from gen.configs import CONFIGS, HNORM  # noqa: E402


def ev_time(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1) / 1e3


def next1(cf):
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    t0 = time.time()
    w = G.wy(n, cf["nd"], cf["seed"])
    M = torch.as_tensor(G.lower_factor(n, cf["seed"] + 7, 0.5)).cuda()
    H1 = torch.as_tensor(w.full()).cuda()
    A = M @ H1 @ M.conj().t()
    B = M @ M.conj().t()
    A = (A + A.conj().t()) / 2
    B = (B + B.conj().t()) / 2
    del H1, M
    Ad, Bd = chfsi.colmajor(n, n), chfsi.colmajor(n, n)
    Ad.copy_(A)
    Bd.copy_(B)
    del A, B
    torch.cuda.empty_cache()
    gen_s = time.time() - t0
    ctx = chfsi.Context(0)
    ctx.reserve(n, n, nev + nex)
    _, t_red = ev_time(lambda: ctx.reduce_generalized(Ad, Bd))
    Xd = chfsi.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
    out, t_solve = ev_time(lambda: ctx.solve_sequence(lambda ell: Ad, 1, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"],
                                                      seed=cf["seed"]))
    C = Xd[:, :nev].contiguous().t().contiguous().t()
    _, t_back = ev_time(lambda: ctx.back_transform(Bd, C))
    ctx.close()
    lam = out["lam"][0]
    err = float(np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev])))
    rep = out["reports"][0]
    print(json.dumps({"row": "NEXT-1 generalised", "n": n, "nev": nev, "nex": nex, "status": out["status"],
                      "t_reduce_s": t_red, "t_solve_s": t_solve, "t_back_transform_s": t_back,
                      "reduce_share": t_red / (t_red + t_solve + t_back), "loops": rep["loops"],
                      "max_rel_eig_err_vs_exact": err, "max_resid_over_tol": float(np.max(out["resid"][0]) / cf["tol"]),
                      "input_gen_s": gen_s}), flush=True)


def next1_panel(cf):
    """NEXT-1 through the row-panel entry points at p = 1 (chfsi_reduce_generalized_panel: ZPOTRF, then
    L^{-H} E, A X, L^{-1}(A X) and the cross-slab hermitisation; chfsi_back_transform_panel)."""
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    M = torch.as_tensor(G.lower_factor(n, cf["seed"] + 7, 0.5)).cuda()
    H1 = torch.as_tensor(w.full()).cuda()
    A = M @ H1 @ M.conj().t()
    B = M @ M.conj().t()
    Ad, Bd = chfsi.colmajor(n, n), chfsi.colmajor(n, n)
    Ad.copy_((A + A.conj().t()) / 2)
    Bd.copy_((B + B.conj().t()) / 2)
    del A, B, H1, M
    torch.cuda.empty_cache()
    Ld = chfsi.colmajor(n, n)
    ctx = chfsi.Context(0)
    ctx.reserve(n, n, nev + nex)
    _, t_red = ev_time(lambda: ctx.reduce_generalized_panel(Ad, Bd, Ld))
    Xd = chfsi.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
    out, t_solve = ev_time(lambda: ctx.solve_sequence(lambda ell: Ad, 1, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"],
                                                      seed=cf["seed"]))
    C = Xd[:, :nev].contiguous().t().contiguous().t()
    _, t_back = ev_time(lambda: ctx.back_transform_panel(Ld, C))
    ctx.close()
    lam = out["lam"][0]
    print(json.dumps({"row": "NEXT-1 generalised, row-panel entry points (p = 1)", "n": n, "nev": nev, "nex": nex,
                      "status": out["status"], "t_reduce_s": t_red, "t_solve_s": t_solve, "t_back_transform_s": t_back,
                      "loops": out["reports"][0]["loops"],
                      "max_rel_eig_err_vs_exact": float(np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev]))),
                      "max_resid_over_tol": float(np.max(out["resid"][0]) / cf["tol"])}), flush=True)


def real_sym_known(n, nd, seed):
    lam = torch.as_tensor(G.spectrum(n, nd), dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(seed)
    H = torch.diag(lam)
    for _ in range(8):  # H <- P H P, P = I - 2 v v^T / v^T v
        v = torch.randn(n, 1, dtype=torch.float64, device="cuda", generator=g)
        v = v / torch.linalg.norm(v)
        Hv = H @ v
        H = H - 2.0 * v @ Hv.t() - 2.0 * Hv @ v.t() + 4.0 * (v.t() @ Hv) * (v @ v.t())
    H = (H + H.t()) / 2
    return H, lam.cpu().numpy()


def next3(cf, nprob=4):
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    t0 = time.time()
    H, lam = real_sym_known(n, cf["nd"], cf["seed"])
    g = torch.Generator(device="cuda").manual_seed(cf["seed"] + 1)
    Hs = []
    for ell in range(nprob):
        if ell > 0:
            Gm = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) / (2 * n) ** 0.5
            H = H + cf["delta"] * HNORM * (Gm + Gm.t()) / 2 ** 0.5
            del Gm
        Hd = chfsi.colmajor(n, n, dtype=torch.float64)
        Hd.copy_(H)
        Hs.append(Hd)
    del H
    torch.cuda.empty_cache()
    gen_s = time.time() - t0
    X0 = torch.randn(n, nev + nex, dtype=torch.float64, device="cuda", generator=g)
    Xd = chfsi.colmajor(n, nev + nex, dtype=torch.float64)
    Xd.copy_(X0)
    ctx = chfsi.Context(0)
    ctx.reserve(n, n, nev + nex)
    out, t_all = ev_time(lambda: ctx.solve_sequence(lambda ell: Hs[ell], nprob, Xd, nev, nex, cf["tol"],
                                                    deg_cap=cf["cap"], seed=cf["seed"], real=True))
    ctx.close()
    reps = out["reports"]
    err = float(np.max(np.abs(out["lam"][0] - lam[:nev]) / np.abs(lam[:nev])))
    k1 = [r["filter_flops"] / max(r["t_filter_kernel"], 1e-12) / 1e12 for r in reps]
    print(json.dumps({"row": "NEXT-3 real symmetric", "n": n, "nev": nev, "nex": nex, "nprob": nprob,
                      "status": out["status"], "t_per_problem_s": [r["t_total"] for r in reps],
                      "loops": [r["loops"] for r in reps], "k1_real_tflops": k1,
                      "k1_frac_of_fp64_peak": [x / 37.07 for x in k1],
                      "max_rel_eig_err_problem1_vs_exact": err,
                      "max_resid_over_tol": float(np.max(out["resid"]) / cf["tol"]), "input_gen_s": gen_s,
                      "total_s": t_all}), flush=True)


def next4(cf, S=8, nprob=3, workers=(1, 2, 4)):
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    base = G.wy(n, cf["nd"], cf["seed"])
    H0 = base.full()
    seqs = []
    for s in range(S):  # sequence s: H1 + a seeded perturbation per problem (distinct k-points)
        Hs = []
        H = H0.copy(order="F")
        for ell in range(nprob):
            G.perturb(H, cf["seed"] + 100 * s, ell + 1, cf["delta"] * HNORM)
            Hs.append(chfsi.to_colmajor(H))
        seqs.append(Hs)
    X0 = G.start_basis(n, nev + nex, cf["seed"])
    for W in workers:
        Xs = [chfsi.to_colmajor(X0) for _ in range(S)]
        sequences = [((lambda ell, s=s: seqs[s][ell]), nprob, Xs[s]) for s in range(S)]
        outs, t = ev_time(lambda: chfsi.solve_batch(0, W, sequences, nev, nex, cf["tol"], deg_cap=cf["cap"],
                                                    seed=cf["seed"]))
        ok = all(o["status"] == 0 for o in outs)
        worst = max(float(np.max(o["resid"])) for o in outs) / cf["tol"]
        print(json.dumps({"row": "NEXT-4 independent sequences", "n": n, "nev": nev, "nex": nex, "sequences": S,
                          "problems_each": nprob, "workers": W, "total_s": t,
                          "eigenproblems_per_s": S * nprob / t, "all_converged": ok, "max_resid_over_tol": worst}),
              flush=True)


def main():
    which = set(sys.argv[1:]) or {"next1", "next1p", "next3", "next4"}
    if "next1" in which:
        next1(CONFIGS["c2"])
    if "next1p" in which:
        next1_panel(CONFIGS["c2"])
    if "next3" in which:
        next3(CONFIGS["c2"])
    if "next4" in which:
        next4(CONFIGS["c1"])


if __name__ == "__main__":
    main()
