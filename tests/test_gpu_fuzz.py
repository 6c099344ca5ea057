"""Seeded random sweep of chfsi_filter configurations against the closed form:
H = Q Lambda Q^H from the compact-WY generator, so Q diag(p_m(Lambda)) Q^H Y0 is exact at any n. Each case
draws the panel count P (1 .. 8 emulated ranks, allgather or peer push, optional column groups), n
(a multiple of P, 64 .. 3000: ragged against every tile height), k (1 .. 400), sorted degrees (random,
all equal, or a ramp), the complex arithmetic (3M / 4M) and sometimes a forced tile variant -- the
persistent / stream-K schedule, its weights, the half-unit MMA skipping and the rank-chunked
contraction meet combinations no hand-written case pins."""
import os

import numpy as np
import pytest

import gen as G
import oracle as O
from test_gpu_multirank import run_ranks, slabs

pytestmark = pytest.mark.gpu

Z3 = ["200", "207", "208"]
Z4 = ["1", "3", "5", "6", "7", "9", "10", "11", "12", "13", "14"]


def draw(seed):
    rng = np.random.default_rng(1404416100 + seed)
    P = int(rng.choice([1, 1, 1, 2, 3, 4, 8]))
    n = P * int(rng.integers(max(64 // P, 8), 3000 // P + 1))
    k = int(rng.integers(1, min(n, 400) + 1))
    kind = int(rng.integers(0, 3))
    if kind == 0:
        deg = sorted(rng.integers(1, 31, k).tolist())
    elif kind == 1:
        deg = [int(rng.integers(1, 31))] * k
    else:
        lo, hi = sorted(rng.integers(1, 31, 2).tolist())
        deg = [lo + round((hi - lo) * j / max(k - 1, 1)) for j in range(k)]
    zmul = int(rng.choice([3, 3, 4]))
    forced = None
    if rng.random() < 0.35:
        forced = str(rng.choice(Z3 if zmul == 3 else Z4))
    push = P > 1 and bool(rng.random() < 0.5)
    group_cols = int(rng.choice([0, 8, 32])) if P > 1 and not push and rng.random() < 0.5 else None
    return dict(P=P, n=n, k=k, deg=deg, zmul=zmul, forced=forced, push=push, group_cols=group_cols,
                wseed=int(rng.integers(1, 1 << 30)), yseed=int(rng.integers(1, 1 << 30)))


@pytest.mark.parametrize("seed", range(64))
def test_filter_fuzz_vs_closed_form(gpu_lib, seed):
    cs = draw(seed)
    P, n, k, deg = cs["P"], cs["n"], cs["k"], cs["deg"]
    w = G.wy(n, max(int(0.9 * n), 1), cs["wseed"])
    rng = np.random.default_rng(cs["yseed"])
    Y0 = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    l1, a, b = w.lam[0] - 0.05, w.lam[min(k, n - 1)], 45.0
    c, e = (a + b) / 2, (b - a) / 2
    env = None
    if cs["forced"] is not None:
        env = "CHFSI_FILTER_VARIANT_Z3" if cs["zmul"] == 3 else "CHFSI_FILTER_VARIANT"
        os.environ[env] = cs["forced"]
    try:
        H = w.full()
        if P == 1:
            ctx = gpu_lib.Context(0)
            ctx.set_complex_mult(cs["zmul"])
            Yd = gpu_lib.to_colmajor(Y0)
            assert ctx.filter(gpu_lib.to_colmajor(H), Yd, deg, l1, c, e) == sum(deg)
            Y = Yd.cpu().numpy()
            ctx.close()
        else:
            Hs, nloc = slabs(gpu_lib, H, P)
            Ys = [gpu_lib.to_colmajor(Y0[r * nloc:(r + 1) * nloc]) for r in range(P)]

            def fn(r, ctx):
                ctx.set_complex_mult(cs["zmul"])
                return ctx.filter(Hs[r], Ys[r], deg, l1, c, e, n=n, row0=r * nloc)

            mv = run_ranks(gpu_lib, P, fn, cs["group_cols"], (n, nloc, k) if cs["push"] else None)
            assert all(m == sum(deg) for m in mv)
            Y = np.concatenate([y.cpu().numpy() for y in Ys], axis=0)
    finally:
        if env:
            os.environ.pop(env, None)
    Yc = O.filter_wy_closed(w, Y0, deg, l1, c, e)
    rel = np.linalg.norm(Y - Yc, axis=0) / np.linalg.norm(Yc, axis=0)
    assert rel.max() <= 1e-11, (cs | {"deg": (min(deg), max(deg))}, float(rel.max()))


def draw_solve(seed):
    rng = np.random.default_rng(1404416200 + seed)
    P = int(rng.choice([1, 1, 2, 4]))
    n = P * int(rng.integers(240 // P, 1600 // P + 1))
    nev = int(rng.integers(4, max(5, n // 20)))
    nex = int(rng.integers(max(4, nev // 4), nev // 2 + 6))  # the configurations use nex = 20-50 % of nev
    cap = int(rng.choice([20, 30, 36, 40]))
    deg0 = int(rng.integers(2, min(cap, 10) + 1))
    zmul = int(rng.choice([3, 3, 4]))
    push = P > 1 and bool(rng.random() < 0.5)
    return dict(P=P, n=n, nev=nev, nex=nex, cap=cap, deg0=deg0, zmul=zmul, push=push,
                nd=int(n * rng.uniform(0.6, 0.95)), wseed=int(rng.integers(1, 1 << 30)),
                nprob=int(rng.integers(1, 4)), delta=float(rng.choice([0.0, 1e-4, 1e-3])))


@pytest.mark.parametrize("seed", range(16))
def test_solve_fuzz(gpu_lib, seed):
    """Seeded random ChFSI sequences (1 .. 3 problems, the later ones perturbed; 1 / 2 / 4 emulated ranks;
    random nev, nex, degree cap, starting degree, 3M / 4M): problem 1's eigenvalues equal the generator's
    exact spectrum to 1e-10 and every problem's residuals ||H x - lambda x|| / ||H||_2 stay <= tol, with
    ||H^(l)||_2 bounded by 40 + the perturbations' norm."""
    from gen.configs import HNORM

    cs = draw_solve(seed)
    P, n, nev, nex, nprob = cs["P"], cs["n"], cs["nev"], cs["nex"], cs["nprob"]
    w = G.wy(n, cs["nd"], cs["wseed"])
    Hl = [w.full()]
    for ell in range(1, nprob):
        H = Hl[-1].copy(order="F")
        if cs["delta"] > 0:
            G.perturb(H, cs["wseed"], ell, cs["delta"] * HNORM)
        Hl.append(H)
    X0 = G.start_basis(n, nev + nex, cs["wseed"])
    tol = 1e-10
    if P == 1:
        ctx = gpu_lib.Context(0)
        ctx.set_complex_mult(cs["zmul"])
        Hd = [gpu_lib.to_colmajor(H) for H in Hl]
        Xd = gpu_lib.to_colmajor(X0)
        out = ctx.solve_sequence(lambda ell: Hd[ell], nprob, Xd, nev, nex, tol, deg_cap=cs["cap"], deg0=cs["deg0"],
                                 seed=cs["wseed"])
        X = Xd.cpu().numpy()
        ctx.close()
    else:
        Hs = [slabs(gpu_lib, H, P)[0] for H in Hl]
        nloc = n // P
        Xs = [gpu_lib.to_colmajor(X0[r * nloc:(r + 1) * nloc]) for r in range(P)]

        def fn(r, ctx):
            ctx.set_complex_mult(cs["zmul"])
            return ctx.solve_sequence(lambda ell: Hs[ell][r], nprob, Xs[r], nev, nex, tol, deg_cap=cs["cap"],
                                      deg0=cs["deg0"], seed=cs["wseed"], n=n, row0=r * nloc)

        outs = run_ranks(gpu_lib, P, fn, None, (n, nloc, nev + nex) if cs["push"] else None)
        for o in outs[1:]:
            assert np.array_equal(o["lam"], outs[0]["lam"])  # identical bits on every rank
        out = outs[0]
        X = np.concatenate([x.cpu().numpy() for x in Xs], axis=0)
    assert out["status"] == 0, cs
    lam = np.asarray(out["lam"])
    assert np.max(np.abs(lam[0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10, cs
    # the final block holds the last problem's eigenvectors (first nev columns, ascending)
    Xn = X[:, :nev]
    Hn = Hl[-1]
    hnorm = HNORM + 2.5 * cs["delta"] * HNORM * (nprob - 1)  # ||G|| ~ 2 per perturbation (d2)
    res = np.linalg.norm(Hn @ Xn - Xn * lam[-1], axis=0) / np.linalg.norm(Xn, axis=0) / hnorm
    assert res.max() <= tol, (cs, float(res.max()))
