"""Parity at BASELINE.json's full sizes (c2: n = 13000, k = 624; c3: n = 30000, k = 1440) in the launch
configuration bench.py times: the filter on H^(1) checked column by column against the oracle's closed
form (every column) and against the oracle's Alg 2 (a sample of columns); the c2 sequence as the bench
solves it through its first timed (perturbed) problem and the first two c3 problems -- exact spectrum on
problem 1, oracle residuals / Kato-Temple bounds / inertia count on the perturbed problems."""
import numpy as np
import pytest

import gen as G
import oracle as O
from gen.configs import CONFIGS, HNORM
from parity_checks import check_perturbed

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def c2():
    cf = CONFIGS["c2"]
    w = G.wy(cf["n"], cf["nd"], cf["seed"])
    H = w.full()
    return cf, w, H


def test_filter_c2_full_width(gpu_lib, c2):
    cf, w, H = c2
    n, k = cf["n"], cf["nev"] + cf["nex"]
    rng = np.random.default_rng(2)
    deg = sorted(rng.integers(1, cf["cap"] + 1, k).tolist())
    Y0 = G.start_basis(n, k, cf["seed"])
    l1, a, b = w.lam[0] - 0.02, w.lam[k], 48.0
    c, e = (a + b) / 2, (b - a) / 2
    ctx = gpu_lib.Context(0)
    Hd = gpu_lib.to_colmajor(H)
    Yd = gpu_lib.to_colmajor(Y0)
    assert ctx.filter(Hd, Yd, deg, l1, c, e) == sum(deg)
    Y = Yd.cpu().numpy()
    del Hd, Yd
    ctx.close()
    Yc = O.filter_wy_closed(w, Y0, deg, l1, c, e)  # every column, closed form (App. A)
    rel = np.linalg.norm(Y - Yc, axis=0) / np.linalg.norm(Yc, axis=0)
    assert rel.max() <= 1e-11, (rel.max(), int(np.argmax(rel)))
    cols = [0, k // 2, k - 1]  # Alg 2 step by step, naive loops
    Yo, _ = O.chebyshev_filter(H, Y0[:, cols], [deg[j] for j in cols], l1, c, e)
    rel = np.linalg.norm(Y[:, cols] - Yo, axis=0) / np.linalg.norm(Yo, axis=0)
    assert rel.max() <= 1e-11


def test_solve_c2_sequence_perturbed(gpu_lib, c2):
    """The c2 sequence exactly as bench.py solves it (H^(1), then H^(l+1) = H^(l) + delta 40 G_l, the
    hand-off of each problem seeding the next, the same options), through problem 4 -- the first problem
    the bench times. Problem 1 against H^(1)'s exact spectrum (1e-10 relative, J) and orthonormality;
    problem 4 (perturbed) against the oracle: residuals, Kato-Temple bounds and the inertia count."""
    from gen.configs import DEG0, LANCZOS_STEPS, MAX_LOOPS

    cf, w, H = c2
    H = H.copy(order="F")
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    nprob = 4
    Hs = [gpu_lib.to_colmajor(H)]
    for ell in range(1, nprob):
        G.perturb(H, cf["seed"], ell, cf["delta"] * HNORM)
        Hs.append(gpu_lib.to_colmajor(H))
    Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
    ctx = gpu_lib.Context(0)
    ctx.reserve(n, n, nev + nex)
    out = ctx.solve_sequence(lambda ell: Hs[ell], nprob, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], deg0=DEG0,
                             max_loops=MAX_LOOPS, lanczos_steps=LANCZOS_STEPS, seed=cf["seed"])
    X = Xd.cpu().numpy()
    del Hs, Xd
    ctx.close()
    assert out["status"] == 0 and all(r["converged"] == nev for r in out["reports"])
    assert np.max(np.abs(out["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    assert np.abs(X[:, :nev].conj().T @ X[:, :nev] - np.eye(nev)).max() <= 1e-12
    assert out["resid"].max() <= cf["tol"]
    check_perturbed(H, out["lam"][-1], X, nev, cf["tol"], cf["seed"] + nprob - 1, inertia=True)


def test_filter_c3_full_width(gpu_lib):
    """c3 size (n = 30000, k = 1440 = 1200 + 240, degree cap 40): the filter on H^(1) against the
    compact-WY closed form on every column (App. A) and the oracle's Alg 2 on two sampled columns."""
    cf = CONFIGS["c3"]
    n, k = cf["n"], cf["nev"] + cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    rng = np.random.default_rng(3)
    deg = sorted(rng.integers(1, cf["cap"] + 1, k).tolist())
    Y0 = G.start_basis(n, k, cf["seed"])
    l1, a, b = w.lam[0] - 0.02, w.lam[k], 48.0
    c, e = (a + b) / 2, (b - a) / 2
    ctx = gpu_lib.Context(0)
    H = w.full()
    Hd = gpu_lib.to_colmajor(H)
    Yd = gpu_lib.to_colmajor(Y0)
    assert ctx.filter(Hd, Yd, deg, l1, c, e) == sum(deg)
    Y = Yd.cpu().numpy()
    del Hd, Yd
    ctx.close()
    Yc = O.filter_wy_closed(w, Y0, deg, l1, c, e)
    rel = np.linalg.norm(Y - Yc, axis=0) / np.linalg.norm(Yc, axis=0)
    assert rel.max() <= 1e-11, (rel.max(), int(np.argmax(rel)))
    cols = [0, k - 1]
    Yo, _ = O.chebyshev_filter(H, Y0[:, cols], [deg[j] for j in cols], l1, c, e)
    rel = np.linalg.norm(Y[:, cols] - Yo, axis=0) / np.linalg.norm(Yo, axis=0)
    assert rel.max() <= 1e-11


def test_solve_c3_sequence_perturbed(gpu_lib):
    """c3 size (n = 30000, nev 1200 + nex 240, cap 40): problems 1 and 2 of the sequence. Problem 1
    against H^(1)'s exact spectrum (1e-10 relative, J) and orthonormality; problem 2 (H^(2) = H^(1) +
    2e-4 40 G_1) against the oracle's residuals and Kato-Temple bounds (the inertia count is left to the
    c2 test: an n = 30000 Bunch-Kaufman factorisation in naive loops takes too long here)."""
    from gen.configs import DEG0, LANCZOS_STEPS, MAX_LOOPS

    cf = CONFIGS["c3"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    Hs = [gpu_lib.to_colmajor(H)]
    G.perturb(H, cf["seed"], 1, cf["delta"] * HNORM)
    Hs.append(gpu_lib.to_colmajor(H))
    Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
    ctx = gpu_lib.Context(0)
    ctx.reserve(n, n, nev + nex)
    out = ctx.solve_sequence(lambda ell: Hs[ell], 2, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], deg0=DEG0,
                             max_loops=MAX_LOOPS, lanczos_steps=LANCZOS_STEPS, seed=cf["seed"])
    X = Xd.cpu().numpy()
    del Hs, Xd
    ctx.close()
    assert out["status"] == 0 and all(r["converged"] == nev for r in out["reports"])
    assert np.max(np.abs(out["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    sample = [0, nev // 2, nev - 1]
    assert np.abs(X[:, sample].conj().T @ X[:, :nev] - np.eye(nev)[sample]).max() <= 1e-12
    check_perturbed(H, out["lam"][1], X, nev, cf["tol"], cf["seed"] + 1, inertia=False)


def _real_sym_known(n, nd, seed):
    """Input construction only (torch on the GPU): H = P_8 ... P_1 diag(lambda) P_1 ... P_8 with seeded
    real Householder reflectors P = I - 2 v v^T, so H's spectrum is exactly gen.spectrum(n, nd)."""
    import torch

    lam = G.spectrum(n, nd)
    g = torch.Generator(device="cuda").manual_seed(seed)
    H = torch.diag(torch.as_tensor(lam, dtype=torch.float64, device="cuda"))
    for _ in range(8):
        v = torch.randn(n, 1, dtype=torch.float64, device="cuda", generator=g)
        v = v / torch.linalg.norm(v)
        Hv = H @ v
        H = H - 2.0 * v @ Hv.t() - 2.0 * Hv @ v.t() + 4.0 * (v.t() @ Hv) * (v @ v.t())
    return (H + H.t()) / 2, lam, g


def test_solve_real_c2_first_problem(gpu_lib):
    """NEXT-3 at the c2 size (n = 13000, nev 520 + 104, cap 36): the real-symmetric solver's first
    eigenproblem against the exact spectrum, orthonormality and naive-oracle residuals on a sample."""
    import torch

    cf = CONFIGS["c2"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    H, lam, g = _real_sym_known(n, cf["nd"], cf["seed"])
    Hd = gpu_lib.colmajor(n, n, dtype=torch.float64)
    Hd.copy_(H)
    Xd = gpu_lib.colmajor(n, nev + nex, dtype=torch.float64)
    Xd.copy_(torch.randn(n, nev + nex, dtype=torch.float64, device="cuda", generator=g))
    del H
    ctx = gpu_lib.Context(0)
    out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], seed=cf["seed"], real=True)
    ctx.close()
    assert out["status"] == 0
    mu = out["lam"][0]
    assert np.max(np.abs(mu - lam[:nev]) / np.abs(lam[:nev])) <= 1e-10
    sample = [0, 1, nev // 2, nev - 1]
    X = Xd.cpu().numpy()[:, :nev]
    assert np.abs(X[:, sample].T @ X - np.eye(nev)[sample]).max() <= 1e-12
    res = O.residuals(Hd.cpu().numpy(), X[:, sample], mu[sample], HNORM)
    assert res.max() <= cf["tol"]


def test_generalized_c2_first_problem(gpu_lib):
    """NEXT-1 at the c2 size: A = M H^(1) M^H, B = M M^H (generator's lower factor M; products formed
    with torch on the GPU, input construction only) -> chfsi_reduce_generalized -> the solver ->
    chfsi_back_transform. Generalised eigenvalues = the exact spectrum of H^(1); generalised residuals
    and B-orthonormality on a sample of eigenvectors."""
    import torch

    cf = CONFIGS["c2"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    M = torch.as_tensor(G.lower_factor(n, cf["seed"] + 7, 0.5)).cuda()
    H1 = torch.as_tensor(w.full()).cuda()
    A = M @ H1 @ M.conj().t()
    B = M @ M.conj().t()
    del H1, M
    Ad, Bd = gpu_lib.colmajor(n, n), gpu_lib.colmajor(n, n)
    Ad.copy_((A + A.conj().t()) / 2)
    Bd.copy_((B + B.conj().t()) / 2)
    del A, B
    torch.cuda.empty_cache()
    A_h, B_h = Ad.cpu().numpy(), Bd.cpu().numpy()  # for the residual check
    ctx = gpu_lib.Context(0)
    ctx.reduce_generalized(Ad, Bd)
    Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
    out = ctx.solve_sequence(lambda ell: Ad, 1, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], seed=cf["seed"])
    sample = [0, nev // 2, nev - 1]
    Cd = Xd[:, sample].contiguous().t().contiguous().t()
    ctx.back_transform(Bd, Cd)
    ctx.close()
    assert out["status"] == 0
    lam = out["lam"][0]
    assert np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    C = Cd.cpu().numpy()
    BC = B_h @ C
    r = np.linalg.norm(A_h @ C - BC * lam[sample], axis=0) / (HNORM * np.linalg.norm(BC, axis=0))
    assert r.max() <= 1e-9
    assert np.abs(C.conj().T @ BC - np.eye(len(sample))).max() <= 1e-10


@pytest.mark.parametrize("k", [256, 1024])
def test_filter_c4_shape_sampled(gpu_lib, k):
    """BASELINE configs[4] shape as the sweep times it: n = 8192 GUE (stream (5, n)), the fixed interval,
    the sorted ramp of degrees 8..40 over k columns (every width from k down to the last few columns,
    3M and the 4M narrow tail); the oracle's Alg 2 on sampled columns (first, middle, last: degrees 8,
    ~24, 40) within the filter tolerance."""
    from gen.configs import C4_INTERVAL, c4_ramp

    n = 8192
    iv = C4_INTERVAL
    c, e = (iv["alpha"] + iv["beta"]) / 2, (iv["beta"] - iv["alpha"]) / 2
    Hh = G.gue(n, 5, G.stream(5, n))
    Y0 = G.start_basis(n, k, 5)
    deg = c4_ramp(k)
    ctx = gpu_lib.Context(0)
    Yd = gpu_lib.to_colmajor(Y0)
    assert ctx.filter(gpu_lib.to_colmajor(Hh), Yd, deg, iv["lambda1"], c, e) == sum(deg)
    cols = [0, k // 2, k - 1]
    Yg = Yd.cpu().numpy()[:, cols]
    ctx.close()
    Yo, _ = O.chebyshev_filter(Hh, Y0[:, cols], [deg[j] for j in cols], iv["lambda1"], c, e)
    rel = np.linalg.norm(Yg - Yo, axis=0) / np.linalg.norm(Yo, axis=0)
    assert rel.max() <= 1e-11, rel
