"""GPU parity of the supporting ChFSI steps (Lanczos, QR, Rayleigh-Ritz) and of the sequence solver
(Alg 1) through the C-ABI, against the oracle and against exactly known spectra (H^(1) from the
generator). Tolerances: BASELINE.json (eigenvalues <= 1e-10 relative, residual <= tol w.r.t. ||H||);
QR / RR to rounding."""
import numpy as np
import pytest

import gen as G
import oracle as O
from gen.configs import CONFIGS, DEG0, HNORM
from parity_checks import check_perturbed

pytestmark = pytest.mark.gpu


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.fixture
def ctx(gpu_lib):
    c = gpu_lib.Context(0)
    yield c
    c.close()


# ---- Lanczos (Alg 1 l3) -------------------------------------------------------------------------------
def test_lanczos_vs_oracle_and_exact(gpu_lib, ctx):
    w = G.wy(512, 480, 1404416100)
    H = w.full()
    Hd = gpu_lib.to_colmajor(H)
    for seed in (0, 5):
        tmin, tmax, beta = ctx.lanczos_bounds(Hd, 25, seed)
        otmin, otmax, obeta = O.lanczos(H, 25, seed)
        assert tmax <= 40.0 + 1e-10 and beta >= 40.0
        assert abs(tmax - otmax) <= 1e-10 * 40 and abs(tmin - otmin) <= 1e-10 * 40
        assert abs(beta - obeta) <= 1e-8 * 40


def test_lanczos_exact_krylov(gpu_lib, ctx):
    Hd = gpu_lib.to_colmajor(np.diag(np.arange(1.0, 6.0)).astype(complex))
    tmin, tmax, beta = ctx.lanczos_bounds(Hd, 5, 1)
    assert tmin == pytest.approx(1.0, abs=1e-12) and tmax == pytest.approx(5.0, abs=1e-12)


# ---- QR (Alg 1 l6) -----------------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,nl", [(300, 40, 0), (300, 40, 11), (1000, 130, 37)])
def test_qr_vs_oracle(gpu_lib, ctx, n, k, nl):
    rng = np.random.default_rng(n + k + nl)
    Y = crand(rng, n, k)
    if nl:
        Y[:, :nl] = np.linalg.qr(Y[:, :nl])[0]
    Yd = gpu_lib.to_colmajor(Y)
    fb = ctx.qr(Yd, nlocked=nl)
    Q = Yd.cpu().numpy()
    assert fb == 0
    assert np.array_equal(Q[:, :nl], Y[:, :nl])  # R15: locked columns untouched
    assert np.abs(Q.conj().T @ Q - np.eye(k)).max() <= 1e-13
    # reference: CGS2 against the locked block, then Householder QR (positive diagonal R: unique)
    A = Y[:, nl:].copy()
    X = Y[:, :nl]
    for _ in range(2):
        A = A - X @ O.zgemm("C", "N", X, A) if nl else A
    Qo, _, _ = O.householder_qr(A)
    assert np.abs(Q[:, nl:] - Qo).max() <= 1e-11


def test_qr_ill_conditioned_block(gpu_lib, ctx):
    rng = np.random.default_rng(9)
    n, k = 200, 12
    Y = crand(rng, n, k)
    Y[:, 5] = Y[:, 4] + 1e-11 * crand(rng, n)  # kappa ~ 1e11
    Yd = gpu_lib.to_colmajor(Y)
    ctx.qr(Yd)
    Q = Yd.cpu().numpy()
    assert np.abs(Q.conj().T @ Q - np.eye(k)).max() <= 1e-13
    P = Q @ Q.conj().T  # span of the well-conditioned leading columns preserved
    assert np.linalg.norm(P @ Y[:, :4] - Y[:, :4]) <= 1e-12 * np.linalg.norm(Y[:, :4])


def test_qr_householder_fallback(gpu_lib, ctx):
    # a zero column makes the Cholesky factorisation of Y^H Y fail -> Householder fallback
    rng = np.random.default_rng(10)
    n, k = 150, 9
    Y = crand(rng, n, k)
    Y[:, 3] = 0
    Yd = gpu_lib.to_colmajor(Y)
    fb = ctx.qr(Yd)
    Q = Yd.cpu().numpy()
    assert fb == 1
    assert np.abs(Q.conj().T @ Q - np.eye(k)).max() <= 1e-13
    P = Q @ Q.conj().T
    keep = [0, 1, 2, 4, 5, 6, 7, 8]
    assert np.linalg.norm(P @ Y[:, keep] - Y[:, keep]) <= 1e-12 * np.linalg.norm(Y[:, keep])
    Qo, _, _ = O.householder_qr(Y[:, :3])  # columns before the zero one: the unique QR
    assert np.abs(Q[:, :3] - Qo).max() <= 1e-12


@pytest.mark.parametrize("case", ["duplicate", "zero", "in_locked_span", "two_dependent"])
def test_qr_rank_deficiency_rule_vs_oracle(gpu_lib, ctx, case):
    """R23 on both sides: a dependent active column is replaced by the R22 vector
    (seed, stream (6 << 16) | column) and the block is orthonormalised again. The GPU result equals the
    oracle's ora_orthonormalize (same replacement count), [X_L | Q] is orthonormal and X_L is untouched
    -- including the Householder fallback with locked columns."""
    rng = np.random.default_rng(21)
    n, ka, seed = 300, 24, 77
    nl = 0 if case == "duplicate" else 9
    XL = np.linalg.qr(crand(rng, n, nl))[0] if nl else None
    Y = crand(rng, n, ka)
    if case == "duplicate":
        Y[:, 6] = Y[:, 5]
    elif case == "zero":
        Y[:, 6] = 0
    elif case == "in_locked_span":
        Y[:, 6] = XL @ crand(rng, nl)
    else:
        Y[:, 6] = XL @ crand(rng, nl)
        Y[:, 17] = 2j * Y[:, 3]
    full = Y if XL is None else np.hstack([XL, Y])
    Yd = gpu_lib.to_colmajor(full)
    fb, replaced = ctx.qr_ex(Yd, nlocked=nl, seed=seed)
    Q = Yd.cpu().numpy()
    Qo, ro = O.orthonormalize(Y, XL, seed=seed)
    assert fb == 1 and replaced == ro == (2 if case == "two_dependent" else 1)
    if nl:
        assert np.array_equal(Q[:, :nl], XL)
    assert np.abs(Q.conj().T @ Q - np.eye(nl + ka)).max() <= 1e-13
    assert np.abs(Q[:, nl:] - Qo).max() <= 1e-11


def test_solve_real_odd_n(gpu_lib, ctx):
    """Real-symmetric solve on one rank with odd n (the H Q operand's TMA stride must be a
    multiple of 16 bytes, so an odd leading dimension is re-strided): eigenvalues = the exact spectrum."""
    n, nev, nex = 301, 12, 6
    lam = np.sort(np.concatenate([np.linspace(-2.0, -1.0, 40), np.linspace(0.0, 10.0, n - 40)]))
    rng = np.random.default_rng(4)
    Qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
    H = (Qm * lam) @ Qm.T
    H = (H + H.T) / 2
    Hd = gpu_lib.to_colmajor(H, real=True)
    Xd = gpu_lib.to_colmajor(rng.standard_normal((n, nev + nex)), real=True)
    out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, nex, 1e-10, deg_cap=30, seed=3, real=True)
    assert out["status"] == 0
    np.testing.assert_allclose(out["lam"][0], lam[:nev], rtol=1e-10)


# ---- Rayleigh-Ritz (Alg 1 l7-9) ------------------------------------------------------------------------
def test_rr_exact_subspace(gpu_lib, ctx):
    n = 400
    w = G.wy(n, 360, 17)
    H = w.full()
    idx = [0, 1, 2, 10, 399]
    X = w.eigvecs(idx)
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(X @ crand(rng, 5, 5))
    Qd = gpu_lib.to_colmajor(Q)
    ritz, res = ctx.rayleigh_ritz(gpu_lib.to_colmajor(H), Qd, normH=HNORM)
    np.testing.assert_allclose(ritz, w.lam[idx], rtol=0, atol=1e-12 * HNORM)
    assert res.max() <= 1e-13


def test_rr_vs_oracle(gpu_lib, ctx):
    n, k = 350, 30
    Gm = G.gue(n, 8, G.stream(5, n))
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(crand(rng, n, k))
    Qd = gpu_lib.to_colmajor(Q)
    ritz, res = ctx.rayleigh_ritz(gpu_lib.to_colmajor(Gm), Qd, normH=2.0)
    ro, Yo = O.rayleigh_ritz(Gm, Q)
    np.testing.assert_allclose(ritz, ro, rtol=0, atol=1e-13)
    Yg = Qd.cpu().numpy()
    # Ritz vectors agree up to phase (simple Ritz values)
    ov = np.abs(np.sum(Yg.conj() * Yo, axis=0))
    assert np.abs(ov - 1).max() <= 1e-10
    ro_res = O.residuals(Gm, Yo, ro, 2.0)
    np.testing.assert_allclose(res, ro_res, rtol=1e-8, atol=1e-15)


@pytest.mark.parametrize("eps", [1e-9, 1e-4, 3e-3])
def test_rr_refinement_eigensolver(gpu_lib, ctx, eps):
    """The Jacobi-type refinement of the k x k eigensolve (chfsi_ctx_set_eigensolver mode 0) on a nearly
    diagonal projected matrix: Q = exact eigenvectors of H^(1) mixed by exp(eps A), A anti-Hermitian, so G =
    Q^H H Q has couplings ~eps. Ritz values agree with the dense ZHEEVD path (mode 1) and the oracle's
    Jacobi (ora_rayleigh_ritz) to 1e-13, with the exact spectrum, and the Ritz vectors agree up to phase."""
    import scipy.linalg

    n, k = 700, 96
    w = G.wy(n, 640, 51)
    H = w.full()
    rng = np.random.default_rng(52)
    idx = sorted(rng.choice(n - 100, k, replace=False))
    A = crand(rng, k, k)
    A = (A - A.conj().T) / 2
    Q = w.eigvecs(idx) @ scipy.linalg.expm(eps * A)
    Hd = gpu_lib.to_colmajor(H)
    out = {}
    for mode in (0, 1):
        ctx.set_eigensolver(mode)
        Qd = gpu_lib.to_colmajor(Q)
        ritz, res = ctx.rayleigh_ritz(Hd, Qd, normH=HNORM)
        out[mode] = (ritz, Qd.cpu().numpy(), res)
    ctx.set_eigensolver(0)
    ro, Yo = O.rayleigh_ritz(H, Q)
    for mode in (0, 1):
        np.testing.assert_allclose(out[mode][0], ro, rtol=0, atol=1e-13)
        np.testing.assert_allclose(out[mode][0], w.lam[idx], rtol=0, atol=1e-12)
        ov = np.abs(np.sum(out[mode][1].conj() * Yo, axis=0))
        assert np.abs(ov - 1).max() <= 1e-10
        assert out[mode][2].max() <= 1e-12
    np.testing.assert_allclose(out[0][0], out[1][0], rtol=0, atol=1e-13)


def test_solve_uses_refinement_and_matches_dense(gpu_lib, ctx):
    """A 3-problem sequence: the later loops' eigensolves run as the refinement (reports count them), and
    the converged eigenvalues equal those of the dense-only solver (mode 1) to 1e-12 relative."""
    cf = CONFIGS["c0"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    Hs = [gpu_lib.to_colmajor(H)]
    for ell in (1, 2):
        G.perturb(H, cf["seed"], ell, 1e-3 * HNORM)
        Hs.append(gpu_lib.to_colmajor(H))
    outs = {}
    for mode in (0, 1):
        ctx.set_eigensolver(mode)
        Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
        outs[mode] = ctx.solve_sequence(lambda ell: Hs[ell], 3, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"],
                                        seed=cf["seed"])
        assert outs[mode]["status"] == 0
    ctx.set_eigensolver(0)
    assert sum(r["eig_refined"] for r in outs[0]["reports"]) > 0
    assert sum(r["eig_refined"] for r in outs[1]["reports"]) == 0
    np.testing.assert_allclose(outs[0]["lam"], outs[1]["lam"], rtol=1e-12)
    ev = np.linalg.eigvalsh(Hs[-1].cpu().numpy())[:nev]
    np.testing.assert_allclose(outs[0]["lam"][-1], ev, rtol=1e-10)


# ---- the sequence solver (Alg 1; Def 1) ---------------------------------------------------------------
def test_solve_c0_exact_and_vs_oracle(gpu_lib, ctx):
    cf = CONFIGS["c0"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    X0 = G.start_basis(n, nev + nex, cf["seed"])
    Hd = gpu_lib.to_colmajor(H)
    Xd = gpu_lib.to_colmajor(X0)
    out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], seed=cf["seed"])
    assert out["status"] == 0
    lam = out["lam"][0]
    assert np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    X = Xd.cpu().numpy()[:, :nev]
    res = np.linalg.norm(H @ X - X * lam, axis=0) / HNORM
    assert res.max() <= cf["tol"]
    assert np.abs(X.conj().T @ X - np.eye(nev)).max() <= 1e-12
    ro = O.chfsi_solve(H, X0, nev, nex, cf["tol"], cf["cap"], seed=cf["seed"])
    assert np.max(np.abs(lam - ro["lam"]) / np.abs(ro["lam"])) <= 1e-10
    rep = out["reports"][0]
    assert rep["converged"] == nev and rep["matvecs_filter"] > 0
    assert rep["filter_flops"] == pytest.approx(8.0 * n * n * rep["matvecs_filter"])


def test_solve_random_start_block_formula(gpu_lib, ctx):
    # R22: random_start draws column j from stream (3 << 16) | j; the oracle builds the same block from
    # its own implementation of the formula, so both solves start from identical bits
    n, nev, nex = 256, 12, 4
    k = nev + nex
    w = G.wy(n, 230, 3)
    H = w.full()
    Hd = gpu_lib.to_colmajor(H)
    Xd = gpu_lib.to_colmajor(np.zeros((n, k)))
    out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, nex, 1e-10, deg_cap=20, seed=42, random_start=True)
    assert out["status"] == 0
    np.testing.assert_allclose(out["lam"][0], w.lam[:nev], rtol=1e-10)
    X0 = np.stack([O.random_vector(n, 42, (3 << 16) | j) for j in range(k)], axis=1)
    ro = O.chfsi_solve(H, X0, nev, nex, 1e-10, 20, seed=42)
    np.testing.assert_allclose(out["lam"][0], ro["lam"], rtol=1e-10)
    # same start bits and the same readings -> the same number of ChFSI loops (trajectory, unpinned
    # in general, agrees on this well-separated case)
    assert out["reports"][0]["loops"] == ro["report"]["loops"]


def test_solve_exact_input_one_loop(gpu_lib, ctx):
    n, nev, nex = 256, 12, 4
    w = G.wy(n, 230, 3)
    H = w.full()
    k = nev + nex
    Hd = gpu_lib.to_colmajor(H)
    # problem 0 converges from the exact eigenvectors; problem 1 (same H) must take one loop
    Xd = gpu_lib.to_colmajor(w.eigvecs(range(k)))
    out = ctx.solve_sequence(lambda ell: Hd, 2, Xd, nev, nex, 1e-10, deg_cap=20, seed=1)
    assert out["status"] == 0
    assert out["reports"][1]["loops"] == 1
    assert out["reports"][1]["matvecs_filter"] <= k * DEG0
    np.testing.assert_allclose(out["lam"][1], w.lam[:nev], rtol=1e-12)


@pytest.mark.slow
def test_solve_c1_sequence(gpu_lib, ctx):
    """c1: n = 4096, 5 correlated problems, nev = 200, nex = 40. Problem 1 against the exact spectrum,
    every problem against numpy.eigvalsh (library routine) and by its residuals (R8, J)."""
    cf = CONFIGS["c1"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    X0 = G.start_basis(n, nev + nex, cf["seed"])
    Hs = []
    for ell in range(cf["nprob"]):
        if ell > 0:
            G.perturb(H, cf["seed"], ell, cf["delta"] * HNORM)
        Hs.append(gpu_lib.to_colmajor(H))
    Xd = gpu_lib.to_colmajor(X0)
    out = ctx.solve_sequence(lambda ell: Hs[ell], cf["nprob"], Xd, nev, nex, cf["tol"], deg_cap=cf["cap"],
                             seed=cf["seed"])
    assert out["status"] == 0
    assert np.max(np.abs(out["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    Hl = Hs[-1].cpu().numpy()
    ev = np.linalg.eigvalsh(Hl)[:nev]
    lam = out["lam"][-1]
    assert np.max(np.abs(lam - ev) / np.abs(ev)) <= 1e-10
    X = Xd.cpu().numpy()[:, :nev]
    nrm = np.abs(np.linalg.eigvalsh(Hl)).max()
    res = np.linalg.norm(Hl @ X - X * lam, axis=0) / nrm
    assert res.max() <= cf["tol"] * 1.01
    # completeness ("the nev smallest"): Sylvester inertia of H - sigma I in the oracle
    # (LDL^H), sigma just above the GPU's largest wanted eigenvalue
    full = np.linalg.eigvalsh(Hl)
    sigma = lam[-1] + min(1e-6, 0.5 * (full[nev] - full[nev - 1]))
    assert O.count_below(Hl, sigma) == nev
    # the last (perturbed) problem against the oracle alone: residuals, Kato-Temple, inertia
    check_perturbed(np.asfortranarray(Hl), lam, Xd.cpu().numpy(), nev, cf["tol"], cf["seed"], inertia=True)
    loops = [r["loops"] for r in out["reports"]]
    assert all(l <= loops[0] for l in loops[1:])  # reuse of the previous eigenvectors pays


def test_ablation_options(gpu_lib, ctx):
    """NEXT-2 ablations: no_reuse restarts every problem from a random block; fixed_degree filters every
    vector with one degree (no Single Optimisation). Both still converge to the exact spectrum."""
    n, nd, nev, nex, delta, seed = 320, 272, 16, 8, 1e-3, 77
    w = G.wy(n, nd, seed)
    H = w.full()
    Hs = []
    for ell in range(3):
        if ell > 0:
            G.perturb(H, seed, ell, delta * HNORM)
        Hs.append(gpu_lib.to_colmajor(H))
    X0 = G.start_basis(n, nev + nex, seed)
    outs = {}
    for label, kw in (("base", {}), ("random", dict(no_reuse=True)), ("fixed", dict(fixed_degree=12))):
        Xd = gpu_lib.to_colmajor(X0)
        outs[label] = ctx.solve_sequence(lambda ell: Hs[ell], 3, Xd, nev, nex, 1e-10, deg_cap=30, seed=seed,
                                         max_loops=200, **kw)
        assert outs[label]["status"] == 0
        ev = np.linalg.eigvalsh(Hs[-1].cpu().numpy())[:nev]
        assert np.max(np.abs(outs[label]["lam"][-1] - ev) / np.abs(ev)) <= 1e-10
    # reuse pays: the random-start arm needs more filter work on the later problems
    base, rnd = outs["base"]["reports"], outs["random"]["reports"]
    assert sum(r["matvecs_filter"] for r in rnd[1:]) > sum(r["matvecs_filter"] for r in base[1:])
    # fixed degree: every filter call uses degree 12 for every vector
    for r in outs["fixed"]["reports"]:
        assert r["matvecs_filter"] % 12 == 0


def test_solve_batch_independent_sequences(gpu_lib, ctx):
    """NEXT-4: independent k-point sequences solved concurrently (chfsi_solve_batch, 2 workers on one
    device) give the same results as solving each sequence alone."""
    n, nd, nev, nex = 384, 340, 12, 6
    seqs, serial = [], []
    for s in range(3):
        w = G.wy(n, nd, 100 + s)
        H = w.full()
        Hs = [gpu_lib.to_colmajor(H)]
        G.perturb(H, 100 + s, 1, 1e-3 * HNORM)
        Hs.append(gpu_lib.to_colmajor(H))
        X0 = G.start_basis(n, nev + nex, 100 + s)
        Xd = gpu_lib.to_colmajor(X0)
        serial.append(ctx.solve_sequence(lambda ell, Hs=Hs: Hs[ell], 2, Xd, nev, nex, 1e-10, deg_cap=24, seed=7))
        seqs.append((lambda ell, Hs=Hs: Hs[ell], 2, gpu_lib.to_colmajor(X0)))
        np.testing.assert_allclose(serial[-1]["lam"][0], w.lam[:nev], rtol=1e-10)
    outs = gpu_lib.solve_batch(0, 2, seqs, nev, nex, 1e-10, deg_cap=24, seed=7)
    for i, (o, s) in enumerate(zip(outs, serial)):
        assert o["status"] == 0
        np.testing.assert_allclose(o["lam"], s["lam"], rtol=1e-13)
        assert [r["loops"] for r in o["reports"]] == [r["loops"] for r in s["reports"]]
        # each sequence's perturbed problem 2 against the oracle (not only against the serial path)
        H2 = np.asfortranarray(seqs[i][0](1).cpu().numpy())
        check_perturbed(H2, o["lam"][1], seqs[i][2].cpu().numpy(), nev, 1e-10, 7, inertia=True)


def test_library_owned_nccl_communicator(gpu_lib):
    """chfsi_nccl_unique_id + chfsi_ctx_create_nccl: NCCL is dlopen-ed, a communicator is created with
    ncclCommInitRank (one rank on this one-GPU box) and destroyed with the context; the solver runs on it."""
    cf = CONFIGS["c0"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    uid = gpu_lib.nccl_unique_id()
    assert len(uid) == 128
    ctx = gpu_lib.Context(0, nccl_id=uid, rank=0, nranks=1)
    w = G.wy(n, cf["nd"], cf["seed"])
    Hd = gpu_lib.to_colmajor(w.full())
    Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + nex, cf["seed"]))
    out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], seed=cf["seed"])
    ctx.close()
    assert out["status"] == 0
    assert np.max(np.abs(out["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10


def test_solve_without_buffer_vectors(gpu_lib, ctx):
    """nex = 0 is rejected (ERR_ARG): the filter interval starts at the largest of the k current values
    (reading R4), which without a buffer vector is the last wanted Ritz value itself -- it would never be
    separated from the damped interval. A small buffer (nex = 8 at the degree cap 40) converges."""
    cf = CONFIGS["c0"]
    n, nev = cf["n"], 40
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    Hd = gpu_lib.to_colmajor(H)
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_ARG"):
        ctx.solve_sequence(lambda ell: Hd, 1, gpu_lib.to_colmajor(G.start_basis(n, nev, cf["seed"])), nev, 0,
                           cf["tol"], deg_cap=cf["cap"], seed=cf["seed"])
    Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + 8, cf["seed"]))
    out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, 8, cf["tol"], deg_cap=40, seed=cf["seed"], max_loops=200)
    assert out["status"] == 0
    assert np.max(np.abs(out["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    X = Xd.cpu().numpy()[:, :nev]
    assert (np.linalg.norm(H @ X - X * out["lam"][0], axis=0) / HNORM).max() <= cf["tol"]
