"""Pins of the oracle's dense building blocks and supporting ChFSI steps: against library routines
(numpy matmul / qr / eigvalsh), SPEC worked examples, exact spectra of the generator's H^(1), and
closed forms. Citations: P:n = PAPER.md line n; S:n = SPEC.md line n."""
import json
import math
import os

import numpy as np
import pytest

import gen as G
import oracle as O

GOLD = [json.loads(l) for l in open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.jsonl"))]


def gold(what):
    return [g for g in GOLD if g["what"] == what]


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_zgemm_vs_numpy():
    rng = np.random.default_rng(0)
    A, B = crand(rng, 37, 23), crand(rng, 23, 19)
    np.testing.assert_allclose(O.zgemm("N", "N", A, B), A @ B, rtol=0, atol=1e-12)
    A2 = crand(rng, 23, 37)
    np.testing.assert_allclose(O.zgemm("C", "N", A2, B), A2.conj().T @ B, rtol=0, atol=1e-12)
    B2 = crand(rng, 19, 23)
    np.testing.assert_allclose(O.zgemm("N", "C", A, B2), A @ B2.conj().T, rtol=0, atol=1e-12)


# ---- Householder QR ---------------------------------------------------------------------------
@pytest.mark.parametrize("g", gold("qr"), ids=lambda g: g["cite"][:11])
def test_qr_golden(g):
    Q, R, d = O.householder_qr(np.array(g["a"], dtype=complex)[:, None])
    np.testing.assert_allclose(np.abs(Q[:, 0]), g["q"], atol=1e-15)
    assert d == 0


@pytest.mark.parametrize("n,k", [(50, 7), (200, 48), (33, 33)])
def test_qr_properties_and_numpy(n, k):
    rng = np.random.default_rng(n + k)
    A = crand(rng, n, k)
    Q, R, d = O.householder_qr(A)
    assert d == 0
    assert np.abs(Q.conj().T @ Q - np.eye(k)).max() <= 1e-13
    assert np.linalg.norm(Q @ R - A) / np.linalg.norm(A) <= 1e-14
    assert np.allclose(np.tril(R, -1), 0)
    assert np.all(np.diag(R).real > 0)
    # unique QR with positive diagonal: equals numpy's up to the diagonal phase it chose
    Qn, Rn = np.linalg.qr(A)
    ph = np.diag(Rn) / np.abs(np.diag(Rn))
    np.testing.assert_allclose(Q, Qn * ph, atol=1e-12)


def test_qr_detects_rank_deficiency():
    rng = np.random.default_rng(5)
    A = crand(rng, 20, 4)
    A[:, 2] = A[:, 0] * (1 - 2j)
    _, _, d = O.householder_qr(A)
    assert d == 1


def _unique_qr(A):
    """numpy QR with the positive-real-diagonal convention (the unique QR of a full-rank A)."""
    Q, R = np.linalg.qr(A)
    return Q * (np.diag(R) / np.abs(np.diag(R)))


def _r22(n, seed, strm):
    """The R22 vector written out from gen's uniform hash (independent of the oracle's own code)."""
    u = np.array([G.uniform(seed, strm, t) for t in range(2 * n)])
    return (2 * u[0::2] - 1) + 1j * (2 * u[1::2] - 1)


@pytest.mark.parametrize("case", ["duplicate", "zero", "in_locked_span"])
def test_orthonormalize_rank_deficiency_rule(case):
    """R23: a numerically dependent active column is replaced by the R22 vector of stream
    (6 << 16) | (nl + j) and the block is orthonormalised again. Pinned against numpy: the result is the
    unique QR of [X_L | Y'] restricted to the active columns, Y' = Y with the column replaced."""
    rng = np.random.default_rng(21)
    n, ka, seed = 120, 9, 77
    nl = 0 if case == "duplicate" else 5
    XL = _unique_qr(crand(rng, n, nl)) if nl else None
    Y = crand(rng, n, ka)
    j = 4
    if case == "duplicate":  # duplicated column
        Y[:, j] = Y[:, j - 1]
    elif case == "zero":
        Y[:, j] = 0
    else:  # lies in span(X_L): nothing is left after the projection against the locked block
        Y[:, j] = XL @ crand(rng, nl)
    Q, replaced = O.orthonormalize(Y, XL, seed=seed)
    assert replaced == 1
    full = Q if XL is None else np.hstack([XL, Q])
    assert np.abs(full.conj().T @ full - np.eye(full.shape[1])).max() <= 1e-13
    Yp = Y.copy()
    Yp[:, j] = _r22(n, seed, (6 << 16) | (nl + j))
    ref = _unique_qr(Yp if XL is None else np.hstack([XL, Yp]))[:, nl:]
    np.testing.assert_allclose(Q, ref, rtol=0, atol=1e-12)


def test_orthonormalize_full_rank_untouched():
    rng = np.random.default_rng(22)
    Y = crand(rng, 80, 12)
    Q, replaced = O.orthonormalize(Y, None, seed=3)
    assert replaced == 0
    np.testing.assert_allclose(Q, _unique_qr(Y), rtol=0, atol=1e-12)


# ---- Jacobi eigensolver -----------------------------------------------------------------------
@pytest.mark.parametrize("g", gold("eig"), ids=lambda g: g["cite"][:11])
def test_jacobi_golden(g):
    w, V = O.jacobi_eig(np.array(g["a"], dtype=complex))
    np.testing.assert_allclose(w, g["w"], atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 17, 64, 120])
def test_jacobi_vs_numpy(n):
    rng = np.random.default_rng(n)
    A = crand(rng, n, n)
    A = A + A.conj().T
    w, V = O.jacobi_eig(A)
    nrm = np.linalg.norm(A, 2)
    np.testing.assert_allclose(w, np.linalg.eigvalsh(A), rtol=0, atol=1e-13 * nrm * max(1, n / 16))
    assert np.linalg.norm(A @ V - V * w) <= 1e-12 * n * np.linalg.norm(A)
    assert np.abs(V.conj().T @ V - np.eye(n)).max() <= 1e-13 * max(1, n / 16)
    # phase convention: the largest-|.| entry of every column is real positive
    for j in range(n):
        i = int(np.argmax(np.abs(V[:, j])))
        assert V[i, j].imag == 0 and V[i, j].real > 0


def test_jacobi_exact_spectrum_h1():
    n = 256
    w_ = G.wy(n, 230, 21)
    H = w_.full()
    w, V = O.jacobi_eig(H)
    np.testing.assert_allclose(w, w_.lam, rtol=0, atol=1e-12 * 40)


def test_count_below_vs_numpy():
    rng = np.random.default_rng(8)
    n = 90
    A = crand(rng, n, n)
    A = (A + A.conj().T) / 2
    ev = np.linalg.eigvalsh(A)
    for s in (-20.0, ev[10] + 1e-3, 0.0, ev[60] - 1e-3, 50.0):
        assert O.count_below(A, s) == int(np.sum(ev < s))


@pytest.mark.parametrize("n", [512, 640])
def test_count_below_near_eigenvalues(n):
    """Bunch-Kaufman inertia at n >= 512 (the completeness gate's sizes scale this up) with shifts
    within 1e-8 of an eigenvalue, on either side (Sylvester's law of inertia vs numpy.eigvalsh)."""
    rng = np.random.default_rng(n)
    A = crand(rng, n, n) / np.sqrt(2 * n)
    A = (A + A.conj().T) / 2
    ev = np.linalg.eigvalsh(A)
    for i in (0, 7, n // 3, n // 2, n - 5):
        gap = min(ev[i] - ev[i - 1] if i else 1.0, ev[i + 1] - ev[i])
        assert gap > 1e-6
        for s in (ev[i] - 1e-8, ev[i] + 1e-8):
            assert O.count_below(A, s) == int(np.sum(ev < s)), (i, s)


def test_count_below_exact_spectrum_h1():
    """H^(1) = Q diag(Lambda) Q^H from the generator has an exactly known spectrum: the count below a
    point halfway between Lambda_i and Lambda_{i+1} is i + 1 (independent of any eigensolver)."""
    n = 600
    w = G.wy(n, 540, 31)
    H = w.full()
    for i in (0, 31, 200, 539, 540, 598):
        s = 0.5 * (w.lam[i] + w.lam[i + 1])
        assert O.count_below(H, s) == i + 1


def test_count_below_needs_pivoting():
    """Cases an unpivoted LDL^H gets wrong: (a) a zero diagonal (every 1x1 pivot of [[0, B], [B^H, 0]]
    at sigma = 0 is 0: the 2x2 pivots are required; the spectrum is +-singular values of B, so exactly
    n/2 are negative); (b) a leading pivot of 1e-14 next to O(1) off-diagonals (element growth 1e14)."""
    rng = np.random.default_rng(12)
    h = 256
    B = crand(rng, h, h)
    Z = np.zeros((2 * h, 2 * h), dtype=complex)
    Z[:h, h:] = B
    Z[h:, :h] = B.conj().T
    assert O.count_below(Z, 0.0) == h
    sv = np.linalg.svd(B, compute_uv=False)  # eigenvalues of Z: -sv (h of them) and +sv
    assert O.count_below(Z, -0.5 * sv.min()) == h
    assert O.count_below(Z, 0.5 * sv.min()) == h
    assert O.count_below(Z, -np.sort(sv)[h // 2] + 1e-9) == h - h // 2
    # (b) a GUE-like matrix whose leading entry is 1e-15 / 1e-17: the unpivoted count returns 255 and
    # 256 here instead of 254 (checked when this pin was written); Bunch-Kaufman interchanges first
    n = 512
    for tiny in (1e-15, 1e-17):
        rng = np.random.default_rng(4)
        A = crand(rng, n, n) / np.sqrt(2 * n)
        A = (A + A.conj().T) / 2
        A[0, 0] = tiny
        ev = np.linalg.eigvalsh(A)
        assert np.min(np.abs(ev)) > 1e-6
        assert O.count_below(A, 0.0) == int(np.sum(ev < 0)) == 254


# ---- Lanczos (Alg 1 l3; R17) ---------------------------------------------------------------
@pytest.mark.parametrize("g", gold("lanczos"), ids=lambda g: g["cite"][:12])
def test_lanczos_golden(g):
    H = np.diag(np.array(g["diag"], dtype=complex))
    tmin, tmax, beta = O.lanczos(H, g["steps"], 1)
    assert tmin == pytest.approx(g["theta_min"], abs=1e-12)
    assert tmax == pytest.approx(g["theta_max"], abs=1e-12)
    assert beta >= g["theta_max"] - 1e-12


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_lanczos_bounds_h1(seed):
    # lambda_max(H^(1)) = 40 exactly: theta_max <= 40 (interlacing) and beta_up >= 40 (safe bound)
    w_ = G.wy(512, 480, 1404416100)
    H = w_.full()
    tmin, tmax, beta = O.lanczos(H, 25, seed)
    assert tmax <= 40.0 + 1e-10
    assert beta >= 40.0
    assert tmin >= -2.0 - 1e-10


def test_random_vector_formula():
    # R22: u_t = (splitmix64(seed ^ (stream << 40) ^ t) >> 11) 2^-53; x_i = (2u_2i - 1) + i(2u_2i+1 - 1)
    M = (1 << 64) - 1

    def sm(x):
        z = (x + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    seed, strm = 1234567, (4 << 16) | 2
    x = O.random_vector(9, seed, strm)
    for i in range(9):
        u0 = (sm(seed ^ (strm << 40) ^ (2 * i)) >> 11) * 2.0**-53
        u1 = (sm(seed ^ (strm << 40) ^ (2 * i + 1)) >> 11) * 2.0**-53
        assert x[i] == complex(2 * u0 - 1, 2 * u1 - 1)


# ---- Rayleigh-Ritz and residuals (Alg 1 l7-10) --------------------------------------------------------
@pytest.mark.parametrize("g", gold("rr_invariant"), ids=lambda g: g["cite"][:12])
def test_rr_golden(g):
    H = np.diag(np.array(g["diag"], dtype=complex))
    n = H.shape[0]
    rng = np.random.default_rng(0)
    E = np.eye(n, dtype=complex)[:, g["cols"]]
    Q, _ = np.linalg.qr(E @ crand(rng, len(g["cols"]), len(g["cols"])))
    ritz, Y = O.rayleigh_ritz(H, Q)
    np.testing.assert_allclose(ritz, g["ritz"], atol=1e-12)


def test_rr_exact_eigvecs_h1():
    n = 300
    w_ = G.wy(n, 270, 99)
    H = w_.full()
    idx = [0, 3, 4, 50, 299]
    X = w_.eigvecs(idx)
    rng = np.random.default_rng(4)
    Q, _ = np.linalg.qr(X @ crand(rng, 5, 5))  # same span, mixed basis
    ritz, Y = O.rayleigh_ritz(H, Q)
    np.testing.assert_allclose(ritz, w_.lam[idx], rtol=0, atol=1e-12 * 40)


def test_rr_ritz_inside_spectrum():
    n = 120
    rng = np.random.default_rng(6)
    A = crand(rng, n, n)
    A = (A + A.conj().T) / 2
    Q, _ = np.linalg.qr(crand(rng, n, 10))
    ritz, Y = O.rayleigh_ritz(A, Q)
    ev = np.linalg.eigvalsh(A)
    assert ritz.min() >= ev[0] - 1e-12 and ritz.max() <= ev[-1] + 1e-12
    assert np.abs(Y.conj().T @ Y - np.eye(10)).max() <= 1e-13


@pytest.mark.parametrize("g", gold("residual"), ids=lambda g: g["cite"][:11])
def test_residual_golden(g):
    H = np.diag(np.array(g["diag"], dtype=complex))
    r = O.residuals(H, np.array(g["y"], dtype=complex)[:, None], [g["lam"]], 1.0)
    assert r[0] == pytest.approx(g["value"], abs=1e-15)


def test_residual_exact_pairs_and_direct():
    n = 200
    w_ = G.wy(n, 180, 5)
    H = w_.full()
    X = w_.eigvecs([1, 7])
    r = O.residuals(H, X, w_.lam[[1, 7]], 40.0)
    assert r.max() <= 1e-15 * n
    rng = np.random.default_rng(1)
    y = crand(rng, n, 1)
    mu = float(np.real(y[:, 0].conj() @ H @ y[:, 0]) / np.real(y[:, 0].conj() @ y[:, 0]))
    r = O.residuals(H, y, [mu], 2.0)
    assert r[0] == pytest.approx(np.linalg.norm(H @ y[:, 0] - mu * y[:, 0]) / (np.linalg.norm(y) * 2.0), rel=1e-13)


# ---- degree model (R21) -------------------------------------------------------------------
@pytest.mark.parametrize("g", gold("degree_literal"), ids=lambda g: g["cite"][:12])
def test_degree_literal_golden(g):
    assert O.degree_literal(g["res"], g["tol"], g["rho"], g["cap"]) == g["m"]


def test_degree_acosh_rule_is_minimal():
    # R21: m = smallest integer with C_m(|t|) >= res/tol (eq:polydef inverted), clamped to [1, cap]
    for t in (-1.01, -1.3, 1.05, 2.0, 6.0):
        for ratio in (1.0, 3.0, 1e3, 1e8, 1e12):
            m = O.degree(ratio * 1e-10, 1e-10, t, 100000)
            assert O.cheb(m, abs(t)) >= ratio * (1 - 1e-12)
            if m > 1:
                assert O.cheb(m - 1, abs(t)) < ratio
    assert O.degree(1.0, 1e-10, 0.5, 36) == 36  # |t| <= 1 -> cap (R5)
    assert O.degree(1.0, 1e-10, 1.0001, 36) == 36  # clamped
    assert O.degree(1e-12, 1e-10, 3.0, 36) == 1  # already converged -> 1


def test_rayleigh_quotients_exact_and_closed_form():
    """ora_rayleigh_quotients: exact eigenpairs of H^(1) (generator) give rho = Lambda_i and zero
    residual; for diagonal H, rho = sum d_r |x_r|^2 / ||x||^2 and the residual is ||(d - rho) x|| / ||x||
    (closed forms evaluated entrywise)."""
    n = 300
    w = G.wy(n, 270, 41)
    idx = [0, 1, 150, 299]
    rho, ra = O.rayleigh_quotients(w.full(), w.eigvecs(idx))
    np.testing.assert_allclose(rho, w.lam[idx], rtol=0, atol=1e-12)
    assert ra.max() <= 1e-12
    rng = np.random.default_rng(42)
    d = rng.uniform(-2, 5, n)
    X = crand(rng, n, 3)
    rho, ra = O.rayleigh_quotients(np.diag(d).astype(complex), X)
    a2 = np.abs(X) ** 2
    rr = (d[:, None] * a2).sum(0) / a2.sum(0)
    np.testing.assert_allclose(rho, rr, rtol=1e-13)
    np.testing.assert_allclose(ra, np.linalg.norm((d[:, None] - rr) * X, axis=0) / np.linalg.norm(X, axis=0), rtol=1e-12)
