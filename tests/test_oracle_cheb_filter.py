"""Pins of the oracle's Chebyshev values, sigma schedule and filter (Alg 2) against what the paper
and the mathematics fix: SPEC worked values, Chebyshev identities, the closed form p_m(H)Y of App. A
(diagonal H and H^(1) = Q Lambda Q^H), the product identity on a dense GUE matrix.
Citations: P:n = PAPER.md line n; S:n = SPEC.md line n."""
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


# ---- eq:polydef -------------------------------------------------------------------------
@pytest.mark.parametrize("g", gold("cheb"), ids=lambda g: g["cite"][:12])
def test_cheb_golden(g):
    assert O.cheb(g["m"], g["t"]) == pytest.approx(g["value"], rel=1e-15, abs=1e-15)


@pytest.mark.parametrize("g", gold("gain"), ids=lambda g: g["cite"][:12])
def test_gain_golden(g):
    assert O.filter_gain(g["m"], g["lam"], g["lambda1"], g["c"], g["e"]) == pytest.approx(g["value"], rel=1e-14)


def test_cheb_identities():
    # C_2m = 2 C_m^2 - 1 and C_m(C_n(t)) = C_mn(t) on both branches (|t|<=1, |t|>1, t<-1)
    for t in (-3.7, -1.2, -0.9, -0.3, 0.0, 0.41, 0.99, 1.0, 1.3, 2.5):
        for m in range(0, 12):
            assert O.cheb(2 * m, t) == pytest.approx(2 * O.cheb(m, t) ** 2 - 1, rel=1e-12, abs=1e-13)
        for m in (2, 3):
            for k in (2, 3):
                assert O.cheb(m, O.cheb(k, t)) == pytest.approx(O.cheb(m * k, t), rel=1e-11, abs=1e-12)
    # explicit polynomials C_4 = 8t^4 - 8t^2 + 1, C_5 = 16t^5 - 20t^3 + 5t
    for t in np.linspace(-3, 3, 61):
        assert O.cheb(4, t) == pytest.approx(8 * t**4 - 8 * t**2 + 1, rel=1e-12, abs=1e-12)
        assert O.cheb(5, t) == pytest.approx(16 * t**5 - 20 * t**3 + 5 * t, rel=1e-12, abs=1e-12)


def test_cheb_growth_outside():
    # |C_m(t)| = (|rho|^m + |rho|^-m)/2 outside [-1,1], |rho| = |t| + sqrt(t^2-1)
    for t in (-5.0, -1.5, 1.01, 3.0):
        r = abs(t) + math.sqrt(t * t - 1)
        for m in (1, 7, 20, 40):
            assert abs(O.cheb(m, t)) == pytest.approx((r**m + r**-m) / 2, rel=1e-12)
    # and |C_m| <= 1 inside
    for t in np.linspace(-1, 1, 41):
        for m in (1, 5, 40):
            assert abs(O.cheb(m, t)) <= 1 + 1e-15


def test_sigma_closed_form():
    # App. A claim 1: sigma_i = C_{i-1}(t1)/C_i(t1), t1 = (lambda1-c)/e (Alg 2 l2, l6: P:682)
    for (l1, a, b) in ((-2.3, -1.2, 40.5), (-2.2, -1.0, 2.2), (0.0, 1.0, 3.0)):
        c, e = (a + b) / 2, (b - a) / 2
        s = O.sigma(40, l1, c, e)
        t1 = (l1 - c) / e
        for i in range(1, 41):
            assert s[i - 1] == pytest.approx(O.cheb(i - 1, t1) / O.cheb(i, t1), rel=1e-14)


@pytest.mark.parametrize("g", gold("tau"), ids=lambda g: g["cite"][:12])
def test_convergence_ratio_golden(g):
    c, e = (g["alpha"] + g["beta"]) / 2, (g["beta"] - g["alpha"]) / 2
    r = O.rho((g["lam"] - c) / e)
    assert r == pytest.approx(g["rho"], rel=1e-14)
    assert 1 / r == pytest.approx(g["tau"], rel=1e-14)


# ---- Alg 2 --------------------------------------------------------------------------------
@pytest.mark.parametrize("g", gold("filter_one_step"), ids=lambda g: g["cite"][:12])
def test_filter_one_step_golden(g):
    H = np.diag(np.array(g["diag"], dtype=complex))
    c, e = (g["alpha"] + g["beta"]) / 2, (g["beta"] - g["alpha"]) / 2
    Y, mv = O.chebyshev_filter(H, np.array(g["y"], dtype=complex)[:, None], [g["m"]], g["gamma"], c, e)
    np.testing.assert_allclose(Y[:, 0], np.array(g["out"], dtype=complex), atol=1e-15)
    assert mv == g["m"]


DEGS = [[1], [40], [1, 1, 2, 3, 3, 8], [2, 5, 5, 20, 36, 40], [1, 64], [7] * 5]


@pytest.mark.parametrize("deg", DEGS, ids=str)
def test_filter_diag_closed_form(deg):
    # App. A: column j equals p_{m_j}(H) y_j; J asks <= 1e-13 relative on diagonal H
    rng = np.random.default_rng(len(deg) * 7 + deg[-1])
    n = 97  # ragged
    d = np.sort(rng.uniform(-2.0, 40.0, n))
    Y0 = crand(rng, n, len(deg))
    l1, a, b = -2.3, -1.2, 40.5
    c, e = (a + b) / 2, (b - a) / 2
    Y, mv = O.chebyshev_filter(np.diag(d.astype(complex)), Y0, deg, l1, c, e)
    Yc = O.filter_diag_closed(d, Y0, deg, l1, c, e)
    rel = np.linalg.norm(Y - Yc, axis=0) / np.linalg.norm(Yc, axis=0)
    assert rel.max() <= 1e-13, rel
    assert mv == sum(deg)


def test_filter_literal_line8_rejected():
    """R1: the literal P:688 trailing term sigma_{i+1} sigma_i Y_i (not Y_{i-1}) fails the closed form."""
    rng = np.random.default_rng(3)
    n = 40
    d = np.sort(rng.uniform(-2.0, 40.0, n))
    y0 = crand(rng, n)
    l1, a, b = -2.3, -1.2, 40.5
    c, e = (a + b) / 2, (b - a) / 2
    s = O.sigma(5, l1, c, e)
    Ht = (np.diag(d) - c * np.eye(n)) / e
    y1 = s[0] * Ht @ y0
    y = y1
    for i in range(1, 5):  # literal: Y_{i+1} = 2 s_{i+1} H~ Y_i - s_{i+1} s_i Y_i
        y = 2 * s[i] * Ht @ y - s[i] * s[i - 1] * y
    yc = O.filter_diag_closed(d, y0[:, None], [5], l1, c, e)[:, 0]
    assert np.linalg.norm(y - yc) / np.linalg.norm(yc) > 1.0
    Yo, _ = O.chebyshev_filter(np.diag(d.astype(complex)), y0[:, None], [5], l1, c, e)
    assert np.linalg.norm(Yo[:, 0] - yc) / np.linalg.norm(yc) < 1e-13


@pytest.mark.parametrize("n,deg", [(300, [1, 3, 20, 20]), (512, [8] * 3 + [20, 40])])
def test_filter_wy_closed_form(n, deg):
    # dense H^(1) = Q diag(lam) Q^H: out = Q diag(p_m(lam)) Q^H y (O(n k 8) closed form), J gate 1e-11
    w = G.wy(n, int(0.9 * n), 11 + n)
    H = w.full()
    rng = np.random.default_rng(n)
    Y0 = crand(rng, n, len(deg))
    lmax = 40.0
    l1, a, b = w.lam[0] - 0.1, w.lam[len(deg) + 5], lmax * 1.1
    c, e = (a + b) / 2, (b - a) / 2
    Y, _ = O.chebyshev_filter(H, Y0, deg, l1, c, e)
    Yc = O.filter_wy_closed(w, Y0, deg, l1, c, e)
    rel = np.linalg.norm(Y - Yc, axis=0) / np.linalg.norm(Yc, axis=0)
    assert rel.max() <= 1e-11, rel


def test_filter_product_identity_dense():
    # C_a C_b = (C_{a+b} + C_{|a-b|})/2  =>  2 C_a(t1) C_b(t1) F_a(F_b(Y)) = C_{a+b}(t1) F_{a+b}(Y)
    #                                                                    + C_{|a-b|}(t1) F_{|a-b|}(Y)
    n = 160
    Gm = G.gue(n, 5, G.stream(5, n))
    rng = np.random.default_rng(1)
    Y0 = crand(rng, n, 2)
    l1, a, b = -2.2, -1.0, 2.2
    c, e = (a + b) / 2, (b - a) / 2
    t1 = (l1 - c) / e

    def F(m, Y):
        if m == 0:
            return Y.copy()
        return O.chebyshev_filter(Gm, Y, [m] * Y.shape[1], l1, c, e)[0]

    for (p, q) in ((3, 5), (7, 7), (10, 4)):
        lhs = 2 * O.cheb(p, t1) * O.cheb(q, t1) * F(p, F(q, Y0))
        rhs = O.cheb(p + q, t1) * F(p + q, Y0) + O.cheb(abs(p - q), t1) * F(abs(p - q), Y0)
        assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-12


def test_filter_column_independence_and_masking():
    # Alg 2 l7: a finished column is carried forward unchanged; each column depends only on itself
    n = 64
    Gm = G.gue(n, 9, G.stream(5, n))
    rng = np.random.default_rng(2)
    deg = [1, 2, 2, 5, 9]
    Y0 = crand(rng, n, len(deg))
    l1, c, e = -2.2, 0.6, 1.6
    Y, mv = O.chebyshev_filter(Gm, Y0, deg, l1, c, e)
    assert mv == sum(deg)
    for j, m in enumerate(deg):
        Yj, _ = O.chebyshev_filter(Gm, Y0[:, j : j + 1], [m], l1, c, e)
        assert np.array_equal(Yj[:, 0], Y[:, j])


def test_filter_argument_errors():
    H = np.eye(4, dtype=complex)
    Y = np.ones((4, 2), dtype=complex)
    with pytest.raises(ValueError):
        O.chebyshev_filter(H, Y, [3, 1], -2.0, 0.0, 1.0)  # unsorted
    with pytest.raises(ValueError):
        O.chebyshev_filter(H, Y, [0, 1], -2.0, 0.0, 1.0)  # zero degree
    with pytest.raises(ValueError):
        O.chebyshev_filter(H, Y, [1, 1], -2.0, 0.0, 0.0)  # e <= 0
