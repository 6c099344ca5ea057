"""Pins of the oracle's generalised front / back end (B = L L^H, H = L^{-1} A L^{-H},
c = L^{-H} y): SPEC worked examples, numpy.linalg.cholesky / scipy-free triangular checks, and a pair
built with a known factor and a known spectrum (gen.generalized_pair)."""
import json
import os

import numpy as np
import pytest

import gen as G
import oracle as O

GOLD = [json.loads(l) for l in open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.jsonl"))]


def gold(what):
    return [g for g in GOLD if g["what"] == what]


@pytest.mark.parametrize("g", gold("cholesky"), ids=lambda g: g["cite"][:11])
def test_cholesky_golden(g):
    L = O.cholesky(np.array(g["b"], dtype=complex))
    np.testing.assert_allclose(L, np.array(g["l"]), atol=1e-15)


@pytest.mark.parametrize("g", gold("reduce"), ids=lambda g: g["cite"][:11])
def test_reduce_golden(g):
    H, L = O.reduce_generalized(np.diag(np.array(g["a"], dtype=complex)), np.diag(np.array(g["b"], dtype=complex)))
    np.testing.assert_allclose(np.diag(H).real, g["h"], atol=1e-15)
    np.testing.assert_allclose(np.diag(L).real, g["l"], atol=1e-15)


@pytest.mark.parametrize("g", gold("back_transform"), ids=lambda g: g["cite"][:11])
def test_back_transform_golden(g):
    c = O.trsm_lower(np.diag(np.array(g["l"], dtype=complex)), np.array(g["y"], dtype=complex)[:, None], adjoint=True)
    np.testing.assert_allclose(c[:, 0], g["c"], atol=1e-15)


def test_cholesky_and_trsm_vs_numpy():
    rng = np.random.default_rng(0)
    n = 60
    X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    B = X @ X.conj().T + n * np.eye(n)
    L = O.cholesky(B)
    np.testing.assert_allclose(L, np.linalg.cholesky(B), atol=1e-12)
    Y = rng.standard_normal((n, 5)) + 1j * rng.standard_normal((n, 5))
    np.testing.assert_allclose(L @ O.trsm_lower(L, Y), Y, atol=1e-11)
    np.testing.assert_allclose(L.conj().T @ O.trsm_lower(L, Y, adjoint=True), Y, atol=1e-11)
    with pytest.raises(ValueError):
        O.cholesky(-np.eye(3, dtype=complex))


def test_reduce_known_factor_and_spectrum():
    n = 240
    w = G.wy(n, 210, 4)
    A, B, M = G.generalized_pair(w, 9)
    H, L = O.reduce_generalized(A, B)
    np.testing.assert_allclose(L, M, atol=1e-13)  # unique Cholesky factor with positive diagonal
    assert np.array_equal(H, H.conj().T)
    np.testing.assert_allclose(np.linalg.eigvalsh(H), w.lam, rtol=0, atol=1e-11 * 40)
    # generalised eigenpairs: c = L^{-H} y with y the eigenvectors of H
    Y = w.eigvecs([0, 1, 2])
    C = O.trsm_lower(L, Y, adjoint=True)
    R = A @ C - (B @ C) * w.lam[:3]
    assert np.linalg.norm(R) / np.linalg.norm(A) <= 1e-12
    assert np.abs(C.conj().T @ B @ C - np.eye(3)).max() <= 1e-12
