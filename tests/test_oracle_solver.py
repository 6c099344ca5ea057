"""Pins of the oracle's ChFSI (Alg 1) on inputs whose answer is known exactly: H^(1) =
Q Lambda Q^H from the generator (converged eigenvalues = Lambda[:nev]), the exact-input fast path
(S:332), completeness via an inertia count, and a short sequence checked against numpy.eigvalsh."""
import numpy as np
import pytest

import gen as G
import oracle as O
from gen.configs import CONFIGS, DEG0


def test_chfsi_c0_exact_spectrum():
    cf = CONFIGS["c0"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    X0 = G.start_basis(n, nev + nex, cf["seed"])
    r = O.chfsi_solve(H, X0, nev, nex, cf["tol"], cf["cap"], seed=cf["seed"])
    assert r["status"] == 0
    lam_ref = w.lam[:nev]
    assert np.max(np.abs(r["lam"] - lam_ref) / np.abs(lam_ref)) <= 1e-10
    X = r["X"][:, :nev]
    # residuals against the exact ||H||_2 = 40 (J: ||HX - X Lambda||/||H|| <= tol)
    res = np.linalg.norm(H @ X - X * r["lam"], axis=0) / 40.0
    assert res.max() <= cf["tol"]
    assert np.abs(X.conj().T @ X - np.eye(nev)).max() <= 1e-12
    # completeness: exactly nev eigenvalues below the midpoint of the nev / nev+1 gap
    sig = 0.5 * (r["lam"][-1] + w.lam[nev])
    assert O.count_below(H, sig) == nev
    rep = r["report"]
    assert rep["converged"] == nev and rep["loops"] >= 1
    assert rep["matvecs_filter"] > 0 and rep["matvecs_total"] >= rep["matvecs_filter"]


def test_chfsi_exact_input_fast_path():
    # exact eigenvectors + exact bounds -> converges in one loop
    n, nev, nex = 256, 12, 4
    w = G.wy(n, 230, 3)
    H = w.full()
    k = nev + nex
    X0 = w.eigvecs(list(range(k)))
    r = O.chfsi_solve(H, X0, nev, nex, 1e-10, 20, seed=1, prev=(w.lam[0], w.lam[k - 1]))
    assert r["status"] == 0
    assert r["report"]["loops"] == 1
    np.testing.assert_allclose(r["lam"], w.lam[:nev], rtol=1e-12)
    assert r["report"]["matvecs_filter"] <= k * DEG0


@pytest.mark.slow
def test_chfsi_short_sequence_vs_numpy():
    # Def 1: problem l's eigenpairs seed problem l+1
    n, nd, nev, nex, delta = 320, 272, 16, 8, 1e-3
    seed = 77
    w = G.wy(n, nd, seed)
    H = w.full()
    X = G.start_basis(n, nev + nex, seed)
    prev = None
    loops = []
    for ell in range(3):
        if ell > 0:
            G.perturb(H, seed, ell, delta * 40.0)
        assert np.array_equal(H, H.conj().T)  # bitwise Hermitian along the sequence
        r = O.chfsi_solve(H, X, nev, nex, 1e-10, 30, seed=seed + ell, prev=prev)
        assert r["status"] == 0
        ev = np.linalg.eigvalsh(H)[:nev]
        assert np.max(np.abs(r["lam"] - ev) / np.abs(ev)) <= 1e-10
        X = r["X"]
        prev = (r["lambda1"], r["lambdak"])
        loops.append(r["report"]["loops"])
    assert loops[1] <= loops[0] and loops[2] <= loops[0]
