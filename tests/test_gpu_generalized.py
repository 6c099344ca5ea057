"""GPU parity of the generalised front / back end (chfsi_reduce_generalized, chfsi_back_transform;
P:541-545) and of a generalised solve (reduce -> chfsi_solve_sequence -> back-transform) on a pair
with a known factor and a known spectrum."""
import numpy as np
import pytest

import gen as G
import oracle as O

pytestmark = pytest.mark.gpu


def test_reduce_and_back_transform_vs_oracle(gpu_lib):
    n = 300
    w = G.wy(n, 270, 6)
    A, B, M = G.generalized_pair(w, 2)
    Ho, Lo = O.reduce_generalized(A, B)
    ctx = gpu_lib.Context(0)
    Ad, Bd = gpu_lib.to_colmajor(A), gpu_lib.to_colmajor(B)
    ctx.reduce_generalized(Ad, Bd)
    H = Ad.cpu().numpy()
    L = np.tril(Bd.cpu().numpy())
    assert np.array_equal(H, H.conj().T)  # exactly Hermitian storage (R13)
    np.testing.assert_allclose(L, Lo, atol=1e-13)
    np.testing.assert_allclose(H, Ho, atol=1e-12)
    rng = np.random.default_rng(1)
    Y = rng.standard_normal((n, 7)) + 1j * rng.standard_normal((n, 7))
    Yd = gpu_lib.to_colmajor(Y)
    ctx.back_transform(Bd, Yd)
    np.testing.assert_allclose(Yd.cpu().numpy(), O.trsm_lower(Lo, Y, adjoint=True), atol=1e-12)
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_ARG"):
        ctx.reduce_generalized(gpu_lib.to_colmajor(np.eye(4)), gpu_lib.to_colmajor(-np.eye(4)))
    ctx.close()


def test_generalized_solve(gpu_lib):
    n, nev, nex = 512, 24, 8
    w = G.wy(n, 480, 12)
    A, B, M = G.generalized_pair(w, 3)
    ctx = gpu_lib.Context(0)
    Ad, Bd = gpu_lib.to_colmajor(A), gpu_lib.to_colmajor(B)
    ctx.reduce_generalized(Ad, Bd)
    Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + nex, 5))
    out = ctx.solve_sequence(lambda ell: Ad, 1, Xd, nev, nex, 1e-10, deg_cap=20, seed=5)
    assert out["status"] == 0
    lam = out["lam"][0]
    assert np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    Cd = Xd[:, :nev].contiguous().t().contiguous().t()
    ctx.back_transform(Bd, Cd)
    C = Cd.cpu().numpy()
    ctx.close()
    # generalised residual and B-orthonormality
    res = np.linalg.norm(A @ C - (B @ C) * lam, axis=0) / (np.linalg.norm(A, 2) * np.linalg.norm(C, axis=0))
    assert res.max() <= 1e-9
    assert np.abs(C.conj().T @ B @ C - np.eye(nev)).max() <= 1e-10
