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


def _ranks(gpu_lib, P, fn):
    if P == 1:
        ctx = gpu_lib.Context(0)
        try:
            return [fn(0, ctx)]
        finally:
            ctx.close()
    from test_gpu_multirank import run_ranks

    return run_ranks(gpu_lib, P, fn)


@pytest.mark.parametrize("P", [1, 2, 3])
def test_reduce_and_back_transform_panels_vs_oracle(gpu_lib, P):
    """Row-panel front / back end (chfsi_reduce_generalized_panel, chfsi_back_transform_panel) on P
    emulated ranks: the assembled H against the oracle's L^{-1} A L^{-H} and exactly Hermitian across the
    ranks' slabs (R13); L identical on every rank and equal to the oracle's Cholesky factor; B untouched;
    the assembled back-transformed rows against the oracle's L^{-H} Y."""
    n = 300
    nloc = n // P
    w = G.wy(n, 270, 6)
    A, B, M = G.generalized_pair(w, 2)
    Ho, Lo = O.reduce_generalized(A, B)
    rng = np.random.default_rng(1)
    Y = rng.standard_normal((n, 7)) + 1j * rng.standard_normal((n, 7))

    def fn(r, ctx):
        cols = slice(r * nloc, (r + 1) * nloc)
        Ap = gpu_lib.to_colmajor(np.asfortranarray(A[:, cols]))
        Bp = gpu_lib.to_colmajor(np.asfortranarray(B[:, cols]))
        L = gpu_lib.colmajor(n, n)
        ctx.reduce_generalized_panel(Ap, Bp, L, n=n, row0=r * nloc)
        Yr = gpu_lib.to_colmajor(Y[cols])
        ctx.back_transform_panel(L, Yr, n=n, row0=r * nloc)
        return Ap.cpu().numpy(), np.tril(L.cpu().numpy()), Yr.cpu().numpy(), Bp.cpu().numpy()

    out = _ranks(gpu_lib, P, fn)
    H = np.concatenate([o[0] for o in out], axis=1)
    assert np.array_equal(H, H.conj().T)
    np.testing.assert_allclose(H, Ho, atol=1e-12)
    for r, o in enumerate(out):
        assert np.array_equal(o[1], out[0][1])
        assert np.array_equal(o[3], B[:, r * nloc:(r + 1) * nloc])
    np.testing.assert_allclose(out[0][1], Lo, atol=1e-13)
    X = np.concatenate([o[2] for o in out], axis=0)
    np.testing.assert_allclose(X, O.trsm_lower(Lo, Y, adjoint=True), atol=1e-12)


def test_reduce_panels_rejects_indefinite_b_on_every_rank(gpu_lib):
    n, P = 64, 2
    nloc = n // P
    B = -np.eye(n, dtype=complex)

    def fn(r, ctx):
        cols = slice(r * nloc, (r + 1) * nloc)
        try:
            ctx.reduce_generalized_panel(gpu_lib.to_colmajor(np.eye(n, dtype=complex)[:, cols]),
                                         gpu_lib.to_colmajor(B[:, cols]), gpu_lib.colmajor(n, n), n=n, row0=r * nloc)
        except gpu_lib.ChfsiError as ex:
            return str(ex)
        return "ok"

    out = _ranks(gpu_lib, P, fn)
    assert all("ERR_ARG" in s for s in out), out


def test_generalized_solve_multirank(gpu_lib):
    """Generalised problem A c = lambda B c with a known spectrum, solved on 2 emulated ranks end to end:
    panel reduction -> chfsi_solve_sequence on the panels -> panel back-transform; eigenvalues against
    the exact spectrum, generalised residuals and B-orthonormality of the assembled eigenvectors."""
    n, nev, nex, P = 512, 24, 8, 2
    nloc = n // P
    w = G.wy(n, 480, 12)
    A, B, M = G.generalized_pair(w, 3)

    def fn(r, ctx):
        cols = slice(r * nloc, (r + 1) * nloc)
        Ap = gpu_lib.to_colmajor(np.asfortranarray(A[:, cols]))
        Bp = gpu_lib.to_colmajor(np.asfortranarray(B[:, cols]))
        L = gpu_lib.colmajor(n, n)
        ctx.reduce_generalized_panel(Ap, Bp, L, n=n, row0=r * nloc)
        Xd = gpu_lib.to_colmajor(G.start_basis(n, nev + nex, 5, r * nloc, nloc))
        out = ctx.solve_sequence(lambda ell: Ap, 1, Xd, nev, nex, 1e-10, deg_cap=20, seed=5, n=n, row0=r * nloc)
        Cd = Xd[:, :nev].contiguous().t().contiguous().t()
        ctx.back_transform_panel(L, Cd, n=n, row0=r * nloc)
        return out, Cd.cpu().numpy()

    res = _ranks(gpu_lib, P, fn)
    for out, _ in res:
        assert out["status"] == 0
        np.testing.assert_array_equal(out["lam"], res[0][0]["lam"])
    lam = res[0][0]["lam"][0]
    assert np.max(np.abs(lam - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    C = np.concatenate([c for _, c in res], axis=0)
    r = np.linalg.norm(A @ C - (B @ C) * lam, axis=0) / (np.linalg.norm(A, 2) * np.linalg.norm(C, axis=0))
    assert r.max() <= 1e-9
    assert np.abs(C.conj().T @ B @ C - np.eye(nev)).max() <= 1e-10
