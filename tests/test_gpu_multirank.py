"""The nranks > 1 data path on one GPU: P emulated ranks (chfsi_local_group, one host thread and one
stream per rank) run the row-panel filter (packed [rank][k_a][nloc] B operands, in-place allgather,
rank-chunked contraction through a 3-D TMA map), Lanczos, QR and Rayleigh-Ritz, and the full solver.
Each rank's output rows are compared with the single-rank result and with the oracle."""
import threading

import numpy as np
import pytest

import gen as G
import oracle as O
from gen.configs import CONFIGS, HNORM

pytestmark = pytest.mark.gpu


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def run_ranks(chfsi, P, fn, group_cols=None, push=None):
    """Run fn(rank, ctx) for rank = 0..P-1 concurrently (one thread + one stream per rank).
    group_cols: column-group width of the filter's comm/compute pipeline (chfsi_ctx_set_pipeline).
    push: (n, nloc, kmax) -> reserve that workspace and switch to the peer-push exchange (collective,
    inside the rank threads)."""
    import torch

    torch.cuda.synchronize()
    g = chfsi.LocalGroup(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [chfsi.Context(0, stream=streams[r], local_group=g, rank=r) for r in range(P)]
    if group_cols is not None:
        for c in ctxs:
            c.set_pipeline(group_cols)
    out = [None] * P
    errs = []

    def work(r):
        try:
            with torch.cuda.stream(streams[r]):
                if push is not None:
                    ctxs[r].reserve(*push)
                    ctxs[r].set_exchange(1)
                out[r] = fn(r, ctxs[r])
                streams[r].synchronize()
        except Exception as ex:  # pragma: no cover - surfaced below
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    torch.cuda.synchronize()
    for c in ctxs:
        c.close()
    g.close()
    if errs:
        raise errs[0]
    return out


def slabs(chfsi, H, P):
    n = H.shape[0]
    nloc = n // P
    return [chfsi.to_colmajor(np.asfortranarray(H[:, r * nloc:(r + 1) * nloc])) for r in range(P)], nloc


@pytest.mark.parametrize("n,P,group_cols,push", [(512, 2, None, False), (600, 4, None, False), (256, 8, None, False),
                                                  (512, 2, 8, False), (600, 4, 10, False), (256, 8, 0, False),
                                                  (512, 2, None, True), (600, 4, None, True), (256, 8, None, True),
                                                  (1000, 8, None, False), (1000, 8, 8, False), (1000, 8, None, True)])
def test_filter_multirank(gpu_lib, n, P, group_cols, push):
    """group_cols: None = default (one group at k = 37), 8 / 10 = 4 / 3 column groups whose
    allgathers overlap the next group's K1 on a separate stream, 0 = pipelining off. push: the
    filter epilogue stores each rank's rows into every rank's next-step operand (peer pointers).
    n = 1000 over 8 ranks gives odd panels (nloc = 125, like c2's 1625 at p = 8)."""
    k = 37
    w = G.wy(n, int(0.9 * n), n + P)
    H = w.full()
    rng = np.random.default_rng(n * P)
    deg = sorted(rng.integers(1, 21, k).tolist())
    Y0 = crand(rng, n, k)
    l1, a, b = w.lam[0] - 0.05, w.lam[k], 45.0
    c, e = (a + b) / 2, (b - a) / 2
    Hs, nloc = slabs(gpu_lib, H, P)
    Ys = [gpu_lib.to_colmajor(Y0[r * nloc:(r + 1) * nloc]) for r in range(P)]

    def fn(r, ctx):
        return ctx.filter(Hs[r], Ys[r], deg, l1, c, e, n=n, row0=r * nloc)

    mv = run_ranks(gpu_lib, P, fn, group_cols, (n, n // P, k) if push else None)
    assert all(m == sum(deg) for m in mv)
    Y = np.concatenate([y.cpu().numpy() for y in Ys], axis=0)
    ctx1 = gpu_lib.Context(0)
    Y1 = gpu_lib.to_colmajor(Y0)
    ctx1.filter(gpu_lib.to_colmajor(H), Y1, deg, l1, c, e)
    ctx1.close()
    Y1 = Y1.cpu().numpy()
    rel1 = np.linalg.norm(Y - Y1, axis=0) / np.linalg.norm(Y1, axis=0)
    assert rel1.max() <= 1e-13  # same kernel, the contraction regrouped by rank chunk
    Yo, _ = O.chebyshev_filter(H, Y0, deg, l1, c, e)
    assert (np.linalg.norm(Y - Yo, axis=0) / np.linalg.norm(Yo, axis=0)).max() <= 1e-11


def test_lanczos_qr_rr_multirank(gpu_lib):
    n, P, k, nl = 512, 2, 24, 5
    w = G.wy(n, 480, 5)
    H = w.full()
    Hs, nloc = slabs(gpu_lib, H, P)
    rng = np.random.default_rng(1)
    Y = crand(rng, n, k)
    Y[:, :nl] = np.linalg.qr(Y[:, :nl])[0]
    Ys = [gpu_lib.to_colmajor(Y[r * nloc:(r + 1) * nloc]) for r in range(P)]

    def fn(r, ctx):
        lz = ctx.lanczos_bounds(Hs[r], 25, 7, n=n, row0=r * nloc)
        fb = ctx.qr(Ys[r], nlocked=nl, n=n, row0=r * nloc)
        ritz, res = ctx.rayleigh_ritz(Hs[r], Ys[r], normH=HNORM, n=n, row0=r * nloc)
        return lz, fb, ritz, res

    out = run_ranks(gpu_lib, P, fn)
    otmin, otmax, obeta = O.lanczos(H, 25, 7)
    for lz, fb, ritz, res in out:
        assert abs(lz[1] - otmax) <= 1e-10 * 40 and abs(lz[0] - otmin) <= 1e-10 * 40
        assert fb == 0
    assert np.array_equal(out[0][2], out[1][2])  # identical bits on every rank (broadcast eigensolve)
    Q = np.concatenate([y.cpu().numpy() for y in Ys], axis=0)
    assert np.abs(Q.conj().T @ Q - np.eye(k)).max() <= 1e-12
    # reference: CGS2 + Householder on the non-locked part, then Rayleigh-Ritz, in the oracle
    A = Y[:, nl:]
    X = Y[:, :nl]
    for _ in range(2):
        A = A - X @ O.zgemm("C", "N", X, A)
    Qo, _, _ = O.householder_qr(A)
    Qfull = np.concatenate([X, Qo], axis=1)
    ro, _ = O.rayleigh_ritz(H, Qfull)
    np.testing.assert_allclose(out[0][2], ro, rtol=0, atol=1e-12 * HNORM)


def test_householder_fallback_multirank(gpu_lib):
    n, P, k = 300, 3, 9
    rng = np.random.default_rng(10)
    Y = crand(rng, n, k)
    Y[:, 3] = 0
    nloc = n // P
    Ys = [gpu_lib.to_colmajor(Y[r * nloc:(r + 1) * nloc]) for r in range(P)]
    out = run_ranks(gpu_lib, P, lambda r, ctx: ctx.qr(Ys[r], n=n, row0=r * nloc))
    assert out == [1] * P
    Q = np.concatenate([y.cpu().numpy() for y in Ys], axis=0)
    assert np.abs(Q.conj().T @ Q - np.eye(k)).max() <= 1e-13


@pytest.mark.parametrize("P,group_cols,push", [(2, None, False), (4, None, False), (4, 12, False), (4, None, True)])
def test_solve_multirank_c0(gpu_lib, P, group_cols, push):
    cf = CONFIGS["c0"]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    X0 = G.start_basis(n, nev + nex, cf["seed"])
    Hs, nloc = slabs(gpu_lib, H, P)
    Xs = [gpu_lib.to_colmajor(X0[r * nloc:(r + 1) * nloc]) for r in range(P)]

    def fn(r, ctx):
        return ctx.solve_sequence(lambda ell: Hs[r], 1, Xs[r], nev, nex, cf["tol"], deg_cap=cf["cap"],
                                  seed=cf["seed"], n=n, row0=r * nloc)

    out = run_ranks(gpu_lib, P, fn, group_cols, (n, n // P, nev + nex) if push else None)
    for o in out:
        assert o["status"] == 0
        assert np.max(np.abs(o["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10
    X = np.concatenate([x.cpu().numpy() for x in Xs], axis=0)[:, :nev]
    res = np.linalg.norm(H @ X - X * out[0]["lam"][0], axis=0) / HNORM
    assert res.max() <= cf["tol"]


@pytest.mark.parametrize("push", [False, True])
def test_solve_multirank_odd_panels_3m(gpu_lib, push):
    """Complex ChFSI over 2 emulated ranks with odd panels (nloc = 255) and a block wide enough for the
    3M kernel (k = 32): filter, H Q of Rayleigh-Ritz and the 3M plane all on odd rank chunks."""
    n, P, nev, nex = 510, 2, 24, 8
    w = G.wy(n, 470, 21)
    H = w.full()
    X0 = G.start_basis(n, nev + nex, 21)
    Hs, nloc = slabs(gpu_lib, H, P)
    Xs = [gpu_lib.to_colmajor(X0[r * nloc:(r + 1) * nloc]) for r in range(P)]

    def fn(r, ctx):
        return ctx.solve_sequence(lambda ell: Hs[r], 1, Xs[r], nev, nex, 1e-10, deg_cap=20, seed=21, n=n,
                                  row0=r * nloc)

    out = run_ranks(gpu_lib, P, fn, None, (n, nloc, nev + nex) if push else None)
    for o in out:
        assert o["status"] == 0
        assert np.max(np.abs(o["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])) <= 1e-10


@pytest.mark.parametrize("push", [False, True])
def test_filter_multirank_tiny_panels(gpu_lib, push):
    """Panels smaller than one K tile (n = 64 over 8 ranks: nloc = 8 rows, 16 real K per rank chunk) and
    a single column, against the oracle."""
    n, P = 64, 8
    w = G.wy(n, 56, 5)
    H = w.full()
    rng = np.random.default_rng(3)
    for k, deg in ((1, [7]), (30, sorted(rng.integers(1, 12, 30).tolist()))):
        Y0 = crand(rng, n, k)
        l1, a, b = w.lam[0] - 0.05, w.lam[min(k, n - 1)], 45.0
        c, e = (a + b) / 2, (b - a) / 2
        Hs, nloc = slabs(gpu_lib, H, P)
        Ys = [gpu_lib.to_colmajor(Y0[r * nloc:(r + 1) * nloc]) for r in range(P)]
        run_ranks(gpu_lib, P, lambda r, ctx: ctx.filter(Hs[r], Ys[r], deg, l1, c, e, n=n, row0=r * nloc), None,
                  (n, nloc, k) if push else None)
        Y = np.concatenate([y.cpu().numpy() for y in Ys], axis=0)
        Yo, _ = O.chebyshev_filter(H, Y0, deg, l1, c, e)
        assert (np.linalg.norm(Y - Yo, axis=0) / np.linalg.norm(Yo, axis=0)).max() <= 1e-11
