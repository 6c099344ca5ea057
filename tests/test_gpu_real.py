"""NEXT-3: the real-symmetric filter (chfsi_filter_real) against the oracle (Alg 2 in complex
arithmetic on real data computes the real recurrence exactly: every imaginary part is 0) and against
the diagonal closed form; all real tile variants, ragged shapes, and the emulated multi-rank path."""
import os

import numpy as np
import pytest

import gen as G
import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["104", "132", "133", "135"])
def rvariant(request):
    os.environ["CHFSI_FILTER_VARIANT_REAL"] = request.param
    yield request.param
    os.environ.pop("CHFSI_FILTER_VARIANT_REAL", None)


def real_sym(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n)) / np.sqrt(2 * n)
    return np.asfortranarray(A + A.T)  # spectrum ~ [-2, 2]


@pytest.mark.parametrize("n,k", [(300, 37), (517, 100), (129, 5)])
def test_filter_real_vs_oracle(gpu_lib, rvariant, n, k):
    H = real_sym(n, n)
    rng = np.random.default_rng(k)
    deg = sorted(rng.integers(1, 25, k).tolist())
    Y0 = np.asfortranarray(rng.standard_normal((n, k)))
    l1, a, b = -2.3, -1.0, 2.3
    c, e = (a + b) / 2, (b - a) / 2
    ctx = gpu_lib.Context(0)
    Yd = gpu_lib.to_colmajor(Y0, real=True)
    assert ctx.filter_real(gpu_lib.to_colmajor(H, real=True), Yd, deg, l1, c, e) == sum(deg)
    Y = Yd.cpu().numpy()
    ctx.close()
    Yo, _ = O.chebyshev_filter(H.astype(complex), Y0.astype(complex), deg, l1, c, e)
    assert np.abs(Yo.imag).max() == 0.0
    rel = np.linalg.norm(Y - Yo.real, axis=0) / np.linalg.norm(Yo.real, axis=0)
    assert rel.max() <= 1e-11


def test_filter_real_diag_closed_form(gpu_lib):
    rng = np.random.default_rng(3)
    n = 211
    d = np.sort(rng.uniform(-2.0, 40.0, n))
    deg = sorted(rng.integers(1, 41, 29).tolist())
    Y0 = rng.standard_normal((n, 29))
    l1, a, b = -2.3, -1.2, 40.5
    c, e = (a + b) / 2, (b - a) / 2
    ctx = gpu_lib.Context(0)
    Yd = gpu_lib.to_colmajor(Y0, real=True)
    ctx.filter_real(gpu_lib.to_colmajor(np.diag(d), real=True), Yd, deg, l1, c, e)
    Y = Yd.cpu().numpy()
    ctx.close()
    Yc = O.filter_diag_closed(d, Y0.astype(complex), deg, l1, c, e).real
    assert (np.linalg.norm(Y - Yc, axis=0) / np.linalg.norm(Yc, axis=0)).max() <= 1e-13


@pytest.mark.parametrize("n,P", [(640, 4), (1000, 8), (1002, 2)])
def test_filter_real_multirank(gpu_lib, n, P):
    """Emulated ranks; (1000, 8) and (1002, 2) have odd panels (nloc = 125, 501): the real A operand's
    rank chunks then start on odd doubles (the library re-strides the panel)."""
    import threading

    import torch

    k = 21
    H = real_sym(n, 11)
    rng = np.random.default_rng(5)
    deg = sorted(rng.integers(1, 15, k).tolist())
    Y0 = rng.standard_normal((n, k))
    l1, c, e = -2.3, 0.65, 1.65
    nloc = n // P
    g = gpu_lib.LocalGroup(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [gpu_lib.Context(0, stream=streams[r], local_group=g, rank=r) for r in range(P)]
    Hs = [gpu_lib.to_colmajor(np.asfortranarray(H[:, r * nloc:(r + 1) * nloc]), real=True) for r in range(P)]
    Ys = [gpu_lib.to_colmajor(Y0[r * nloc:(r + 1) * nloc], real=True) for r in range(P)]
    torch.cuda.synchronize()
    errs = []

    def work(r):
        try:
            with torch.cuda.stream(streams[r]):
                ctxs[r].filter_real(Hs[r], Ys[r], deg, l1, c, e, n=n, row0=r * nloc)
                streams[r].synchronize()
        except Exception as ex:
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    torch.cuda.synchronize()
    [cx.close() for cx in ctxs]
    g.close()
    assert not errs, errs
    Y = np.concatenate([y.cpu().numpy() for y in Ys], axis=0)
    Yo, _ = O.chebyshev_filter(H.astype(complex), Y0.astype(complex), deg, l1, c, e)
    assert (np.linalg.norm(Y - Yo.real, axis=0) / np.linalg.norm(Yo.real, axis=0)).max() <= 1e-11


def real_known(n, nd, seed):
    """Real symmetric H = Q diag(lam) Q^T, Q a product of 8 real Householder reflectors (numpy)."""
    import gen as G

    lam = G.spectrum(n, nd)
    rng = np.random.default_rng(seed)
    Q = np.eye(n)
    for _ in range(8):
        v = rng.standard_normal((n, 1))
        Q = Q - 2.0 * (Q @ v) @ v.T / (v.T @ v).item()
    H = Q @ np.diag(lam) @ Q.T
    return np.asfortranarray((H + H.T) / 2), lam


def test_solve_real_known_spectrum_and_vs_oracle(gpu_lib):
    n, nd, nev, nex = 512, 480, 32, 16
    H, lam = real_known(n, nd, 4)
    X0 = np.asfortranarray(np.random.default_rng(1).standard_normal((n, nev + nex)))
    ctx = gpu_lib.Context(0)
    Hd = gpu_lib.to_colmajor(H, real=True)
    Xd = gpu_lib.to_colmajor(X0, real=True)
    out = ctx.solve_sequence(lambda ell: Hd, 1, Xd, nev, nex, 1e-10, deg_cap=20, seed=3, real=True)
    X = Xd.cpu().numpy()[:, :nev]
    ctx.close()
    assert out["status"] == 0
    got = out["lam"][0]
    assert np.max(np.abs(got - lam[:nev]) / np.abs(lam[:nev])) <= 1e-10
    res = np.linalg.norm(H @ X - X * got, axis=0) / 40.0
    assert res.max() <= 1e-10
    assert np.abs(X.T @ X - np.eye(nev)).max() <= 1e-12
    ro = O.chfsi_solve(H.astype(complex), X0.astype(complex), nev, nex, 1e-10, 20, seed=3)
    assert np.max(np.abs(got - ro["lam"]) / np.abs(ro["lam"])) <= 1e-10
    assert out["reports"][0]["filter_flops"] == pytest.approx(2.0 * n * n * out["reports"][0]["matvecs_filter"])


def test_solve_real_multirank_odd_panels(gpu_lib):
    """Real-symmetric ChFSI over 2 emulated ranks with odd panels (nloc = 255): every step of the path
    (Lanczos, filter on the re-strided A operand, QR, Rayleigh-Ritz) on row panels, against the known
    spectrum of H = Q diag(lambda) Q^T."""
    import threading

    import torch

    n, P, nev, nex = 510, 2, 16, 8
    H, lam = real_known(n, 470, 9)
    X0 = np.asfortranarray(np.random.default_rng(2).standard_normal((n, nev + nex)))
    nloc = n // P
    g = gpu_lib.LocalGroup(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [gpu_lib.Context(0, stream=streams[r], local_group=g, rank=r) for r in range(P)]
    Hs = [gpu_lib.to_colmajor(np.asfortranarray(H[:, r * nloc:(r + 1) * nloc]), real=True) for r in range(P)]
    Xs = [gpu_lib.to_colmajor(np.asfortranarray(X0[r * nloc:(r + 1) * nloc]), real=True) for r in range(P)]
    torch.cuda.synchronize()
    outs, errs = [None] * P, []

    def work(r):
        try:
            with torch.cuda.stream(streams[r]):
                outs[r] = ctxs[r].solve_sequence(lambda ell: Hs[r], 1, Xs[r], nev, nex, 1e-10, deg_cap=20, seed=3,
                                                 real=True, n=n, row0=r * nloc)
                streams[r].synchronize()
        except Exception as ex:
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    torch.cuda.synchronize()
    [cx.close() for cx in ctxs]
    g.close()
    assert not errs, errs
    for o in outs:
        assert o["status"] == 0
        assert np.max(np.abs(o["lam"][0] - lam[:nev]) / np.abs(lam[:nev])) <= 1e-10


def test_filter_real_every_last_unit_residue(gpu_lib, rvariant):
    """Real tiles skip the MMA tiles of the inactive half of the last column unit (WNC 16 or 32 real
    columns): every residue of the active width modulo 16 / 32 at one degree, against the closed form."""
    rng = np.random.default_rng(int(rvariant))
    n = 777
    d = np.sort(rng.uniform(-2.0, 40.0, n))
    l1, a, b = -2.3, -1.2, 40.5
    c, e = (a + b) / 2, (b - a) / 2
    ctx = gpu_lib.Context(0)
    Hd = gpu_lib.to_colmajor(np.diag(d), real=True)
    for k in list(range(65, 97)) + [150]:
        Y0 = rng.standard_normal((n, k))
        Yd = gpu_lib.to_colmajor(Y0, real=True)
        ctx.filter_real(Hd, Yd, [4] * k, l1, c, e)
        Yc = O.filter_diag_closed(d, Y0.astype(complex), [4] * k, l1, c, e).real
        rel = np.linalg.norm(Yd.cpu().numpy() - Yc, axis=0) / np.linalg.norm(Yc, axis=0)
        assert rel.max() <= 1e-13, k
    ctx.close()
