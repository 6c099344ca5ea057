"""GPU parity of chfsi_filter (K1 through the C-ABI) against the oracle (Alg 2, naive C) and against
the closed forms of App. A. Tolerances from BASELINE.json: filter <= 1e-11 relative per column (error
budget sqrt(n) eps per step x <= 40 steps), diagonal closed form <= 1e-13."""
import os

import numpy as np
import pytest

import gen as G
import oracle as O
from gen.configs import C4_INTERVAL, CONFIGS, c4_ramp

pytestmark = pytest.mark.gpu
# every built K1 variant the step model can select: 3M (the default complex arithmetic, ids >= 200) and
# 4M real embedding (ids < 100); the A/B-only variants are compiled with -DCHFSI_K1_AB only
VARIANTS = ["200", "207", "208", "1", "3", "5", "6", "7", "9", "10", "11", "12", "13", "14"]


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.fixture
def ctx(gpu_lib):
    c = gpu_lib.Context(0)
    yield c
    c.close()


@pytest.fixture(params=VARIANTS)
def variant(request, ctx):
    z3 = int(request.param) >= 200
    env = "CHFSI_FILTER_VARIANT_Z3" if z3 else "CHFSI_FILTER_VARIANT"
    ctx.set_complex_mult(3 if z3 else 4)
    os.environ[env] = request.param
    yield request.param
    os.environ.pop(env, None)


def run_filter(chfsi, ctx, H, Y0, deg, l1, c, e):
    Hd = chfsi.to_colmajor(H)
    Yd = chfsi.to_colmajor(Y0)
    mv = ctx.filter(Hd, Yd, deg, l1, c, e)
    assert mv == sum(deg)
    return Yd.cpu().numpy()


def colrel(A, B):
    return np.linalg.norm(A - B, axis=0) / np.linalg.norm(B, axis=0)


def test_filter_diag_closed_form(gpu_lib, ctx, variant):
    rng = np.random.default_rng(1)
    n = 203  # ragged in every tile dimension
    d = np.sort(rng.uniform(-2.0, 40.0, n))
    deg = sorted(rng.integers(1, 41, 37).tolist())
    Y0 = crand(rng, n, len(deg))
    l1, a, b = -2.3, -1.2, 40.5
    c, e = (a + b) / 2, (b - a) / 2
    Y = run_filter(gpu_lib, ctx, np.diag(d.astype(complex)), Y0, deg, l1, c, e)
    Yc = O.filter_diag_closed(d, Y0, deg, l1, c, e)
    assert colrel(Y, Yc).max() <= 1e-13


@pytest.mark.parametrize("n,k", [(512, 48), (300, 37), (129, 5)])
def test_filter_dense_vs_oracle(gpu_lib, ctx, variant, n, k):
    w = G.wy(n, int(0.9 * n), n + k)
    H = w.full()
    rng = np.random.default_rng(n * k)
    deg = sorted(rng.integers(1, 21, k).tolist())
    Y0 = crand(rng, n, k)
    l1, a, b = w.lam[0] - 0.05, w.lam[k], 45.0
    c, e = (a + b) / 2, (b - a) / 2
    Y = run_filter(gpu_lib, ctx, H, Y0, deg, l1, c, e)
    Yo, _ = O.chebyshev_filter(H, Y0, deg, l1, c, e)
    assert colrel(Y, Yo).max() <= 1e-11
    Yc = O.filter_wy_closed(w, Y0, deg, l1, c, e)
    assert colrel(Y, Yc).max() <= 1e-11


@pytest.mark.parametrize("forced", ["13", None])
def test_filter_column_independence(gpu_lib, ctx, forced):
    """A column filtered alone equals the same column filtered inside a block (Alg 2 treats columns
    independently; the degree masking never mixes them). Bitwise when both calls run the same tile
    variant and hence the same contraction order (forced variant 13: one N tile for k <= 8, so the
    persistent / stream-K schedule is identical); to rounding when the chooser picks different variants
    for the block and the single column (a different stream-K split re-associates the k sum)."""
    n = 257
    Gm = G.gue(n, 3, G.stream(5, n))
    rng = np.random.default_rng(4)
    deg = [1, 2, 2, 6, 9, 9, 13]
    Y0 = crand(rng, n, len(deg))
    iv = C4_INTERVAL
    c, e = (iv["alpha"] + iv["beta"]) / 2, (iv["beta"] - iv["alpha"]) / 2
    if forced:
        ctx.set_complex_mult(4)
        os.environ["CHFSI_FILTER_VARIANT"] = forced
    try:
        Y = run_filter(gpu_lib, ctx, Gm, Y0, deg, iv["lambda1"], c, e)
        for j in (0, 3, 6):
            Yj = run_filter(gpu_lib, ctx, Gm, Y0[:, j:j + 1], [deg[j]], iv["lambda1"], c, e)
            if forced:
                assert np.array_equal(Yj[:, 0], Y[:, j])
            else:
                assert colrel(Yj, Y[:, j:j + 1]).max() <= 1e-14
    finally:
        os.environ.pop("CHFSI_FILTER_VARIANT", None)


def test_filter_ld_and_panel_views(gpu_lib, ctx):
    # ld > rows for Y and H (sub-views of larger allocations)
    import torch

    n, k = 130, 9
    w = G.wy(n, 100, 2)
    H = w.full()
    rng = np.random.default_rng(2)
    Y0 = crand(rng, n, k)
    deg = [3] * 4 + [7] * 5
    l1, a, b = w.lam[0] - 0.1, w.lam[20], 44.0
    c, e = (a + b) / 2, (b - a) / 2
    Hbig = gpu_lib.colmajor(n + 6, n + 3)
    Hbig[:n, :n].copy_(torch.as_tensor(H))
    Ybig = gpu_lib.colmajor(n + 10, k)
    Ybig.fill_(complex(1234.5, -6789.25))  # guard band: rows n..n+9 of every column must stay untouched
    Ybig[:n].copy_(torch.as_tensor(Y0))
    Hguard = Hbig.clone()
    ctx.filter(Hbig[:n, :n], Ybig[:n], deg, l1, c, e)
    Yo, _ = O.chebyshev_filter(H, Y0, deg, l1, c, e)
    assert colrel(Ybig[:n].cpu().numpy(), Yo).max() <= 1e-11
    assert bool((Ybig[n:] == complex(1234.5, -6789.25)).all())  # no write outside the caller's view
    assert torch.equal(Hbig, Hguard)  # H is read-only


def test_filter_errors(gpu_lib, ctx):
    n = 16
    H = gpu_lib.to_colmajor(np.eye(n))
    Y = gpu_lib.to_colmajor(np.ones((n, 2)))
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_ARG"):
        ctx.filter(H, Y, [3, 1], -2.0, 0.0, 1.0)
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_ARG"):
        ctx.filter(H, Y, [1, 1], -2.0, 0.0, 0.0)
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_ARG"):
        ctx.filter(H, Y, [1, 1], 0.5, 0.0, 1.0)  # lambda1 inside [alpha, beta]
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_ARG"):
        ctx.filter(H, Y, [1, 65], -2.0, 0.0, 1.0)  # degree > CHFSI_MAX_DEGREE
    Y2 = gpu_lib.to_colmajor(np.full((n, 2), np.nan))
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_NONFINITE"):
        ctx.filter(H, Y2, [1, 2], -2.0, 0.0, 1.0)
    assert ctx.filter(H, gpu_lib.colmajor(n, 0), [], -2.0, 0.0, 1.0) == 0  # empty block


def test_filter_c1_shape_sampled(gpu_lib, ctx):
    # c1 shape (n = 4096, k = 240) with the c4 ramp degrees 8..40; oracle on a column sample
    n, k = 4096, 240
    Gm = G.gue(n, 7, G.stream(5, n))
    Y0 = G.start_basis(n, k, 7)
    deg = c4_ramp(k)
    iv = C4_INTERVAL
    c, e = (iv["alpha"] + iv["beta"]) / 2, (iv["beta"] - iv["alpha"]) / 2
    Y = run_filter(gpu_lib, ctx, Gm, Y0, deg, iv["lambda1"], c, e)
    cols = [0, 1, 119, 238, 239]
    Yo, _ = O.chebyshev_filter(Gm, Y0[:, cols], [deg[j] for j in cols], iv["lambda1"], c, e)
    assert colrel(Y[:, cols], Yo).max() <= 1e-11


@pytest.mark.parametrize("n,k", [(1000, 64), (515, 21)])
def test_filter_3m_matches_4m_and_oracle(gpu_lib, n, k):
    """Gauss 3M (default) and the 4M real embedding compute the same Alg 2 result: both within the
    filter tolerance of the oracle, and within a few ulps (normwise) of each other."""
    Gm = G.gue(n, 11, G.stream(5, n))
    rng = np.random.default_rng(n + k)
    Y0 = crand(rng, n, k)
    deg = sorted(rng.integers(1, 31, k).tolist())
    iv = C4_INTERVAL
    c, e = (iv["alpha"] + iv["beta"]) / 2, (iv["beta"] - iv["alpha"]) / 2
    out = {}
    for mults in (3, 4):
        cx = gpu_lib.Context(0)
        cx.set_complex_mult(mults)
        out[mults] = run_filter(gpu_lib, cx, Gm, Y0, deg, iv["lambda1"], c, e)
        cx.close()
    assert colrel(out[3], out[4]).max() <= 1e-12
    cols = [0, k // 2, k - 1]
    Yo, _ = O.chebyshev_filter(Gm, Y0[:, cols], [deg[j] for j in cols], iv["lambda1"], c, e)
    for mults in (3, 4):
        assert colrel(out[mults][:, cols], Yo).max() <= 1e-11


def test_filter_rejects_partial_panel_on_one_rank(gpu_lib, ctx):
    """nranks == 1 owns every row: a panel with nloc < n or row0 != 0 is CHFSI_ERR_ARG (the B operand of
    a single rank is its own state, so a partial panel would read rows it does not hold)."""
    n = 64
    H = gpu_lib.to_colmajor(np.eye(n))
    Y = gpu_lib.to_colmajor(np.ones((n // 2, 2)))
    with pytest.raises(gpu_lib.ChfsiError, match="ERR_ARG"):
        ctx.filter(H[:, : n // 2], Y, [1, 1], -2.0, 0.0, 1.0, n=n, row0=0)


@pytest.mark.parametrize("deg_kind", ["all_one", "all_max", "one_and_max"])
def test_filter_degree_extremes(gpu_lib, ctx, deg_kind):
    """Degree edge cases of Alg 2: every column finishing at step 1 (only the a3 step, no recurrence),
    every column at CHFSI_MAX_DEGREE = 64, and both in one block (a 1-step column next to 63 more steps of
    a 64-step one) -- against the closed form on a diagonal H (App. A, <= 1e-13)."""
    rng = np.random.default_rng(11)
    n, k = 173, 11
    d = np.sort(rng.uniform(-2.0, 40.0, n))
    deg = {"all_one": [1] * k, "all_max": [64] * k, "one_and_max": [1] * 5 + [64] * 6}[deg_kind]
    Y0 = crand(rng, n, k)
    l1, a, b = -2.3, -1.2, 40.5
    c, e = (a + b) / 2, (b - a) / 2
    Y = run_filter(gpu_lib, ctx, np.diag(d.astype(complex)), Y0, deg, l1, c, e)
    Yc = O.filter_diag_closed(d, Y0, deg, l1, c, e)
    assert colrel(Y, Yc).max() <= 1e-13


@pytest.mark.parametrize("env,vid,mults", [("CHFSI_FILTER_VARIANT_Z3", "200", 3), ("CHFSI_FILTER_VARIANT", "7", 4),
                                           ("CHFSI_FILTER_VARIANT_Z3", "207", 3)])
def test_filter_stream_k_hybrid_schedule(gpu_lib, ctx, env, vid, mults):
    """Persistent schedule with a small stream-K remainder: n = 2000, k = 480 under a 128 x 48 tile is
    16 x 10 = 160 tiles on 148 CTAs (remainder 12 < 148 / 2). The default schedule folds one
    data-parallel wave into the stream-K tail (12 + 148 tail tiles, at most two contributors each);
    CHFSI_SK_HYBRID=0 keeps the plain split (12 tail tiles over all 148 CTAs). Both within the filter
    tolerance of the compact-WY closed form (App. A) and of each other (they only re-associate the k sum).
    z207 (64 x 64 tiles: 32 x 8 = 256 tiles, remainder 108) keeps the plain split."""
    n, k = 2000, 480
    w = G.wy(n, int(0.9 * n), 31)
    H = w.full()
    rng = np.random.default_rng(31)
    deg = sorted(rng.integers(2, 9, k).tolist())
    Y0 = crand(rng, n, k)
    l1, a, b = w.lam[0] - 0.05, w.lam[k], 45.0
    c, e = (a + b) / 2, (b - a) / 2
    ctx.set_complex_mult(mults)
    out = {}
    os.environ[env] = vid
    try:
        for hy in ("1", "0"):
            os.environ["CHFSI_SK_HYBRID"] = hy
            out[hy] = run_filter(gpu_lib, ctx, H, Y0, deg, l1, c, e)
    finally:
        os.environ.pop(env, None)
        os.environ.pop("CHFSI_SK_HYBRID", None)
    Yc = O.filter_wy_closed(w, Y0, deg, l1, c, e)
    for hy in ("1", "0"):
        assert colrel(out[hy], Yc).max() <= 1e-11
    assert colrel(out["1"], out["0"]).max() <= 1e-13


@pytest.mark.parametrize("vid", ["200", "207", "7", "1"])
def test_filter_every_last_unit_residue(gpu_lib, ctx, vid):
    """The kernel skips the MMA tiles of the inactive half of the block's last column unit (WNC = 16
    columns: z200 / z207 skip 8 of 16, 4M v7 / v1 skip 8 of 16 complex columns). Every residue of the
    active width modulo the unit -- all steps at the same width (one degree for every column), and a
    width over several N tiles -- against the diagonal closed form."""
    z3 = int(vid) >= 200
    env = "CHFSI_FILTER_VARIANT_Z3" if z3 else "CHFSI_FILTER_VARIANT"
    ctx.set_complex_mult(3 if z3 else 4)
    os.environ[env] = vid
    try:
        rng = np.random.default_rng(int(vid))
        n = 1100
        d = np.sort(rng.uniform(-2.0, 40.0, n))
        Hd = gpu_lib.to_colmajor(np.diag(d.astype(complex)))
        l1, a, b = -2.3, -1.2, 40.5
        c, e = (a + b) / 2, (b - a) / 2
        for k in list(range(33, 49)) + [100, 105, 153]:
            Y0 = crand(rng, n, k)
            deg = [3] * k
            Yd = gpu_lib.to_colmajor(Y0)
            assert ctx.filter(Hd, Yd, deg, l1, c, e) == 3 * k
            Yc = O.filter_diag_closed(d, Y0, deg, l1, c, e)
            assert colrel(Yd.cpu().numpy(), Yc).max() <= 1e-13, k
    finally:
        os.environ.pop(env, None)


@pytest.mark.parametrize("n,k", [(300, 37), (517, 100)])
def test_filter_guard_bands_every_variant(gpu_lib, ctx, variant, n, k):
    """Out-of-bounds write check without a sanitizer (compute-sanitizer is unavailable on the GPU pool):
    Y is a view of a larger allocation with guard rows below every column and guard columns after the
    block, H a view with guard rows and columns; after a filter call with ragged tiles in M, N and K,
    every guard value is bit-identical and H is unchanged, for every tile variant."""
    import torch

    w = G.wy(n, int(0.9 * n), n + k)
    H = w.full()
    rng = np.random.default_rng(n + k)
    Y0 = crand(rng, n, k)
    deg = sorted(rng.integers(1, 16, k).tolist())
    l1, a, b = w.lam[0] - 0.05, w.lam[k], 45.0
    c, e = (a + b) / 2, (b - a) / 2
    sentinel = complex(1234.5, -6789.25)
    Hbig = gpu_lib.colmajor(n + 9, n + 5)
    Hbig.fill_(sentinel)
    Hbig[:n, :n].copy_(torch.as_tensor(H))
    Hguard = Hbig.clone()
    Ybig = gpu_lib.colmajor(n + 13, k + 3)
    Ybig.fill_(sentinel)
    Ybig[:n, :k].copy_(torch.as_tensor(Y0))
    ctx.filter(Hbig[:n, :n], Ybig[:n, :k], deg, l1, c, e)
    assert bool((Ybig[n:, :] == sentinel).all())      # guard rows of every column
    assert bool((Ybig[:, k:] == sentinel).all())      # guard columns after the block
    assert torch.equal(Hbig, Hguard)                  # H (and its guards) read-only
    Yo, _ = O.chebyshev_filter(H, Y0, deg, l1, c, e)
    assert colrel(Ybig[:n, :k].cpu().numpy(), Yo).max() <= 1e-11
