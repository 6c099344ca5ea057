"""Python binding of libchfsi.so -- the B200-native ChFSI library (arXiv:1404.4161).

Argument marshalling only: every step runs in the library's CUDA kernels (or cuBLAS / cuSOLVER /
NCCL calls it makes). PyTorch supplies device memory, streams and the NCCL communicator. There is no
CPU fallback: importing this module on a machine without the built library raises, and creating a
context without a B200 raises.

Matrices are column-major complex128: pass (rows x cols) torch tensors with stride (1, ld), e.g. from
`colmajor(rows, cols)` or `t.t().contiguous().t()` -- the same memory layout as the C-ABI
(include/chfsi.h).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CHFSI_LIB: another build of the same library (A/B measurements of two builds in one session)
LIB_PATH = os.environ.get("CHFSI_LIB") or os.path.join(_HERE, "libchfsi.so")
MAX_DEGREE = 64

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_NONFINITE", 3: "ERR_NOCONV", 4: "ERR_QR", 5: "ERR_CUDA", 6: "ERR_NCCL",
          7: "ERR_NOMEM"}

EXPORTS = ("chfsi_ctx_create", "chfsi_ctx_create_local", "chfsi_ctx_create_nccl", "chfsi_nccl_unique_id", "chfsi_ctx_reserve", "chfsi_ctx_destroy",
           "chfsi_last_error", "chfsi_kernel_launches", "chfsi_ctx_set_pipeline", "chfsi_ctx_set_complex_mult", "chfsi_ctx_set_eigensolver", "chfsi_ctx_set_exchange", "chfsi_local_group_create", "chfsi_local_group_destroy",
           "chfsi_filter", "chfsi_filter_real", "chfsi_lanczos_bounds", "chfsi_qr", "chfsi_qr_ex", "chfsi_rayleigh_ritz", "chfsi_solve_sequence",
           "chfsi_reduce_generalized", "chfsi_back_transform", "chfsi_reduce_generalized_panel", "chfsi_back_transform_panel",
           "chfsi_solve_batch", "chfsi_solve_sequence_real")


class ChfsiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Opts(ctypes.Structure):
    _fields_ = [("nev", ctypes.c_int32), ("nex", ctypes.c_int32), ("deg0", ctypes.c_int32),
                ("deg_cap", ctypes.c_int32), ("max_loops", ctypes.c_int32), ("lanczos_steps", ctypes.c_int32),
                ("tol", ctypes.c_double), ("seed", ctypes.c_uint64), ("random_start", ctypes.c_int32),
                ("no_reuse", ctypes.c_int32), ("fixed_degree", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("loops", ctypes.c_int32), ("qr_fallbacks", ctypes.c_int32), ("capped", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("matvecs_filter", ctypes.c_int64), ("matvecs_total", ctypes.c_int64),
                ("filter_flops", ctypes.c_double), ("t_lanczos", ctypes.c_double), ("t_filter", ctypes.c_double),
                ("t_qr", ctypes.c_double), ("t_rr", ctypes.c_double), ("t_resid", ctypes.c_double),
                ("t_opt", ctypes.c_double), ("t_total", ctypes.c_double), ("theta_min", ctypes.c_double),
                ("theta_max", ctypes.c_double), ("beta_up", ctypes.c_double), ("normH", ctypes.c_double),
                ("t_filter_kernel", ctypes.c_double), ("filter_launches", ctypes.c_int64),
                ("qr_replaced", ctypes.c_int32), ("reseeded", ctypes.c_int32), ("eig_refined", ctypes.c_int32),
                ("eig_dense", ctypes.c_int32), ("t_eig", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Sequence(ctypes.Structure):
    pass


GET_H = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p),
                         ctypes.POINTER(ctypes.c_int64))

Sequence._fields_ = [("nprob", ctypes.c_int32), ("get_h", GET_H), ("user", ctypes.c_void_p), ("X", ctypes.c_void_p),
                     ("ldx", ctypes.c_int64), ("lambda_", ctypes.POINTER(ctypes.c_double)),
                     ("resid", ctypes.POINTER(ctypes.c_double)), ("reports", ctypes.POINTER(Report)),
                     ("status", ctypes.c_int)]

_lib = None


def lib():
    """Load libchfsi.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: build it with `make` or __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        i64, u64, i32, dbl, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        pd, pi64, pi32 = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)
        L.chfsi_ctx_create.argtypes = [ctypes.POINTER(vp), i32, vp, vp, i32, i32]
        L.chfsi_ctx_create_local.argtypes = [ctypes.POINTER(vp), i32, vp, vp, i32]
        L.chfsi_ctx_create_nccl.argtypes = [ctypes.POINTER(vp), i32, vp, ctypes.c_char_p, i32, i32]
        L.chfsi_ctx_create_nccl.restype = ctypes.c_int
        L.chfsi_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.chfsi_nccl_unique_id.restype = ctypes.c_int
        L.chfsi_local_group_create.argtypes = [ctypes.POINTER(vp), i32]
        L.chfsi_local_group_destroy.argtypes = [vp]
        L.chfsi_local_group_destroy.restype = None
        L.chfsi_ctx_reserve.argtypes = [vp, i64, i64, i64]
        L.chfsi_ctx_destroy.argtypes = [vp]
        L.chfsi_ctx_destroy.restype = None
        L.chfsi_last_error.argtypes = [vp]
        L.chfsi_last_error.restype = ctypes.c_char_p
        L.chfsi_kernel_launches.argtypes = [vp]
        L.chfsi_kernel_launches.restype = i64
        L.chfsi_ctx_set_pipeline.argtypes = [vp, i32, i32]
        L.chfsi_ctx_set_pipeline.restype = ctypes.c_int
        L.chfsi_ctx_set_complex_mult.argtypes = [vp, i32]
        L.chfsi_ctx_set_complex_mult.restype = ctypes.c_int
        L.chfsi_ctx_set_exchange.argtypes = [vp, i32]
        L.chfsi_ctx_set_eigensolver.argtypes = [vp, i32]
        L.chfsi_ctx_set_eigensolver.restype = ctypes.c_int
        L.chfsi_ctx_set_exchange.restype = ctypes.c_int
        L.chfsi_filter.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, i64, pi32, dbl, dbl, dbl, pi64]
        L.chfsi_filter_real.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, i64, pi32, dbl, dbl, dbl, pi64]
        L.chfsi_filter_real.restype = ctypes.c_int
        L.chfsi_lanczos_bounds.argtypes = [vp, i64, i64, i64, vp, i64, i32, u64, pd, pd, pd]
        L.chfsi_qr.argtypes = [vp, i64, i64, i64, vp, i64, i64, i64, pi32]
        L.chfsi_qr_ex.argtypes = [vp, i64, i64, i64, vp, i64, i64, i64, u64, pi32, pi32]
        L.chfsi_qr_ex.restype = ctypes.c_int
        L.chfsi_rayleigh_ritz.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, i64, dbl, pd, pd]
        L.chfsi_solve_sequence.argtypes = [vp, i64, i64, i64, i32, GET_H, vp, ctypes.POINTER(Opts), vp, i64, pd, pd,
                                           ctypes.POINTER(Report)]
        L.chfsi_reduce_generalized.argtypes = [vp, i64, vp, i64, vp, i64]
        L.chfsi_back_transform.argtypes = [vp, i64, vp, i64, vp, i64, i64]
        L.chfsi_reduce_generalized_panel.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, vp, i64]
        L.chfsi_back_transform_panel.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, i64]
        L.chfsi_solve_sequence_real.argtypes = L.chfsi_solve_sequence.argtypes
        L.chfsi_solve_sequence_real.restype = ctypes.c_int
        L.chfsi_solve_batch.argtypes = [i32, i32, i64, ctypes.POINTER(Opts), ctypes.POINTER(Sequence), i32]
        for name in ("chfsi_solve_batch", "chfsi_reduce_generalized", "chfsi_back_transform",
                     "chfsi_reduce_generalized_panel", "chfsi_back_transform_panel", "chfsi_ctx_create", "chfsi_ctx_create_local", "chfsi_local_group_create", "chfsi_ctx_reserve", "chfsi_filter", "chfsi_lanczos_bounds", "chfsi_qr",
                     "chfsi_rayleigh_ritz", "chfsi_solve_sequence"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def colmajor(rows: int, cols: int, device="cuda", dtype=None):
    """An uninitialised (rows x cols) column-major complex128 tensor (stride (1, rows))."""
    import torch

    dtype = dtype or torch.complex128
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def to_colmajor(a, device="cuda", real=False):
    """Copy a numpy / torch (rows x cols) array into a column-major complex128 (real: float64) device tensor."""
    import torch

    t = torch.as_tensor(np.asarray(a) if not isinstance(a, torch.Tensor) else a)
    dt = torch.float64 if real else torch.complex128
    out = colmajor(t.shape[0], t.shape[1], device=device, dtype=dt)
    out.copy_(t.real.to(dt) if (real and t.is_complex()) else t.to(dt))
    return out


def _mat(t, rows=None, cols=None, name="matrix", real=False):
    """(pointer, ld) of a column-major complex128 (real=True: float64) CUDA tensor."""
    import torch

    want = torch.float64 if real else torch.complex128
    if not isinstance(t, torch.Tensor) or t.dtype != want or not t.is_cuda or t.dim() != 2:
        raise TypeError(f"{name}: need a 2-D {want} CUDA tensor")
    if rows is not None and t.shape[0] != rows or cols is not None and t.shape[1] != cols:
        raise ValueError(f"{name}: shape {tuple(t.shape)} != ({rows}, {cols})")
    if t.shape[1] > 1 and t.stride(0) != 1 or t.shape[1] <= 1 and t.shape[0] > 1 and t.stride(0) != 1:
        raise ValueError(f"{name}: must be column-major (stride (1, ld))")
    ld = t.stride(1) if t.shape[1] > 1 else max(t.shape[0], 1)
    return ctypes.c_void_p(t.data_ptr()), ld


class LocalGroup:
    """P emulated ranks on one device (chfsi_local_group): drive each rank's Context from its own
    thread, each on its own stream. Runs the nranks > 1 data path on a single GPU."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        st = lib().chfsi_local_group_create(ctypes.byref(h), nranks)
        if st != 0:
            raise ChfsiError(st, "chfsi_local_group_create failed")
        self.h, self.nranks = h, nranks

    def close(self):
        if getattr(self, "h", None):
            lib().chfsi_local_group_destroy(self.h)
            self.h = None


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for Context(nccl_id=...) (rank 0 creates it; broadcast it to all ranks)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().chfsi_nccl_unique_id(buf)
    if st != 0:
        raise ChfsiError(st, "chfsi_nccl_unique_id failed (NCCL unavailable?)")
    return buf.raw


class Context:
    """A library context on one device (one per rank). Work runs on `stream` (default: torch's current
    stream). For nranks > 1 pass `nccl_id` (bytes from nccl_unique_id(), broadcast to all ranks: the
    library creates its own NCCL communicator), or `nccl_comm` (an existing ncclComm_t as int), or a
    LocalGroup (emulated ranks on one device)."""

    def __init__(self, device: int = 0, stream=None, nccl_comm: int | None = None, rank: int = 0, nranks: int = 1,
                 local_group: LocalGroup | None = None, nccl_id: bytes | None = None):
        import torch

        L = lib()
        self.device = device
        self.rank = rank
        self.nranks = local_group.nranks if local_group else nranks
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        if local_group is not None:
            st = L.chfsi_ctx_create_local(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream),
                                          local_group.h, rank)
        elif nccl_id is not None:
            st = L.chfsi_ctx_create_nccl(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream),
                                         ctypes.c_char_p(bytes(nccl_id)), rank, nranks)
        else:
            st = L.chfsi_ctx_create(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream),
                                    ctypes.c_void_p(nccl_comm or 0), rank, nranks)
        if st != 0:
            raise ChfsiError(st, "chfsi_ctx_create failed (no B200 / CUDA device?)")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().chfsi_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0 and st != 3:
            raise ChfsiError(st, lib().chfsi_last_error(self.h).decode())
        return st

    @property
    def kernel_launches(self) -> int:
        return lib().chfsi_kernel_launches(self.h)

    def reserve(self, n, nloc, kmax):
        self._check(lib().chfsi_ctx_reserve(self.h, n, nloc, kmax))

    def set_complex_mult(self, mults: int = 3):
        """Complex filter / H Q arithmetic: 3 = Gauss 3M (default), 4 = 4M real embedding
        (chfsi_ctx_set_complex_mult)."""
        self._check(lib().chfsi_ctx_set_complex_mult(self.h, mults))

    def set_eigensolver(self, mode: int = 0):
        """Rayleigh-Ritz k x k eigensolve: 0 = Jacobi-type refinement with the dense fallback (default),
        1 = dense ZHEEVD only (chfsi_ctx_set_eigensolver)."""
        self._check(lib().chfsi_ctx_set_eigensolver(self.h, mode))

    def set_exchange(self, mode: int):
        """nranks > 1, collective: 0 = pipelined allgather, 1 = peer push from the filter epilogue
        (chfsi_ctx_set_exchange; reserve() first)."""
        self._check(lib().chfsi_ctx_set_exchange(self.h, mode))

    def set_pipeline(self, group_cols: int = 128, sm_reserve: int = 0):
        """nranks > 1: column groups of >= group_cols overlap their allgather with the next group's
        filter kernel (chfsi_ctx_set_pipeline; 0 = one group)."""
        self._check(lib().chfsi_ctx_set_pipeline(self.h, group_cols, sm_reserve))

    # -- Alg 2 -------------------------------------------------------------------------------------
    def filter(self, Hp, Y, deg, lambda1, c, e, n=None, row0=0):
        """In place: Y <- filtered block (chfsi_filter). Returns the mat-vec count sum(deg)."""
        nloc, k = Y.shape
        n = n or Hp.shape[0]
        hp, ldh = _mat(Hp, n, nloc, "Hp")
        yp, ldy = _mat(Y, nloc, k, "Y")
        d = (ctypes.c_int32 * max(k, 1))(*[int(x) for x in deg])
        mv = ctypes.c_int64()
        self._check(lib().chfsi_filter(self.h, n, row0, nloc, hp, ldh, yp, ldy, k, d, lambda1, c, e, ctypes.byref(mv)))
        return mv.value

    def filter_real(self, Hp, Y, deg, lambda1, c, e, n=None, row0=0):
        """Real-symmetric Alg 2 (chfsi_filter_real): float64 column-major Hp (n x nloc) and Y (nloc x k)."""
        nloc, k = Y.shape
        n = n or Hp.shape[0]
        hp, ldh = _mat(Hp, n, nloc, "Hp", real=True)
        yp, ldy = _mat(Y, nloc, k, "Y", real=True)
        d = (ctypes.c_int32 * max(k, 1))(*[int(x) for x in deg])
        mv = ctypes.c_int64()
        self._check(lib().chfsi_filter_real(self.h, n, row0, nloc, hp, ldh, yp, ldy, k, d, lambda1, c, e,
                                            ctypes.byref(mv)))
        return mv.value

    # -- Alg 1 l3 ----------------------------------------------------------------------------------
    def lanczos_bounds(self, Hp, steps=25, seed=0, n=None, row0=0):
        n = n or Hp.shape[0]
        nloc = Hp.shape[1]
        hp, ldh = _mat(Hp, n, nloc, "Hp")
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self._check(lib().chfsi_lanczos_bounds(self.h, n, row0, nloc, hp, ldh, steps, seed, ctypes.byref(a),
                                               ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    # -- Alg 1 l6 ----------------------------------------------------------------------------------
    def qr(self, Y, nlocked=0, n=None, row0=0):
        nloc, k = Y.shape
        n = n or nloc
        yp, ldy = _mat(Y, nloc, k, "Y")
        fb = ctypes.c_int32()
        self._check(lib().chfsi_qr(self.h, n, row0, nloc, yp, ldy, k, nlocked, ctypes.byref(fb)))
        return fb.value

    def qr_ex(self, Y, nlocked=0, seed=0, n=None, row0=0):
        """chfsi_qr_ex: QR with the rank-deficiency rule R23; returns (used_fallback, replaced)."""
        nloc, k = Y.shape
        n = n or nloc
        yp, ldy = _mat(Y, nloc, k, "Y")
        fb, rep = ctypes.c_int32(), ctypes.c_int32()
        self._check(lib().chfsi_qr_ex(self.h, n, row0, nloc, yp, ldy, k, nlocked, seed, ctypes.byref(fb),
                                      ctypes.byref(rep)))
        return fb.value, rep.value

    # -- Alg 1 l7-9 --------------------------------------------------------------------------------
    def rayleigh_ritz(self, Hp, Q, normH=None, n=None, row0=0):
        nloc, k = Q.shape
        n = n or Hp.shape[0]
        hp, ldh = _mat(Hp, n, nloc, "Hp")
        qp, ldq = _mat(Q, nloc, k, "Q")
        ritz = np.zeros(k)
        res = np.zeros(k) if normH else None
        self._check(lib().chfsi_rayleigh_ritz(
            self.h, n, row0, nloc, hp, ldh, qp, ldq, k, float(normH or 0.0),
            ritz.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if res is not None else None))
        return ritz, res

    # -- generalised front / back end ------------------------------------------------
    def reduce_generalized(self, A, B):
        """In place: B <- L (lower Cholesky factor), A <- H = L^{-1} A L^{-H}."""
        n = A.shape[0]
        ap, lda = _mat(A, n, n, "A")
        bp, ldb = _mat(B, n, n, "B")
        self._check(lib().chfsi_reduce_generalized(self.h, n, ap, lda, bp, ldb))

    def back_transform(self, L, X):
        """In place: X <- L^{-H} X (generalised eigenvectors)."""
        n, k = X.shape
        lp, ldl = _mat(L, n, n, "L")
        xp, ldx = _mat(X, n, k, "X")
        self._check(lib().chfsi_back_transform(self.h, n, lp, ldl, xp, ldx, k))

    def reduce_generalized_panel(self, Ap, Bp, L, n=None, row0=0):
        """Row-panel form (collective): Ap (n x nloc) <- this rank's slab of H = L^{-1} A L^{-H};
        Bp (n x nloc) is read only; L (n x n) <- the full Cholesky factor (lower triangle)."""
        n = n or Ap.shape[0]
        nloc = Ap.shape[1]
        ap, lda = _mat(Ap, n, nloc, "Ap")
        bp, ldb = _mat(Bp, n, nloc, "Bp")
        lp, ldl = _mat(L, n, n, "L")
        self._check(lib().chfsi_reduce_generalized_panel(self.h, n, row0, nloc, ap, lda, bp, ldb, lp, ldl))

    def back_transform_panel(self, L, X, n=None, row0=0):
        """Row-panel back-transformation (collective): X (this rank's nloc x k rows) <- its rows of L^{-H} X."""
        nloc, k = X.shape
        n = n or L.shape[0]
        lp, ldl = _mat(L, n, n, "L")
        xp, ldx = _mat(X, nloc, k, "X")
        self._check(lib().chfsi_back_transform_panel(self.h, n, row0, nloc, lp, ldl, xp, ldx, k))

    # -- Alg 1 over a sequence ----------------------------------------------------------------------
    def solve_sequence(self, get_h, nprob, X, nev, nex, tol, deg_cap=40, deg0=8, max_loops=50, lanczos_steps=25,
                       seed=0, random_start=False, n=None, row0=0, no_reuse=False, fixed_degree=0, real=False):
        """get_h(ell) -> column-major CUDA tensor Hp (n x nloc) of problem ell (kept alive by the caller
        until the next call). real=True: real symmetric H and X (float64; chfsi_solve_sequence_real).
        Returns dict(status, lam (nprob x nev), resid, reports)."""
        nloc, k = X.shape
        assert k == nev + nex
        n = n or nloc
        xp, ldx = _mat(X, nloc, k, "X", real=real)
        keep = {}

        def cb(user, ell, hp_out, ldh_out):
            try:
                t = get_h(int(ell))
                p, ld = _mat(t, n, nloc, "Hp", real=real)
                keep["h"] = t
                hp_out[0] = p.value
                ldh_out[0] = ld
                return 0
            except Exception as ex:  # surfaced as ERR_ARG through the C-ABI
                keep["exc"] = ex
                return 1

        cbf = GET_H(cb)
        opts = Opts(nev, nex, deg0, deg_cap, max_loops, lanczos_steps, tol, seed, 1 if random_start else 0,
                    1 if no_reuse else 0, int(fixed_degree))
        lam = np.zeros(nprob * nev)
        res = np.zeros(nprob * nev)
        reps = (Report * nprob)()
        fn = lib().chfsi_solve_sequence_real if real else lib().chfsi_solve_sequence
        st = fn(self.h, n, row0, nloc, nprob, cbf, None, ctypes.byref(opts), xp, ldx,
                                        lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), reps)
        if "exc" in keep:
            raise keep["exc"]
        self._check(st)
        return dict(status=st, lam=lam.reshape(nprob, nev), resid=res.reshape(nprob, nev),
                    reports=[r.as_dict() for r in reps])


def solve_batch(device, workers, sequences, nev, nex, tol, deg_cap=40, deg0=8, max_loops=50, lanczos_steps=25,
                seed=0):
    """Independent sequences (k-points) concurrently on one device (chfsi_solve_batch).
    sequences: list of (get_h(ell) -> column-major Hp tensor, nprob, X tensor). Returns a list of
    dict(status, lam, resid, reports)."""
    import torch

    torch.cuda.synchronize(device)
    count = len(sequences)
    arr = (Sequence * count)()
    keep = []
    outs = []
    for i, (get_h, nprob, X) in enumerate(sequences):
        n, k = X.shape
        xp, ldx = _mat(X, n, k, "X")
        tensors = {}

        def cb(user, ell, hp_out, ldh_out, get_h=get_h, tensors=tensors, n=n):
            try:
                t = get_h(int(ell))
                p, ld = _mat(t, n, n, "Hp")
                tensors[int(ell)] = t
                hp_out[0] = p.value
                ldh_out[0] = ld
                return 0
            except Exception:
                return 1

        cbf = GET_H(cb)
        lam = np.zeros(nprob * nev)
        res = np.zeros(nprob * nev)
        reps = (Report * nprob)()
        keep += [cbf, lam, res, reps, tensors]
        arr[i] = Sequence(nprob, cbf, None, xp.value, ldx, lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                          res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), reps, 0)
        outs.append((lam, res, reps, nprob))
    n = sequences[0][2].shape[0]
    opts = Opts(nev, nex, deg0, deg_cap, max_loops, lanczos_steps, tol, seed, 0, 0, 0)
    st = lib().chfsi_solve_batch(device, workers, n, ctypes.byref(opts), arr, count)
    if st not in (0, 3):
        raise ChfsiError(st, "chfsi_solve_batch failed")
    return [dict(status=arr[i].status, lam=lam.reshape(nprob, nev), resid=res.reshape(nprob, nev),
                 reports=[r.as_dict() for r in reps]) for i, (lam, res, reps, nprob) in enumerate(outs)]


def filter_flops(n: int, deg) -> float:
    """Algorithmic flops of one filter call: 8 n^2 sum(deg) (complex MAC = 8 real flops)."""
    return 8.0 * n * n * float(sum(int(d) for d in deg))
