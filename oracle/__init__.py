"""TEST INFRASTRUCTURE ONLY: ctypes binding of the plain CPU oracle (oracle/oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package. The product path (paper_1404_4161_b200) never imports it and shares no code with it.
Arrays are numpy complex128 / float64 in Fortran (column-major) order.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


class Opts(ctypes.Structure):
    _fields_ = [("nev", ctypes.c_int32), ("nex", ctypes.c_int32), ("deg0", ctypes.c_int32),
                ("deg_cap", ctypes.c_int32), ("max_loops", ctypes.c_int32), ("lanczos_steps", ctypes.c_int32),
                ("tol", ctypes.c_double), ("seed", ctypes.c_uint64)]


class Report(ctypes.Structure):
    _fields_ = [("loops", ctypes.c_int32), ("capped", ctypes.c_int32), ("qr_replaced", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("matvecs_filter", ctypes.c_int64),
                ("matvecs_total", ctypes.c_int64), ("theta_min", ctypes.c_double),
                ("theta_max", ctypes.c_double), ("beta_up", ctypes.c_double), ("normH", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make oracle/liboracle.so`")
        L = ctypes.CDLL(path)
        i64, u64, i32, dbl, ptr, ch = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double,
                                       ctypes.c_void_p, ctypes.c_char)
        ld = ctypes.c_longdouble
        L.ora_cheb.argtypes = [i32, ld]
        L.ora_cheb.restype = ld
        L.ora_filter_gain.argtypes = [i32, ld, ld, ld, ld]
        L.ora_filter_gain.restype = ld
        L.ora_sigma.argtypes = [i32, dbl, dbl, dbl, ptr]
        L.ora_filter.argtypes = [i64, ptr, i64, ptr, i64, i64, ptr, dbl, dbl, dbl, ptr]
        L.ora_filter.restype = i32
        L.ora_filter_diag_closed.argtypes = [i64, ptr, ptr, i64, i64, ptr, dbl, dbl, dbl]
        L.ora_filter_wy_closed.argtypes = [i64, ptr, ptr, ptr, ptr, i64, i64, ptr, dbl, dbl, dbl]
        L.ora_zgemm.argtypes = [ch, ch, i64, i64, i64, ptr, i64, ptr, i64, ptr, i64]
        L.ora_householder_qr.argtypes = [i64, i64, ptr, i64, ptr, i64, ptr, i64]
        L.ora_householder_qr.restype = i32
        L.ora_jacobi_eig.argtypes = [i64, ptr, i64, ptr, ptr, i64]
        L.ora_jacobi_eig.restype = i32
        L.ora_random_vector.argtypes = [i64, u64, u64, ptr]
        L.ora_lanczos.argtypes = [i64, ptr, i64, i32, u64, ptr, ptr, ptr]
        L.ora_lanczos.restype = i32
        L.ora_rayleigh_ritz.argtypes = [i64, ptr, i64, ptr, i64, i64, ptr]
        L.ora_rayleigh_ritz.restype = i32
        L.ora_residuals.argtypes = [i64, ptr, i64, ptr, i64, i64, ptr, dbl, ptr]
        L.ora_rayleigh_quotients.argtypes = [i64, ptr, i64, ptr, i64, i64, ptr, ptr]
        L.ora_degree.argtypes = [dbl, dbl, dbl, i32]
        L.ora_degree.restype = i32
        L.ora_degree_literal.argtypes = [dbl, dbl, dbl, i32]
        L.ora_degree_literal.restype = i32
        L.ora_rho.argtypes = [dbl]
        L.ora_rho.restype = dbl
        L.ora_chfsi_solve.argtypes = [i64, ptr, i64, ctypes.POINTER(Opts), ptr, i64, i32, ptr, ptr, ptr, ptr,
                                      ctypes.POINTER(Report)]
        L.ora_chfsi_solve.restype = i32
        L.ora_cholesky.argtypes = [i64, ptr, i64, ptr, i64]
        L.ora_cholesky.restype = i32
        L.ora_trsm_lower.argtypes = [i64, i64, ptr, i64, ptr, i64, i32]
        L.ora_reduce_generalized.argtypes = [i64, ptr, i64, ptr, i64, ptr, i64, ptr, i64]
        L.ora_reduce_generalized.restype = i32
        L.ora_orthonormalize.argtypes = [i64, ptr, i64, ptr, i64, u64, ptr]
        L.ora_orthonormalize.restype = i32
        L.ora_count_below.argtypes = [i64, ptr, i64, dbl]
        L.ora_count_below.restype = i64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _cf(a, dtype=np.complex128):
    a = np.asarray(a, dtype=dtype)
    return np.asfortranarray(a)


def cheb(m: int, t: float) -> float:
    return float(lib().ora_cheb(m, t))


def filter_gain(m, lam, lambda1, c, e) -> float:
    return float(lib().ora_filter_gain(m, lam, lambda1, c, e))


def sigma(mmax: int, lambda1: float, c: float, e: float) -> np.ndarray:
    s = np.empty(mmax, dtype=np.float64)
    lib().ora_sigma(mmax, lambda1, c, e, _p(s))
    return s


def _deg(deg):
    return np.ascontiguousarray(np.asarray(deg, dtype=np.int32))


def chebyshev_filter(H, Y0, deg, lambda1, c, e):
    """Alg 2. Returns (Y_m, matvecs)."""
    H = _cf(H)
    Y = _cf(Y0).copy(order="F")
    d = _deg(deg)
    n, k = Y.shape
    mv = ctypes.c_int64(0)
    st = lib().ora_filter(n, _p(H), H.shape[0], _p(Y), n, k, _p(d), lambda1, c, e, ctypes.byref(mv))
    if st == 1:
        raise ValueError("ora_filter: bad arguments")
    return Y, mv.value


def filter_diag_closed(d, Y0, deg, lambda1, c, e):
    d = np.ascontiguousarray(d, dtype=np.float64)
    Y = _cf(Y0).copy(order="F")
    lib().ora_filter_diag_closed(Y.shape[0], _p(d), _p(Y), Y.shape[0], Y.shape[1], _p(_deg(deg)), lambda1, c, e)
    return Y


def filter_wy_closed(wy, Y0, deg, lambda1, c, e):
    Y = _cf(Y0).copy(order="F")
    lib().ora_filter_wy_closed(wy.n, _p(wy.lam), _p(wy.V), _p(wy.T), _p(Y), Y.shape[0], Y.shape[1],
                               _p(_deg(deg)), lambda1, c, e)
    return Y


def zgemm(ta, tb, A, B):
    A = _cf(A)
    B = _cf(B)
    m = A.shape[0] if ta == "N" else A.shape[1]
    kk = A.shape[1] if ta == "N" else A.shape[0]
    n = B.shape[1] if tb == "N" else B.shape[0]
    C = np.empty((m, n), dtype=np.complex128, order="F")
    lib().ora_zgemm(ta.encode(), tb.encode(), m, n, kk, _p(A), A.shape[0], _p(B), B.shape[0], _p(C), m)
    return C


def householder_qr(A):
    A = _cf(A)
    n, k = A.shape
    Q = np.empty((n, k), dtype=np.complex128, order="F")
    R = np.empty((k, k), dtype=np.complex128, order="F")
    defic = lib().ora_householder_qr(n, k, _p(A), n, _p(Q), n, _p(R), k)
    return Q, R, defic


def orthonormalize(Y, XL=None, seed=0):
    """Alg 1 l6 with the rank-deficiency rule R23. Returns (Q, replaced); raises if R23 failed."""
    Y = _cf(Y).copy(order="F")
    n, ka = Y.shape
    nl = 0 if XL is None else XL.shape[1]
    X = _cf(XL) if nl else np.zeros((n, 1), dtype=np.complex128, order="F")
    rep = ctypes.c_int32(0)
    st = lib().ora_orthonormalize(n, _p(X), nl, _p(Y), ka, seed, ctypes.byref(rep))
    if st:
        raise RuntimeError("ora_orthonormalize: still rank deficient after 3 replacement rounds")
    return Y, rep.value


def jacobi_eig(A):
    A = _cf(A)
    n = A.shape[0]
    w = np.empty(n, dtype=np.float64)
    V = np.empty((n, n), dtype=np.complex128, order="F")
    sw = lib().ora_jacobi_eig(n, _p(A), n, _p(w), _p(V), n)
    if sw < 0:
        raise RuntimeError("Jacobi did not converge")
    return w, V


def random_vector(n, seed, strm):
    x = np.empty(n, dtype=np.complex128)
    lib().ora_random_vector(n, seed, strm, _p(x))
    return x


def lanczos(H, steps, seed):
    H = _cf(H)
    a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    st = lib().ora_lanczos(H.shape[0], _p(H), H.shape[0], steps, seed, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    if st:
        raise RuntimeError("Lanczos failed")
    return a.value, b.value, c.value


def rayleigh_ritz(H, Q):
    H = _cf(H)
    Q = _cf(Q).copy(order="F")
    n, k = Q.shape
    ritz = np.empty(k, dtype=np.float64)
    lib().ora_rayleigh_ritz(n, _p(H), H.shape[0], _p(Q), n, k, _p(ritz))
    return ritz, Q


def residuals(H, X, lam, normH):
    H = _cf(H)
    X = _cf(X)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    r = np.empty(X.shape[1], dtype=np.float64)
    lib().ora_residuals(X.shape[0], _p(H), H.shape[0], _p(X), X.shape[0], X.shape[1], _p(lam), normH, _p(r))
    return r


def rayleigh_quotients(H, X):
    """(rho, resid_abs): Rayleigh quotients of the columns of X and ||H x - rho x|| / ||x||."""
    H = _cf(H)
    X = _cf(X)
    k = X.shape[1]
    rho = np.empty(k)
    ra = np.empty(k)
    lib().ora_rayleigh_quotients(X.shape[0], _p(H), H.shape[0], _p(X), X.shape[0], k, _p(rho), _p(ra))
    return rho, ra


def degree(res, tol, t, cap):
    return lib().ora_degree(res, tol, t, cap)


def degree_literal(res, tol, rho, cap):
    return lib().ora_degree_literal(res, tol, rho, cap)


def rho(t):
    return lib().ora_rho(t)


def chfsi_solve(H, X0, nev, nex, tol, cap, deg0=8, max_loops=50, lanczos_steps=25, seed=0,
                prev=None):
    """Alg 1 for one problem. prev = (lambda1, lambdak) of the previous problem or None.
    Returns dict(status, lam, resid, X (hand-off block), lambda1, lambdak, report)."""
    H = _cf(H)
    X = _cf(X0).copy(order="F")
    n, k = X.shape
    assert k == nev + nex
    o = Opts(nev, nex, deg0, cap, max_loops, lanczos_steps, tol, seed)
    l1 = ctypes.c_double(prev[0] if prev else 0.0)
    lk = ctypes.c_double(prev[1] if prev else 0.0)
    lam = np.zeros(nev)
    res = np.zeros(nev)
    rep = Report()
    st = lib().ora_chfsi_solve(n, _p(H), H.shape[0], ctypes.byref(o), _p(X), n, 1 if prev else 0,
                               ctypes.byref(l1), ctypes.byref(lk), _p(lam), _p(res), ctypes.byref(rep))
    if st == 1:
        raise ValueError("ora_chfsi_solve: bad arguments")
    return dict(status=st, lam=lam, resid=res, X=X, lambda1=l1.value, lambdak=lk.value, report=rep.as_dict())


def count_below(H, sigma_):
    H = _cf(H)
    return lib().ora_count_below(H.shape[0], _p(H), H.shape[0], sigma_)


def cholesky(B):
    B = _cf(B)
    n = B.shape[0]
    L = np.empty((n, n), dtype=np.complex128, order="F")
    st = lib().ora_cholesky(n, _p(B), n, _p(L), n)
    if st:
        raise ValueError(f"not positive definite at pivot {st - 1}")
    return L


def trsm_lower(L, X, adjoint=False):
    L = _cf(L)
    X = _cf(X).copy(order="F")
    lib().ora_trsm_lower(L.shape[0], X.shape[1], _p(L), L.shape[0], _p(X), X.shape[0], 1 if adjoint else 0)
    return X


def reduce_generalized(A, B):
    """(H, L): B = L L^H, H = L^{-1} A L^{-H}."""
    A = _cf(A)
    B = _cf(B)
    n = A.shape[0]
    H = np.empty((n, n), dtype=np.complex128, order="F")
    L = np.empty((n, n), dtype=np.complex128, order="F")
    st = lib().ora_reduce_generalized(n, _p(A), n, _p(B), n, _p(H), n, _p(L), n)
    if st:
        raise ValueError(f"B not positive definite at pivot {st - 1}")
    return H, L
