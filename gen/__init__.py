"""Seeded synthetic input generator (gen/gen.c), shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic; see gen.h for the construction (SURVEY.md 8(d) d2 and
DESIGN.md "Input recipe"). Arrays are numpy complex128 in Fortran (column-major) order.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

NREF = 8


def stream(major: int, minor: int = 0) -> int:
    return (major << 16) | minor


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make gen/libgen.so` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        i64, u64, i32, dbl, ptr = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        L.gen_splitmix64.argtypes = [u64]
        L.gen_splitmix64.restype = u64
        L.gen_uniform.argtypes = [u64, u64, u64]
        L.gen_uniform.restype = dbl
        L.gen_spectrum.argtypes = [i64, i64, ptr]
        L.gen_wy.argtypes = [i64, u64, ptr, ptr]
        L.gen_wy_aux.argtypes = [i64, ptr, ptr, ptr, ptr, ptr, ptr]
        L.gen_h1_panel.argtypes = [i64, ptr, ptr, ptr, ptr, i64, i64, ptr, i64]
        L.gen_eigvecs.argtypes = [i64, ptr, ptr, ptr, i64, ptr, i64]
        L.gen_gue_panel.argtypes = [i64, u64, u64, i64, i64, ptr, i64]
        L.gen_perturb_panel.argtypes = [i64, u64, i32, dbl, i64, i64, ptr, i64]
        L.gen_start_basis.argtypes = [i64, i64, u64, i64, i64, ptr, i64]
        L.gen_lower_factor.argtypes = [i64, u64, dbl, ptr, i64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def spectrum(n: int, nd: int) -> np.ndarray:
    lam = np.empty(n, dtype=np.float64)
    lib().gen_spectrum(n, nd, _p(lam))
    return lam


@dataclass
class WY:
    """H^(1) = Q diag(lam) Q^H with Q = I - V T V^H (8 reflectors)."""

    n: int
    lam: np.ndarray
    V: np.ndarray
    T: np.ndarray
    B: np.ndarray
    A: np.ndarray
    D: np.ndarray

    def panel(self, c0: int, ncols: int, out: np.ndarray | None = None) -> np.ndarray:
        """Columns [c0, c0+ncols) of H^(1) (n x ncols, Fortran order)."""
        if out is None:
            out = np.empty((self.n, ncols), dtype=np.complex128, order="F")
        assert out.flags.f_contiguous and out.shape == (self.n, ncols)
        lib().gen_h1_panel(self.n, _p(self.lam), _p(self.B), _p(self.A), _p(self.D), c0, ncols, _p(out), self.n)
        return out

    def full(self) -> np.ndarray:
        return self.panel(0, self.n)

    def eigvecs(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        X = np.empty((self.n, len(idx)), dtype=np.complex128, order="F")
        lib().gen_eigvecs(self.n, _p(self.V), _p(self.B), _p(idx), len(idx), _p(X), self.n)
        return X


def wy(n: int, nd: int, seed: int, lam: np.ndarray | None = None) -> WY:
    L = lib()
    if lam is None:
        lam = spectrum(n, nd)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    V = np.empty((n, NREF), dtype=np.complex128, order="F")
    T = np.empty((NREF, NREF), dtype=np.complex128, order="F")
    L.gen_wy(n, seed, _p(V), _p(T))
    B = np.empty_like(V)
    A = np.empty_like(V)
    D = np.empty_like(V)
    L.gen_wy_aux(n, _p(lam), _p(V), _p(T), _p(B), _p(A), _p(D))
    return WY(n, lam, V, T, B, A, D)


def gue(n: int, seed: int, strm: int, c0: int = 0, ncols: int | None = None) -> np.ndarray:
    ncols = n if ncols is None else ncols
    G = np.empty((n, ncols), dtype=np.complex128, order="F")
    lib().gen_gue_panel(n, seed, strm, c0, ncols, _p(G), n)
    return G


def perturb(H: np.ndarray, seed: int, ell: int, scale: float, c0: int = 0) -> np.ndarray:
    """In place: H[:, panel] += scale * G_ell[:, panel] (H holds columns c0..c0+H.shape[1])."""
    assert H.flags.f_contiguous and H.dtype == np.complex128
    lib().gen_perturb_panel(H.shape[0], seed, ell, scale, c0, H.shape[1], _p(H), H.shape[0])
    return H


def start_basis(n: int, k: int, seed: int, r0: int = 0, nrows: int | None = None) -> np.ndarray:
    nrows = n if nrows is None else nrows
    Y = np.empty((nrows, k), dtype=np.complex128, order="F")
    lib().gen_start_basis(n, k, seed, r0, nrows, _p(Y), nrows)
    return Y


def uniform(seed: int, strm: int, idx: int) -> float:
    return lib().gen_uniform(seed, strm, idx)


def lower_factor(n: int, seed: int, scale: float = 0.5) -> np.ndarray:
    M = np.empty((n, n), dtype=np.complex128, order="F")
    lib().gen_lower_factor(n, seed, scale, _p(M), n)
    return M


def generalized_pair(wy: WY, seed: int, scale: float = 0.5):
    """(A, B, M): B = M M^H (HPD, Cholesky factor M), A = M H^(1) M^H -- generalised eigenvalues = wy.lam,
    generalised eigenvectors M^{-H} Q e_i. Products formed with numpy (input construction only)."""
    M = lower_factor(wy.n, seed, scale)
    H = wy.full()
    B = np.asfortranarray(M @ M.conj().T)
    A = M @ H @ M.conj().T
    A = np.asfortranarray((A + A.conj().T) / 2)  # exact Hermitian storage (R13)
    B = np.asfortranarray((B + B.conj().T) / 2)
    return A, B, M
