"""Seeded synthetic inputs for BASELINE.json configs C1–C5 (input plumbing only).

This package is shared by tests/, bench.py and __graft_entry__.smoke().  It holds
no GMRES arithmetic: matrices, random vectors and b = A·x_true come from the
C++ generator in ``inputs/gen.cpp`` (counter-based RNG, OpenMP, deterministic
for any thread count).  Recipe and readings: DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.cpp")
_LIB = os.path.join(_HERE, "libgmres_gen.so")
_lib = None

# power-law exponent that gives mean row length 30 on [4, 2000]
C3_ALPHA = 1.8743


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c++17", "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, u64, i32, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        vp = ctypes.c_void_p
        L.gen_stencil_n.argtypes = [i32, i64]; L.gen_stencil_n.restype = i64
        L.gen_stencil_nnz.argtypes = [i32, i64]; L.gen_stencil_nnz.restype = i64
        L.gen_stencil.argtypes = [i32, i64, vp, vp, vp, vp]; L.gen_stencil.restype = i32
        L.gen_randdd_rowptr.argtypes = [i64, u64, dbl, i32, i32, vp]; L.gen_randdd_rowptr.restype = i64
        L.gen_randdd_fill.argtypes = [i64, u64, vp, vp, vp]; L.gen_randdd_fill.restype = i32
        L.gen_uniform.argtypes = [i64, u64, u64, dbl, dbl, vp]; L.gen_uniform.restype = None
        L.gen_matvec.argtypes = [i64, vp, vp, vp, vp, vp]; L.gen_matvec.restype = None
        L.gen_u01.argtypes = [u64, u64, u64]; L.gen_u01.restype = dbl
        L.gen_normal.argtypes = [u64, u64, u64]; L.gen_normal.restype = dbl
        L.gen_num_threads.argtypes = []; L.gen_num_threads.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class CSR:
    row_ptr: np.ndarray  # int32[n+1]
    col: np.ndarray      # int32[nnz]
    val: np.ndarray      # float64[nnz]

    @property
    def n(self) -> int:
        return self.row_ptr.shape[0] - 1

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        n = self.n
        A = np.zeros((n, n))
        for i in range(n):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            A[i, self.col[s:e]] = self.val[s:e]
        return A


def stencil(kind: int, N: int, beta=(0.0, 0.0, 0.0)) -> CSR:
    L = lib()
    n = L.gen_stencil_n(kind, N)
    nnz = L.gen_stencil_nnz(kind, N)
    rp = np.empty(n + 1, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    b = np.ascontiguousarray(np.array(list(beta) + [0.0] * (3 - len(beta)), np.float64))
    rc = L.gen_stencil(kind, N, _p(b), _p(rp), _p(col), _p(val))
    if rc != 0:
        raise ValueError(f"gen_stencil({kind},{N}) failed")
    return CSR(rp, col, val)


def randdd(n: int, seed: int, alpha: float = C3_ALPHA, kmin: int = 4, kmax: int = 2000) -> CSR:
    L = lib()
    rp = np.empty(n + 1, np.int32)
    nnz = L.gen_randdd_rowptr(n, seed, alpha, kmin, kmax, _p(rp))
    if nnz < 0:
        raise ValueError("gen_randdd_rowptr failed")
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    if L.gen_randdd_fill(n, seed, _p(rp), _p(col), _p(val)) != 0:
        raise ValueError("gen_randdd_fill failed")
    return CSR(rp, col, val)


def uniform(n: int, seed: int, stream: int = 0, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().gen_uniform(n, seed, stream, lo, hi, _p(out))
    return out


def matvec(A: CSR, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    b = np.empty(A.n, np.float64)
    lib().gen_matvec(A.n, _p(A.row_ptr), _p(A.col), _p(A.val), _p(x), _p(b))
    return b


@dataclass
class Problem:
    name: str
    A: CSR
    b: np.ndarray
    x_true: np.ndarray | None
    m: int
    tol: float = 1e-10
    meta: dict = field(default_factory=dict)


def make(name: str, scale: int | None = None) -> Problem:
    """Build a BASELINE.json config.  ``scale`` shrinks the grid (N) or n for
    oracle-sized variants (e.g. make("C2", 32) = the C2 recipe on a 32³ grid)."""
    if name == "C1":
        N = scale or 64
        A = stencil(5, N, (20.0, 20.0, 0.0))
        xt = uniform(A.n, 0)
        return Problem(name, A, matvec(A, xt), xt, 30, meta={"kind": "5pt", "N": N, "beta": [20, 20]})
    if name in ("C2", "C5"):
        N = scale or 128
        A = stencil(7, N, (10.0, 5.0, 2.0))
        xt = uniform(A.n, 1)
        return Problem(name, A, matvec(A, xt), xt, 50, meta={"kind": "7pt", "N": N, "beta": [10, 5, 2]})
    if name == "C3":
        n = scale or 4_000_000
        A = randdd(n, 2)
        b = uniform(n, 2)
        return Problem(name, A, b, None, 50, meta={"kind": "randdd", "n": n, "alpha": C3_ALPHA})
    if name == "C4":
        N = scale or 256
        A = stencil(27, N, (20.0, 10.0, 5.0))
        xt = uniform(A.n, 3)
        return Problem(name, A, matvec(A, xt), xt, 100, meta={"kind": "27pt", "N": N, "beta": [20, 10, 5]})
    raise KeyError(name)
