"""CPU oracle for mixed-precision restarted GMRES(m) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2011_01850_b200`` never imports it (checked by tests/test_layout.py).

Thin ctypes wrappers over ``oracle/oracle.cpp`` (plain single-threaded C++
following Alg. 1; see oracle.h for every entry point).
Pins: tests/test_oracle.py.  Parity unpinned: cycle counts beyond the weak
expectation of PAPER.md:434-435.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

FP64, MIXED = 0, 1
MGS, CGSR = 0, 1
F_CGS1, F_RESID32, F_UPDATE32, F_ACC32 = 1, 2, 4, 8
F_ILU0, F_ILU32 = 16, 32   # preconditioner (§8 f2, reading R24); default Jacobi
OK, NOT_CONVERGED = 0, 1


class _Result(ctypes.Structure):
    _fields_ = [("cycles", ctypes.c_int32), ("inner_iters", ctypes.c_int32),
                ("history_len", ctypes.c_int32), ("inner_len", ctypes.c_int32),
                ("final_relres", ctypes.c_double)]


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_use_omp = False


def build(force: bool = False, omp: bool = False) -> str:
    """Compile the oracle.  omp=True builds liboracle_omp.so (-fopenmp): the same
    source with its element-parallel loops (ORACLE_PAR, oracle.cpp) spread over
    threads and every reduction kept sequential — bitwise equal to the default
    single-threaded build (tests/test_oracle.py)."""
    out = _LIB_OMP if omp else _LIB
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
        # -ffp-contract=off: every W operation rounds on its own (no FMA fusion);
        # SSE2 arithmetic on x86-64 (no x87 extended precision).
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
               "-std=c++17"] + (["-fopenmp"] if omp else []) + ["-o", out, _SRC]
        subprocess.check_call(cmd)
    return out


def use_omp(flag: bool = True) -> None:
    """Route every later call through the OpenMP build (full-size golden runs only)."""
    global _use_omp, _lib
    if flag != _use_omp:
        _use_omp = flag
        _lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build(omp=_use_omp))
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.oracle_spmv64.argtypes = [i64, vp, vp, vp, vp, vp]; L.oracle_spmv64.restype = None
        L.oracle_spmv32.argtypes = [i64, vp, vp, vp, vp, vp]; L.oracle_spmv32.restype = None
        L.oracle_dinv.argtypes = [i64, vp, vp, vp, vp, vp]; L.oracle_dinv.restype = i32
        L.oracle_cast32.argtypes = [i64, vp, vp]; L.oracle_cast32.restype = i32
        L.oracle_ilu0.argtypes = [i32, i64, vp, vp, vp, vp, vp]; L.oracle_ilu0.restype = i32
        L.oracle_ilu0_apply.argtypes = [i32, i64, vp, vp, vp, vp, vp]; L.oracle_ilu0_apply.restype = None
        L.oracle_jacobi_spmv.argtypes = [i32, i64, vp, vp, vp, vp, vp, vp]; L.oracle_jacobi_spmv.restype = None
        L.oracle_resid.argtypes = [i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]; L.oracle_resid.restype = i32
        L.oracle_dot.argtypes = [i32, i64, vp, vp]; L.oracle_dot.restype = dbl
        L.oracle_mgs.argtypes = [i32, i64, i32, vp, i64, vp, vp]; L.oracle_mgs.restype = None
        L.oracle_cgsr.argtypes = [i32, i64, i32, vp, i64, vp, vp, i32]; L.oracle_cgsr.restype = None
        L.oracle_scale.argtypes = [i32, i64, vp, dbl, vp]; L.oracle_scale.restype = None
        L.oracle_givens.argtypes = [dbl, dbl, vp, vp, vp]; L.oracle_givens.restype = None
        L.oracle_hess_step.argtypes = [i32, vp, vp, vp, vp]; L.oracle_hess_step.restype = dbl
        L.oracle_backsolve.argtypes = [i32, vp, i64, vp, vp]; L.oracle_backsolve.restype = i32
        L.oracle_xupdate.argtypes = [i32, i64, i32, vp, i64, vp, vp]; L.oracle_xupdate.restype = None
        L.oracle_arnoldi.argtypes = [i32, i32, i32, i64, vp, vp, vp, vp, vp, i32, dbl, vp, i64,
                                     vp, vp, vp, vp, vp, vp]
        L.oracle_arnoldi.restype = i32
        L.oracle_gmres_solve.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32, dbl, i32, i32, dbl, i32, i32,
                                         vp, vp, ctypes.c_int32, vp, ctypes.c_int32]
        L.oracle_gmres_solve.restype = i32
        L.oracle_gmres_solve_policy.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32, dbl, i32, i32, dbl, i32, i32,
                                                vp, vp, ctypes.c_int32, vp, ctypes.c_int32, i32, dbl, dbl]
        L.oracle_gmres_solve_policy.restype = i32
        L.oracle_gmres_solve_orth.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32, dbl, i32, i32, dbl, i32, i32,
                                              vp, vp, ctypes.c_int32, vp, ctypes.c_int32, i32, dbl, dbl, i32, dbl,
                                              vp, ctypes.c_int32]
        L.oracle_gmres_solve_orth.restype = i32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def wdtype(prec: int):
    return np.float32 if prec == MIXED else np.float64


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ------------------------------------------------------------- components
def spmv64(A, x):
    y = np.empty(A.n)
    lib().oracle_spmv64(A.n, _p(A.row_ptr), _p(A.col), _p(_c(A.val, np.float64)), _p(_c(x, np.float64)), _p(y))
    return y


def spmv32(A, val32, x32):
    y = np.empty(A.n, np.float32)
    v, x = _c(val32, np.float32), _c(x32, np.float32)
    lib().oracle_spmv32(A.n, _p(A.row_ptr), _p(A.col), _p(v), _p(x), _p(y))
    return y


def dinv(A):
    d = np.empty(A.n)
    bad = np.zeros(1, np.int64)
    rc = lib().oracle_dinv(A.n, _p(A.row_ptr), _p(A.col), _p(_c(A.val, np.float64)), _p(d), _p(bad))
    if rc != 0:
        raise ZeroDivisionError(f"zero diagonal at row {int(bad[0])}")
    return d


def cast32(a):
    a = _c(a, np.float64)
    out = np.empty(a.shape, np.float32)
    rc = lib().oracle_cast32(a.size, _p(a), _p(out))
    if rc != 0:
        raise OverflowError("value outside fp32 range")
    return out


def working_copy(A, prec):
    """(aW, dinvW) as the solver builds them (reading R11)."""
    d = dinv(A)
    if prec == MIXED:
        return cast32(A.val), d.astype(np.float32)
    return _c(A.val, np.float64), d


def ilu0(prec, A, aW=None):
    """ILU(0) factors of A_W in W (reading R24): one array on A's
    pattern, strict lower part = L (unit diagonal implicit), the rest = U."""
    dt = wdtype(prec)
    aW = working_copy(A, prec)[0] if aW is None else _c(aW, dt)
    f = np.empty(A.nnz, dt)
    bad = np.zeros(1, np.int64)
    rc = lib().oracle_ilu0(prec, A.n, _p(A.row_ptr), _p(A.col), _p(aW), _p(f), _p(bad))
    if rc != 0:
        raise ZeroDivisionError(f"ILU(0): zero or missing pivot at row {int(bad[0])}")
    return f


def ilu0_apply(prec, A, f, z):
    """U⁻¹ L⁻¹ z in W (forward, then backward substitution)."""
    dt = wdtype(prec)
    out = np.empty(A.n, dt)
    lib().oracle_ilu0_apply(prec, A.n, _p(A.row_ptr), _p(A.col), _p(_c(f, dt)), _p(_c(z, dt)), _p(out))
    return out


def jacobi_spmv(prec, A, aW, dinvW, v):
    dt = wdtype(prec)
    w = np.empty(A.n, dt)
    lib().oracle_jacobi_spmv(prec, A.n, _p(A.row_ptr), _p(A.col), _p(_c(aW, dt)), _p(_c(dinvW, dt)),
                             _p(_c(v, dt)), _p(w))
    return w


def resid(prec, A, b, x, dinvW):
    dt = wdtype(prec)
    r = np.empty(A.n, dt)
    zz = np.zeros(1); rr = np.zeros(1)
    rc = lib().oracle_resid(prec, A.n, _p(A.row_ptr), _p(A.col), _p(_c(A.val, np.float64)),
                            _p(_c(b, np.float64)), _p(_c(x, np.float64)), _p(_c(dinvW, dt)), _p(r), _p(zz), _p(rr))
    return rc, r, float(zz[0]), float(rr[0])


def dot(prec, x, y):
    dt = wdtype(prec)
    x, y = _c(x, dt), _c(y, dt)
    return lib().oracle_dot(prec, x.size, _p(x), _p(y))


def _colmajor(V, dt):
    """V given as (n, j) array → column-major buffer with ld = n."""
    return np.asfortranarray(V, dtype=dt)


def mgs(prec, V, w):
    dt = wdtype(prec)
    n, j = V.shape
    Vc = _colmajor(V, dt)
    w2 = _c(w, dt).copy()
    h = np.zeros(j)
    lib().oracle_mgs(prec, n, j, _p(Vc), n, _p(w2), _p(h))
    return w2, h


def cgsr(prec, V, w, passes=2):
    dt = wdtype(prec)
    n, j = V.shape
    Vc = _colmajor(V, dt)
    w2 = _c(w, dt).copy()
    h = np.zeros(j)
    lib().oracle_cgsr(prec, n, j, _p(Vc), n, _p(w2), _p(h), passes)
    return w2, h


def scale(prec, w, inv):
    dt = wdtype(prec)
    w = _c(w, dt)
    v = np.empty_like(w)
    lib().oracle_scale(prec, w.size, _p(w), float(inv), _p(v))
    return v


def givens(a, b):
    c = np.zeros(1); s = np.zeros(1); r = np.zeros(1)
    lib().oracle_givens(float(a), float(b), _p(c), _p(s), _p(r))
    return float(c[0]), float(s[0]), float(r[0])


def hess_step(j, h, cs, sn, s):
    """In-place a6 step on float64 arrays; returns |s_{j+1}|."""
    return lib().oracle_hess_step(j, _p(h), _p(cs), _p(sn), _p(s))


def backsolve(R, s):
    """R: (J, J) upper triangular (any layout), s: (J,) → y."""
    J = R.shape[0]
    Rc = np.asfortranarray(R, dtype=np.float64)
    y = np.zeros(J)
    rc = lib().oracle_backsolve(J, _p(Rc), J, _p(_c(s, np.float64)), _p(y))
    if rc != 0:
        raise ZeroDivisionError("singular R")
    return y


def xupdate(prec, V, y, x):
    dt = wdtype(prec)
    n, J = V.shape
    Vc = _colmajor(V, dt)
    x2 = _c(x, np.float64).copy()
    lib().oracle_xupdate(prec, n, J, _p(Vc), n, _p(_c(y, np.float64)), _p(x2))
    return x2


@dataclass
class Cycle:
    V: np.ndarray      # (n, J+1) W
    Hbar: np.ndarray   # (J+1, J) unrotated
    R: np.ndarray      # (J+1, J) rotated
    s: np.ndarray      # (J+1,)
    J: int
    breakdown: bool
    inner: np.ndarray  # (J,) |s_{j+1}|/β


def arnoldi(prec, ortho, A, r, m, thr=0.0, flags=0, aW=None, dinvW=None):
    dt = wdtype(prec)
    if aW is None:
        aW, dinvW = working_copy(A, prec)
    n = A.n
    V = np.zeros((m + 1) * n, dt)
    Hbar = np.zeros((m + 1) * m); R = np.zeros((m + 1) * m); s = np.zeros(m + 1)
    J = np.zeros(1, np.int32); bd = np.zeros(1, np.int32); ih = np.zeros(m)
    rc = lib().oracle_arnoldi(prec, ortho, flags, n, _p(A.row_ptr), _p(A.col), _p(_c(aW, dt)), _p(_c(dinvW, dt)),
                              _p(_c(r, dt)), m, float(thr), _p(V), n, _p(Hbar), _p(R), _p(s), _p(J), _p(bd), _p(ih))
    if rc != 0:
        raise RuntimeError(f"oracle_arnoldi rc={rc}")
    Jn = int(J[0])
    Vm = V.reshape(m + 1, n).T
    Hm = Hbar.reshape(m, m + 1).T
    Rm = R.reshape(m, m + 1).T
    return Cycle(Vm[:, :Jn + 1].copy(), Hm[:Jn + 1, :Jn].copy(), Rm[:Jn + 1, :Jn].copy(), s[:Jn + 1].copy(),
                 Jn, bool(bd[0]), ih[:Jn].copy())


@dataclass
class SolveResult:
    status: int
    x: np.ndarray
    cycles: int
    inner_iters: int
    history: np.ndarray
    inner: np.ndarray
    final_relres: float


THRESHOLD, TWOSTAGE, STALL, ORTHLOSS = 0, 1, 2, 3   # restart policies (oracle.h; R6, R22, R23)


def solve(A, b, x0=None, m=30, tol=1e-10, ortho=CGSR, prec=MIXED, delta=None, max_cycles=10000, flags=0,
          inner_cap=200000, policy=THRESHOLD, stall_factor=1.001, stall_frac=0.05, orth_kind=0, orth_thresh=1.0):
    if delta is None:
        delta = 1e-6 if (prec == MIXED and policy != STALL) else 0.0
    n = A.n
    x = np.zeros(n)
    hist = np.zeros(max_cycles + 2)
    inner = np.zeros(inner_cap)
    res = _Result()
    x0c = None if x0 is None else _c(x0, np.float64)
    orth = np.zeros(inner_cap)
    rc = lib().oracle_gmres_solve_orth(n, _p(A.row_ptr), _p(A.col), _p(_c(A.val, np.float64)),
                                       _p(_c(b, np.float64)), _p(x0c), _p(x), m, tol, ortho, prec, delta,
                                       max_cycles, flags, ctypes.byref(res), _p(hist), hist.size, _p(inner),
                                       inner.size, int(policy), float(stall_factor), float(stall_frac),
                                       int(orth_kind), float(orth_thresh), _p(orth), orth.size)
    if rc < 0:
        raise RuntimeError(f"oracle_gmres_solve error {rc}")
    out = SolveResult(rc, x, res.cycles, res.inner_iters, hist[:min(res.history_len, hist.size)].copy(),
                      inner[:min(res.inner_len, inner.size)].copy(), res.final_relres)
    out.orth = orth[:min(res.inner_len, orth.size)].copy() if policy == ORTHLOSS else None
    return out


def backward_error(A, b, x):
    """Normwise backward error ‖b − A x‖₂ / (‖A‖_F ‖x‖₂ + ‖b‖₂) (the paper's
    stopping metric at PAPER.md:317, 431-433 is named but not defined — reading Q5/Q17).
    Report only; the stop test is ‖b − Ax‖/‖b‖ (reading R5).  Pins: tests/test_oracle.py."""
    z = np.asarray(b, np.float64) - spmv64(A, x)
    na = float(np.sqrt(np.sum(np.asarray(A.val, np.float64) ** 2)))
    den = na * float(np.linalg.norm(x)) + float(np.linalg.norm(b))
    return float(np.linalg.norm(z) / den) if den > 0 else 0.0
