"""ctypes binding for include/gmres.h (argument marshalling only).

Names follow the C ABI: ``Solver`` wraps ``gmres_create``/``gmres_destroy``;
``Solver.solve`` → ``gmres_solve`` (host numpy arrays), ``Solver.solve_device``
→ ``gmres_solve_device`` (torch CUDA tensors, current stream); ``k_*`` are the
per-step component entry points used by the parity tests.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("G200_LIB") or os.path.join(_HERE, "libgmres.so")  # (G200_LIB: dev A/B builds)
_lib = None

MGS, CGSR = 0, 1
JACOBI, ILU0, ILU0_FP32 = 0, 1, 2   # preconditioners (gmres_opts.precond; ILU0_FP32: fp64 solver, fp32 ILU)
THRESHOLD, TWOSTAGE, STALL, ORTHLOSS = 0, 1, 2, 3   # restart policies (gmres_opts.restart_policy)
FROBENIUS, SPECTRAL = 0, 1                          # gmres_opts.orth_norm (policy 3)
FP64, MIXED = 0, 1
STATUS = {0: "OK", 1: "NOT_CONVERGED", -1: "EINVAL", -2: "EBADCSR", -3: "EZERODIAG", -4: "EFP32RANGE",
          -5: "ENONFINITE", -6: "ENOMEM", -7: "ECUDA", -8: "ETIMEOUT"}


class GmresError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class _Result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("cycles", ctypes.c_int32), ("inner_iters", ctypes.c_int32),
                ("history_len", ctypes.c_int32), ("final_relres", ctypes.c_double), ("device_ms", ctypes.c_double),
                ("kernel_ms", ctypes.c_double), ("final_backward_err", ctypes.c_double)]


class _Opts(ctypes.Structure):
    _fields_ = [("delta", ctypes.c_double), ("max_cycles", ctypes.c_int32), ("record_inner", ctypes.c_int32),
                ("lanes_per_row", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32), ("profile", ctypes.c_int32),
                ("tune", ctypes.c_int32), ("restart_policy", ctypes.c_int32), ("stall_factor", ctypes.c_double),
                ("stall_frac", ctypes.c_double), ("orth_thresh", ctypes.c_double), ("precond", ctypes.c_int32),
                ("orth_norm", ctypes.c_int32)]


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libgmres.so; raise if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA library is required; there is no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    pR, pO = ctypes.POINTER(_Result), ctypes.POINTER(_Opts)
    L.gmres_create.argtypes = [vp, vp, vp, i64, i64, ctypes.POINTER(vp)]
    L.gmres_create.restype = ctypes.c_int
    L.gmres_solve.argtypes = [vp, vp, vp, vp, i32, dbl, i32, i32, pO, pR, vp, i32, ctypes.POINTER(i32)]
    L.gmres_solve.restype = ctypes.c_int
    L.gmres_solve_device.argtypes = [vp, vp, vp, vp, i32, dbl, i32, i32, pO, pR, vp, i32, ctypes.POINTER(i32), vp]
    L.gmres_solve_device.restype = ctypes.c_int
    L.gmres_get_inner_history.argtypes = [vp, vp, i32, ctypes.POINTER(i32)]
    L.gmres_get_inner_history.restype = ctypes.c_int
    L.gmres_get_cycle_iters.argtypes = [vp, vp, i32, ctypes.POINTER(i32)]
    L.gmres_get_cycle_iters.restype = ctypes.c_int
    L.gmres_get_phase_ns.argtypes = [vp, vp, i32]
    L.gmres_get_plan.argtypes = [vp, vp, i32]
    L.gmres_ilu0_factor.argtypes = [vp, i32, vp]
    L.gmres_ilu0_factor.restype = ctypes.c_int
    L.gmres_k_ilu_apply.argtypes = [vp, i32, vp, vp, i32]
    L.gmres_k_ilu_apply.restype = ctypes.c_int
    L.gmres_ilu0_levels.argtypes = [vp, vp, vp]
    L.gmres_ilu0_levels.restype = ctypes.c_int
    L.gmres_get_plan.restype = ctypes.c_int
    L.gmres_get_basis.argtypes = [vp, i32, i32, vp, i64]
    L.gmres_get_basis.restype = ctypes.c_int
    L.gmres_get_phase_ns.restype = ctypes.c_int
    L.gmres_last_error.argtypes = [vp]
    L.gmres_last_error.restype = ctypes.c_char_p
    L.gmres_destroy.argtypes = [vp]
    L.gmres_destroy.restype = None
    L.gmres_k_spmv.argtypes = [vp, i32, vp, vp]
    L.gmres_k_resid.argtypes = [vp, i32, vp, vp, vp, vp]
    L.gmres_k_ortho.argtypes = [vp, i32, i32, i32, vp, i64, vp, vp]
    L.gmres_k_ortho_ex.argtypes = [vp, i32, i32, i32, vp, i64, vp, vp, i32, ctypes.POINTER(i32)]
    L.gmres_k_xupdate.argtypes = [vp, i32, i32, vp, i64, vp, vp, i32]
    L.gmres_k_hessenberg.argtypes = [vp, i32, i32, vp, dbl, vp, vp, vp]
    L.gmres_k_cast32.argtypes = [vp]
    for f in ("gmres_k_spmv", "gmres_k_resid", "gmres_k_ortho", "gmres_k_ortho_ex", "gmres_k_xupdate", "gmres_k_hessenberg",
              "gmres_k_cast32"):
        getattr(L, f).restype = ctypes.c_int
    p64 = ctypes.POINTER(i64)
    L.gmres_dist_partition.argtypes = [vp, i64, i32, i64, vp]
    L.gmres_dist_ghosts.argtypes = [vp, vp, i64, i64, vp, i64, p64]
    L.gmres_dist_sends.argtypes = [i64, i64, vp, i64, vp, i64, p64]
    L.gmres_plan_mtiles.argtypes = [vp, i64, vp, i32, vp, i64, p64, vp, vp, i64, p64, vp]
    L.gmres_create_dist.argtypes = [vp, vp, vp, i64, i64, i64, i32, i32, ctypes.POINTER(vp)]
    L.gmres_dist_export.argtypes = [vp, vp, i64, p64]
    L.gmres_dist_import.argtypes = [vp, vp, vp]
    L.gmres_dist_link_local.argtypes = [vp, i32]
    L.gmres_solve_virtual.argtypes = [vp, i32, vp, vp, vp, i32, dbl, i32, i32, pO, vp]
    for f in ("gmres_dist_partition", "gmres_dist_ghosts", "gmres_dist_sends", "gmres_plan_mtiles", "gmres_create_dist",
              "gmres_dist_export", "gmres_dist_import", "gmres_dist_link_local", "gmres_solve_virtual"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(a.data_ptr())  # torch tensor


def _prec(p) -> int:
    if isinstance(p, str):
        return {"fp64": FP64, "mixed": MIXED}[p.lower()]
    return int(p)


def _ortho(o) -> int:
    if isinstance(o, str):
        return {"mgs": MGS, "cgsr": CGSR}[o.lower()]
    return int(o)


def ld_for(n: int) -> int:
    """Leading dimension the component entry points require for V (n rounded to 256)."""
    return (n + 255) // 256 * 256


@dataclass
class SolveResult:
    status: int
    cycles: int
    inner_iters: int
    final_relres: float
    device_ms: float
    history: np.ndarray
    kernel_ms: float = 0.0
    cycle_iters: np.ndarray | None = None
    x: object = None
    inner: np.ndarray | None = None
    phase_ns: np.ndarray | None = None
    meta: dict = field(default_factory=dict)
    final_backward_err: float = float("nan")

    @property
    def status_name(self) -> str:
        return STATUS.get(self.status, str(self.status))


class Solver:
    """gmres_create(csr_fp64) — copies A to the current CUDA device."""

    def __init__(self, row_ptr, col, val):
        self._lib = load_library()
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        self.n = self.row_ptr.shape[0] - 1
        self.nnz = int(col.shape[0])
        h = ctypes.c_void_p()
        rc = self._lib.gmres_create(_p(self.row_ptr), _p(col), _p(val), self.n, self.nnz, ctypes.byref(h))
        if rc != 0:
            raise GmresError(rc, self._lib.gmres_last_error(None).decode())
        self._h = h

    @classmethod
    def from_csr(cls, A):
        return cls(A.row_ptr, A.col, A.val)

    @classmethod
    def from_csr_dist(cls, row_ptr, col, val, n_global, row_begin, nranks, rank):
        """gmres_create_dist: this rank's rows (local CSR, global columns) of a row-partitioned matrix."""
        self = cls.__new__(cls)
        self._lib = load_library()
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        self.n = self.row_ptr.shape[0] - 1
        self.nnz = int(col.shape[0])
        self.row_begin, self.n_global, self.nranks, self.rank = int(row_begin), int(n_global), int(nranks), int(rank)
        h = ctypes.c_void_p()
        rc = self._lib.gmres_create_dist(_p(self.row_ptr), _p(col), _p(val), self.n_global, self.row_begin, self.n,
                                         self.nranks, self.rank, ctypes.byref(h))
        if rc != 0:
            raise GmresError(rc, self._lib.gmres_last_error(None).decode())
        self._h = h
        return self

    def export_blob(self) -> bytes:
        """gmres_dist_export: ghost list + CUDA IPC handles of this rank (to all-gather)."""
        ln = ctypes.c_int64()
        self._ck(self._lib.gmres_dist_export(self._h, None, 0, ctypes.byref(ln)))
        buf = np.zeros(ln.value, np.uint8)
        self._ck(self._lib.gmres_dist_export(self._h, _p(buf), buf.size, ctypes.byref(ln)))
        return buf.tobytes()

    def import_blobs(self, blobs):
        """gmres_dist_import: the blobs of all ranks, in rank order."""
        off = np.zeros(len(blobs) + 1, np.int64)
        off[1:] = np.cumsum([len(b) for b in blobs])
        cat = np.frombuffer(b"".join(blobs), np.uint8).copy()
        self._ck(self._lib.gmres_dist_import(self._h, _p(cat), _p(off)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.gmres_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self, rc):
        return GmresError(rc, self._lib.gmres_last_error(self._h).decode())

    @staticmethod
    def _opts(delta, max_cycles, record_inner, lanes, ctas_per_sm, profile=False, tune=0, policy=0,
              stall_factor=0.0, stall_frac=0.0, orth_thresh=0.0, precond=0, orth_norm=0):
        o = _Opts()
        o.orth_norm = int(orth_norm)
        o.precond = int(precond)
        o.orth_thresh = float(orth_thresh)
        o.restart_policy = int(policy)
        o.stall_factor = float(stall_factor)
        o.stall_frac = float(stall_frac)
        o.delta = -1.0 if delta is None else float(delta)
        o.max_cycles = 0 if max_cycles is None else int(max_cycles)
        o.record_inner = 1 if record_inner else 0
        o.lanes_per_row = int(lanes)
        o.ctas_per_sm = int(ctas_per_sm)
        o.profile = 1 if profile else 0
        o.tune = int(tune)
        return o

    def _finish(self, rc, res, hist, hl, record_inner):
        if rc < 0:
            raise self._err(rc)
        inner = None
        if record_inner:
            ln = ctypes.c_int32()
            self._lib.gmres_get_inner_history(self._h, None, 0, ctypes.byref(ln))
            inner = np.zeros(ln.value)
            self._lib.gmres_get_inner_history(self._h, _p(inner), ln.value, ctypes.byref(ln))
        ph = np.zeros(16)
        self._lib.gmres_get_phase_ns(self._h, _p(ph), 16)
        ln = ctypes.c_int32()
        self._lib.gmres_get_cycle_iters(self._h, None, 0, ctypes.byref(ln))
        cj = np.zeros(ln.value, np.int32)
        self._lib.gmres_get_cycle_iters(self._h, _p(cj), ln.value, ctypes.byref(ln))
        return SolveResult(res.status, res.cycles, res.inner_iters, res.final_relres, res.device_ms,
                           hist[:min(hl.value, hist.size)].copy(), kernel_ms=res.kernel_ms, cycle_iters=cj,
                           inner=inner, phase_ns=ph, final_backward_err=res.final_backward_err)

    def solve(self, b, x0=None, m=30, tol=1e-10, ortho=CGSR, precision=MIXED, delta=None, max_cycles=None,
              record_inner=False, lanes=0, ctas_per_sm=0, out=None, policy=THRESHOLD,
              orth_thresh=0.0, precond=0, tune=0, stall_factor=0.0, orth_norm=0) -> SolveResult:
        """gmres_solve: host arrays in, host x out (h2d/d2h inside the call).  `out` may be a
        preallocated (e.g. pinned) float64 array of length n."""
        b = np.ascontiguousarray(b, np.float64)
        x0c = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        if out is not None:
            assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == self.n
            x = out
        else:
            x = np.zeros(self.n)
        mc = 10000 if not max_cycles else int(max_cycles)
        hist = np.zeros(mc + 2)
        hl = ctypes.c_int32()
        res = _Result()
        o = self._opts(delta, max_cycles, record_inner, lanes, ctas_per_sm, tune=tune, policy=policy,
                       orth_thresh=orth_thresh, precond=precond, stall_factor=stall_factor, orth_norm=orth_norm)
        rc = self._lib.gmres_solve(self._h, _p(b), _p(x0c), _p(x), int(m), float(tol), _ortho(ortho),
                                   _prec(precision), ctypes.byref(o), ctypes.byref(res), _p(hist), hist.size,
                                   ctypes.byref(hl))
        out = self._finish(rc, res, hist, hl, record_inner)
        out.x = x
        return out

    def solve_device(self, b, x, x0=None, m=30, tol=1e-10, ortho=CGSR, precision=MIXED, delta=None,
                     max_cycles=None, record_inner=False, lanes=0, ctas_per_sm=0, stream=None,
                     profile=False, tune=0, policy=THRESHOLD, precond=0) -> SolveResult:
        """gmres_solve_device on torch CUDA float64 tensors (x is written in place).
        precond: JACOBI (0) or ILU0 (1, §8 f2)."""
        import torch
        for t in (b, x) + ((x0,) if x0 is not None else ()):
            assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and t.numel() == self.n
        st = stream if stream is not None else torch.cuda.current_stream()
        mc = 10000 if not max_cycles else int(max_cycles)
        hist = np.zeros(mc + 2)
        hl = ctypes.c_int32()
        res = _Result()
        o = self._opts(delta, max_cycles, record_inner, lanes, ctas_per_sm, profile, tune, policy, precond=precond)
        rc = self._lib.gmres_solve_device(self._h, _p(b), _p(x0), _p(x), int(m), float(tol), _ortho(ortho),
                                          _prec(precision), ctypes.byref(o), ctypes.byref(res), _p(hist), hist.size,
                                          ctypes.byref(hl), ctypes.c_void_p(st.cuda_stream))
        out = self._finish(rc, res, hist, hl, record_inner)
        out.x = x
        return out

    def ilu0_factor(self, precision):
        """gmres_ilu0_factor: ILU(0) factors of A_W on the device (torch tensor, nnz W values)."""
        import torch
        f = torch.empty(self.nnz, dtype=torch.float32 if precision == MIXED else torch.float64, device="cuda")
        rc = self._lib.gmres_ilu0_factor(self._h, _prec(precision), _p(f))
        if rc < 0:
            raise self._err(rc)
        return f

    def ilu_apply(self, z, precision, tune=0):
        """gmres_k_ilu_apply: U⁻¹L⁻¹ z with the last factors of this precision (torch tensors);
        tune bit 16 (65536): the level-synchronous schedule instead of the sync-free one."""
        import torch
        out = torch.empty_like(z)
        rc = self._lib.gmres_k_ilu_apply(self._h, _prec(precision), _p(z), _p(out), int(tune))
        if rc < 0:
            raise self._err(rc)
        return out

    def ilu0_levels(self):
        lo, up = ctypes.c_int32(), ctypes.c_int32()
        rc = self._lib.gmres_ilu0_levels(self._h, ctypes.byref(lo), ctypes.byref(up))
        if rc < 0:
            raise self._err(rc)
        return lo.value, up.value

    PLAN_KEYS = ("ctas", "lanes", "mgs_variant", "ring", "w_smem_chunks", "stage_bytes", "smem", "csr_stream",
                 "row_tile")

    def plan(self) -> dict:
        """Launch plan of the last solve (gmres_get_plan): grid, SpMV lanes, MGS variant, staging sizes."""
        buf = np.zeros(len(self.PLAN_KEYS), np.int32)
        k = self._lib.gmres_get_plan(self._h, _p(buf), len(buf))
        if k < 0:
            raise RuntimeError("gmres_get_plan failed")
        return dict(zip(self.PLAN_KEYS, buf[:k].tolist()))

    def basis(self, ncols, precision, col0=0):
        """gmres_get_basis: columns of the last solve's Krylov basis as a (ncols, n) torch tensor."""
        import torch
        dt = torch.float32 if _prec(precision) == MIXED else torch.float64
        out = torch.empty((int(ncols), self.n), dtype=dt, device="cuda")
        self._ck(self._lib.gmres_get_basis(self._h, int(col0), int(ncols), _p(out), self.n))
        return out

    # ------------------------------------------------------ components
    def _ck(self, rc):
        if rc != 0:
            raise self._err(rc)

    def k_cast32(self):
        self._ck(self._lib.gmres_k_cast32(self._h))

    def k_spmv(self, precision, v, w):
        self._ck(self._lib.gmres_k_spmv(self._h, _prec(precision), _p(v), _p(w)))

    def k_resid(self, precision, b, x, r):
        out = np.zeros(2)
        self._ck(self._lib.gmres_k_resid(self._h, _prec(precision), _p(b), _p(x), _p(r), _p(out)))
        return float(out[0]), float(out[1])

    def k_ortho(self, precision, ortho, j, V, ldv, w, mgs_variant=-1, return_variant=False):
        """gmres_k_ortho_ex: h_{1..j} and h[j] = ‖w‖ (w orthogonalised in place); mgs_variant −1 = the
        solve's choice, 0 sweep, 1 resident, 2 chunk ring, 3 streamed."""
        h = np.zeros(j + 1)
        used = ctypes.c_int32()
        self._ck(self._lib.gmres_k_ortho_ex(self._h, _prec(precision), _ortho(ortho), int(j), _p(V), int(ldv), _p(w),
                                            _p(h), int(mgs_variant), ctypes.byref(used)))
        return (h, used.value) if return_variant else h

    def k_xupdate(self, precision, J, V, ldv, y, x, blocked=False):
        y = np.ascontiguousarray(y, np.float64)
        self._ck(self._lib.gmres_k_xupdate(self._h, _prec(precision), int(J), _p(V), int(ldv), _p(y), _p(x),
                                           int(bool(blocked))))

    def k_hessenberg(self, m, J, Hbar, beta):
        Hc = np.asfortranarray(Hbar, np.float64)  # (m+1, m) column-major
        assert Hc.shape == (m + 1, m)
        R = np.zeros((m + 1) * m)
        s = np.zeros(J + 1)
        y = np.zeros(J)
        self._ck(self._lib.gmres_k_hessenberg(self._h, int(m), int(J), Hc.ctypes.data_as(ctypes.c_void_p),
                                              float(beta), _p(R), _p(s), _p(y)))
        return R.reshape(m, m + 1).T, s, y


# ------------------------------------------------------------ row partition (§8 e)
def dist_partition(row_ptr, nranks: int, align: int = 256) -> np.ndarray:
    """gmres_dist_partition: row boundaries [0, …, n] of an nnz-balanced split at multiples of align (host)."""
    L = load_library()
    rp = np.ascontiguousarray(row_ptr, np.int32)
    out = np.zeros(nranks + 1, np.int64)
    rc = L.gmres_dist_partition(_p(rp), rp.size - 1, int(nranks), int(align), _p(out))
    if rc != 0:
        raise GmresError(rc, L.gmres_last_error(None).decode())
    return out


def plan_mtiles(row_ptr, cta_rows):
    """gmres_plan_mtiles: merge-path tiles of a G-CTA row split (host) →
    (tiles (T, 4), tile_off (G+1), splits (S, 4), split_off (G+1))."""
    L = load_library()
    rp = np.ascontiguousarray(row_ptr, np.int32)
    rb = np.ascontiguousarray(cta_rows, np.int32)
    G = rb.size - 1
    nt, ns = ctypes.c_int64(), ctypes.c_int64()
    rc = L.gmres_plan_mtiles(_p(rp), rp.size - 1, _p(rb), G, None, 0, ctypes.byref(nt), None, None, 0,
                             ctypes.byref(ns), None)
    if rc != 0:
        raise GmresError(rc, L.gmres_last_error(None).decode())
    tiles = np.zeros((nt.value, 4), np.int32)
    splits = np.zeros((max(ns.value, 1), 4), np.int32)
    toff = np.zeros(G + 1, np.int32)
    soff = np.zeros(G + 1, np.int32)
    rc = L.gmres_plan_mtiles(_p(rp), rp.size - 1, _p(rb), G, _p(tiles), nt.value, ctypes.byref(nt), _p(toff),
                             _p(splits), ns.value, ctypes.byref(ns), _p(soff))
    if rc != 0:
        raise GmresError(rc, L.gmres_last_error(None).decode())
    return tiles, toff, splits[:ns.value], soff


def dist_ghosts(row_ptr, col, row_begin: int) -> np.ndarray:
    """gmres_dist_ghosts: sorted global columns of a rank's local rows outside them (host)."""
    L = load_library()
    rp = np.ascontiguousarray(row_ptr, np.int32)
    c = np.ascontiguousarray(col, np.int32)
    cnt = ctypes.c_int64()
    L.gmres_dist_ghosts(_p(rp), _p(c), rp.size - 1, int(row_begin), None, 0, ctypes.byref(cnt))
    out = np.zeros(cnt.value, np.int32)
    rc = L.gmres_dist_ghosts(_p(rp), _p(c), rp.size - 1, int(row_begin), _p(out), out.size, ctypes.byref(cnt))
    if rc != 0:
        raise GmresError(rc, L.gmres_last_error(None).decode())
    return out


def dist_sends(row_begin: int, n_local: int, peer_ghosts) -> np.ndarray:
    """gmres_dist_sends: this rank's local rows a peer gathers (host)."""
    L = load_library()
    pg = np.ascontiguousarray(peer_ghosts, np.int32)
    cnt = ctypes.c_int64()
    L.gmres_dist_sends(int(row_begin), int(n_local), _p(pg), pg.size, None, 0, ctypes.byref(cnt))
    out = np.zeros(cnt.value, np.int32)
    rc = L.gmres_dist_sends(int(row_begin), int(n_local), _p(pg), pg.size, _p(out), out.size, ctypes.byref(cnt))
    if rc != 0:
        raise GmresError(rc, L.gmres_last_error(None).decode())
    return out


def split_rows(A, bounds):
    """Local CSR pieces (row_ptr, col, val) of the row blocks [bounds[q], bounds[q+1]) (global columns)."""
    parts = []
    for q in range(len(bounds) - 1):
        r0, r1 = int(bounds[q]), int(bounds[q + 1])
        e0, e1 = int(A.row_ptr[r0]), int(A.row_ptr[r1])
        parts.append((A.row_ptr[r0:r1 + 1] - e0, A.col[e0:e1], A.val[e0:e1]))
    return parts


def link_local(solvers):
    """gmres_dist_link_local: in-process ranks on one device."""
    L = load_library()
    arr = (ctypes.c_void_p * len(solvers))(*[s._h.value for s in solvers])
    rc = L.gmres_dist_link_local(arr, len(solvers))
    if rc != 0:
        raise GmresError(rc, L.gmres_last_error(solvers[0]._h).decode())


def solve_virtual(solvers, bs, xs, x0s=None, m=30, tol=1e-10, ortho=CGSR, precision=MIXED, delta=None,
                  max_cycles=None, lanes=0, tune=0):
    """gmres_solve_virtual: all in-process ranks in one cooperative launch (torch float64 tensors)."""
    L = load_library()
    P = len(solvers)
    H = (ctypes.c_void_p * P)(*[s._h.value for s in solvers])
    B = (ctypes.c_void_p * P)(*[b.data_ptr() for b in bs])
    X = (ctypes.c_void_p * P)(*[x.data_ptr() for x in xs])
    X0 = None if x0s is None else (ctypes.c_void_p * P)(*[x.data_ptr() for x in x0s])
    res = (_Result * P)()
    o = Solver._opts(delta, max_cycles, False, lanes, 0, False, tune)
    rc = L.gmres_solve_virtual(H, P, B, X0, X, int(m), float(tol), _ortho(ortho), _prec(precision), ctypes.byref(o),
                               res)
    if rc < 0:
        raise GmresError(rc, L.gmres_last_error(solvers[0]._h).decode())
    return [SolveResult(r.status, r.cycles, r.inner_iters, r.final_relres, r.device_ms, np.zeros(0),
                        kernel_ms=r.kernel_ms) for r in res]
