"""Host-side checks that need no GPU: the C-ABI library loads and exports every
symbol include/gmres.h declares; the product never touches the oracle; the
binding fails loudly without its library; no forbidden CUDA APIs are named."""
import ctypes
import importlib
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2011_01850_b200")
LIB = os.path.join(PKG, "libgmres.so")
HDR = os.path.join(ROOT, "include", "gmres.h")


def header_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gmres_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2011_01850_b200 import build
        build.build()
    return LIB


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("gmres_create", "gmres_solve", "gmres_solve_device", "gmres_destroy", "gmres_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gmres_[a-z0-9_]+)", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    L = ctypes.CDLL(lib)  # loads without a GPU (static cudart, no device call at load)
    for f in header_functions():
        assert hasattr(L, f)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_string_without_gpu(lib):
    L = ctypes.CDLL(lib)
    L.gmres_last_error.restype = ctypes.c_char_p
    L.gmres_create.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
    h = ctypes.c_void_p()
    # invalid CSR is rejected on the host before any device call
    import numpy as np
    rp = np.array([0, 2, 1], np.int32)
    col = np.array([0, 1], np.int32)
    val = np.ones(2)
    rc = L.gmres_create(rp.ctypes.data, col.ctypes.data, val.ctypes.data, 2, 2, ctypes.byref(h))
    assert rc == -2 and b"row_ptr" in L.gmres_last_error(None)


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), fn
                assert "liboracle" not in txt, fn


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2011_01850_b200 import gmres as G
    monkeypatch.setattr(G, "_LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(G, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        G.load_library()


def test_bench_byte_model_closed_form():
    # one full C2 cycle (J = m = 50), mixed MGS = 19.3 GB, CGSR = 42.4 GB
    import bench
    n, nnz = 2097152, 14581760
    one = bench.model_bytes(n, nnz, 4, 0, [50]) - (12 * nnz + 4 * (n + 1) + 16 * n + 8 * n)
    assert abs(one / 1e9 - 19.3) < 0.1
    one = bench.model_bytes(n, nnz, 4, 1, [50]) - (12 * nnz + 4 * (n + 1) + 16 * n + 8 * n)
    assert abs(one / 1e9 - 42.4) < 0.1
