"""Build libgmres.so (the C-ABI library) in-tree with nvcc for sm_100a.

The device code is one header (csrc/gmres_kernels.cuh); its template
instantiations are spread over several translation units (csrc/ks_*.cu,
csrc/kc_*.cu — see csrc/ktab.h) that are compiled in parallel and linked with
the host side (csrc/gmres_capi.cu) into one shared library with a static cudart.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.environ.get("G200_OBJ_DIR") or os.path.join(HERE, "_obj")
LIB = os.environ.get("G200_LIB_OUT") or os.path.join(HERE, "libgmres.so")
SOURCES = [os.path.join(CSRC, "gmres_capi.cu")] + sorted(glob.glob(os.path.join(CSRC, "ks_*.cu"))) + \
    sorted(glob.glob(os.path.join(CSRC, "kc_*.cu")))
HEADERS = [os.path.join(CSRC, "gmres_kernels.cuh"), os.path.join(CSRC, "ktab.h"), os.path.join(ROOT, "include", "gmres.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
] + os.environ.get("G200_DEFINES", "").split()  # dev A/B builds only (e.g. -DG200_NTB=3)


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.splitext(os.path.basename(src))[0] + ".o")


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in deps)


def stale() -> bool:
    return _stale(LIB, SOURCES + HEADERS)


def _compile(src: str, verbose: bool) -> str:
    out = _obj(src)
    cmd = [nvcc()] + NVCC_FLAGS + (["-Xptxas=-v"] if verbose else []) + \
        ["-I", os.path.join(ROOT, "include"), "-c", "-o", out, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    msg = (r.stdout + r.stderr).strip()
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{msg}")
    return msg


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    todo = [s for s in SOURCES if force or _stale(_obj(s), [s] + HEADERS)]
    print(f"[build] nvcc {' '.join(ARCH)}: {len(todo)} of {len(SOURCES)} translation units", file=sys.stderr)
    jobs = int(os.environ.get("G200_BUILD_JOBS", "0")) or max(1, min(len(todo), os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(jobs) as ex:
        for src, msg in zip(todo, ex.map(lambda s: _compile(s, verbose), todo)):
            if msg:
                print(f"[build] {os.path.basename(src)}:\n{msg}", file=sys.stderr)
    cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + [_obj(s) for s in SOURCES]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="-f" in sys.argv or "-v" in sys.argv, verbose="-v" in sys.argv)
