"""Full-size oracle records (VERDICT r1 'next' 1b): run the CPU oracle — and ONLY
the oracle (oracle/ + the seeded generators in inputs/) — on the full BASELINE.json
configs and write one JSON per case to tests/golden/full_size/<case>.json.

    OMP_NUM_THREADS=4 python tools/make_golden.py C4 [C2 C3 C5 C1 ...]

Uses oracle.use_omp(): the OpenMP build of oracle/oracle.cpp, bitwise equal to the
single-threaded build (only element-parallel loops are threaded; every reduction
is sequential — tests/test_oracle.py::test_omp_build_bitwise).  Recorded per case:
cycles, inner iterations, the per-cycle residual history, the final relative
residual recomputed with the oracle's fp64 SpMV, the SPEC normwise backward error
(S:96), wall time and the threads used.  tests/test_gpu_parity.py asserts the GPU's
restart counts against these files (BASELINE.json: "restart count within ±10 % of
the oracle's").
"""
import hashlib
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import inputs  # noqa: E402
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "full_size")

# (config, m values) — C5 is the C2 matrix at the restart-length sweep of BASELINE.json configs[4]
CASES = {
    "C1": [30], "C2": [50], "C3": [50], "C4": [100], "C5": [10, 25, 100, 200],
}


def case_key(cfg, prec, ortho, m):
    return f"{cfg}_{'mixed' if prec == O.MIXED else 'fp64'}_{'mgs' if ortho == O.MGS else 'cgsr'}_m{m}"


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(cfg, only=None):
    P = inputs.make(cfg)
    src = open(os.path.join(os.path.dirname(O.__file__), "oracle.cpp"), "rb").read()
    for m in CASES[cfg]:
        for prec in (O.MIXED, O.FP64):
            for ortho in (O.MGS, O.CGSR):
                key = case_key(cfg, prec, ortho, m)
                path = os.path.join(OUT, key + ".json")
                if os.path.exists(path) or (only and key not in only):
                    continue
                t0 = time.time()
                r = O.solve(P.A, P.b, m=m, tol=P.tol, ortho=ortho, prec=prec, inner_cap=1)
                dt = time.time() - t0
                z = P.b - O.spmv64(P.A, r.x)
                relres = float(np.linalg.norm(z) / np.linalg.norm(P.b))
                rec = {
                    "case": key, "config": cfg, "n": P.A.n, "nnz": P.A.nnz, "m": m, "tol": P.tol,
                    "precision": "mixed" if prec == O.MIXED else "fp64", "ortho": "mgs" if ortho == O.MGS else "cgsr",
                    "delta": 1e-6 if prec == O.MIXED else 0.0, "status": r.status, "cycles": r.cycles,
                    "inner_iters": r.inner_iters, "history": [float(v) for v in r.history],
                    "final_relres_recomputed": relres, "backward_err": O.backward_error(P.A, P.b, r.x),
                    "seconds": dt, "threads": int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count(),
                    "build": "liboracle_omp.so (bitwise equal to liboracle.so)", "host_cpu": cpu_model(),
                    "oracle_cpp_sha256": hashlib.sha256(src).hexdigest(),
                    "generator": f"inputs.make({cfg!r})",
                }
                with open(path + ".tmp", "w") as f:
                    json.dump(rec, f, indent=1)
                os.replace(path + ".tmp", path)
                print(key, r.status, r.cycles, r.inner_iters, f"{relres:.3e}", f"{dt:.1f}s", flush=True)


if __name__ == "__main__":
    O.use_omp(True)
    os.makedirs(OUT, exist_ok=True)
    args = sys.argv[1:] or list(CASES)
    cfgs = [a for a in args if a in CASES]
    only = [a for a in args if a not in CASES] or None
    for c in cfgs:
        run(c, only)
