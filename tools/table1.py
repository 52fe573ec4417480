"""Synthetic analogue of Table 1: iterations before
the Arnoldi residual stalls in the first three restart cycles of mixed-precision
MGS-GMRES with a fixed restart length, on the seeded synthetic matrices (the
paper's SuiteSparse matrices are not in this container).

Protocol (reading R22 / DESIGN.md §2): policy THRESHOLD with δ = 0 and no reachable
tolerance (1e-30, 3 cycles: restart at j = m exactly, as the paper's fixed-restart
convergence runs), the device's per-inner-step |s_{j+1}|/β recorded; "stall" = the
paper's definition: the first inner step i of a cycle after which the
next ⌈0.05·m⌉ steps improve the Arnoldi residual by less than a factor 1.001.  The
same from the CPU oracle on the same inputs.  Also the device's STALL restart policy
(the detector running inside the solve kernel): its first cycle lengths.

    python tools/table1.py [out.json]     (GPU; writes profiles/r02_table1.json)
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle as O  # noqa: E402
from paper_2011_01850_b200 import gmres as G  # noqa: E402

CASES = [("C1", 64, 250), ("C2", 32, 200), ("C4", 24, 150), ("C3", 30000, 60)]


def split_cycles(inner, lengths):
    out, k = [], 0
    for J in lengths:
        out.append(np.concatenate([[1.0], inner[k:k + J]]))
        k += J
    return out


def stall_point(h, m, f=1.001, frac=0.05):
    """First i with h[i + w]·f > h[i], w = ⌈frac·m⌉; None if no stall."""
    w = max(1, math.ceil(frac * m))
    for i in range(0, len(h) - w):
        if h[i + w] * f > h[i]:
            return i
    return None


def oracle_cycle_lengths(inner):
    """Cycle boundaries of the oracle's inner history: |s|/β restarts at 1 each cycle."""
    J, c = [], 0
    for t in range(len(inner)):
        if t > 0 and inner[t] > inner[t - 1] * (1 + 1e-12):
            J.append(c)
            c = 0
        c += 1
    J.append(c)
    return J


def run(name, scale, m):
    P = inputs.make(name, scale)
    S = G.Solver.from_csr(P.A)
    r = S.solve(P.b, m=m, tol=1e-30, ortho=G.MGS, precision=G.MIXED, delta=0.0, record_inner=True, max_cycles=3)
    ref = O.solve(P.A, P.b, m=m, tol=1e-30, ortho=O.MGS, prec=O.MIXED, delta=0.0, max_cycles=3)
    gpu = [stall_point(h, m) for h in split_cycles(r.inner, list(r.cycle_iters))[:3]]
    orc = [stall_point(h, m) for h in split_cycles(ref.inner, oracle_cycle_lengths(ref.inner))[:3]]
    st = S.solve(P.b, m=m, tol=1e-30, ortho=G.MGS, precision=G.MIXED, policy=G.STALL, max_cycles=3)
    st_o = O.solve(P.A, P.b, m=m, tol=1e-30, ortho=O.MGS, prec=O.MIXED, policy=O.STALL, max_cycles=3)
    return {"config": name, "scale": scale, "n": P.A.n, "m": m,
            "stall_iters_gpu": gpu, "stall_iters_oracle": orc,
            "cycles_gpu": r.cycles, "cycles_oracle": ref.cycles,
            "stall_policy_cycle_lengths_gpu": [int(v) for v in st.cycle_iters[:3]],
            "stall_policy_cycle_lengths_oracle": oracle_cycle_lengths(st_o.inner)[:3]}


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "r02_table1.json")
    rows = [run(*c) for c in CASES]
    for r in rows:
        print(r)
    with open(out, "w") as f:
        json.dump({"source": "tools/table1.py (PAPER.md:348-366, SURVEY.md §8 f4)", "rows": rows}, f, indent=1)
