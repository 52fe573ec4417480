"""BASELINE.json C5: restart-length sweep on the 128³ 7-point matrix (1 GPU).

For m ∈ {10, 25, 50, 100, 200} × {MGS, CGSR} × {fp64, mixed (δ = 1e-6: restart after
each single-precision-accuracy gain)}: time to ‖b − Ax‖/‖b‖ ≤ 1e-10
(median of 3 after a warm-up, device time incl. the A32 cast), restart count, inner
iterations, and the loss of orthogonality ‖I − VᵀV‖ (Frobenius and max-abs) of the
first cycle's final basis — computed untimed from gmres_get_basis with an fp64 Gram
matrix.  Writes one JSON document (stdout, and the path given as argv[1]).
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2011_01850_b200 import gmres as G  # noqa: E402

P = inputs.make("C5")
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
x = torch.zeros_like(b)
rows = []
for m in (10, 25, 50, 100, 200):
    for ortho in (G.MGS, G.CGSR):
        for prec in (G.FP64, G.MIXED):
            S.solve_device(b, x, m=m, ortho=ortho, precision=prec)  # warm
            rs = [S.solve_device(b, x, m=m, ortho=ortho, precision=prec) for _ in range(3)]
            r = rs[-1]
            tts = statistics.median(q.device_ms for q in rs)
            # first cycle's basis (untimed)
            c1 = S.solve_device(b, x, m=m, ortho=ortho, precision=prec, max_cycles=1)
            J = int(c1.cycle_iters[0])
            V = S.basis(J, prec).double()            # J × n
            Gm = V @ V.T
            E = torch.eye(J, dtype=torch.float64, device=V.device) - Gm
            row = {"m": m, "ortho": "MGS" if ortho == G.MGS else "CGSR", "precision": "fp64" if prec == G.FP64 else "mixed",
                   "status": r.status, "tts_ms": tts, "cycles": r.cycles, "inner_iters": r.inner_iters,
                   "final_relres": r.final_relres, "first_cycle_J": J,
                   "orth_loss_fro": float(torch.linalg.norm(E)), "orth_loss_max": float(E.abs().max())}
            rows.append(row)
            print(json.dumps(row), flush=True)
for m in (10, 25, 50, 100, 200):
    for o in ("MGS", "CGSR"):
        t = {r["precision"]: r["tts_ms"] for r in rows if r["m"] == m and r["ortho"] == o}
        print(f"m={m:3d} {o:4s} mixed-over-fp64 TTS speedup {t['fp64'] / t['mixed']:.2f}", flush=True)
doc = {"config": "C5: C2's 7-pt 128^3 matrix, seed 1, tol 1e-10, Jacobi; 1 GPU", "rows": rows}
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(doc, f, indent=1)
