"""Quick per-variant timing of the fused solve on one config (dev tool)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs
from paper_2011_01850_b200 import gmres as G
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import model_bytes

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
scale = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
lanes = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(os.environ.get("REPS", "2"))
P = inputs.make(name, scale)
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda(); x = torch.zeros_like(b)
m = P.m
print(f"{name} n={P.A.n} nnz={P.A.nnz} m={m} lanes={lanes}")
for prec in (G.MIXED, G.FP64):
    for ortho in (G.MGS, G.CGSR):
        best = None
        for _ in range(reps):
            r = S.solve_device(b, x, m=m, ortho=ortho, precision=prec, lanes=lanes, profile=bool(int(os.environ.get("PROFILE", "0"))), tune=int(os.environ.get("TUNE", "0")))
            if best is None or r.kernel_ms < best.kernel_ms: best = r
        r = best
        wb = 4 if prec == G.MIXED else 8
        mb = model_bytes(P.A.n, P.A.nnz, wb, ortho, r.cycle_iters)
        ph = r.phase_ns[:5] / 1e6
        print(f"{'mixed' if prec else 'fp64 '} {'MGS ' if ortho == 0 else 'CGSR'} st={r.status} cyc={r.cycles} inner={r.inner_iters} "
              f"tts={r.device_ms:8.2f}ms kern={r.kernel_ms:8.2f}ms model={mb/1e9:7.1f}GB -> {mb/r.kernel_ms/1e6:7.0f} GB/s  "
              f"per-iter {r.kernel_ms/r.inner_iters*1e3:6.1f}us  phases resid/spmv/ortho/givens/upd(ms) "
              + " ".join(f"{v:.1f}" for v in ph) + f" relres={r.final_relres:.2e}"
              + (f" spmv/CTA max {r.phase_ns[5]/1e6:.1f} mean {r.phase_ns[6]/1e6:.1f}ms" if r.phase_ns[5] else "")
              + (" sub(ms) " + " ".join(f"{v/1e6:.1f}" for v in r.phase_ns[8:14]) if r.phase_ns[8] else ""))
