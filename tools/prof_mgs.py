"""Profile-slot breakdown of the MGS ortho phase (dev tool): prof_mgs.py [lib.so] [C2] [scale]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    G._LIB_PATH = os.path.abspath(sys.argv[1]); sys.argv.pop(1)
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else None
P = inputs.make(name, scale)
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
for prec in (G.MIXED, G.FP64):
    for prof in (False, True):
        best = None
        for _ in range(2):
            x = torch.zeros_like(b)
            r = S.solve_device(b, x, m=P.m, ortho=G.MGS, precision=prec, profile=prof, tune=int(os.environ.get("TUNE", "0")))
            if best is None or r.kernel_ms < best.kernel_ms: best = r
        ph = best.phase_ns / 1e6
        print(f"{G._LIB_PATH.split('/')[-1]} {name} {'mixed' if prec else 'fp64'} prof={int(prof)} st={best.status} cyc={best.cycles} "
              f"kern={best.kernel_ms:.2f} ms  spmv={ph[1]:.1f} ortho={ph[2]:.1f} s8={ph[8]:.1f} dot={ph[9]:.1f} red+upd={ph[10]:.1f} ar_n={int(best.phase_ns[13])} skew_us={best.phase_ns[11]/max(1,best.phase_ns[13])/1e3:.2f} prop_us={best.phase_ns[12]/max(1,best.phase_ns[13])/1e3:.2f}", flush=True)
