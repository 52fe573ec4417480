"""Profile-slot breakdown of the streamed MGS (dev tool): prof_stream.py NAME [scale] [tune]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
name = sys.argv[1]; scale = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
tune = int(sys.argv[3]) if len(sys.argv) > 3 else 0
mc = int(sys.argv[4]) if len(sys.argv) > 4 else 1
P = inputs.make(name, scale)
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
for prec in (G.MIXED, G.FP64):
    for prof in (False, True):
        x = torch.zeros_like(b)
        r = S.solve_device(b, x, m=P.m, ortho=G.MGS, precision=prec, profile=prof, tune=tune, max_cycles=mc)
        ph = r.phase_ns / 1e6
        print(f"{name} {scale} {'mixed' if prec else 'fp64'} prof={int(prof)} plan={S.plan()} inner={r.inner_iters} kern={r.kernel_ms:.2f} ms "
              f"spmv={ph[1]:.1f} ortho={ph[2]:.1f} pump={ph[11]:.1f} wait={ph[12]:.1f} ar={ph[13]:.1f}", flush=True)
