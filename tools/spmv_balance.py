"""Per-CTA SpMV time balance inside the solve (profile mode): max vs mean over CTAs (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
P = inputs.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
for prec in (G.MIXED, G.FP64):
    for tune in (0,):
        x = torch.zeros_like(b)
        r = S.solve_device(b, x, m=P.m, ortho=G.MGS, precision=prec, profile=True, max_cycles=2, tune=tune)
        ph = r.phase_ns / 1e6
        it = r.inner_iters
        print(f"{'mixed' if prec else 'fp64'} inner={it} spmv phase {ph[1]:.2f} ms = {1e3*ph[1]/it:.1f} us/iter; "
              f"per-CTA own spmv max {1e3*ph[5]/it:.1f} us, mean {1e3*ph[6]/it:.1f} us; plan {S.plan()}", flush=True)
