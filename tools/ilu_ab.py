"""ILU apply A/B: per-inner-iteration time of one 50-step cycle with and without the row work (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
P = inputs.make("C2")
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
for ortho in (G.MGS, G.CGSR):
    for prec in (G.MIXED, G.FP64):
        for tune in (0, 65536):
            x = torch.zeros_like(b)
            r = S.solve_device(b, x, m=50, ortho=ortho, precision=prec, precond=G.ILU0, max_cycles=1, delta=0.0,
                               tol=1e-30, tune=tune)
            x = torch.zeros_like(b)
            r = S.solve_device(b, x, m=50, ortho=ortho, precision=prec, precond=G.ILU0, max_cycles=1, delta=0.0,
                               tol=1e-30, tune=tune)
            print(f"{'MGS ' if ortho == 0 else 'CGSR'} {'mixed' if prec else 'fp64 '} tune={tune:5d} inner={r.inner_iters} "
                  f"kern={r.kernel_ms:8.2f} ms  per-iter={1e3 * r.kernel_ms / max(1, r.inner_iters):8.1f} us  plan={S.plan()['mgs_variant']},{S.plan()['smem']}",
                  flush=True)
