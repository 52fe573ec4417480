"""ILU(0)-preconditioned solve timings vs Jacobi on one config (dev tool): ilu_time.py [C2] [scale]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else None
P = inputs.make(name, scale)
S = G.Solver.from_csr(P.A)
print(name, "n", P.A.n, "levels", S.ilu0_levels(), flush=True)
b = torch.from_numpy(P.b).cuda()
for prec in (G.MIXED, G.FP64):
    for ortho in (G.MGS, G.CGSR):
        for pc in (G.JACOBI, G.ILU0):
            best = None
            for _ in range(2):
                x = torch.zeros_like(b)
                r = S.solve_device(b, x, m=P.m, ortho=ortho, precision=prec, precond=pc)
                if best is None or r.device_ms < best.device_ms: best = r
            r = best
            print(f"{'mixed' if prec else 'fp64 '} {'MGS ' if ortho == 0 else 'CGSR'} {'ILU0' if pc else 'Jac '} st={r.status} "
                  f"cyc={r.cycles} inner={r.inner_iters} tts={r.device_ms:9.2f} ms kern={r.kernel_ms:9.2f} ms "
                  f"per-iter={1e3 * r.kernel_ms / max(1, r.inner_iters):8.1f} us relres={r.final_relres:.2e}", flush=True)
