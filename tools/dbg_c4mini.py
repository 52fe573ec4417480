"""C4mini fp64 MGS debugging (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs, oracle as O
from paper_2011_01850_b200 import gmres as G
P = inputs.make("C4", 20)
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
for prec in (G.FP64, G.MIXED):
    for ortho in (G.MGS, G.CGSR):
        for tune in (0, 4, 256):
            x = torch.zeros_like(b)
            r = S.solve_device(b, x, m=50, ortho=ortho, precision=prec, tune=tune, max_cycles=40)
            print(prec, ortho, tune, r.status, r.cycles, r.inner_iters, f"{r.final_relres:.2e}", list(r.cycle_iters[:4]))
ref = O.solve(P.A, P.b, m=50, ortho=O.MGS, prec=O.FP64)
print("oracle", ref.cycles, ref.inner_iters)
