"""Small solves covering every phase (both streams, both layouts, MGS resident and sweep,
all policies, virtual ranks) for compute-sanitizer runs (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs
from paper_2011_01850_b200 import gmres as G
cases = [("C1", None, 20), ("C2", 12, 20), ("C3", 3000, 20), ("C4", 8, 20)]
for name, scale, m in cases:
    P = inputs.make(name, scale)
    S = G.Solver.from_csr(P.A)
    b = torch.from_numpy(P.b).cuda()
    for prec in (G.MIXED, G.FP64):
        for ortho in (G.MGS, G.CGSR):
            for policy in (0, 1, 2, 3):
                if policy == 3 and ortho == G.CGSR:
                    continue
                x = torch.zeros_like(b)
                r = S.solve_device(b, x, m=m, ortho=ortho, precision=prec, policy=policy, max_cycles=3,
                                   tune=4 if (name == "C2" and ortho == G.MGS and policy == 1) else 0)
                print(name, prec, ortho, policy, r.status, r.cycles, flush=True)
    S.close()
P = inputs.make("C2", 16)
A = P.A
bounds = G.dist_partition(A.row_ptr, 2, 256)
Ss = [G.Solver.from_csr_dist(rp, c, v, A.n, bounds[q], 2, q) for q, (rp, c, v) in enumerate(G.split_rows(A, bounds))]
G.link_local(Ss)
bs = [torch.from_numpy(P.b[bounds[q]:bounds[q + 1]].copy()).cuda() for q in range(2)]
xs = [torch.zeros_like(t) for t in bs]
r = G.solve_virtual(Ss, bs, xs, m=20, ortho=G.CGSR, precision=G.MIXED, max_cycles=3)
print("virtual", r[0].status, r[0].cycles)
torch.cuda.synchronize()
print("DONE")
