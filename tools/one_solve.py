"""One fused solve of a config/variant (for ncu captures): python tools/one_solve.py C2 mixed cgsr [max_cycles] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
name = sys.argv[1]; prec = G.MIXED if sys.argv[2] == "mixed" else G.FP64
ortho = G.MGS if sys.argv[3] == "mgs" else G.CGSR
mc = int(sys.argv[4]) if len(sys.argv) > 4 else 1
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
P = inputs.make(name)
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda(); x = torch.zeros_like(b)
for _ in range(reps):
    r = S.solve_device(b, x, m=P.m, ortho=ortho, precision=prec, max_cycles=mc)
print(name, sys.argv[2], sys.argv[3], "status", r.status, "cycles", r.cycles, "inner", r.inner_iters, "kernel_ms", r.kernel_ms)
