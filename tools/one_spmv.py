import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
P = inputs.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
S = G.Solver.from_csr(P.A)
v = torch.rand(P.A.n, dtype=torch.float32, device="cuda"); w = torch.empty_like(v)
for _ in range(3): S.k_spmv(G.MIXED, v, w)
torch.cuda.synchronize(); print("ok")
