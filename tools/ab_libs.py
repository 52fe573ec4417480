"""A/B of several builds of libgmres.so on C2 (dev tool): ab_libs.py lib1.so lib2.so ..."""
import sys, os, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2:  # one process per library (the binding loads one library per process)
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, lib], check=False)
    sys.exit(0)
import torch, inputs
from paper_2011_01850_b200 import gmres as G
G._LIB_PATH = os.path.abspath(sys.argv[1])
P = inputs.make("C2")
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
out = []
for prec in (G.MIXED, G.FP64):
    for ortho in (G.MGS, G.CGSR):
        best = None
        for _ in range(3):
            x = torch.zeros_like(b)
            r = S.solve_device(b, x, m=P.m, ortho=ortho, precision=prec)
            best = r.kernel_ms if best is None else min(best, r.kernel_ms)
        out.append(f"{'mix' if prec else 'f64'}-{'mgs' if ortho == 0 else 'cgsr'} {best:7.2f}")
print(os.path.basename(sys.argv[1]), " | ".join(out), flush=True)
