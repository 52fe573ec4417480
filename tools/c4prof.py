"""C4 MGS A/B of library builds and tune bits (dev tool):
   c4prof.py [lib.so] [tune ...] — mixed and fp64 MGS kernel time and phases (profile=PROF env)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    G._LIB_PATH = os.path.abspath(sys.argv.pop(1))
tunes = [int(t) for t in sys.argv[1:]] or [0]
prof = bool(int(os.environ.get("PROF", "0")))
P = inputs.make(os.environ.get("CFG", "C4"))
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
for tune in tunes:
    for prec in (G.MIXED, G.FP64):
        x = torch.zeros_like(b)
        r = S.solve_device(b, x, m=P.m, ortho=G.MGS, precision=prec, profile=prof, tune=tune)
        print(f"{os.path.basename(G._LIB_PATH)} tune={tune} {'mixed' if prec else 'fp64'} st={r.status} cyc={r.cycles} "
              f"inner={r.inner_iters} kern={r.kernel_ms:.1f}ms relres={r.final_relres:.2e} phases(ms)="
              + " ".join(f"{v/1e6:.1f}" for v in r.phase_ns[:14]), flush=True)
