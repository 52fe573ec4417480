"""Row-tile pass microbenchmark (dev tool): python tools/micro_tile.py [tune ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
P = inputs.make("C2")
n = P.A.n; S = G.Solver.from_csr(P.A); ld = G.ld_for(n)
tunes = [int(t) for t in sys.argv[1:]] or [0, 2048]
for prec, wb, dt in ((G.MIXED, 4, torch.float32), (G.FP64, 8, torch.float64)):
    V = torch.rand(51, ld, dtype=dt, device="cuda") * 1e-3
    w = torch.rand(ld, dtype=dt, device="cuda")
    for tune in tunes:
        out = []
        for nc in (10, 25, 50):
            for mode in (3, 4, 5):
                ns = S.k_micro(prec, mode | (tune << 8), 10, nc, V, ld, w) / 10
                out.append(f"M{mode-2}j{nc}:{nc*wb*n/ns:5.0f}")
        print(f"prec={prec} tune={tune:5d} GB/s(V once) " + " ".join(out))
