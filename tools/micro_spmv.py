"""SpMV-phase microbenchmark over tune settings (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, inputs
from paper_2011_01850_b200 import gmres as G
P = inputs.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
n = P.A.n; nnz = P.A.nnz; S = G.Solver.from_csr(P.A); ld = G.ld_for(n)
tunes = [int(t) for t in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["512", "0", str(1 << 12), str(2 << 12), str(5 << 12), str(7 << 12)])]
for prec, wb, dt in ((G.MIXED, 4, torch.float32), (G.FP64, 8, torch.float64)):
    V = torch.rand(3, ld, dtype=dt, device="cuda") * 1e-3
    w = torch.rand(ld, dtype=dt, device="cuda")
    for tune in tunes:
        it = 50
        r = []
        for what, extra in ((6, 2 * wb * n), (7, 3 * wb * n), (8, 4 * wb * n)):
            ns = S.k_micro(prec, what | (tune << 8), it, 1, V, ld, w) / it
            r.append(f"what{what} {ns/1e3:6.1f}us {((wb+4)*nnz+4*n+extra)/ns:5.0f}GB/s")
        print(f"prec={prec} tune={tune:6d} " + "  ".join(r))
