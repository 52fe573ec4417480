"""In-kernel microbenchmarks of barrier / all-reduce / MGS sweep / tile passes (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs
TUNE = int(os.environ.get('TUNE', '0'))
TUNE = int(os.environ.get('TUNE', '0'))
from paper_2011_01850_b200 import gmres as G
P = inputs.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
n = P.A.n; S = G.Solver.from_csr(P.A); ld = G.ld_for(n)
for prec, wb, dt in ((G.MIXED, 4, torch.float32), (G.FP64, 8, torch.float64)):
    V = torch.rand(51, ld, dtype=dt, device="cuda") * 1e-3
    w = torch.rand(ld, dtype=dt, device="cuda")
    it = 200
    ns = S.k_micro(prec, 0 | (TUNE << 8), it, 1, V, ld, w); print(f"prec={prec} grid barrier      {ns/it/1e3:7.2f} us")
    ns = S.k_micro(prec, 1 | (TUNE << 8), it, 1, V, ld, w); print(f"prec={prec} allreduce(1)      {ns/it/1e3:7.2f} us")
    ns = S.k_micro(prec, 2 | (TUNE << 8), it, 1, V, ld, w); print(f"prec={prec} mgs sweep         {ns/it/1e3:7.2f} us  {3*wb*n/(ns/it):7.0f} GB/s (3 vectors)")
    it = 50
    nnz = P.A.nnz
    ns = S.k_micro(prec, 6 | (TUNE << 8), it, 1, V, ld, w); print(f"prec={prec} csr stream (no gather) {ns/it/1e3:7.2f} us  {((wb+4)*nnz+4*n+2*wb*n)/(ns/it):7.0f} GB/s")
    ns = S.k_micro(prec, 7 | (TUNE << 8), it, 1, V, ld, w); print(f"prec={prec} spmv phase (L=1)     {ns/it/1e3:7.2f} us  {((wb+4)*nnz+4*n+3*wb*n)/(ns/it):7.0f} GB/s")
    ns = S.k_micro(prec, 8 | (TUNE << 8), it, 1, V, ld, w); print(f"prec={prec} spmv phase + vcol    {ns/it/1e3:7.2f} us  {((wb+4)*nnz+4*n+4*wb*n)/(ns/it):7.0f} GB/s")
    if os.environ.get("ONLY_SPMV"): continue
    for nc in (1, 10, 25, 50):
        for mode in (3, 4, 5):
            ns = S.k_micro(prec, mode, 20, nc, V, ld, w)
            t = ns / 20
            byt = (nc + 1) * wb * n + (0 if mode == 3 else wb * n)
            print(f"prec={prec} tile MODE{mode-2} j={nc:3d} {t/1e3:8.1f} us  {byt/t:7.0f} GB/s")
