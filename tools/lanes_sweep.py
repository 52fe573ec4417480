"""SpMV lanes-per-row sweep on one config (dev tool): python tools/lanes_sweep.py C4 [scale] — one
profiled mixed CGSR cycle per lanes value; prints the SpMV phase time per inner iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2011_01850_b200 import gmres as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scale = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
P = inputs.make(name, scale)
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
x = torch.zeros_like(b)
nnz, n = P.A.nnz, P.A.n
for prec in (G.MIXED, G.FP64):
    wb = 4 if prec == G.MIXED else 8
    spmv_bytes = (wb + 4) * nnz + 4 * (n + 1) + 3 * wb * n
    for lanes in (1, 2, 4, 8, 16):
        best = None
        for _ in range(2):
            r = S.solve_device(b, x, m=P.m, ortho=G.CGSR, precision=prec, lanes=lanes, max_cycles=1, profile=True)
            if best is None or r.phase_ns[1] < best.phase_ns[1]:
                best = r
        per = best.phase_ns[1] / 1e3 / best.inner_iters
        print(f"{name} {'mixed' if prec else 'fp64 '} lanes={lanes:2d} plan={S.plan()['csr_stream']} inner={best.inner_iters} "
              f"spmv {per:7.1f} us/iter -> {spmv_bytes / per / 1e3:6.0f} GB/s", flush=True)
