import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs, oracle as O
from paper_2011_01850_b200 import gmres as G
A = inputs.make("C1").A
S = G.Solver.from_csr(A)
rng = np.random.default_rng(2)
b = rng.uniform(-1, 1, A.n) * 1e3
x = rng.uniform(-1, 1, A.n) * 1e-2
for prec in (G.FP64, G.MIXED):
    _, dW = O.working_copy(A, prec)
    rc, r_o, zz_o, rr_o = O.resid(prec, A, b, x, dW)
    rd = torch.empty(A.n, dtype=torch.float32 if prec else torch.float64, device="cuda")
    zz, rr = S.k_resid(prec, torch.from_numpy(b).cuda(), torch.from_numpy(x).cuda(), rd)
    r = rd.cpu().numpy()
    bad = np.nonzero(np.abs(r - r_o) > 1e-6 * np.abs(r_o).max())[0]
    print("prec", prec, "zz", zz, zz_o, "rr", rr, rr_o, "nbad", bad.size, bad[:20], bad[-5:] if bad.size else "")
    if bad.size:
        i = bad[0]; print("row", i, r[i], r_o[i])
D = A.to_dense()
z = b - D @ x
print("numpy zz", (z * z).sum(), "bb", (b * b).sum())
bd = torch.from_numpy(b).cuda(); xd = torch.from_numpy(x).cuda(); xo = torch.zeros_like(bd)
for prec in (G.FP64, G.MIXED):
    for t in range(3):
        r = S.solve_device(bd, xo, x0=xd, m=5, precision=prec, max_cycles=1, tol=1e-300)
        print("solve hist0", r.history[0], "expected", np.sqrt((z*z).sum()) / np.sqrt((b*b).sum()))
    for t in range(3):
        rd = torch.empty(A.n, dtype=torch.float32 if prec else torch.float64, device="cuda")
        print("k_resid", S.k_resid(prec, bd, xd, rd))
