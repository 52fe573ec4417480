import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs, oracle as O
from paper_2011_01850_b200 import gmres as G
A = inputs.make("C1").A; n = A.n; S = G.Solver.from_csr(A); ld = G.ld_for(n)
for prec in (G.FP64,):
    for j in (1, 2, 3, 4, 5, 8):
        rng = np.random.default_rng(3 + j)
        Q, _ = np.linalg.qr(rng.standard_normal((n, j)))
        w0 = Q @ rng.standard_normal(j) + 0.3 * rng.standard_normal(n)
        w_o, h_o = O.cgsr(prec, Q, w0)
        Vp = np.zeros((j, ld)); Vp[:, :n] = Q.T
        wd = torch.from_numpy(w0.copy()).cuda()
        h = S.k_ortho(prec, G.CGSR, j, torch.from_numpy(Vp).cuda(), ld, wd)
        c1 = Q.T @ w0
        print(j, "h", h[:j], "ora", h_o, "c1", c1, "hn", h[j], np.linalg.norm(w_o), "werr", np.abs(wd.cpu().numpy() - w_o).max())
