"""Bit-equality of the MGS variants on one config (dev check): mgs_agree.py N prec"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs
from paper_2011_01850_b200 import gmres as G
N = int(sys.argv[1]); prec = G.MIXED if sys.argv[2] == "mixed" else G.FP64
P = inputs.make("C2", N)
S = G.Solver.from_csr(P.A)
bd = torch.from_numpy(P.b).cuda()
out = []
for tune in (0, 4, 524288):
    xd = torch.zeros_like(bd)
    r = S.solve_device(bd, xd, m=30, ortho=G.MGS, precision=prec, max_cycles=3, tol=1e-14, tune=tune)
    out.append((tune, S.plan()["mgs_variant"], r.status, r.cycles, list(r.cycle_iters), r.final_relres, r.kernel_ms, xd.cpu().numpy()))
for o in out:
    print(N, sys.argv[2], "tune", o[0], "variant", o[1], "st", o[2], "cyc", o[3], o[4], "relres %.6e" % o[5], "ms %.2f" % o[6],
          "bitequal_to_sweep", np.array_equal(o[7], out[1][7]))
