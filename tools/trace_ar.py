"""All-reduce timeline of a C2 mixed MGS solve (dev tool).  Needs the G200_TRACE hook of
commit 3 before the one that added this file (per-CTA timestamps written in allreduce1 and
dumped by finish_solve); the hook is not in the product kernel (a branch in the hot
all-reduce).  Result: profiles/r02_mgs_allreduce_trace.txt."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs
from paper_2011_01850_b200 import gmres as G
P = inputs.make("C2")
S = G.Solver.from_csr(P.A)
b = torch.from_numpy(P.b).cuda()
x = torch.zeros_like(b)
TUNE = int(sys.argv[1]) if len(sys.argv) > 1 else 0
S.solve_device(b, x, m=50, ortho=G.MGS, precision=G.MIXED, max_cycles=1, tune=TUNE)
os.environ["G200_TRACE"] = "/tmp/tr.bin"
x.zero_()
r = S.solve_device(b, x, m=50, ortho=G.MGS, precision=G.MIXED, max_cycles=1, tune=TUNE)
print("tune", TUNE, "kernel_ms", r.kernel_ms, "ortho_ms", r.phase_ns[2] / 1e6)
G148 = 148
t = np.fromfile("/tmp/tr.bin", dtype=np.uint64).reshape(512, -1, 4)[:, :G148, :].astype(np.float64)
ok = (t > 0).all(axis=(1, 2))
t = t[ok]
print("ARs traced", t.shape[0])
ent, arr, det, done = t[..., 0], t[..., 1], t[..., 2], t[..., 3]
e = slice(40, 400)
print("entry spread (max-min over CTAs) us:", np.median((ent.max(1) - ent.min(1))[e]) / 1e3)
print("arrival spread us:", np.median((arr.max(1) - arr.min(1))[e]) / 1e3)
print("entry->arrival (own) median us:", np.median((arr - ent)[e]) / 1e3)
print("last arrival -> detect (median over CTAs) us:", np.median((det - arr.max(1, keepdims=True))[e]) / 1e3)
print("detect -> sum done us:", np.median((done - det)[e]) / 1e3)
print("done -> next entry us:", np.median((ent[1:] - done[:-1])[40:399]) / 1e3)
print("step period (CTA0) us:", np.median(np.diff(ent[:, 0])[40:399]) / 1e3)
which = np.argmax(arr, axis=1)[e]
print("last-arriving CTAs (top):", np.bincount(which, minlength=148).argsort()[::-1][:10], np.sort(np.bincount(which, minlength=148))[::-1][:10])
