"""Component microbenchmarks on C2-sized data (dev tool): µs per call and GB/s."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs
from paper_2011_01850_b200 import gmres as G
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
P = inputs.make(name)
A = P.A; n = A.n; nnz = A.nnz
S = G.Solver.from_csr(A)
ld = G.ld_for(n)
def timeit(f, reps=20):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    return min(ts), float(np.median(ts))
for prec, wb, dt in ((G.MIXED, 4, torch.float32), (G.FP64, 8, torch.float64)):
    v = torch.rand(n, dtype=dt, device="cuda"); w = torch.empty_like(v)
    S.solve_device(torch.from_numpy(P.b).cuda(), torch.zeros(n, dtype=torch.float64, device="cuda"), m=50, precision=prec, max_cycles=1)
    mn, md = timeit(lambda: S.k_spmv(prec, v, w))
    byt = (wb + 4) * nnz + 4 * (n + 1) + 3 * wb * n
    print(f"prec={prec} spmv   {mn:8.1f}us (med {md:8.1f})  {byt/mn/1e3:7.0f} GB/s model")
    b = torch.from_numpy(P.b).cuda(); x = torch.rand(n, dtype=torch.float64, device="cuda")
    mn, md = timeit(lambda: S.k_resid(prec, b, x, w))
    byt = 12 * nnz + 4 * (n + 1) + 16 * n + 2 * wb * n
    print(f"prec={prec} resid  {mn:8.1f}us (med {md:8.1f})  {byt/mn/1e3:7.0f} GB/s model")
    V = torch.rand(51, ld, dtype=dt, device="cuda") * 1e-3
    wcopy = torch.rand(n, dtype=dt, device="cuda")
    base, _ = timeit(lambda: w.copy_(wcopy))
    for ortho in (G.MGS, G.CGSR):
        for j in (1, 10, 25, 50):
            def f():
                w.copy_(wcopy)
                S.k_ortho(prec, ortho, j, V, ld, w)
            mn, md = timeit(f, 10)
            byt = (wb * n * j + wb * n) if ortho == 0 else (3 * wb * n * j + 5 * wb * n)
            print(f"prec={prec} {'MGS ' if ortho == 0 else 'CGSR'} j={j:3d} {mn:8.1f}us (med {md:8.1f})  {byt/mn/1e3:7.0f} GB/s model  ({(mn)/ (j+1 if ortho==0 else 3):6.1f} us/reduction)")
