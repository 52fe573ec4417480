"""GPU ↔ oracle parity through the C ABI (libgmres.so), on seeded inputs.

Per-step parity (rows a1–a8 of SURVEY.md §8) compares each component entry
point — which runs the same device code as the fused solve kernel — with the
oracle's step on identical inputs.  End-to-end parity checks the final
residual recomputed by the oracle (‖b − A x‖/‖b‖ ≤ 1e-10) and the restart
count within ±10 % of the oracle's (BASELINE.json).
"""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_01850_b200 import gmres as G  # noqa: E402

DEV = "cuda:0"


def tdev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def wdt(prec):
    return np.float32 if prec == G.MIXED else np.float64


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    G.load_library()  # fails loudly if the library is missing
    yield


MATS = {
    "c1": lambda: inputs.make("C1").A,
    "c2mini": lambda: inputs.make("C2", 24).A,
    "c3mini": lambda: inputs.make("C3", 20000).A,
    "c4mini": lambda: inputs.make("C4", 14).A,
    "ragged": lambda: inputs.stencil(5, 37, (3.0, -2.0, 0.0)),   # n = 1369: not a multiple of 32
}


@pytest.fixture(scope="module", params=sorted(MATS))
def mat(request):
    A = MATS[request.param]()
    return request.param, A, G.Solver.from_csr(A)


# ------------------------------------------------------------------ a2 SpMV
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_spmv_parity(mat, prec):
    name, A, S = mat
    rng = np.random.default_rng(1)
    aW, dW = O.working_copy(A, prec)
    v = rng.uniform(-1, 1, A.n).astype(wdt(prec))
    w_o = O.jacobi_spmv(prec, A, aW, dW, v)
    vd = tdev(v)
    wd = torch.empty_like(vd)
    S.k_spmv(prec, vd, wd)
    w = wd.cpu().numpy()
    rel = np.linalg.norm(w.astype(np.float64) - w_o) / np.linalg.norm(w_o)
    assert rel <= (1e-12 if prec == G.FP64 else 1e-5), rel   # BASELINE.json per-kernel bar
    # componentwise: |ŵ_i − w_i| ≤ γ_{k+1} |dinv_i| (|A||v|)_i, any summation order
    u = 2.0 ** -53 if prec == G.FP64 else 2.0 ** -24
    absAv = np.zeros(A.n)
    for i in range(A.n):
        s, e = A.row_ptr[i], A.row_ptr[i + 1]
        absAv[i] = np.abs(aW[s:e].astype(np.float64) * v[A.col[s:e]].astype(np.float64)).sum()
    k = np.diff(A.row_ptr) + 1
    gam = k * u / (1 - k * u)
    exact = np.array([math.fsum(aW[A.row_ptr[i]:A.row_ptr[i + 1]].astype(np.float64) *
                                v[A.col[A.row_ptr[i]:A.row_ptr[i + 1]]].astype(np.float64)) for i in range(A.n)])
    exact *= dW.astype(np.float64)
    assert np.all(np.abs(w - exact) <= 2 * gam * np.abs(dW) * absAv + 1e-300)


# ------------------------------------------------------------------ a1 residual
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_resid_parity(mat, prec):
    name, A, S = mat
    rng = np.random.default_rng(2)
    b = rng.uniform(-1, 1, A.n) * 1e3
    x = rng.uniform(-1, 1, A.n) * 1e-2
    _, dW = O.working_copy(A, prec)
    rc, r_o, zz_o, rr_o = O.resid(prec, A, b, x, dW)
    assert rc == 0
    rd = torch.empty(A.n, dtype=torch.float32 if prec == G.MIXED else torch.float64, device=DEV)
    zz, rr = S.k_resid(prec, tdev(b), tdev(x), rd)
    r = rd.cpu().numpy()
    assert zz == pytest.approx(zz_o, rel=1e-12)
    assert rr == pytest.approx(rr_o, rel=1e-12 if prec == G.FP64 else 1e-6)
    rel = np.linalg.norm(r.astype(np.float64) - r_o) / np.linalg.norm(r_o)
    assert rel <= (1e-12 if prec == G.FP64 else 1e-6)


# ------------------------------------------------------------------ a3/a4/a5
# every MGS variant the solves run (1 resident ring, 2 chunk ring, 3 streamed, 0 sweep),
# steps up to the bench's m = 50, C4's m = 100 and C5's m = 200
ORTHO_CASES = [(G.MGS, v) for v in (1, 2, 3, 0)] + [(G.CGSR, -1)]


@pytest.mark.parametrize("ortho,variant", ORTHO_CASES, ids=["mgs_resident", "mgs_chunk", "mgs_stream", "mgs_sweep", "cgsr"])
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
@pytest.mark.parametrize("j", [1, 7, 33, 50, 100, 200])
def test_ortho_parity(mat, prec, ortho, variant, j):
    name, A, S = mat
    n = A.n
    ld = G.ld_for(n)
    rng = np.random.default_rng(3 + j)
    Q, _ = np.linalg.qr(rng.standard_normal((n, j)))
    Vw = Q.astype(wdt(prec))
    w0 = (Q @ rng.standard_normal(j) + 0.3 * rng.standard_normal(n)).astype(wdt(prec))
    proc = O.mgs if ortho == G.MGS else O.cgsr
    w_o, h_o = proc(prec, Vw, w0)
    hn_o = math.sqrt(O.dot(prec, w_o, w_o))
    Vpad = np.zeros((j, ld), wdt(prec))
    Vpad[:, :n] = Vw.T
    Vd = tdev(Vpad)
    wd = tdev(w0)
    h, used = S.k_ortho(prec, ortho, j, Vd, ld, wd, mgs_variant=variant, return_variant=True)
    assert used == variant
    w = wd.cpu().numpy().astype(np.float64)
    nw = np.linalg.norm(w0.astype(np.float64))
    tol = 1e-12 if prec == G.FP64 else 1e-5
    assert np.linalg.norm(h[:j] - h_o) <= tol * nw
    assert np.linalg.norm(w - w_o) <= tol * nw
    assert h[j] == pytest.approx(hn_o, rel=1e-10 if prec == G.FP64 else 1e-4)


# ------------------------------------------------------------------ a8 update
@pytest.mark.parametrize("blocked", [False, True])
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_xupdate_parity(mat, prec, blocked):
    name, A, S = mat
    n = A.n
    ld = G.ld_for(n)
    J = 13
    rng = np.random.default_rng(4)
    V = rng.standard_normal((n, J)).astype(wdt(prec))
    y = rng.standard_normal(J)
    x = rng.standard_normal(n)
    x_o = O.xupdate(prec, V, y, x)
    Vpad = np.zeros((J, ld), wdt(prec))
    Vpad[:, :n] = V.T
    xd = tdev(x)
    S.k_xupdate(prec, J, tdev(Vpad), ld, y, xd, blocked=blocked)
    assert np.allclose(xd.cpu().numpy(), x_o, rtol=1e-14, atol=1e-14 * np.abs(x_o).max())


# ------------------------------------------------------------------ a6/a7 Givens + back-solve
@pytest.mark.parametrize("m,J", [(1, 1), (12, 12), (50, 31)])
def test_hessenberg_parity(m, J):
    A = inputs.make("C1", 8).A
    S = G.Solver.from_csr(A)
    rng = np.random.default_rng(5)
    H = np.triu(rng.standard_normal((m + 1, m)), -1)
    H[np.arange(m), np.arange(m)] += 3.0
    beta = 1.7
    R, s, y = S.k_hessenberg(m, J, H, beta)
    cs, sn, so = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    so[0] = beta
    Ro = np.zeros((m + 1, m))
    for j in range(1, J + 1):
        h = np.zeros(m + 1)
        h[:j + 1] = H[:j + 1, j - 1]
        O.hess_step(j, h, cs, sn, so)
        Ro[:, j - 1] = h
    yo = O.backsolve(Ro[:J, :J], so[:J])
    assert np.allclose(R[:, :J], Ro[:, :J], rtol=1e-13, atol=1e-13)
    assert np.allclose(s[:J + 1], so[:J + 1], rtol=1e-13, atol=1e-15)
    assert np.allclose(y, yo, rtol=1e-12, atol=1e-13)


# ------------------------------------------------------------------ end to end
def check_solution(A, b, x, tol=1e-10):
    r = b - O.spmv64(A, x)
    return np.linalg.norm(r) / np.linalg.norm(b)


E2E = {
    "C1": lambda: inputs.make("C1"),
    "C2mini": lambda: inputs.make("C2", 32),
    "C3mini": lambda: inputs.make("C3", 30000),
    "C4mini": lambda: inputs.make("C4", 20),
}


@pytest.fixture(scope="module", params=sorted(E2E))
def prob(request):
    P = E2E[request.param]()
    return P, G.Solver.from_csr(P.A)


@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_solve_end_to_end(prob, ortho, prec):
    P, S = prob
    m = min(P.m, 50)
    res = S.solve(P.b, m=m, tol=1e-10, ortho=ortho, precision=prec, record_inner=True)
    ref = O.solve(P.A, P.b, m=m, tol=1e-10, ortho=ortho, prec=prec)
    assert res.status == 0, res.status_name
    assert ref.status == O.OK
    rel = check_solution(P.A, P.b, res.x)
    assert rel <= 1e-10, rel
    assert res.final_relres == pytest.approx(rel, rel=1e-3, abs=1e-13)
    # normwise backward error of the returned x, recomputed by the oracle
    assert res.final_backward_err == pytest.approx(O.backward_error(P.A, P.b, res.x), rel=1e-3)
    assert abs(res.cycles - ref.cycles) <= 0.1 * ref.cycles, (res.cycles, ref.cycles)
    # diagnostic: per-cycle history tracks the oracle's
    k = min(len(res.history), len(ref.history))
    assert np.all(np.abs(np.log10(res.history[:k]) - np.log10(ref.history[:k])) <= 0.5)
    # within a cycle the Arnoldi residual is monotone non-increasing
    assert res.inner is not None and res.inner.size == res.inner_iters


@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_first_cycle_tracks_oracle(ortho, prec):
    P = inputs.make("C1")
    S = G.Solver.from_csr(P.A)
    res = S.solve(P.b, m=30, ortho=ortho, precision=prec, max_cycles=1, record_inner=True)
    ref = O.solve(P.A, P.b, m=30, ortho=ortho, prec=prec, max_cycles=1)
    assert res.status == 1 and ref.status == O.NOT_CONVERGED
    n = min(res.inner.size, ref.inner.size)
    assert abs(res.inner.size - ref.inner.size) <= 1
    tol = 1e-8 if prec == G.FP64 else 1e-3
    mask = ref.inner[:n] > (1e-12 if prec == G.FP64 else 1e-5)
    assert np.all(np.abs(res.inner[:n][mask] - ref.inner[:n][mask]) <= tol * ref.inner[:n][mask])
    assert np.allclose(res.x, ref.x, rtol=0, atol=(1e-9 if prec == G.FP64 else 1e-5) * np.abs(ref.x).max())


# ------------------------------------------------------------------ edge cases
def test_special_cases():
    P = inputs.make("C1", 16)
    S = G.Solver.from_csr(P.A)
    r = S.solve(np.zeros(P.A.n), m=10)
    assert r.status == 0 and r.cycles == 0 and not r.x.any()
    r = S.solve(P.b, x0=P.x_true, m=10)
    assert r.status == 0 and r.cycles == 0
    # A = I: one inner step with breakdown, one cycle
    n = 77
    I = inputs.CSR(np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.ones(n))
    SI = G.Solver.from_csr(I)
    b = np.linspace(1, 2, n)
    for prec in (G.FP64, G.MIXED):
        r = SI.solve(b, m=5, precision=prec)
        assert r.status == 0 and r.inner_iters == r.cycles and np.allclose(r.x, b, rtol=1e-12)
    # tiny dense DD system (n < 32: one partial row block)
    rng = np.random.default_rng(9)
    D = rng.standard_normal((5, 5))
    np.fill_diagonal(D, np.abs(D).sum(1) + 1)
    rp = np.arange(0, 26, 5, dtype=np.int32)
    col = np.tile(np.arange(5, dtype=np.int32), 5)
    Sd = G.Solver(rp, col, D.ravel())
    bb = rng.standard_normal(5)
    for ortho in (G.MGS, G.CGSR):
        r = Sd.solve(bb, m=5, ortho=ortho, precision=G.FP64, tol=1e-13)
        assert np.allclose(r.x, np.linalg.solve(D, bb), rtol=1e-11)


def test_errors():
    A = inputs.make("C1", 6).A
    val = A.val.copy()
    d = [e for e in range(A.row_ptr[3], A.row_ptr[4]) if A.col[e] == 3][0]
    val[d] = 0.0
    with pytest.raises(G.GmresError, match="EZERODIAG.*row 3"):
        G.Solver(A.row_ptr, A.col, val)
    bad = A.col.copy()
    bad[[0, 1]] = bad[[1, 0]]
    with pytest.raises(G.GmresError, match="EBADCSR"):
        G.Solver(A.row_ptr, bad, A.val)
    big = A.val.copy()
    big[0] = 1e39
    S = G.Solver(A.row_ptr, A.col, big)
    with pytest.raises(G.GmresError, match="EFP32RANGE"):
        S.solve(np.ones(A.n), precision=G.MIXED)
    S = G.Solver.from_csr(A)
    with pytest.raises(G.GmresError, match="EINVAL"):
        S.solve(np.ones(A.n), m=0)
    with pytest.raises(G.GmresError, match="EINVAL"):
        S.solve(np.ones(A.n), tol=-1.0)
    with pytest.raises(G.GmresError, match="stall_factor"):          # f must exceed 1
        S.solve(np.ones(A.n), policy=G.STALL, stall_factor=1.0)
    with pytest.raises(G.GmresError, match="lanes_per_row"):         # no 8-lane ILU/monitor kernels
        S.solve(np.ones(A.n), precond=G.ILU0, lanes=8)
    r = S.solve(np.ones(A.n), m=2, max_cycles=1, tol=1e-14)
    assert r.status == 1 and r.cycles == 1   # NOT_CONVERGED, x = last iterate


# ------------------------------------------------------------------ full size (BASELINE.json configs)
# The bench's launch configuration at the configs' full sizes: the converged
# residual recomputed by the oracle's fp64 SpMV (a property that holds at any
# size), mixed vs fp64 restart counts, and SpMV rows sampled and computed one
# by one by the oracle's rule (the oracle cannot run whole C3/C4 solves in
# seconds).  C3 exercises lanes-per-row > 1 and the direct (long-row) chunks.
FULL = {"C2": (50, [G.FP64, G.MIXED]), "C3": (50, [G.FP64, G.MIXED]), "C4": (100, [G.MIXED, G.FP64])}


def _sampled_spmv_rows(P, S, prec, rng, nsample=3000):
    A = P.A
    wt = np.float32 if prec == G.MIXED else np.float64
    v = rng.uniform(-1, 1, A.n).astype(wt)
    wd = torch.empty(A.n, dtype=torch.float32 if prec == G.MIXED else torch.float64, device=DEV)
    S.k_spmv(prec, tdev(v), wd)
    w = wd.cpu().numpy()
    aW = A.val.astype(wt)
    dW = O.dinv(A).astype(wt)
    u = 2.0 ** -24 if prec == G.MIXED else 2.0 ** -53
    rows = np.concatenate([rng.integers(0, A.n, nsample), [0, A.n - 1]])
    rows = np.concatenate([rows, np.argsort(np.diff(A.row_ptr))[-20:]])   # the longest rows
    for i in rows:
        s, e = A.row_ptr[i], A.row_ptr[i + 1]
        prod = aW[s:e].astype(np.float64) * v[A.col[s:e]].astype(np.float64)
        exact = math.fsum(prod) * float(dW[i])
        scale = float(np.abs(prod).sum() * abs(dW[i]))
        k = e - s + 1
        assert abs(float(w[i]) - exact) <= 2 * k * u * scale + 1e-300, (i, e - s)


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full_size")


def golden(cfg, prec, ortho, m):
    """Oracle record of a full-size config (tools/make_golden.py: the CPU oracle only)."""
    key = f"{cfg}_{'mixed' if prec == G.MIXED else 'fp64'}_{'mgs' if ortho == G.MGS else 'cgsr'}_m{m}"
    with open(os.path.join(GOLDEN, key + ".json")) as f:
        return json.load(f)


def within_10pct(c, ref):
    """BASELINE.json: "restart count within ±10 % of the oracle's" (below 10 cycles: equal)."""
    return abs(c - ref) <= 0.1 * ref


@pytest.mark.slow
@pytest.mark.parametrize("name", sorted(FULL))
def test_full_size(name):
    P = inputs.make(name)
    m, _ = FULL[name]
    S = G.Solver.from_csr(P.A)
    bd = tdev(P.b)
    for ortho in (G.MGS, G.CGSR):
        for prec in (G.MIXED, G.FP64):
            xd = torch.zeros_like(bd)
            r = S.solve_device(bd, xd, m=m, ortho=ortho, precision=prec)
            assert r.status == 0, r.status_name
            rel = check_solution(P.A, P.b, xd.cpu().numpy())
            assert rel <= 1e-10, (name, ortho, prec, rel)
            assert r.final_relres == pytest.approx(rel, rel=1e-3, abs=1e-13)
            ref = golden(name, prec, ortho, m)
            assert ref["status"] == 0 and ref["final_relres_recomputed"] <= 1e-10
            assert within_10pct(r.cycles, ref["cycles"]), (name, ortho, prec, r.cycles, ref["cycles"])
            # inner iterations: the same up to the fp32/fp64 rounding order of the last cycle
            assert abs(r.inner_iters - ref["inner_iters"]) <= max(3, 0.05 * ref["inner_iters"]), \
                (r.inner_iters, ref["inner_iters"])
    rng = np.random.default_rng(11)
    for prec in (G.MIXED, G.FP64):
        _sampled_spmv_rows(P, S, prec, rng)
    S.close()


@pytest.mark.slow
@pytest.mark.parametrize("m", [10, 25, 100, 200])
def test_c5_restart_sweep_matches_oracle(m):
    """BASELINE.json configs[4]: the C2 matrix at m ∈ {10, 25, 100, 200} (m = 50 is C2) —
    restart counts within ±10 % of the oracle's for MGS/CGSR × fp64/mixed."""
    P = inputs.make("C5")
    S = G.Solver.from_csr(P.A)
    bd = tdev(P.b)
    for ortho in (G.MGS, G.CGSR):
        for prec in (G.MIXED, G.FP64):
            xd = torch.zeros_like(bd)
            r = S.solve_device(bd, xd, m=m, ortho=ortho, precision=prec)
            assert r.status == 0, r.status_name
            assert check_solution(P.A, P.b, xd.cpu().numpy()) <= 1e-10
            ref = golden("C5", prec, ortho, m)
            assert within_10pct(r.cycles, ref["cycles"]), (m, ortho, prec, r.cycles, ref["cycles"])
    S.close()


# ------------------------------------------------------------------ MGS variants (DESIGN.md §5 a3)
# The global sweep, the whole-vector TMA ring and the chunk ring perform the
# same operations in the same order per element and per thread partial
# (reading R9), so their solves agree bit for bit; sizes are
# picked so each ring engages (fp64 chunk ring: > 8 register vectors of w per
# thread; the ragged grid side 109 leaves a partial last chunk).
@pytest.mark.slow
@pytest.mark.parametrize("prec,k,variant", [(G.MIXED, 64, 1), (G.FP64, 64, 1), (G.FP64, 109, 2), (G.MIXED, 137, 2),
                                            (G.FP64, 128, 2), (G.MIXED, 160, 2)])
def test_mgs_variants_agree(prec, k, variant):
    P = inputs.make("C2", k)
    S = G.Solver.from_csr(P.A)
    bd = tdev(P.b)
    xs, its = [], []
    # tune bit 2: force the global sweep; bit 19: force the streamed MGS (w in shared + global memory);
    # bit 8: a two-buffer ring for the resident MGS (its copies go in the all-reduce, not at the
    # start of the step: another schedule, the same arithmetic)
    # bit 28: the three-buffer ring's copies in the all-reduce too (gmres.h)
    cases = ((0, variant), (4, 0), (524288, 3)) + (((256, 1), (268435456, 1)) if variant == 1 else ())
    for tune, want in cases:
        xd = torch.zeros_like(bd)
        r = S.solve_device(bd, xd, m=30, ortho=G.MGS, precision=prec, max_cycles=3, tol=1e-14, tune=tune)
        assert r.status in (0, 1), r.status_name
        plan = S.plan()
        assert plan["mgs_variant"] == want, plan
        xs.append(xd.cpu().numpy())
        its.append((r.cycles, list(r.cycle_iters), r.final_relres))
    assert all(t == its[0] for t in its)
    assert all(np.array_equal(xs[0], x) for x in xs[1:])
    S.close()


# ------------------------------------------------------------------ basis getter (C5 orthogonality report)
@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])   # column-major / row-blocked basis layouts
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_basis_matches_oracle_first_cycle(ortho, prec):
    P = inputs.make("C2", 16)
    A = P.A
    S = G.Solver.from_csr(A)
    m = 20
    bd = tdev(P.b)
    xd = torch.zeros_like(bd)
    r = S.solve_device(bd, xd, m=m, ortho=ortho, precision=prec, max_cycles=1, tol=1e-14, delta=0.0)
    J = int(r.cycle_iters[0])
    V = S.basis(J, prec).cpu().numpy().astype(np.float64).T          # n × J
    aW, dW = O.working_copy(A, prec)
    r0 = O.resid(prec, A, P.b, np.zeros(A.n), dW)[1]
    cyc = O.arnoldi(prec, ortho, A, r0, m, 0.0)
    assert cyc.J == J
    Vo = cyc.V[:, :J].astype(np.float64)
    err = np.linalg.norm(V - Vo, axis=0)
    # fp64: rounding-order differences only; fp32: they grow slowly along the cycle
    assert np.all(err[:5] <= (1e-12 if prec == G.FP64 else 1e-5)), err[:5]
    assert np.allclose(np.linalg.norm(V, axis=0), 1.0, atol=1e-12 if prec == G.FP64 else 1e-6)
    loss = np.abs(np.eye(J) - V.T @ V).max()
    loss_o = np.abs(np.eye(J) - Vo.T @ Vo).max()
    assert loss <= 10 * loss_o + (1e-13 if prec == G.FP64 else 1e-6), (loss, loss_o)


# ------------------------------------------------------------------ restart policies (§8 f1, f4; reading R22)
def _cycle_lengths(inner):
    J, c = [], 0
    for t in range(len(inner)):
        if t > 0 and inner[t] > inner[t - 1] * (1 + 1e-12):
            J.append(c)
            c = 0
        c += 1
    J.append(c)
    return J


@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
def test_twostage_policy_matches_oracle(ortho):
    P = inputs.make("C2", 24)
    S = G.Solver.from_csr(P.A)
    r = S.solve(P.b, m=150, ortho=ortho, precision=G.MIXED, delta=1e-3, policy=G.TWOSTAGE)
    ref = O.solve(P.A, P.b, m=150, ortho=ortho, prec=O.MIXED, delta=1e-3, policy=O.TWOSTAGE)
    assert r.status == 0 and check_solution(P.A, P.b, r.x) <= 1e-10
    Jo = _cycle_lengths(ref.inner)
    J = list(r.cycle_iters)
    assert J[0] == Jo[0] and all(j == J[0] for j in J[1:-1]) and J[-1] <= J[0]
    assert abs(r.cycles - ref.cycles) <= max(1, 0.1 * ref.cycles)


@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
def test_stall_policy_matches_oracle(ortho):
    P = inputs.make("C2", 24)
    S = G.Solver.from_csr(P.A)
    m = 150
    r = S.solve(P.b, m=m, ortho=ortho, precision=G.MIXED, policy=G.STALL, record_inner=True)
    ref = O.solve(P.A, P.b, m=m, ortho=ortho, prec=O.MIXED, policy=O.STALL)
    assert r.status == 0 and check_solution(P.A, P.b, r.x) <= 1e-10
    J, Jo = list(r.cycle_iters), _cycle_lengths(ref.inner)
    assert abs(J[0] - Jo[0]) <= 3, (J, Jo)
    # the device took its exit at the first stall of its own |s| history
    w = math.ceil(0.05 * m)
    first = np.concatenate([[1.0], r.inner[:J[0]]])
    stall = [j for j in range(w, len(first)) if first[j] * 1.001 > first[j - w]]
    if J[0] < m and not stall:   # exit by convergence (need), as for CGSR
        assert first[-1] <= 1e-10 * 10
    elif stall:
        assert stall[0] == J[0]


@pytest.mark.parametrize("norm,thresh", [(0, 0.05), (0, 1.0), (1, 0.05), (1, 0.5)],
                         ids=["fro-0.05", "fro-1.0", "spec-0.05", "spec-0.5"])
def test_orthloss_policy_matches_oracle(norm, thresh):
    """f3 (reading R23): the device's monitor — ‖S_k‖_F or ‖S_k‖₂ by 10 power iterations
     — ends the MGS cycles where the oracle's does."""
    P = inputs.make("C2", 24)
    S = G.Solver.from_csr(P.A)
    m = 150
    r = S.solve(P.b, m=m, ortho=G.MGS, precision=G.MIXED, policy=G.ORTHLOSS, orth_thresh=thresh, delta=0.0,
                orth_norm=norm)
    ref = O.solve(P.A, P.b, m=m, ortho=O.MGS, prec=O.MIXED, policy=O.ORTHLOSS, orth_thresh=thresh, delta=0.0,
                  orth_kind=norm)
    assert r.status == 0 and check_solution(P.A, P.b, r.x) <= 1e-10
    J, Jo = list(r.cycle_iters), _cycle_lengths(ref.inner)
    assert abs(J[0] - Jo[0]) <= 2, (J, Jo)
    assert abs(r.cycles - ref.cycles) <= max(1, 0.1 * ref.cycles)


# ------------------------------------------------------------------ f4: Table-1 analogue
@pytest.mark.parametrize("name,scale,m", [("C2", 24, 150), ("C4", 16, 120)])
def test_table1_stall_points_match_oracle(name, scale, m):
    """Iterations before the Arnoldi residual stalls in the first three
    forced-restart cycles of mixed MGS: device histories vs the oracle's, and the paper's
    observation that the stall point repeats from cycle to cycle."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import table1
    row = table1.run(name, scale, m)
    g, o = row["stall_iters_gpu"], row["stall_iters_oracle"]
    assert len(g) >= 2 and None not in g and None not in o, row
    for a, b in zip(g, o):
        assert abs(a - b) <= max(2, 0.2 * b), row      # ±20 %
    assert max(g) - min(g) <= max(3, 0.2 * max(g)), row   # about the same after each restart



# ------------------------------------------------------------------ reading R27
FX_OFF = 1 << 25  # tune bit: the fp64 partial all-reduce instead of the fixed-point word


@pytest.mark.parametrize("name,scale,rowscale", [("C1", None, 1.0), ("C2", 24, 1.0), ("C3", 20000, 1.0),
                                                 ("C1", None, 1e8)], ids=["c1", "c2mini", "c3mini", "c1_scaled"])
def test_fixed_point_projections(name, scale, rowscale):
    """Reading R27: the mixed solve's MGS projections sum per-CTA partials quantised to
    2^-42·B (B ≥ 2√(‖D⁻¹A‖₁‖D⁻¹A‖∞), a power of two) as exact integers.  Against the fp64
    partial all-reduce (tune bit 25) and the oracle: same cycles, the first cycle's Arnoldi
    residuals equal far inside the fp32 rounding of w, x to 1e-10.  Rows scaled by 1e8 leave
    D⁻¹A — and so B and the quantisation — unchanged (the bound is Jacobi-scale invariant)."""
    P = inputs.make(name, scale)
    A, b = P.A, P.b
    if rowscale != 1.0:
        rs = rowscale ** np.linspace(0.0, 1.0, A.n)  # rows scaled by 1 … 1e8
        A = inputs.CSR(A.row_ptr, A.col, A.val * np.repeat(rs, np.diff(A.row_ptr)))
        b = b * rs
    S = G.Solver.from_csr(A)
    m = min(P.m, 50)
    r_fx = S.solve(b, m=m, ortho=G.MGS, precision=G.MIXED, record_inner=True)
    r_64 = S.solve(b, m=m, ortho=G.MGS, precision=G.MIXED, record_inner=True, tune=FX_OFF)
    ref = O.solve(A, b, m=m, tol=1e-10, ortho=G.MGS, prec=G.MIXED)
    assert r_fx.status == 0 and r_64.status == 0, (r_fx.status_name, r_64.status_name)
    assert check_solution(A, b, r_fx.x) <= 1e-10
    assert r_fx.cycles == r_64.cycles
    assert abs(r_fx.cycles - ref.cycles) <= 0.1 * ref.cycles, (r_fx.cycles, ref.cycles)
    J = int(r_fx.cycle_iters[0])
    a, c = r_fx.inner[:J], r_64.inner[:J]
    mask = c > 1e-5 * c[0]
    assert np.all(np.abs(a[mask] - c[mask]) <= 1e-4 * c[mask])


def test_fixed_point_projection_nonfinite_flagged():
    """Reading R27: a partial outside the bound (only non-finite data can produce one) sets
    the error flag; the component entry point reports GMRES_ENONFINITE."""
    A = inputs.make("C1").A
    S = G.Solver.from_csr(A)
    n, j = A.n, 4
    ld = G.ld_for(n)
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.standard_normal((n, j)))
    Vpad = np.zeros((j, ld), np.float32)
    Vpad[:, :n] = Q.T
    Vpad[2, 7] = np.nan
    w0 = rng.standard_normal(n).astype(np.float32)
    with pytest.raises(G.GmresError) as e:
        S.k_ortho(G.MIXED, G.MGS, j, tdev(Vpad), ld, tdev(w0))
    assert "fixed-point" in str(e.value) or "NONFINITE" in str(e.value).upper()
