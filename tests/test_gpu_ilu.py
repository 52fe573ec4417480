"""§8 f2: ILU(0) preconditioner on the GPU vs the oracle (reading R24).

The factorisation (one thread per row, IKJ order) and the level-scheduled
triangular solves perform the oracle's operations in the oracle's order, so
factors and M⁻¹z agree bit for bit; the preconditioned solves agree to the
end-to-end bar of tests/test_gpu_parity.py (final residual ≤ 1e-10 recomputed
in fp64, restart count within ±10 %, first-cycle Arnoldi residuals).
"""
import numpy as np
import pytest

import inputs
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_01850_b200 import gmres as G  # noqa: E402


def tdev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def check_solution(A, b, x):
    return float(np.linalg.norm(b - O.spmv64(A, x)) / np.linalg.norm(b))


def random_dd_csr(n, seed, per_row=6):
    """Ragged nonsymmetric sparse matrix: random off-diagonal columns, strictly
    diagonally dominant (pivots stay away from zero)."""
    rng = np.random.default_rng(seed)
    rp, cols, vals = [0], [], []
    for i in range(n):
        c = np.unique(np.concatenate([rng.integers(0, n, rng.integers(0, per_row + 1)), [i]]))
        v = rng.standard_normal(c.size)
        v[c == i] = 0.0
        v[c == i] = 1.5 * np.abs(v).sum() + 1.0
        cols.extend(c.tolist()); vals.extend(v.tolist()); rp.append(len(cols))
    return inputs.CSR(np.array(rp, np.int32), np.array(cols, np.int32), np.array(vals))


MATS = {
    "c1": lambda: inputs.make("C1").A,                     # 5-pt 64², 127 levels
    "c2mini": lambda: inputs.make("C2", 17).A,             # 7-pt 17³ (ragged n = 4913)
    "c4mini": lambda: inputs.make("C4", 9).A,              # 27-pt
    "random": lambda: random_dd_csr(3001, 5),              # irregular rows and levels
    "c3mini": lambda: inputs.make("C3", 6000).A,           # power-law rows (up to 1902 non-zeros)
}


@pytest.fixture(scope="module", params=sorted(MATS))
def mat(request):
    A = MATS[request.param]()
    return request.param, A, G.Solver.from_csr(A)


@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_ilu0_factors_bit_exact(mat, prec):
    _, A, S = mat
    f = S.ilu0_factor(prec).cpu().numpy()
    ref = O.ilu0(prec, A)
    assert f.dtype == ref.dtype
    assert np.array_equal(f, ref)


@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
@pytest.mark.parametrize("tune", [0, 65536], ids=["sync_free", "level_sync"])
def test_ilu0_apply_bit_exact(mat, prec, tune):
    """Both triangular-solve schedules — the sync-free default and the level-synchronous
    fallback (tune bit 16) — reproduce the oracle's substitutions bit for bit."""
    _, A, S = mat
    S.ilu0_factor(prec)
    dt = np.float32 if prec == G.MIXED else np.float64
    z = np.random.default_rng(3).uniform(-1, 1, A.n).astype(dt)
    y = S.ilu_apply(tdev(z), prec, tune=tune).cpu().numpy()
    ref = O.ilu0_apply(prec, A, O.ilu0(prec, A), z)
    assert np.array_equal(y, ref)


def test_level_counts_closed_form():
    # natural-order stencils: level of grid point (i, j, k) = i + j + k in both solves
    for N in (5, 12):
        S = G.Solver.from_csr(inputs.stencil(7, N, (1.0, 2.0, 3.0)))
        assert S.ilu0_levels() == (3 * (N - 1) + 1, 3 * (N - 1) + 1)
        S = G.Solver.from_csr(inputs.stencil(5, N, (1.0, 2.0, 0.0)))
        assert S.ilu0_levels() == (2 * (N - 1) + 1, 2 * (N - 1) + 1)


E2E = {
    "C1": lambda: inputs.make("C1"),
    "C2mini": lambda: inputs.make("C2", 24),
    "C4mini": lambda: inputs.make("C4", 12),
    "C3mini": lambda: inputs.make("C3", 6000),             # power-law rows: the merge-path SpMV + ILU kernels
}


@pytest.fixture(scope="module", params=sorted(E2E))
def prob(request):
    P = E2E[request.param]()
    return P, G.Solver.from_csr(P.A)


@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_ilu_solve_end_to_end(prob, ortho, prec):
    P, S = prob
    m = min(P.m, 50)
    res = S.solve(P.b, m=m, tol=1e-10, ortho=ortho, precision=prec, record_inner=True, precond=G.ILU0)
    ref = O.solve(P.A, P.b, m=m, tol=1e-10, ortho=ortho, prec=prec, flags=O.F_ILU0)
    jac = O.solve(P.A, P.b, m=m, tol=1e-10, ortho=ortho, prec=prec)
    assert res.status == 0, res.status_name
    assert ref.status == O.OK
    rel = check_solution(P.A, P.b, res.x)
    assert rel <= 1e-10, rel
    assert res.final_relres == pytest.approx(rel, rel=1e-3, abs=1e-13)
    assert abs(res.cycles - ref.cycles) <= max(1, 0.1 * ref.cycles), (res.cycles, ref.cycles)
    assert res.inner_iters < jac.inner_iters          # the stronger preconditioner pays
    # first cycle (the later ones start from x's rounding, which differs): Arnoldi
    # residuals track the oracle's
    j1 = min(int(res.cycle_iters[0]), ref.inner.size, 10)
    tol = 1e-6 if prec == G.FP64 else 1e-2
    assert np.allclose(res.inner[:j1], ref.inner[:j1], rtol=tol, atol=0)


@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
def test_fp32_ilu_in_fp64_solver(prob, ortho):
    """The paper's third arm: the fp64 solver with an fp32 ILU(0) of
    RN32(A) applied as RN32(in) → fp32 substitutions → fp64 (oracle F_ILU32)."""
    P, S = prob
    m = min(P.m, 50)
    res = S.solve(P.b, m=m, tol=1e-10, ortho=ortho, precision=G.FP64, record_inner=True, precond=G.ILU0_FP32)
    ref = O.solve(P.A, P.b, m=m, tol=1e-10, ortho=ortho, prec=O.FP64, flags=O.F_ILU32)
    assert res.status == 0, res.status_name
    assert ref.status == O.OK
    rel = check_solution(P.A, P.b, res.x)
    assert rel <= 1e-10, rel
    assert abs(res.cycles - ref.cycles) <= max(1, 0.1 * ref.cycles), (res.cycles, ref.cycles)
    j1 = min(int(res.cycle_iters[0]), ref.inner.size, 10)
    assert np.allclose(res.inner[:j1], ref.inner[:j1], rtol=1e-6, atol=0)
    res2 = S.solve(P.b, m=m, tol=1e-10, ortho=ortho, precision=G.FP64, precond=G.ILU0_FP32, tune=65536)
    assert res2.status == 0 and check_solution(P.A, P.b, res2.x) <= 1e-10   # level-synchronous schedule


def test_ilu_solve_errors():
    P = inputs.make("C1", 8)
    S = G.Solver.from_csr(P.A)
    with pytest.raises(G.GmresError):
        S.solve(P.b, precond=7)
    with pytest.raises(G.GmresError):
        S.solve(P.b, precond=G.ILU0, policy=G.ORTHLOSS)
    with pytest.raises(G.GmresError, match="precision GMRES_FP64"):
        S.solve(P.b, precond=G.ILU0_FP32, precision=G.MIXED)
    with pytest.raises(G.GmresError):                  # apply before any factorisation
        G.Solver.from_csr(P.A).ilu_apply(tdev(P.b), G.FP64)
    # zero pivot: u_22 = 1 − 1·1 = 0 (row 1); the solve reports it before any cycle
    A = inputs.CSR(np.array([0, 2, 4], np.int32), np.array([0, 1, 0, 1], np.int32), np.array([1.0, 1.0, 1.0, 1.0]))
    S2 = G.Solver.from_csr(A)
    with pytest.raises(G.GmresError, match="row 1"):
        S2.solve(np.array([1.0, 2.0]), precond=G.ILU0, precision=G.FP64)
    with pytest.raises(G.GmresError, match="row 1"):
        S2.ilu0_factor(G.FP64)
