"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Nothing here re-types the oracle's formulas: every check is a closed form, an
invariant (Arnoldi relation, orthogonality, minimal-residual property), a
textbook/library routine on a tiny case (dense LU / least squares via numpy),
or a worked example from SPEC.md (cited).  Each is chosen so that a dropped
term, wrong sign/index or transposed operand in the oracle fails at least one.
"""
import math

import numpy as np
import pytest

import inputs
import oracle as O

# ------------------------------------------------------------------ helpers


def csr_from_dense(D):
    n = D.shape[0]
    rp = [0]
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(D[i])[0]
        cols.extend(nz.tolist())
        vals.extend(D[i, nz].tolist())
        rp.append(len(cols))
    return inputs.CSR(np.array(rp, np.int32), np.array(cols, np.int32), np.array(vals, np.float64))


def random_dd(n, seed, density=0.3, plus=1.0):
    """F1 fixture: random sparse, strictly diagonally dominant."""
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((n, n)) * (rng.random((n, n)) < density)
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, 1.1 * np.abs(D).sum(axis=1) + plus)
    return D


def lapl1d(n):
    return np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)


# ------------------------------------------------------------------- SpMV


def test_spmv_worked_examples():
    # I₃·[1,2,3] = [1,2,3]; tridiag(-1,2,-1)·1 = [1,0,0,1]
    assert np.array_equal(O.spmv64(csr_from_dense(np.eye(3)), np.array([1.0, 2, 3])), [1, 2, 3])
    assert np.array_equal(O.spmv64(csr_from_dense(lapl1d(4)), np.ones(4)), [1, 0, 0, 1])


@pytest.mark.parametrize("n,seed", [(8, 0), (33, 1), (64, 2)])
def test_spmv64_dense(n, seed):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.5)
    x = rng.standard_normal(n)
    y = O.spmv64(csr_from_dense(D), x)
    assert np.linalg.norm(y - D @ x) <= 1e-14 * np.linalg.norm(D @ x) * 10


def test_spmv32_componentwise_bound():
    # |ŷ_i − y_i| ≤ γ_k (|A||x|)_i, γ_k = k u/(1 − k u), u = 2⁻²⁴ (any summation order)
    rng = np.random.default_rng(3)
    A = inputs.randdd(2000, 11, kmax=200)
    a32 = A.val.astype(np.float32)
    x32 = rng.uniform(-1, 1, A.n).astype(np.float32)
    y = O.spmv32(A, a32, x32)
    u = 2.0 ** -24
    for i in range(0, A.n, 7):
        s, e = A.row_ptr[i], A.row_ptr[i + 1]
        prods = a32[s:e].astype(np.float64) * x32[A.col[s:e]].astype(np.float64)  # exact in fp64
        exact = math.fsum(prods)
        k = e - s
        gam = k * u / (1 - k * u)
        assert abs(float(y[i]) - exact) <= gam * np.abs(prods).sum() + 1e-45


def test_jacobi_spmv_scales_rows():
    # M = diag(A): M⁻¹A has unit diagonal, so M⁻¹A e_i has 1 in row i
    D = random_dd(12, 4)
    A = csr_from_dense(D)
    aW, dW = O.working_copy(A, O.FP64)
    for i in (0, 5, 11):
        e = np.zeros(12); e[i] = 1.0
        w = O.jacobi_spmv(O.FP64, A, aW, dW, e)
        assert np.allclose(w, D[:, i] / np.diag(D), rtol=1e-15, atol=0)
        assert w[i] == 1.0


# ----------------------------------------------------------- dot / norm


def test_dot_examples():
    # dot([1,0],[0,1]) = 0 ; norm2([3,4]) = 5
    assert O.dot(O.FP64, np.array([1.0, 0.0]), np.array([0.0, 1.0])) == 0.0
    assert math.sqrt(O.dot(O.FP64, np.array([3.0, 4.0]), np.array([3.0, 4.0]))) == 5.0
    rng = np.random.default_rng(5)
    x = rng.standard_normal(10000).astype(np.float32)
    y = rng.standard_normal(10000).astype(np.float32)
    exact = math.fsum((x.astype(np.float64) * y.astype(np.float64)).tolist())
    bound = 10000 * 2.0 ** -53 * float(np.abs(x.astype(np.float64) * y).sum())
    assert abs(O.dot(O.MIXED, x, y) - exact) <= bound  # fp64 accumulator (reading R9)


# ---------------------------------------------------------------- Givens


def test_givens_examples():
    # rot(1,0) = (1,0); rot(3,4) = (0.6,0.8), ρ = 5
    assert O.givens(1.0, 0.0) == (1.0, 0.0, 1.0)
    c, s, r = O.givens(3.0, 4.0)
    assert (c, s, r) == pytest.approx((0.6, 0.8, 5.0), rel=1e-15)
    rng = np.random.default_rng(6)
    for a, b in rng.standard_normal((50, 2)):
        c, s, r = O.givens(a, b)
        assert c * c + s * s == pytest.approx(1.0, abs=1e-15)
        assert c * a + s * b == pytest.approx(r, rel=1e-14)
        assert -s * a + c * b == pytest.approx(0.0, abs=1e-14 * abs(r))


def test_hess_step_matches_lstsq():
    # |s_{j+1}| = min_y ‖β e₁ − H̄_j y‖ at every j (Prop. 6.9 cited at PAPER.md:243)
    rng = np.random.default_rng(7)
    m, beta = 12, 2.5
    H = np.triu(rng.standard_normal((m + 1, m)), -1)
    cs, sn, s = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    s[0] = beta
    for j in range(1, m + 1):
        h = np.zeros(m + 1)
        h[:j + 1] = H[:j + 1, j - 1]
        res = O.hess_step(j, h, cs, sn, s)
        Hj = H[:j + 1, :j]
        rhs = np.zeros(j + 1); rhs[0] = beta
        y, *_ = np.linalg.lstsq(Hj, rhs, rcond=None)
        ls = np.linalg.norm(rhs - Hj @ y)
        assert res == pytest.approx(ls, rel=1e-10, abs=1e-14)
        assert h[j] == 0.0
    # the rotated columns form R = Qᵀ H̄ (upper triangular): |det| and column norms preserved
    assert np.all(np.abs(s) <= beta)


def test_backsolve():
    # R = [2], s = [4] → y = 2 ; random upper triangular vs LAPACK solve
    assert np.allclose(O.backsolve(np.array([[2.0]]), np.array([4.0])), [2.0])
    rng = np.random.default_rng(8)
    R = np.triu(rng.standard_normal((20, 20))) + 5 * np.eye(20)
    s = rng.standard_normal(20)
    assert np.allclose(O.backsolve(R, s), np.linalg.solve(R, s), rtol=1e-13, atol=1e-13)


def test_xupdate():
    rng = np.random.default_rng(9)
    V = rng.standard_normal((100, 7)).astype(np.float32)
    y = rng.standard_normal(7)
    x = rng.standard_normal(100)
    out = O.xupdate(O.MIXED, V, y, x)
    exact = x + V.astype(np.float64) @ y
    assert np.allclose(out, exact, rtol=1e-14, atol=1e-14)


# ------------------------------------------------------------- MGS / CGSR


@pytest.mark.parametrize("proc", ["mgs", "cgsr"])
def test_ortho_worked_examples(proc):
    f = getattr(O, proc)
    # V = [e₁], w = [1,1,0] → h₁ = 1, w' = [0,1,0]
    V = np.array([[1.0], [0.0], [0.0]])
    w, h = f(O.FP64, V, np.array([1.0, 1.0, 0.0]))
    assert np.array_equal(w, [0.0, 1.0, 0.0]) and np.array_equal(h, [1.0])
    # w ⟂ span(V) → h = 0, w unchanged
    V = np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0], [0.0, 0.0]])
    w0 = np.array([0.0, 0.0, 3.0, -2.0])
    w, h = f(O.FP64, V, w0)
    assert np.array_equal(w, w0) and np.array_equal(h, [0.0, 0.0])


@pytest.mark.parametrize("proc", ["mgs", "cgsr"])
@pytest.mark.parametrize("prec,tol", [(O.FP64, 1e-13), (O.MIXED, 2e-5)])
def test_ortho_invariants(proc, prec, tol):
    rng = np.random.default_rng(10)
    n, j = 300, 9
    Q, _ = np.linalg.qr(rng.standard_normal((n, j)))
    Vw = Q.astype(O.wdtype(prec))
    V = Vw.astype(np.float64)
    w0 = rng.standard_normal(n).astype(O.wdtype(prec))
    w, h = getattr(O, proc)(prec, Vw, w0)
    w = w.astype(np.float64)
    nw = np.linalg.norm(w0)
    assert np.abs(V.T @ w).max() <= tol * nw                      # w' ⟂ V
    assert np.linalg.norm(w0 - (w + V @ h)) <= tol * nw            # w = w' + V h (no dropped term)
    assert np.linalg.norm(h - V.T @ w0.astype(np.float64)) <= tol * nw  # h = Vᵀw for orthonormal V


def test_cgsr_reorthogonalisation_restores_orthogonality():
    # F2: V 10×3 orthonormal, w = V c + τ g, τ = 1e-12.
    fails1 = 0
    for seed in range(20):
        rng = np.random.default_rng(100 + seed)
        V, _ = np.linalg.qr(rng.standard_normal((10, 3)))
        c = rng.standard_normal(3); c /= np.linalg.norm(c)
        g = rng.standard_normal(10); g /= np.linalg.norm(g)
        w0 = V @ c + 1e-12 * g
        w1, _ = O.cgsr(O.FP64, V, w0, passes=1)
        w2, _ = O.cgsr(O.FP64, V, w0, passes=2)
        fails1 += np.linalg.norm(V.T @ w1) / np.linalg.norm(w1) >= 1e-6
        assert np.linalg.norm(V.T @ w2) <= 1e-13 * np.linalg.norm(w2)
    assert fails1 == 20  # a single CGS pass does not restore orthogonality


# --------------------------------------------------------------- Arnoldi


@pytest.mark.parametrize("ortho", [O.MGS, O.CGSR])
def test_arnoldi_relation_and_orthogonality(ortho):
    # ‖M⁻¹A V_J − V_{J+1} H̄_J‖_F ≤ 1e-12 ‖M⁻¹A‖_F ; ‖I − VᵀV‖_max ≤ 1e-12
    n, m = 60, 20
    D = random_dd(n, 21)
    A = csr_from_dense(D)
    MA = D / np.diag(D)[:, None]
    r = np.random.default_rng(22).standard_normal(n)
    cyc = O.arnoldi(O.FP64, ortho, A, r, m)
    assert cyc.J == m and not cyc.breakdown
    V = cyc.V
    lhs = MA @ V[:, :m]
    rhs = V @ cyc.Hbar
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(MA)
    loss = [np.abs(np.eye(j + 1) - V[:, :j + 1].T @ V[:, :j + 1]).max() for j in range(1, m + 1)]
    if ortho == O.CGSR:
        assert max(loss) <= 1e-12  # CGSR keeps orthogonality
    else:
        # MGS: orthogonal while the basis is well conditioned, then loses orthogonality in
        # inverse proportion to the Arnoldi residual (Paige et al.)
        assert all(l <= 1e-12 for l, s in zip(loss, cyc.inner) if s >= 1e-3)
        assert max(l * s for l, s in zip(loss, cyc.inner)) <= 1e-13
    assert np.allclose(V[:, 0], r / np.linalg.norm(r), rtol=0, atol=1e-15)
    # per-step |s_{j+1}|/β equals the dense least-squares residual
    beta = np.linalg.norm(r)
    for j in range(1, m + 1):
        Hj = cyc.Hbar[:j + 1, :j]
        rhs = np.zeros(j + 1); rhs[0] = beta
        y, *_ = np.linalg.lstsq(Hj, rhs, rcond=None)
        assert cyc.inner[j - 1] * beta == pytest.approx(np.linalg.norm(rhs - Hj @ y), rel=1e-9, abs=1e-13 * beta)
    # monotone within the cycle (BASELINE.json)
    assert np.all(np.diff(cyc.inner) <= 1e-14 * cyc.inner[:-1])


@pytest.mark.parametrize("ortho", [O.MGS, O.CGSR])
def test_minimal_residual_property(ortho):
    # u = argmin_{u ∈ K_J} ‖M⁻¹(b − A u)‖, dense LS over a numpy Krylov basis
    n, J = 30, 6
    D = random_dd(n, 31)
    MA = D / np.diag(D)[:, None]
    b = np.random.default_rng(32).standard_normal(n)
    A = csr_from_dense(D)
    res = O.solve(A, b, m=J, tol=1e-300, ortho=ortho, prec=O.FP64, max_cycles=1)
    u = res.x
    r0 = b / np.diag(D)
    K = np.empty((n, J))
    K[:, 0] = r0
    for i in range(1, J):
        K[:, i] = MA @ K[:, i - 1]
    Q, _ = np.linalg.qr(K)
    c, *_ = np.linalg.lstsq(MA @ Q, r0, rcond=None)
    best = np.linalg.norm(r0 - MA @ Q @ c)
    got = np.linalg.norm(r0 - MA @ u)
    assert got == pytest.approx(best, rel=1e-8)
    assert np.linalg.norm(u - Q @ c) <= 1e-8 * np.linalg.norm(u)


# --------------------------------------------------------------- solves


@pytest.mark.parametrize("ortho", [O.MGS, O.CGSR])
@pytest.mark.parametrize("n,seed", [(5, 100), (10, 101), (30, 102), (64, 103), (200, 104)])
def test_solve_matches_dense_lu(ortho, n, seed):
    D = random_dd(n, seed)
    xt = np.random.default_rng(seed + 1).uniform(-1, 1, n)
    b = D @ xt
    A = csr_from_dense(D)
    res = O.solve(A, b, m=min(n, 30), tol=1e-12, ortho=ortho, prec=O.FP64)
    assert res.status == O.OK
    x_lu = np.linalg.solve(D, b)
    assert np.linalg.norm(res.x - x_lu) <= 1e-8 * np.linalg.norm(x_lu)
    assert np.linalg.norm(b - D @ res.x) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("ortho", [O.MGS, O.CGSR])
def test_exact_convergence_in_n_steps(ortho):
    # unrestarted (m ≥ n) fp64 GMRES on a tiny system terminates within n inner steps
    for seed, n in [(200, 8), (201, 15), (202, 25)]:
        D = random_dd(n, seed, density=0.8, plus=0.0) + np.triu(np.ones((n, n)), 1) * 0.3
        b = np.random.default_rng(seed).standard_normal(n)
        A = csr_from_dense(D)
        res = O.solve(A, b, m=n, tol=1e-12, ortho=ortho, prec=O.FP64, max_cycles=1)
        assert res.cycles == 1 and res.inner_iters <= n
        assert np.linalg.norm(res.x - np.linalg.solve(D, b)) <= 1e-10 * np.linalg.norm(res.x)


def test_special_cases():
    n = 6
    b = np.arange(1.0, n + 1)
    # A = I → one inner step with lucky breakdown h_{2,1} = 0
    I = csr_from_dense(np.eye(n))
    cyc = O.arnoldi(O.FP64, O.MGS, I, b, 5)
    assert cyc.J == 1 and cyc.breakdown and cyc.Hbar[1, 0] == 0.0
    res = O.solve(I, b, m=5, prec=O.FP64)
    assert res.cycles == 1 and res.inner_iters == 1 and np.allclose(res.x, b, rtol=1e-15)
    # diagonal A with Jacobi: M⁻¹A = I → one step
    # mixed (power-of-two diagonal so that dinv32·a32 = 1 exactly): every cycle is one
    # inner step; the fp32 rounding of v₁ is removed by one more refinement cycle
    Dg = csr_from_dense(np.diag([2.0, 4.0, 8.0, 0.5, 16.0, 0.25]))
    res = O.solve(Dg, b, m=5, prec=O.MIXED)
    assert res.status == O.OK and res.cycles == 2 and res.inner_iters == 2
    Dg = csr_from_dense(np.diag([2.0, 4.0, 8.0, 3.0, 5.0, 7.0]))
    res = O.solve(Dg, b, m=5, prec=O.FP64)
    assert res.cycles == 1 and res.inner_iters == 1
    # diag(2,4)·[1,1] = [2,4]
    res = O.solve(csr_from_dense(np.diag([2.0, 4.0])), np.array([2.0, 4.0]), m=2, prec=O.FP64)
    assert np.allclose(res.x, [1.0, 1.0], rtol=1e-15)
    # b = 0 → x = 0, 0 cycles
    P = inputs.make("C1", 8)
    res = O.solve(P.A, np.zeros(P.A.n), m=5)
    assert res.cycles == 0 and not res.x.any()
    # x0 already meets tol → 0 cycles
    res = O.solve(P.A, P.b, x0=P.x_true, m=5)
    assert res.cycles == 0 and res.history[0] <= 1e-10


def test_invalid_inputs():
    D = random_dd(5, 1)
    D[2, 2] = 0.0
    A = csr_from_dense(D)
    with pytest.raises(RuntimeError):
        O.solve(A, np.ones(5), m=3)
    with pytest.raises(ZeroDivisionError, match="row 2"):
        O.dinv(A)
    bad = inputs.CSR(np.array([0, 2, 3], np.int32), np.array([1, 0, 1], np.int32), np.ones(3))
    with pytest.raises(RuntimeError):
        O.solve(bad, np.ones(2), m=2)
    with pytest.raises(OverflowError):
        O.cast32(np.array([1e39]))
    # StallDetect's factor must exceed 1: with 1 the stall test can never fire
    good = inputs.make("C1", 8)
    with pytest.raises(RuntimeError):
        O.solve(good.A, good.b, m=10, policy=O.STALL, stall_factor=1.0)
    assert O.solve(good.A, good.b, m=10, policy=O.STALL, stall_factor=1.001).status == O.OK


# ------------------------------------------------------ mixed-precision claims


@pytest.fixture(scope="module")
def c1():
    return inputs.make("C1")


@pytest.mark.parametrize("ortho", [O.MGS, O.CGSR])
def test_mixed_reaches_double_accuracy(c1, ortho):
    # fp64 residual + update, fp32 elsewhere, reaches fp64 accuracy
    m = O.solve(c1.A, c1.b, m=30, ortho=ortho, prec=O.MIXED)
    d = O.solve(c1.A, c1.b, m=30, ortho=ortho, prec=O.FP64)
    assert m.status == O.OK and m.final_relres <= 1e-10
    assert d.status == O.OK and d.final_relres <= 1e-10
    # forced-restart regime: mixed and double take the same number of cycles
    assert m.cycles == d.cycles
    # iterative refinement view: ρ_K ≤ (max δ_k)^K ρ_0, slack ×10
    h = m.history
    dk = h[1:] / h[:-1]
    assert np.all(dk < 1)
    assert h[-1] <= 10 * dk.max() ** (len(h) - 1) * h[0]
    # history matches the recomputed true residual
    assert m.final_relres == pytest.approx(np.linalg.norm(c1.b - O.spmv64(c1.A, m.x)) / np.linalg.norm(c1.b),
                                           rel=1e-6)


@pytest.mark.parametrize("flags", [O.F_RESID32 | O.F_UPDATE32, O.F_RESID32, O.F_UPDATE32])
def test_fp32_refinement_variables_cap_accuracy(c1, flags):
    # fp32 residual or fp32 update cannot improve past single-precision accuracy
    r = O.solve(c1.A, c1.b, m=30, ortho=O.CGSR, prec=O.MIXED, flags=flags, max_cycles=40)
    assert r.status == O.NOT_CONVERGED
    assert r.history.min() > 1e-8


def test_single_cgs_pass_still_converges_in_mixed(c1):
    # the correction variables alone in fp32 still converge: fp32 accumulators too
    r = O.solve(c1.A, c1.b, m=30, ortho=O.MGS, prec=O.MIXED, flags=O.F_ACC32)
    assert r.status == O.OK and r.final_relres <= 1e-10


# ---------------------------------------------------------------- restart policies (reading R22)
def _cycle_lengths(inner):
    """Cycle lengths from the per-inner |s_{j+1}|/β history: |s| is non-increasing within a
    cycle (Givens), so every increase marks a restart."""
    J, c = [], 0
    for t in range(len(inner)):
        if t > 0 and inner[t] > inner[t - 1] * (1 + 1e-12):
            J.append(c)
            c = 0
        c += 1
    J.append(c)
    return J


def test_twostage_restart_repeats_first_cycle_length():
    """f1: first restart on an Arnoldi improvement δ, then every cycle restarts
    at the first cycle's iteration count; the last cycle may stop earlier (converged)."""
    P = inputs.make("C2", 24)
    delta = 1e-3
    for ortho in (O.MGS, O.CGSR):
        r = O.solve(P.A, P.b, m=150, ortho=ortho, prec=O.MIXED, policy=O.TWOSTAGE, delta=delta)
        assert r.status == O.OK and r.final_relres <= 1e-10
        J = _cycle_lengths(r.inner)
        assert len(J) == r.cycles and sum(J) == r.inner_iters
        J1 = J[0]
        assert J1 < 150 and all(j == J1 for j in J[1:-1]) and J[-1] <= J1
        # the first cycle ended on the δ rule: |s_{J1+1}|/β ≤ δ < |s_{J1}|/β
        assert r.inner[J1 - 1] <= delta < r.inner[J1 - 2]
        # against the threshold policy, which keeps restarting on δ
        r0 = O.solve(P.A, P.b, m=150, ortho=ortho, prec=O.MIXED, policy=O.THRESHOLD, delta=delta)
        assert _cycle_lengths(r0.inner)[0] == J1 and _cycle_lengths(r0.inner)[1] != J1


def test_stall_restart_fires_exactly_at_the_first_stall():
    """f4: restart when |s| improves by less than ×1.001 over the
    last ⌈5 % · m⌉ inner iterations — checked against the recorded |s| history."""
    P = inputs.make("C2", 24)
    m, factor = 150, 1.001
    w = math.ceil(0.05 * m)
    r = O.solve(P.A, P.b, m=m, ortho=O.MGS, prec=O.MIXED, policy=O.STALL)
    assert r.status == O.OK and r.final_relres <= 1e-10
    J = _cycle_lengths(r.inner)
    first = np.concatenate([[1.0], r.inner[:J[0]]])   # |s_1|/β = 1, then |s_{j+1}|/β
    stall = [j for j in range(w, len(first)) if first[j] * factor > first[j - w]]
    assert J[0] < m and stall and stall[0] == J[0]      # MGS stagnates: the stall ends the cycle
    # without the stall test the same cycle runs to m (MGS's Arnoldi residual stagnates)
    r0 = O.solve(P.A, P.b, m=m, ortho=O.MGS, prec=O.MIXED, policy=O.THRESHOLD, delta=0.0)
    assert _cycle_lengths(r0.inner)[0] == m
    # CGSR: the stall is not visible in the Arnoldi residual
    rc = O.solve(P.A, P.b, m=m, ortho=O.CGSR, prec=O.MIXED, policy=O.STALL)
    rc0 = O.solve(P.A, P.b, m=m, ortho=O.CGSR, prec=O.MIXED, policy=O.THRESHOLD, delta=0.0)
    assert _cycle_lengths(rc.inner) == _cycle_lengths(rc0.inner)


def test_orthloss_monitor_matches_dense_definition():
    """f3: the incremental S_k = (I+U_k)⁻¹U_k of the monitor equals the
    dense definition from the cycle's basis; ‖S‖_F exactly, ‖S‖₂ by 10 power iterations from
    below; Frobenius ≥ spectral; the cycle ends at the first step whose norm reaches the
    threshold (reading R23)."""
    P = inputs.make("C2", 16)
    m = 60
    for kind in (0, 1):
        r = O.solve(P.A, P.b, m=m, ortho=O.MGS, prec=O.MIXED, policy=O.ORTHLOSS, orth_kind=kind,
                    orth_thresh=10.0, delta=0.0, max_cycles=1)
        aW, dW = O.working_copy(P.A, O.MIXED)
        r0 = O.resid(O.MIXED, P.A, P.b, np.zeros(P.A.n), dW)[1]
        cyc = O.arnoldi(O.MIXED, O.MGS, P.A, r0, m, 0.0)
        V = cyc.V.astype(np.float64)                       # n × (J+1)
        J = len(r.orth)
        assert J == cyc.J
        for j in (1, 5, 20, J - 1):                        # monitor value after inner step j
            k = j + 1
            U = np.triu(V[:, :k].T @ V[:, :k], 1)
            S = np.linalg.solve(np.eye(k) + U, U)
            fro, two = np.linalg.norm(S), np.linalg.norm(S, 2)
            if kind == 0:
                assert r.orth[j - 1] == pytest.approx(fro, rel=1e-9, abs=1e-13)
            else:
                assert r.orth[j - 1] <= two * (1 + 1e-9) + 1e-13
                assert r.orth[j - 1] >= 0.5 * two - 1e-13
            assert two <= 1 + 1e-9 and fro >= two - 1e-12
    # the trigger: first step whose Frobenius norm reaches the threshold
    r = O.solve(P.A, P.b, m=m, ortho=O.MGS, prec=O.MIXED, policy=O.ORTHLOSS, orth_thresh=0.05, delta=0.0,
                max_cycles=1)
    hit = np.nonzero(r.orth >= 0.05)[0]
    assert hit.size and len(r.orth) == hit[0] + 1 < m


# ------------------------------------------------------------------- ILU(0) (§8 f2, reading R24)
def _factors_dense(A, f):
    """Split the combined factor array into dense unit-lower L and upper U."""
    n = A.n
    L, U = np.eye(n), np.zeros((n, n))
    for i in range(n):
        for e in range(A.row_ptr[i], A.row_ptr[i + 1]):
            j = int(A.col[e])
            if j < i:
                L[i, j] = f[e]
            else:
                U[i, j] = f[e]
    return L, U


def lapl2d(k):
    """5-point Laplacian on a k×k grid (SPEC's 2-D Poisson pin)."""
    T = lapl1d(k)
    return np.kron(np.eye(k), T) + np.kron(T, np.eye(k))


def test_ilu0_trivial_cases():
    # diagonal matrix: L = I, U = A (SPEC precond examples); diag(2,4) applied to [2,4] is [1,1]
    A = csr_from_dense(np.diag([2.0, 3.0]))
    assert np.array_equal(O.ilu0(O.FP64, A), [2.0, 3.0])
    A = csr_from_dense(np.diag([2.0, 4.0]))
    assert np.array_equal(O.ilu0_apply(O.FP64, A, O.ilu0(O.FP64, A), np.array([2.0, 4.0])), [1.0, 1.0])
    A = csr_from_dense(np.eye(5))
    z = np.arange(5.0)
    for prec in (O.FP64, O.MIXED):
        assert np.array_equal(O.ilu0_apply(prec, A, O.ilu0(prec, A), z), z)


@pytest.mark.parametrize("D", [lapl1d(5), random_dd(40, 3, density=0.0) + np.diag(np.full(39, -0.7), 1)
                               + np.diag(np.full(39, 0.4), -1)], ids=["tridiag5", "tridiag40"])
def test_ilu0_is_exact_lu_without_fill(D):
    # tridiagonal: LU has no fill, so ILU(0) = the exact LU (dense product equals A everywhere)
    A = csr_from_dense(D)
    f = O.ilu0(O.FP64, A)
    L, U = _factors_dense(A, f)
    assert np.allclose(L @ U, D, rtol=0, atol=1e-14 * np.abs(D).max())
    x = np.random.default_rng(1).uniform(-1, 1, A.n)
    y = O.ilu0_apply(O.FP64, A, f, D @ x)
    assert np.linalg.norm(y - x) <= 1e-12 * np.linalg.norm(x)
    # and it matches the dense solve
    assert np.allclose(y, np.linalg.solve(D, D @ x), rtol=0, atol=1e-12)


def test_ilu0_lower_triangular_is_exact():
    rng = np.random.default_rng(4)
    D = np.tril(rng.standard_normal((12, 12)) * (rng.random((12, 12)) < 0.4), -1) + np.diag(rng.uniform(2, 3, 12))
    A = csr_from_dense(D)
    x = rng.uniform(-1, 1, 12)
    y = O.ilu0_apply(O.FP64, A, O.ilu0(O.FP64, A), D @ x)
    assert np.linalg.norm(y - x) <= 1e-12 * np.linalg.norm(x)


def test_ilu0_pattern_identity_2d_poisson():
    # SPEC: (LU)[i,j] = A[i,j] on the pattern (relative 1e-13), nnz(F) = nnz(A);
    # off the pattern LU carries the dropped fill (it is incomplete: not A)
    D = lapl2d(4)
    A = csr_from_dense(D)
    f = O.ilu0(O.FP64, A)
    assert f.size == A.nnz
    L, U = _factors_dense(A, f)
    P = L @ U
    mask = D != 0
    assert np.allclose(P[mask], D[mask], rtol=1e-13, atol=0)
    assert np.abs(P[~mask]).max() > 0.05
    # full LU would differ from ILU(0) on this pattern (the incomplete factor is not exact)
    x = np.ones(A.n)
    assert np.linalg.norm(O.ilu0_apply(O.FP64, A, f, D @ x) - x) > 1e-6


def test_ilu0_fp32_matches_fp64_to_fp32_roundoff():
    # SPEC: factorising in LOW then applying equals HIGH to LOW round-off (rel 1e-5), 16×16
    D = random_dd(16, 7, density=0.4)
    A = csr_from_dense(D)
    f64, f32 = O.ilu0(O.FP64, A), O.ilu0(O.MIXED, A)
    assert f32.dtype == np.float32
    assert np.allclose(f32, f64, rtol=1e-5, atol=0)
    z = np.random.default_rng(2).uniform(-1, 1, 16)
    y64 = O.ilu0_apply(O.FP64, A, f64, z)
    y32 = O.ilu0_apply(O.MIXED, A, f32, z.astype(np.float32))
    assert np.allclose(y32, y64, rtol=1e-5, atol=1e-6 * np.abs(y64).max())


def test_ilu0_zero_pivot_names_the_row():
    with pytest.raises(ZeroDivisionError, match="row 1"):
        O.ilu0(O.FP64, csr_from_dense(np.array([[1.0, 1.0], [1.0, 1.0]])))   # u_22 = 1 − 1·1 = 0
    with pytest.raises(ZeroDivisionError, match="row 0"):
        O.ilu0(O.FP64, csr_from_dense(np.array([[0.0, 1.0], [1.0, 2.0]])))   # no diagonal in row 0


def test_ilu_gmres_exact_preconditioner_one_step():
    # M = LU = A (tridiagonal, no fill): M⁻¹A = I, so the first Arnoldi step exits (J = 1)
    D = lapl1d(30) + np.diag(np.linspace(0.1, 0.5, 29), 1)
    A = csr_from_dense(D)
    b = D @ np.random.default_rng(3).uniform(-1, 1, 30)
    r = O.solve(A, b, m=10, ortho=O.MGS, prec=O.FP64, flags=O.F_ILU0)
    assert r.inner_iters == 1 and r.final_relres <= 1e-13


@pytest.mark.parametrize("prec,flags", [(O.FP64, O.F_ILU0), (O.MIXED, O.F_ILU0), (O.FP64, O.F_ILU32)])
@pytest.mark.parametrize("ortho", [O.MGS, O.CGSR])
def test_ilu_gmres_converges_faster_than_jacobi(prec, flags, ortho):
    # C1-recipe problem (5-pt convection-diffusion): ILU(0) needs fewer inner iterations,
    # and the mixed / fp32-ILU solves still reach 1e-10
    P = inputs.make("C1", 16)
    rj = O.solve(P.A, P.b, m=30, ortho=ortho, prec=prec)
    ri = O.solve(P.A, P.b, m=30, ortho=ortho, prec=prec, flags=flags)
    assert ri.final_relres <= 1e-10 and rj.final_relres <= 1e-10
    assert ri.inner_iters < rj.inner_iters
    assert np.linalg.norm(ri.x - P.x_true) <= 1e-8 * np.linalg.norm(P.x_true)


# ------------------------------------------------------------------ a1 residual
# Alg. 1 lines 86/90: z = b − A x in fp64, then
# r = M⁻¹ RN_W(z) in W with M = diag(A) (readings R10, R11).  Pinned against a
# library SpMV (scipy.sparse), elementwise, at x ≠ 0 on a matrix whose diagonal
# varies row to row (so a missing or misplaced dinv, a sign error or a dropped
# b would each fail), in both precisions.
@pytest.mark.parametrize("prec", [O.FP64, O.MIXED])
@pytest.mark.parametrize("kind", ["randdd", "ragged_stencil"])
def test_resid_pinned_against_library_spmv(prec, kind):
    sp = pytest.importorskip("scipy.sparse")
    A = inputs.randdd(3001, 7) if kind == "randdd" else inputs.stencil(7, 9, (3.0, -2.0, 1.0))
    n = A.n
    rng = np.random.default_rng(21)
    x = rng.uniform(-1, 1, n)
    b = rng.uniform(-1, 1, n) * np.abs(A.val).max()
    M = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(n, n))
    z_lib = b - M @ x
    diag = M.diagonal()
    assert np.ptp(diag) > 0 or kind == "ragged_stencil"
    dW = (1.0 / diag).astype(np.float32 if prec == O.MIXED else np.float64)
    rc, r, zz, rr = O.resid(prec, A, b, x, dW)
    assert rc == 0
    # z: componentwise γ-bound of an fp64 row sum in any order, |b_i| + (|A||x|)_i
    k = np.diff(A.row_ptr) + 2
    u = 2.0 ** -53
    bound = k * u / (1 - k * u) * (np.abs(b) + abs(M) @ np.abs(x))
    assert zz == pytest.approx(float(np.dot(z_lib, z_lib)), rel=1e-12)
    # r_i = RN_W(dinv_i · RN_W(z_i)): the library z rounded through the same two W operations
    if prec == O.MIXED:
        r_lib = (dW * z_lib.astype(np.float32)).astype(np.float32)
        # |z − z_lib| ≤ bound moves RN32(z) by at most one ulp; dinv·(·) adds one rounding
        ulp = np.spacing(np.abs(r_lib).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(r.astype(np.float64) - r_lib) <= 2 * ulp + 2 * np.abs(dW) * bound)
    else:
        r_lib = dW * z_lib
        assert np.all(np.abs(r - r_lib) <= np.abs(dW) * bound + 2 * u * np.abs(r_lib))
    assert rr == pytest.approx(float(np.dot(r.astype(np.float64), r.astype(np.float64))), rel=1e-12)
    assert rr == pytest.approx(float(np.dot(r_lib.astype(np.float64), r_lib.astype(np.float64))),
                               rel=1e-12 if prec == O.FP64 else 1e-6)
    # special cases: x solving A x = b exactly (b = A x) → z ≈ 0; b = 0 → z = −A x
    rc, _, zz0, _ = O.resid(prec, A, M @ x, x, dW)
    assert rc == 0 and math.sqrt(zz0) <= 1e-13 * np.linalg.norm(M @ x)
    rc, r1, zz1, _ = O.resid(O.FP64, A, np.zeros(n), x, np.ones(n))
    assert np.allclose(r1, -(M @ x), rtol=1e-13, atol=1e-13 * np.abs(M @ x).max())


def test_resid_error_codes():
    A = inputs.stencil(5, 6, (1.0, 1.0, 0.0))
    n = A.n
    d = O.dinv(A)
    x = np.zeros(n)
    b = np.ones(n)
    b[5] = 1e39          # |z_5| > FLT_MAX: the cast of the residual to fp32 overflows (reading R10)
    assert O.resid(O.MIXED, A, b, x, d.astype(np.float32))[0] == -4
    assert O.resid(O.FP64, A, b, x, d)[0] == 0
    x[3] = np.inf        # non-finite residual
    assert O.resid(O.FP64, A, np.ones(n), x, d)[0] == -5


# ------------------------------------------------------------------ normwise backward error (Q5/Q17)
def test_backward_error_properties():
    D = random_dd(40, 3)
    A = csr_from_dense(D)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(40)
    xs = np.linalg.solve(D, b)
    assert O.backward_error(A, b, xs) <= 1e-15          # exact solution → ~u
    assert O.backward_error(A, b, np.zeros(40)) == pytest.approx(1.0)   # x = 0 → ‖b‖/‖b‖
    x = xs + 1e-3 * rng.standard_normal(40)
    e = O.backward_error(A, b, x)
    # invariant under scaling the system (A, b) → (cA, cb)
    A2 = inputs.CSR(A.row_ptr, A.col, 8.0 * A.val)
    assert O.backward_error(A2, 8.0 * b, x) == pytest.approx(e, rel=1e-14)
    # Rigal–Gaches: the smallest normwise perturbation ‖ΔA‖_F/‖A‖_F = ‖Δb‖/‖b‖ = η making x exact
    # has η = e; check the explicit perturbation ΔA = η‖A‖_F r xᵀ/(‖r‖‖x‖), Δb = −η‖b‖ r/‖r‖
    r = b - D @ x
    na, nx, nb = np.linalg.norm(D), np.linalg.norm(x), np.linalg.norm(b)
    dA = e * na * np.outer(r, x) / (np.linalg.norm(r) * nx)
    db = -e * nb * r / np.linalg.norm(r)
    assert np.linalg.norm((D + dA) @ x - (b + db)) <= 1e-12 * nb


# ------------------------------------------------------------------ OpenMP oracle build
def test_omp_build_bitwise():
    """liboracle_omp.so (used for the full-size golden records) equals the
    single-threaded build bit for bit: only element-parallel loops are threaded."""
    P = inputs.make("C3", 12000)
    Q = inputs.make("C2", 20)
    try:
        for prob in (P, Q):
            for prec in (O.MIXED, O.FP64):
                for ortho in (O.MGS, O.CGSR):
                    O.use_omp(False)
                    a = O.solve(prob.A, prob.b, m=prob.m, ortho=ortho, prec=prec)
                    O.use_omp(True)
                    c = O.solve(prob.A, prob.b, m=prob.m, ortho=ortho, prec=prec)
                    assert (a.cycles, a.inner_iters) == (c.cycles, c.inner_iters)
                    assert np.array_equal(a.x.view(np.uint64), c.x.view(np.uint64))
                    assert np.array_equal(a.history, c.history) and np.array_equal(a.inner, c.inner)
    finally:
        O.use_omp(False)
