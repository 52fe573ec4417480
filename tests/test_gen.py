"""Pins for the seeded input generators (inputs/gen.cpp).

Closed forms: nnz counts, and the consistency of the central-difference
convection–diffusion stencils with −Δu + β·∇u on linear and quadratic functions
(exact for central differences), which catches sign, scaling and index slips.
"""
import numpy as np
import pytest

import inputs


def interior_mask(N, dims):
    idx = np.arange(N ** dims)
    i = idx % N
    j = (idx // N) % N
    m = (i > 0) & (i < N - 1) & (j > 0) & (j < N - 1)
    if dims == 3:
        k = idx // (N * N)
        m &= (k > 0) & (k < N - 1)
    return m


def coords(N, dims):
    h = 1.0 / (N + 1)
    idx = np.arange(N ** dims)
    xs = [(idx % N + 1) * h, ((idx // N) % N + 1) * h]
    if dims == 3:
        xs.append((idx // (N * N) + 1) * h)
    return xs


def spmv(A, x):
    return inputs.matvec(A, x)


@pytest.mark.parametrize("kind,N", [(5, 6), (5, 64), (7, 5), (7, 17), (27, 4), (27, 9)])
def test_stencil_nnz_closed_form(kind, N):
    A = inputs.stencil(kind, N, (1.0, 2.0, 3.0))
    expect = {5: 5 * N * N - 4 * N, 7: 7 * N ** 3 - 6 * N * N, 27: (3 * N - 2) ** 3}[kind]
    assert A.nnz == expect
    # sorted unique columns, diagonal present
    for i in range(A.n):
        c = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0) and i in c


def test_config_sizes():
    L = inputs.lib()
    assert L.gen_stencil_nnz(5, 64) == 20224            # C1
    assert L.gen_stencil_nnz(7, 128) == 14581760        # C2
    assert L.gen_stencil_nnz(27, 256) == 449455096      # C4 = 766³
    assert L.gen_stencil_n(27, 256) == 16777216


def test_c1_coefficients():
    # BASELINE.json C1: h = 1/65, β = (20,20): diag 16900, W/S −4875, E/N −3575
    A = inputs.stencil(5, 64, (20.0, 20.0, 0.0))
    r = 64 * 10 + 10
    c = A.col[A.row_ptr[r]:A.row_ptr[r + 1]]
    v = A.val[A.row_ptr[r]:A.row_ptr[r + 1]]
    d = dict(zip(c.tolist(), v.tolist()))
    assert d[r] == pytest.approx(16900.0, rel=1e-14)
    assert d[r - 1] == pytest.approx(-4875.0, rel=1e-14)
    assert d[r + 1] == pytest.approx(-3575.0, rel=1e-14)
    assert d[r - 64] == pytest.approx(-4875.0, rel=1e-14)
    assert d[r + 64] == pytest.approx(-3575.0, rel=1e-14)


@pytest.mark.parametrize("kind,N,dims", [(5, 12, 2), (7, 9, 3), (27, 8, 3)])
def test_stencil_consistency(kind, N, dims):
    beta = (3.0, -2.0, 5.0)
    A = inputs.stencil(kind, N, beta)
    inner = interior_mask(N, dims)
    X = coords(N, dims)
    scale = np.abs(A.val).max()
    # constant: interior row sums = 0
    assert np.abs(spmv(A, np.ones(A.n))[inner]).max() <= 1e-12 * scale
    for d in range(dims):
        # linear u = x_d: −Δu = 0, β·∇u = β_d
        y = spmv(A, X[d])
        assert np.allclose(y[inner], beta[d], rtol=0, atol=1e-9 * scale)
        # quadratic u = x_d²: −Δu = −2, β·∇u = 2 β_d x_d
        y2 = spmv(A, X[d] ** 2)
        assert np.allclose(y2[inner], -2.0 + 2.0 * beta[d] * X[d][inner], rtol=0, atol=1e-8 * scale)


@pytest.mark.parametrize("kind", [5, 7, 27])
def test_beta_zero_symmetric(kind):
    A = inputs.stencil(kind, 5, (0.0, 0.0, 0.0))
    D = A.to_dense()
    assert np.array_equal(D, D.T)


def test_randdd_properties():
    n = 100_000
    A = inputs.randdd(n, 7)
    lens = np.diff(A.row_ptr)
    assert lens.min() >= 4 and lens.max() <= 2000
    assert abs(lens.mean() - 30.0) < 1.5           # α = 1.8743 → mean 30
    assert np.median(lens) == 8
    for i in range(0, n, 997):
        s, e = A.row_ptr[i], A.row_ptr[i + 1]
        c, v = A.col[s:e], A.val[s:e]
        assert np.all(np.diff(c) > 0)
        dpos = np.nonzero(c == i)[0]
        assert dpos.size == 1
        off = np.abs(np.delete(v, dpos)).sum()
        assert v[dpos[0]] == pytest.approx(1.1 * off, rel=1e-14)


def test_determinism():
    a = inputs.randdd(5000, 3)
    b = inputs.randdd(5000, 3)
    assert np.array_equal(a.col, b.col) and np.array_equal(a.val, b.val)
    u = inputs.uniform(1000, 5)
    assert np.array_equal(u, inputs.uniform(1000, 5))
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.1
    assert not np.array_equal(u, inputs.uniform(1000, 6))


def test_problem_rhs():
    P = inputs.make("C1")
    assert np.allclose(P.A.to_dense() @ P.x_true, P.b, rtol=1e-13, atol=1e-9)
