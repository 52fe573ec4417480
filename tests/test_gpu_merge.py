"""Merge-path CSR stream (BASELINE.json north_star (a): "vectorised
warp-per-row and merge-path CSR SpMV"), through the C ABI.

Irregular matrices (rows longer than the block stream's 64 non-zeros) run the
merge-path tiles: equal non-zeros per lane, rows split across lanes and tiles,
crossing rows summed from per-tile partials after the CTA barrier.  The
matrices below stress what that split can get wrong: rows spanning many tiles
(up to n non-zeros), rows of one non-zero (the 31-rows-per-tile cut), long and
short rows interleaved, mostly-empty grids (n < CTAs · 32), the power-law rows of
C3.  SpMV (Alg. 1) and the residual (line 86) are
compared with the oracle element by element; whole solves with the oracle's
recomputed residual and restart count; the chunk stream (tune bit 22) is the
A/B reference path.
"""
import math
import os
import sys

import numpy as np
import pytest

import inputs
import oracle as O

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_01850_b200 import gmres as G  # noqa: E402

DEV = "cuda:0"
CHUNK_STREAM = 4194304  # tune bit 22: the per-warp chunk stream instead of the merge-path tiles


from merge_mats import MATS  # noqa: E402


@pytest.fixture(scope="module", params=sorted(MATS))
def mat(request):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    G.load_library()
    A = MATS[request.param]()
    return request.param, A, G.Solver.from_csr(A)


def tdev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_merge_spmv_parity(mat, prec):
    name, A, S = mat
    rng = np.random.default_rng(5)
    aW, dW = O.working_copy(A, prec)
    v = rng.uniform(-1, 1, A.n).astype(np.float32 if prec == G.MIXED else np.float64)
    w_o = O.jacobi_spmv(prec, A, aW, dW, v)
    wd = torch.empty(A.n, dtype=torch.float32 if prec == G.MIXED else torch.float64, device=DEV)
    S.k_spmv(prec, tdev(v), wd)
    w = wd.cpu().numpy()
    rel = np.linalg.norm(w.astype(np.float64) - w_o) / np.linalg.norm(w_o)
    assert rel <= (1e-12 if prec == G.FP64 else 1e-5), rel   # BASELINE.json per-kernel bar
    # componentwise, any summation order: |ŵ_i − w_i| ≤ γ_{k+1} |dinv_i| (|A||v|)_i (+ the final scaling)
    u = 2.0 ** -53 if prec == G.FP64 else 2.0 ** -24
    rpx = A.row_ptr
    prod = aW.astype(np.float64) * v[A.col].astype(np.float64)
    absAv = np.add.reduceat(np.abs(prod), rpx[:-1])
    exact = np.array([math.fsum(prod[rpx[i]:rpx[i + 1]]) for i in range(A.n)]) * dW.astype(np.float64)
    k = np.diff(rpx) + 1
    gam = k * u / (1 - k * u)
    bad = np.abs(w - exact) > 2 * gam * np.abs(dW) * absAv + 1e-300
    assert not bad.any(), (name, np.nonzero(bad)[0][:10])


@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_merge_resid_parity(mat, prec):
    name, A, S = mat
    rng = np.random.default_rng(6)
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
    assert rel <= (1e-12 if prec == G.FP64 else 1e-6), rel


@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_merge_solve_matches_oracle(mat, ortho, prec):
    name, A, S = mat
    x_true = inputs.uniform(A.n, 7)
    b = inputs.matvec(A, x_true)
    ref = O.solve(A, b, m=30, tol=1e-10, ortho=ortho, prec=O.MIXED if prec == G.MIXED else O.FP64)
    bd = tdev(b)
    out = {}
    for tune in (0, CHUNK_STREAM):
        x = torch.zeros_like(bd)
        res = S.solve_device(bd, x, m=30, tol=1e-10, ortho=ortho, precision=prec, tune=tune)
        assert S.plan()["csr_stream"] == (0 if tune else 2), S.plan()
        xh = x.cpu().numpy()
        rel = np.linalg.norm(b - O.spmv64(A, xh)) / np.linalg.norm(b)
        assert res.status == 0 and rel <= 1e-10, (name, tune, res.status_name, rel)
        assert abs(res.cycles - ref.cycles) <= int(0.1 * ref.cycles), (res.cycles, ref.cycles)
        out[tune] = res
    # the two CSR streams differ only in the summation order of row sums
    assert abs(out[0].inner_iters - out[CHUNK_STREAM].inner_iters) <= max(1, out[CHUNK_STREAM].inner_iters // 20)
