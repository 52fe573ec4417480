"""Seeded irregular test matrices for the merge-path CSR stream (test inputs only:
numpy generators, no arithmetic of the method).  C3's power-law rows come from
inputs.make; the others stress what a non-zero split across lanes and tiles can
get wrong."""
import numpy as np

import inputs


def _dd(rowlens, seed):
    """Diagonally dominant CSR with the given row lengths (diagonal included, sorted
    distinct columns, N(0,1) off-diagonal values, a_ii = 1.1·Σ|a_ij| as C3)."""
    rng = np.random.default_rng(seed)
    n = len(rowlens)
    rp = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for i, k in enumerate(rowlens):
        k = int(min(max(k, 1), n))
        others = rng.choice(n - 1, size=k - 1, replace=False)
        others = others + (others >= i)             # skip the diagonal
        c = np.sort(np.concatenate([others, [i]])).astype(np.int32)
        v = rng.standard_normal(k)
        d = np.searchsorted(c, i)
        v[d] = 0.0
        v[d] = 1.1 * np.abs(v).sum() + (1.0 if k == 1 else 0.0)
        cols.append(c)
        vals.append(v)
        rp[i + 1] = rp[i] + k
    return inputs.CSR(rp.astype(np.int32), np.concatenate(cols), np.concatenate(vals))


def _longrows():
    rng = np.random.default_rng(11)
    n = 6000
    k = rng.integers(2, 41, n)
    k[[0, 17, 2999, 3000, 5999]] = [n, 4000, n, 3001, n]   # rows spanning up to 24 tiles
    k[100:110] = [257, 511, 1024, 256, 255, 9, 258, 1, 2000, 767]
    return _dd(k, 1)


def _diag1():
    rng = np.random.default_rng(12)
    n = 9000
    k = np.where(rng.uniform(size=n) < 0.6, 1, rng.integers(65, 400, n))   # 60 % diagonal-only rows
    return _dd(k, 2)


MATS = {
    "c3mini": lambda: inputs.make("C3", 20000).A,
    "longrows": _longrows,
    "diag1": _diag1,
    "tiny": lambda: _dd(np.r_[100, np.full(99, 3)], 3),       # n = 100: most CTAs own no row
}
