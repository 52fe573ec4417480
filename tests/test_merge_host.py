"""Host-side plan of the merge-path CSR stream, no GPU:
gmres_plan_mtiles is the planner the solves use.  The kernel's correctness rests
on these invariants — every non-zero of a CTA in exactly one tile, in order; a
tile's positions within 256 of its 8-aligned base (8 per lane) and at most 31
rows (one row_ptr entry per lane); a tile's first row the row of its first
non-zero; every row that spans tiles listed once with the tiles of its first and
last non-zero, being the last row of the first and the first (open-left) row of
the others, which hold nothing else in between (the carry slots the fix-up
sums, gmres_kernels.cuh csr_merge_stream)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from merge_mats import MATS  # noqa: E402

from paper_2011_01850_b200 import gmres as G  # noqa: E402


def _check(A, rb):
    rp = A.row_ptr.astype(np.int64)
    tiles, toff, splits, soff = G.plan_mtiles(A.row_ptr, rb)
    Gn = rb.size - 1
    assert toff[-1] == len(tiles) and soff[-1] == len(splits)
    row_tiles = {}  # row → tiles holding its non-zeros
    for g in range(Gn):
        r0, r1 = min(rb[g], A.n), min(rb[g + 1], A.n)
        ent = tiles[toff[g]:toff[g + 1]]
        assert len(ent) >= 1 and tuple(ent[-1][:2]) == (r1, rp[r1])   # sentinel
        pos = rp[r0]
        for t in range(len(ent) - 1):
            c = toff[g] + t
            row, s, nr = int(ent[t][0]), int(ent[t][1]), int(ent[t][2])
            ne = int(ent[t + 1][1])
            assert s == pos and ne > s, (g, t)                          # contiguous, non-empty
            assert ne - (s & ~7) <= 256                                 # 32 lanes × 8 positions
            assert rp[row] <= s < rp[row + 1]                           # first row holds s
            last = int(np.searchsorted(rp, ne - 1, side="right")) - 1  # row holding ne − 1
            assert nr == last - row + 1 and 1 <= nr <= 31
            for r in range(row, last + 1):
                row_tiles.setdefault(r, []).append(c)
            pos = ne
        assert pos == rp[r1]
        # split rows of this CTA: exactly the rows whose non-zeros span tiles
        want = sorted(r for r, ts in row_tiles.items() if r0 <= r < r1 and len(ts) > 1)
        got = splits[soff[g]:soff[g + 1]]
        assert sorted(int(x[0]) for x in got) == want
        for r, tf, tl, _ in got:
            ts = row_tiles[int(r)]
            assert (tf, tl) == (ts[0], ts[-1]) and ts == list(range(tf, tl + 1))
            # tile tf: r is its last row; later tiles: r is the first row, open-left;
            # tiles strictly between hold only r
            assert int(np.searchsorted(rp, int(tiles[tf + 1][1]) - 1, side="right")) - 1 == r
            for c in range(tf + 1, tl + 1):
                assert tiles[c][0] == r and tiles[c][1] > rp[r]
            for c in range(tf + 1, tl):
                assert tiles[c][2] == 1
    return tiles, splits


@pytest.mark.parametrize("name", sorted(MATS))
@pytest.mark.parametrize("G_", [1, 7, 148])
def test_mtiles_invariants(name, G_):
    A = MATS[name]()
    nvec = -(-A.n // 256) * 256
    # the solve's CTA split: boundaries at multiples of 32 rows balancing rows + nnz
    tot = A.n + A.nnz
    cost = np.arange(0, nvec + 1, 32) + A.row_ptr[np.minimum(np.arange(0, nvec + 1, 32), A.n)]
    b = [0] + [int(np.searchsorted(cost, tot * g / G_) * 32) for g in range(1, G_)] + [nvec]
    b = np.maximum.accumulate(np.minimum(np.array(b), nvec)).astype(np.int32)
    tiles, splits = _check(A, b)
    if name == "longrows":  # rows of 4000-6000 non-zeros span ≥ 16 tiles
        assert max(int(t) - int(f) for _, f, t, _ in splits) >= 15


def test_mtiles_rejects_empty_rows():
    rp = np.array([0, 1, 1, 2], np.int32)
    with pytest.raises(G.GmresError):
        G.plan_mtiles(rp, np.array([0, 3], np.int32))
