"""Host logic of the row-partitioned solve on CPU, multi-process.

Two (and three) `gloo` processes each take their row block of a matrix, compute
its ghost list with the library's host planner (gmres_dist_ghosts, no GPU),
all-gather the ghost lists, derive what they push to every peer
(gmres_dist_sends) and emulate the kernel's halo push with gloo send/recv.
The distributed SpMV rows assembled from own + received entries must equal
the global SpMV rows, and the pushes a rank receives must cover exactly its
ghost list — the invariants the GPU halo push relies on.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
from paper_2011_01850_b200 import gmres as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(kind):
    if kind == "stencil":
        return inputs.make("C2", 12).A        # 7-pt, n = 1728
    if kind == "stencil27":
        return inputs.make("C4", 10).A        # 27-pt, n = 1000
    return inputs.make("C3", 3000).A          # random DD, ghosts almost everywhere


def _worker(rank, world, port, kind, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        A = _matrix(kind)
        bounds = G.dist_partition(A.row_ptr, world, 256)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        rp, col, val = G.split_rows(A, bounds)[rank]
        ghosts = G.dist_ghosts(rp, col, r0)
        # the planner's ghosts are exactly the out-of-block columns of the local rows
        ref = np.unique(col[(col < r0) | (col >= r1)])
        assert np.array_equal(ghosts, ref)
        allg = [None] * world
        dist.all_gather_object(allg, ghosts.tolist())
        sends = {q: G.dist_sends(r0, r1 - r0, np.asarray(allg[q], np.int32)) for q in range(world) if q != rank}
        # what each peer pushes to me (computed by the same planner on my ghost list)
        recvs = {q: G.dist_sends(int(bounds[q]), int(bounds[q + 1] - bounds[q]), ghosts) for q in range(world)
                 if q != rank}
        got = np.sort(np.concatenate([bounds[q] + r for q, r in recvs.items()])) if recvs else np.zeros(0, np.int64)
        assert np.array_equal(got, ghosts.astype(np.int64))
        # halo push emulated with gloo point-to-point (the kernel uses peer stores)
        rng = np.random.default_rng(7)
        x = rng.uniform(-1, 1, A.n)
        full = np.full(A.n, np.nan)
        full[r0:r1] = x[r0:r1]
        for q in range(world):
            if q == rank:
                continue
            out = torch.from_numpy(x[r0:r1][sends[q]].copy())
            inc = torch.empty(recvs[q].size, dtype=torch.float64)
            if rank < q:
                dist.send(out, q)
                dist.recv(inc, q)
            else:
                dist.recv(inc, q)
                dist.send(out, q)
            full[int(bounds[q]) + recvs[q]] = inc.numpy()
        y = np.array([np.dot(val[rp[i]:rp[i + 1]], full[col[rp[i]:rp[i + 1]]]) for i in range(r1 - r0)])
        y_ref = inputs.matvec(A, x)[r0:r1]
        assert np.all(np.isfinite(y)), "a gathered column was not delivered"
        assert np.allclose(y, y_ref, rtol=1e-13, atol=1e-13 * np.abs(y_ref).max())
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("kind", ["stencil", "stencil27", "randdd"])
@pytest.mark.parametrize("world", [2, 3])
def test_halo_plan_gloo(kind, world):
    G.load_library()  # host functions only: no GPU needed
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_partition_properties():
    A = inputs.make("C3", 5000).A
    for P in (1, 2, 4, 8):
        b = G.dist_partition(A.row_ptr, P, 256)
        assert b[0] == 0 and b[-1] == A.n and np.all(np.diff(b) > 0)
        assert np.all(b[1:-1] % 256 == 0)
        cost = np.diff(b) + np.diff(A.row_ptr[b])
        assert cost.max() <= cost.mean() * 1.2 + 256 + 2000   # rows+nnz balanced up to one block


def test_sends_host():
    g = np.array([3, 10, 11, 500, 700], np.int32)
    assert np.array_equal(G.dist_sends(256, 512, g), np.array([500 - 256, 700 - 256]))
    assert G.dist_sends(0, 3, g).size == 0
