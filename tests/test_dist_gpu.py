"""Row-partitioned solve on one B200 through "virtual ranks".

P ranks, each a gmres_create_dist context holding its own row block (local
CSR rows, global columns), are linked in-process and solved in ONE
cooperative launch (sms/P CTAs per rank) by the same kernel code the
one-process-per-GPU path runs: cross-rank all-reduces of the Gram–Schmidt
dots, halo pushes of the gathered vectors into the peers' copies.  Parity:
oracle-recomputed ‖b − Ax‖/‖b‖ ≤ 1e-10 on the assembled x, restart count
within ±10 % of the oracle's (BASELINE.json), and every rank reports the
same cycles / inner iterations / residual (replicated control flow).
"""
import numpy as np
import pytest

import inputs
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_01850_b200 import gmres as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    G.load_library()
    yield


PROBS = {
    "C2mini": lambda: inputs.make("C2", 24),      # 7-pt stencil: ghosts = neighbouring planes
    "C3mini": lambda: inputs.make("C3", 20000),   # random DD: ghosts almost everywhere
    "C4mini": lambda: inputs.make("C4", 16),      # 27-pt stencil
}


def dist_solve(P, nranks, **kw):
    A = P.A
    bounds = G.dist_partition(A.row_ptr, nranks, 256)
    parts = G.split_rows(A, bounds)
    S = [G.Solver.from_csr_dist(rp, c, v, A.n, bounds[q], nranks, q) for q, (rp, c, v) in enumerate(parts)]
    G.link_local(S)
    bs = [torch.from_numpy(P.b[bounds[q]:bounds[q + 1]].copy()).cuda() for q in range(nranks)]
    xs = [torch.zeros_like(b) for b in bs]
    res = G.solve_virtual(S, bs, xs, **kw)
    x = np.concatenate([t.cpu().numpy() for t in xs])
    for s in S:
        s.close()
    return res, x, bounds


@pytest.mark.parametrize("name", sorted(PROBS))
@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
@pytest.mark.parametrize("prec", [G.FP64, G.MIXED])
def test_virtual_ranks_solve(name, nranks, ortho, prec):
    P = PROBS[name]()
    m = min(P.m, 50)
    res, x, bounds = dist_solve(P, nranks, m=m, tol=1e-10, ortho=ortho, precision=prec)
    assert len(set(np.diff(bounds) > 0)) == 1
    ref = O.solve(P.A, P.b, m=m, tol=1e-10, ortho=ortho, prec=prec)
    assert all(r.status == 0 for r in res), [r.status for r in res]
    rel = np.linalg.norm(P.b - O.spmv64(P.A, x)) / np.linalg.norm(P.b)
    assert rel <= 1e-10, rel
    # replicated control flow: identical decisions and sums on every rank
    assert len({(r.cycles, r.inner_iters, r.final_relres) for r in res}) == 1
    assert abs(res[0].cycles - ref.cycles) <= 0.1 * ref.cycles, (res[0].cycles, ref.cycles)
    assert res[0].final_relres == pytest.approx(rel, rel=1e-3, abs=1e-13)


@pytest.mark.parametrize("name", ["C2mini", "C3mini"])
@pytest.mark.parametrize("ortho", [G.MGS, G.CGSR])
def test_virtual_ranks_system_scope(name, ortho):
    """The multi-GPU memory-order path on one device: tune bit 21 forces the system-scope
    release/acquire (red.release.sys / ld.acquire.sys) the IPC ranks use; same decisions and
    the same x bit for bit as the GPU-scope run (only the ordering scope differs).  C3mini also
    exercises the whole-row-block halo pushes (each rank gathers > half of the other's rows)."""
    P = PROBS[name]()
    kw = dict(m=40, tol=1e-10, ortho=ortho, precision=G.MIXED)
    r_gpu, x_gpu, _ = dist_solve(P, 2, **kw)
    r_sys, x_sys, _ = dist_solve(P, 2, tune=2097152, **kw)
    assert all(r.status == 0 for r in r_sys)
    assert [(r.cycles, r.inner_iters) for r in r_sys] == [(r.cycles, r.inner_iters) for r in r_gpu]
    assert np.array_equal(x_sys, x_gpu)
    assert np.linalg.norm(P.b - O.spmv64(P.A, x_sys)) / np.linalg.norm(P.b) <= 1e-10


def test_virtual_ranks_match_single_rank():
    """Same matrix, 1 rank vs 2 ranks: same restart count and inner iterations (stencil, fp64)."""
    P = inputs.make("C2", 24)
    S1 = G.Solver.from_csr(P.A)
    b = torch.from_numpy(P.b).cuda()
    x = torch.zeros_like(b)
    r1 = S1.solve_device(b, x, m=30, tol=1e-10, ortho=G.CGSR, precision=G.FP64)
    res, x2, _ = dist_solve(P, 2, m=30, tol=1e-10, ortho=G.CGSR, precision=G.FP64)
    assert res[0].cycles == r1.cycles and abs(res[0].inner_iters - r1.inner_iters) <= 1
    assert np.linalg.norm(x2 - x.cpu().numpy()) <= 1e-8 * np.linalg.norm(x2)


def test_virtual_ranks_repeat_solves():
    """Monotonic arrival counters: back-to-back solves on the same linked contexts."""
    P = inputs.make("C2", 16)
    A = P.A
    bounds = G.dist_partition(A.row_ptr, 2, 256)
    S = [G.Solver.from_csr_dist(rp, c, v, A.n, bounds[q], 2, q) for q, (rp, c, v) in enumerate(G.split_rows(A, bounds))]
    G.link_local(S)
    bs = [torch.from_numpy(P.b[bounds[q]:bounds[q + 1]].copy()).cuda() for q in range(2)]
    for ortho in (G.MGS, G.CGSR, G.MGS):
        xs = [torch.zeros_like(b) for b in bs]
        res = G.solve_virtual(S, bs, xs, m=20, tol=1e-10, ortho=ortho, precision=G.MIXED)
        x = np.concatenate([t.cpu().numpy() for t in xs])
        assert res[0].status == 0
        assert np.linalg.norm(P.b - O.spmv64(A, x)) / np.linalg.norm(P.b) <= 1e-10


def test_dist_errors():
    P = inputs.make("C2", 16)
    A = P.A
    parts = G.split_rows(A, [0, 1000, A.n])  # 1000 is not a multiple of 256
    with pytest.raises(G.GmresError):
        G.Solver.from_csr_dist(*parts[0], A.n, 0, 2, 0)
    bounds = G.dist_partition(A.row_ptr, 2, 256)
    S = [G.Solver.from_csr_dist(rp, c, v, A.n, bounds[q], 2, q) for q, (rp, c, v) in enumerate(G.split_rows(A, bounds))]
    b = torch.from_numpy(P.b[:bounds[1]].copy()).cuda()
    with pytest.raises(G.GmresError):   # not linked
        S[0].solve_device(b, torch.zeros_like(b))
    G.link_local(S)
    with pytest.raises(G.GmresError):   # virtual ranks are solved together
        S[0].solve_device(b, torch.zeros_like(b))


def _ipc_worker(rank, port, errq):
    import os
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        A = inputs.make("C2", 16).A
        bounds = G.dist_partition(A.row_ptr, 2, 256)
        rp, c, v = G.split_rows(A, bounds)[rank]
        S = G.Solver.from_csr_dist(rp, c, v, A.n, bounds[rank], 2, rank)
        blobs = [None, None]
        dist.all_gather_object(blobs, S.export_blob())
        S.import_blobs(blobs)        # opens the peer's CUDA IPC handles
        dist.barrier()
        S.close()
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def test_ipc_export_import_two_processes():
    """One process per GPU plumbing: blobs (ghosts + CUDA IPC handles) exchanged and
    opened by two processes.  (Both share cuda:0 here, so no solve is launched:
    kernels of different processes that wait on one another must not share a GPU.)"""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, errq)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(180)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in ps)
