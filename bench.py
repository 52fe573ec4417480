#!/usr/bin/env python
"""bench.py — B200 benchmark of mixed-precision restarted GMRES(m) (arXiv 2011.01850).

Workload (BASELINE.json configs[1], "C2"): 3-D 7-point convection–diffusion on a
128³ grid (n = 2,097,152, nnz = 14,581,760, β = (10,5,2), h = 1/129), b = A·x_true
with x_true ~ U(−1,1) seed 1, x0 = 0, Jacobi, GMRES(m = 50), tol 1e-10.
One STEP = one pass of the whole hot path (every row of SURVEY.md §8(a)): a
mixed-precision MGS solve and a mixed-precision CGSR solve, each from x0 = 0 to
‖b − A x‖/‖b‖ ≤ 1e-10, each including its fp32 copy of A.

metric: GMRES restart cycles/s over the step (higher is better); the JSON line
also carries time-to-solution per variant, the fp64 arm for the mixed-over-fp64
speedup, the HBM roofline of the fused solve kernel, the CPU oracle baseline,
an end-to-end figure through gmres_solve with host buffers, and SM clocks.
Inputs (A 183 MB + V 428 MB per solve) exceed the 126 MB L2, so no flush is
needed between steps.  `--impl reference` times the CPU oracle instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD = "C2"
M = 50
TOL = 1e-10
FALLBACK_HBM_GBS = 6650.0


# ---------------------------------------------------------------- byte model
def model_bytes(n, nnz, wb, ortho, cycle_iters, cast=False):
    """Algorithmic HBM bytes of one solve.

    Per inner step j: SpMV_j = (wb+4)·nnz + 4(n+1) + 3·wb·n;
    MGS_j = wb·n·j + wb·n; CGSR_j = 3·wb·n·j + 5·wb·n.
    Per cycle: RESID = 12·nnz + 4(n+1) + 16n + 2·wb·n; UPDATE = wb·n·J + 16n.
    Plus the final residual (the converged stop test) and, in mixed mode, the
    A32 cast (8·nnz read + 4·nnz written) when `cast`.
    """
    spmv = (wb + 4) * nnz + 4 * (n + 1) + 3 * wb * n
    resid = 12 * nnz + 4 * (n + 1) + 16 * n + 2 * wb * n
    total = 0
    for J in cycle_iters:
        for j in range(1, int(J) + 1):
            orth = (wb * n * j + wb * n) if ortho == 0 else (3 * wb * n * j + 5 * wb * n)
            total += spmv + orth
        total += resid + wb * n * int(J) + 16 * n
    total += resid
    if cast:
        total += 12 * nnz
    return total


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- arms
def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def oracle_sample(prob, budget_cycles=1):
    """Time the CPU oracle (as it stands, 1 thread) on a bounded sample of the
    workload: `budget_cycles` restart cycle(s) of the mixed MGS and the mixed
    CGSR solve from x0 = 0.  Returns (cycles/s, seconds, sample text)."""
    import oracle as O
    t0 = time.perf_counter()
    cyc = 0
    for ortho in (O.MGS, O.CGSR):
        r = O.solve(prob.A, prob.b, m=M, tol=TOL, ortho=ortho, prec=O.MIXED, max_cycles=budget_cycles)
        cyc += r.cycles
    dt = time.perf_counter() - t0
    return cyc / dt, dt, (f"{budget_cycles} restart cycle(s) of the mixed MGS and of the mixed CGSR solve "
                          f"(m={M}) on the full {WORKLOAD} matrix, oracle single-threaded, incl. its A32 cast")


def golden_tts(cfg, m, variants=None):
    """The oracle's full time-to-solution records (tests/golden/full_size, tools/make_golden.py)."""
    out = {}
    for prec in ("mixed", "fp64"):
        for ortho in ("mgs", "cgsr"):
            p = os.path.join(ROOT, "tests", "golden", "full_size", f"{cfg}_{prec}_{ortho}_m{m}.json")
            if not os.path.exists(p):
                continue
            g = json.load(open(p))
            rec = {"seconds": g["seconds"], "threads": g["threads"], "cycles": g["cycles"],
                   "inner_iters": g["inner_iters"], "host_cpu": g.get("host_cpu")}
            if variants and f"{prec}_{ortho}" in variants:
                rec["gpu_cycles"] = variants[f"{prec}_{ortho}"]["cycles"]
                rec["gpu_tts_ms"] = variants[f"{prec}_{ortho}"]["tts_ms"]
            out[f"{prec}_{ortho}"] = rec
    return out


def extra_config(name, m, peak):
    """One config of BASELINE.json at full size: every variant once (after a warm-up solve),
    time-to-solution, restart counts next to the oracle's golden records, model GB/s and the
    fraction of the measured HBM peak of the fused solve kernel."""
    import torch
    import inputs
    from paper_2011_01850_b200 import gmres as G
    P = inputs.make(name)
    S = G.Solver.from_csr(P.A)
    b = torch.from_numpy(P.b).cuda()
    out = {"n": P.A.n, "nnz": P.A.nnz, "m": m}
    for prec in (G.MIXED, G.FP64):
        for ortho in (G.MGS, G.CGSR):
            x = torch.zeros_like(b)
            S.solve_device(b, x, m=m, tol=TOL, ortho=ortho, precision=prec, max_cycles=1)  # warm-up
            x.zero_()
            r = S.solve_device(b, x, m=m, tol=TOL, ortho=ortho, precision=prec)
            wb = 4 if prec == G.MIXED else 8
            mb = model_bytes(P.A.n, P.A.nnz, wb, ortho, r.cycle_iters)
            key = ("mixed_" if prec == G.MIXED else "fp64_") + ("mgs" if ortho == 0 else "cgsr")
            gold = golden_tts(name, m).get(key, {})
            out[key] = {"status": r.status_name, "tts_ms": r.device_ms, "kernel_ms": r.kernel_ms,
                        "cycles": r.cycles, "inner_iters": r.inner_iters, "final_relres": r.final_relres,
                        "final_backward_err": r.final_backward_err, "oracle_cycles": gold.get("cycles"),
                        "oracle_inner_iters": gold.get("inner_iters"), "model_GB": mb / 1e9,
                        "model_GBps": mb / (r.kernel_ms * 1e-3) / 1e9,
                        "frac_of_peak": mb / (r.kernel_ms * 1e-3) / 1e9 / peak,
                        "mgs_variant": S.plan().get("mgs_variant") if ortho == 0 else None,
                        "phase_ms": {k: v / 1e6 for k, v in zip(["resid", "spmv", "ortho", "givens", "update"],
                                                                  r.phase_ns[:5])}}
    out["mixed_over_fp64_tts_speedup"] = {o: out[f"fp64_{o}"]["tts_ms"] / out[f"mixed_{o}"]["tts_ms"]
                                          for o in ("mgs", "cgsr")}
    S.close()
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return
    import inputs
    prob = inputs.make(WORKLOAD)
    times, vals = [], []
    for i in range(args.warmup + args.steps):
        v, dt, sample = oracle_sample(prob, 1)
        if i >= args.warmup:
            times.append(dt)
            vals.append(v)
    value = sum(2 for _ in times) / sum(times)
    line = {
        "impl": "reference", "metric": metric_name(), "value": value, "unit": "cycles/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (mixed)",
        "data": "synthetic", "config": config(),
        "cpu_baseline": {"value": value, "unit": "cycles/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cores": cpu_cores()},
        "e2e": {"value": value, "unit": "cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name():
    return ("GMRES restart cycles/s (time-to-1e-10 solves; C2 128^3 7-pt, m=50, mixed fp32/fp64, "
            "one MGS + one CGSR solve per step)")


def config():
    return {"workload": "C2: 3-D 7-pt convection-diffusion 128^3 (n=2097152, nnz=14581760), beta=(10,5,2), "
                        "b=A*x_true (U(-1,1) seed 1), x0=0, Jacobi, GMRES(m=50), tol 1e-10",
            "step": "mixed MGS solve + mixed CGSR solve, each to 1e-10 incl. the A32 cast",
            "l2": "inputs larger than L2 (A 183 MB + V 428 MB per solve); no flush",
            "parallelism": "1 GPU"}


def run_ours(args, rank, world, local_rank):
    import torch
    import inputs
    from paper_2011_01850_b200 import gmres as G

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    prob = inputs.make(WORKLOAD)
    A = prob.A
    if world == 1:
        S = G.Solver.from_csr(A)
        r0, r1 = 0, A.n
    else:
        # row partition over the GPUs: rank q owns rows [bounds[q], bounds[q+1]);
        # exchange buffers are shared over NVLink via CUDA IPC (blobs all-gathered here)
        bounds = G.dist_partition(A.row_ptr, world, 256)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        rp, col, val = G.split_rows(A, bounds)[rank]
        S = G.Solver.from_csr_dist(rp, col, val, A.n, r0, world, rank)
        blobs = [None] * world
        torch.distributed.all_gather_object(blobs, S.export_blob())
        S.import_blobs(blobs)
        torch.distributed.barrier()
    n, nnz = S.n, S.nnz  # this rank's rows
    b = torch.from_numpy(prob.b[r0:r1].copy()).to(dev)
    x = torch.zeros_like(b)
    stream = torch.cuda.current_stream()

    def step(prec=G.MIXED, out=None):
        cyc = 0
        for ortho in (G.MGS, G.CGSR):
            r = S.solve_device(b, x, m=M, tol=TOL, ortho=ortho, precision=prec, stream=stream)
            if r.status != 0:
                raise RuntimeError(f"solve failed: {r.status_name}")
            cyc += r.cycles
            if out is not None:
                out.append((ortho, r))
        return cyc

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    per = []
    total_cycles = 0
    for _ in range(args.steps):
        total_cycles += step(out=per)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    if world > 1:  # one global problem: every rank ran the same cycles; time = max over ranks
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    value = total_cycles / (elapsed_ms / 1e3)

    # roofline of the dominant kernel (the fused solve kernel: one launch per solve)
    peak, peak_src = measured_peak()
    ach, kms, byts = [], [], []
    variants = {}
    for ortho, r in per:
        mb = model_bytes(n, nnz, 4, ortho, r.cycle_iters)
        byts.append(mb)
        kms.append(r.kernel_ms)
        ach.append(mb / (r.kernel_ms * 1e-3) / 1e9)
    for ortho, r in per[-2:]:
        name = "mixed_" + ("mgs" if ortho == 0 else "cgsr")
        variants[name] = {"tts_ms": r.device_ms, "kernel_ms": r.kernel_ms, "cycles": r.cycles,
                          "inner_iters": r.inner_iters, "final_relres": r.final_relres,
                          "final_backward_err": r.final_backward_err,
                          "model_GBps": model_bytes(n, nnz, 4, ortho, r.cycle_iters, cast=True) / (r.device_ms * 1e-3) / 1e9,
                          "phase_ms": {k: v / 1e6 for k, v in zip(["resid", "spmv", "ortho", "givens", "update"],
                                                                    r.phase_ns[:5])}}
    achieved = sum(byts) / (sum(kms) * 1e-3) / 1e9
    # DRAM traffic per launch: the traffic/algorithmic ratio ncu measured for each
    # variant's launch (profiles/traffic.json) applied to the timed launches
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and world == 1:
        try:
            tj = json.load(open(tp))
            tr = [tj["mgs" if o == 0 else "cgsr"]["ratio"] * mb for (o, _), mb in zip(per, byts)]
            traffic = sum(tr) / len(tr)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src,
                "kernel": "g200::solve_kernel<float,1,false> (fused persistent solve, 1 launch per solve)",
                "algorithmic_bytes_per_launch": sum(byts) / len(byts), "frac_of_8TBps": achieved / 8000.0}

    # fp64 arm (mixed-over-fp64 time-to-solution speedup, BASELINE.json target)
    fp64 = []
    step(G.FP64)
    for _ in range(max(1, min(args.steps, 3))):
        step(G.FP64, out=fp64)
    for ortho, r in fp64[-2:]:
        name = "fp64_" + ("mgs" if ortho == 0 else "cgsr")
        variants[name] = {"tts_ms": r.device_ms, "kernel_ms": r.kernel_ms, "cycles": r.cycles,
                          "inner_iters": r.inner_iters, "final_relres": r.final_relres,
                          "model_GBps": model_bytes(n, nnz, 8, ortho, r.cycle_iters) / (r.device_ms * 1e-3) / 1e9}
    speedup = {o: variants[f"fp64_{o}"]["tts_ms"] / variants[f"mixed_{o}"]["tts_ms"] for o in ("mgs", "cgsr")}

    # §8 f2: the paper's preconditioner, ILU(0), on the same problem —
    # one solve per variant outside the timed step, factorisation included
    ilu = {}
    if world == 1 and not args.no_ilu:
        lo, up = S.ilu0_levels()  # one-time host level analysis (per context, like gmres_create)
        for prec in (G.MIXED, G.FP64):
            for ortho in (G.MGS, G.CGSR):
                xi = torch.zeros_like(x)
                r = S.solve_device(b, xi, m=M, tol=TOL, ortho=ortho, precision=prec, precond=G.ILU0)
                assert r.status == 0, r.status_name
                ilu[("mixed_" if prec == G.MIXED else "fp64_") + ("mgs" if ortho == 0 else "cgsr")] = {
                    "tts_ms": r.device_ms, "cycles": r.cycles, "inner_iters": r.inner_iters,
                    "us_per_inner": 1e3 * r.kernel_ms / max(1, r.inner_iters), "final_relres": r.final_relres}
        ilu["levels"] = {"lower": lo, "upper": up}

    # the paper's third arm: the fp64 solver with an fp32 ILU(0)
    if world == 1 and not args.no_ilu:
        for ortho in (G.MGS, G.CGSR):
            xi = torch.zeros_like(x)
            r = S.solve_device(b, xi, m=M, tol=TOL, ortho=ortho, precision=G.FP64, precond=G.ILU0_FP32)
            assert r.status == 0, r.status_name
            ilu["fp64_ilu32_" + ("mgs" if ortho == 0 else "cgsr")] = {
                "tts_ms": r.device_ms, "cycles": r.cycles, "inner_iters": r.inner_iters,
                "us_per_inner": 1e3 * r.kernel_ms / max(1, r.inner_iters), "final_relres": r.final_relres}

    # e2e through gmres_solve with pinned host buffers (h2d b, d2h x inside every call)
    hb = torch.from_numpy(prob.b[r0:r1].copy()).pin_memory()
    hb_np = hb.numpy()
    hx_np = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    e2e_cycles = 0
    for ortho in (G.MGS, G.CGSR):
        S.solve(hb_np, m=M, tol=TOL, ortho=ortho, precision=G.MIXED, out=hx_np)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for ortho in (G.MGS, G.CGSR):
            r = S.solve(hb_np, m=M, tol=TOL, ortho=ortho, precision=G.MIXED, out=hx_np)
            e2e_cycles += r.cycles
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": e2e_cycles / e2e_s, "unit": "cycles/s", "h2d_bytes_per_step": 2 * 8 * n,
           "d2h_bytes_per_step": 2 * 8 * n, "api": "gmres_solve (pinned host b in, pinned host x out)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, dt, sample = oracle_sample(prob, 1)
        cpu = {"value": v, "unit": "cycles/s", "cores": 1, "kind": "oracle", "sample": sample,
               "seconds": dt, "host_cores": cpu_cores(),
               # the oracle's whole time-to-solution on this workload, recorded once by
               # tools/make_golden.py (OpenMP build, bitwise equal to the 1-thread one),
               # next to the GPU's restart counts of this run
               "full_tts_recorded": golden_tts("C2", M, variants)}

    # the other BASELINE.json configs at full size (untimed: one solve per variant after a warm-up)
    extra = None
    if rank == 0 and world == 1 and not args.no_extra:
        S.close()
        S = None
        extra = {name: extra_config(name, m, peak) for name, m in (("C3", 50), ("C4", 100))}

    if rank == 0:
        cfg = config()
        cfg["parallelism"] = (f"row partition over {world} GPUs (rank 0: rows {r0}..{r1}); dot/norm all-reduces "
                              "and SpMV halo as NVLink peer stores inside the persistent kernel") if world > 1 \
            else "1 GPU"
        line = {
            "metric": metric_name(), "value": value, "unit": "cycles/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f32 (Arnoldi) + f64 (residual, update)",
            "data": "synthetic", "config": cfg,
            "tts_ms": {k: v["tts_ms"] for k, v in variants.items()},
            "mixed_over_fp64_tts_speedup": speedup,
            "variants": variants,
            "ilu0_untimed": ilu or None,
            "roofline": roofline,
            "extra_configs": extra,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": 4 * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if S is not None:
        S.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--no-ilu", action="store_true", help="skip the untimed ILU(0) solves (§8 f2)")
    ap.add_argument("--no-extra", action="store_true", help="skip the untimed full-size C3 / C4 solves")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
