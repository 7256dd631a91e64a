#!/usr/bin/env python3
"""bench.py -- AJM (arXiv 2407.03272, Alg. 3) on B200: iterations/s, achieved HBM GB/s, time to 1e-6.

Workload (BASELINE.json configs[1], the config the metric is quoted on): FP64 3D 7-point Poisson
Laplacian on a 128^3 Dirichlet grid (n = 2,097,152, nnz = 14,581,760), x* ~ U(-1,1) (seed 2),
b = Q x*, x0 = 0, eq-J-diag metric, adaptive restart on, tol 1e-6 on ||b - Qx||/||b||.
A "step" = one complete ajm_solve to tol (every Alg. 3 iteration on the device, ~330 passes).
value = whole-job AJM iterations/s (sum over ranks of iterations / max-over-ranks device time).

--impl reference times the CPU oracle (oracle/, plain C, literal two-SpMV Alg. 3) on this box's
host cores on a bounded sample of the same workload (this tier's reference arm).
Multi-GPU (torchrun, one process per GPU): by default N independent replicas of the solve, one per
GPU ("scaling": "weak") -- the north_star's path is one GPU and SURVEY.md §8(e) says "replicas
only".  --parallel shard runs the paper's row-block partition instead (Alg. 3 lines 3-5, §4.4;
DESIGN.md §6): ONE solve of the same system sharded over the N GPUs, halo entries and the five
partial sums exchanged every pass over peer memory (CUDA IPC / NVLink) by the solver kernel
itself ("scaling": "strong").
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

METRIC = "AJM iterations/s + achieved HBM GB/s (% of B200 peak); time to 1e-6 rel. residual"
UNIT = "iterations/s"
# BASELINE.json configs; the default (configs[1], the config the metric is quoted on) is the bench
# line; the others are reported with --config K (every config as a roofline fraction, north_star)
WORKLOADS = {
    1: dict(tol=0.0, maxit=2000, bound="latency",
            workload="poisson2d_64: 2D 5-pt Dirichlet Laplacian 64^2 (n=4096, nnz=20224), FP64 CSR, "
                     "x*~U(-1,1) seed 1, b=Qx*, x0=0, eq-J-diag, restart on, K0=2, 2000 iterations "
                     "(BASELINE.json configs[0]; 0.49 MB per pass: L2/latency-bound, not HBM)"),
    2: dict(tol=1e-6, maxit=5000, bound="hbm",
            workload="poisson3d_128: 3D 7-pt Dirichlet Laplacian 128^3 (n=2097152, nnz=14581760), FP64 CSR, "
                     "x*~U(-1,1) seed 2, b=Qx*, x0=0, eq-J-diag, restart on, K0=2, solve to 1e-6 rel. residual "
                     "(BASELINE.json configs[1])"),
    3: dict(tol=1e-6, maxit=5000, bound="hbm",
            workload="er_1m_deg16: weighted Erdos-Renyi Laplacian n=1M, 8M edges, w~U(0.1,1), singular SPSD, "
                     "x*~N(0,1)-mean seed 1003, b=Lx*, x0=0, eq-J-diag, restart on, solve to 1e-6 "
                     "(BASELINE.json configs[2])"),
    4: dict(tol=1e-6, maxit=5000, bound="hbm",
            workload="chunglu_4m_deg20: Chung-Lu gamma=2.1 Laplacian n=4M mean degree 20 (max row ~1e5) "
                     "+1e-3 I, w~U(0.1,1), x*~U(-1,1) seed 1004, x0=0, eq-J-diag, restart on, solve to 1e-6 "
                     "(BASELINE.json configs[3])"),
    5: dict(tol=1e-6, maxit=5000, bound="hbm",
            workload="aniso27_256: anisotropic 27-pt stencil 256^3 (n=16777216, nnz=449455096), w=(1,1,1e-2), "
                     "diag=row-abs-sum+1e-6, x*~U(-1,1) seed 5, x0=0, eq-J-diag, restart on, solve to 1e-6 "
                     "(BASELINE.json configs[4])"),
}
WORKLOAD = WORKLOADS[2]["workload"]
NOMINAL_HBM_GBS = 8000.0
GATHER_PEAK_GPS = 282.0  # random 8-byte gathers/s from an L2-resident array, measured
# The paper's own performance statements, quoted with its hardware (context, not the target;
# BASELINE.md §1). Its results are figures only, so there is no number to divide by.
PAPER_CONTEXT = {
    "published_speedups": None,
    "note": "PAPER.md §4.4 (lines 771-811) calls setup/solve/matvec 'scalable' up to 121 MPI "
            "processes over 100 iterations on Zaratan (dual AMD EPYC 7763 per node, HDR-100 IB, "
            "petsc4py CSR) but prints no speed-up values; §4.1-4.3 ran on a 2.2 GHz quad-core "
            "i7 laptop with figures only",
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload: str):
    """ncu DRAM bytes per pass of the solver kernel on this workload (profiles/ncu_traffic.json,
    committed from an `ncu --set full` capture; one record per workload name)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
    except Exception:
        return None
    recs = tr if isinstance(tr, list) else [tr]
    for r in recs:
        if r.get("workload") == workload:
            return r
    return None


# ------------------------------------------------------------------------------------------------
# distributed plumbing (one process per GPU; replicas)
# ------------------------------------------------------------------------------------------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, backend):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist if world > 1 else None


def reduce_job(iters: float, ms: float, dist=None, device=None):
    """Whole-job aggregate: iterations summed over ranks, time = max over ranks."""
    if dist is None:
        return iters, ms
    import torch
    t = torch.tensor([iters], dtype=torch.float64, device=device)
    m = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return float(t.item()), float(m.item())


def barrier(dist, device=None):
    if dist is not None:
        import torch
        if device is not None and device.type == "cuda":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


# ------------------------------------------------------------------------------------------------
# clocks during the timed region
# ------------------------------------------------------------------------------------------------

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
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
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# workload
# ------------------------------------------------------------------------------------------------

def make_problem(cfg=2):
    import synth
    return synth.config_problem(cfg)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def layout_bytes_per_iter(info, jblock=None) -> float:
    """Bytes one pass of THIS layout must move at minimum: every stored SELL entry including its
    padding (8-byte value + the streamed column index: 4 B int32 or 1 B byte code; 1 B in all for
    pair-coded entries, whose code also names the value), the warp
    segments' CSR entries (12 B), and the seven n-vectors (D replaced by bs doubles of J^-1 with
    block J).  Differs from the algorithmic model (12 nnz + 56 n + 4(n+1)) by the byte codes, the
    padding and the row offsets SELL does not need."""
    return ((info["val_bytes"] + info["col_bytes"]) * info["sell_elems"] + 12.0 * info["seg_nnz"]
            + (48.0 + 8.0 * (jblock or 1)) * info["n"])


def kernel_name(info) -> str:
    """The persistent solver kernel the handle launches."""
    if info["mode"] == 6:
        return "ajm_resident_kernel (single thread-block cluster, whole solve on chip; one launch per solve)"
    if info["band_staged"]:
        return "ajm_band_kernel (pair-coded entries, x~ bands + row operands TMA-staged; one launch per solve)"
    enc = "pair-coded entries" if info["val_bytes"] == 0 else ("byte-coded columns" if info["col_bytes"] == 1
                                                              else "int32 columns")
    return f"ajm_solve_kernel ({enc}; persistent, one launch per solve)"


def cpu_baseline_run(p, cfg=2, budget_s=12.0, nthreads=None):
    """The oracle as it stands (literal two-SpMV Alg. 3), on host cores, on a bounded sample of the
    workload: the first T iterations of the same solve, T sized to ~budget_s seconds."""
    import oracle
    nt = nthreads or (os.cpu_count() or 1)
    oracle.set_threads(nt)
    t0 = time.perf_counter()
    oracle.solve(p.Q, p.b, tol=0.0, maxit=3, restart=True)
    per_it = (time.perf_counter() - t0) / 3.0
    T = int(max(5, min(1000, budget_s / max(per_it, 1e-6))))
    t0 = time.perf_counter()
    r = oracle.solve(p.Q, p.b, tol=0.0, maxit=T, restart=True)
    dt = time.perf_counter() - t0
    return {"value": r.iterations / dt, "unit": UNIT, "cores": nt, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"first {T} iterations of the config-{cfg} solve (literal two-SpMV Alg. 3, "
                      f"plain C FP64, {nt} OpenMP threads), {dt:.2f} s wall"}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0  # rank 0 alone runs the CPU reference arm
    W = WORKLOADS[args.config]
    p = make_problem(args.config)
    import oracle
    nt = os.cpu_count() or 1
    oracle.set_threads(nt)
    # each step: a bounded sample (S iterations) of the workload's solve
    t0 = time.perf_counter()
    oracle.solve(p.Q, p.b, tol=0.0, maxit=2, restart=True)
    per_it = (time.perf_counter() - t0) / 2.0
    S = int(max(2, min(200, 8.0 / max(per_it, 1e-6))))
    for _ in range(args.warmup):
        oracle.solve(p.Q, p.b, tol=0.0, maxit=S, restart=True)
    iters, t_total = 0, 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = oracle.solve(p.Q, p.b, tol=0.0, maxit=S, restart=True)
        t_total += time.perf_counter() - t0
        iters += r.iterations
    v = iters / t_total
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": W["workload"], "sample_iterations_per_step": S},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nt, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"{S} iterations of the config-{args.config} solve per step (literal two-SpMV "
                                   f"Alg. 3, plain C FP64, {nt} OpenMP threads)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def timed_solves(solver, kw, steps, warmup, stream, dist=None, dev=None, clocks=None):
    """W untimed solves, then K solves bracketed by barrier + synchronize, CUDA events on the
    launching stream.  Returns (iterations, passes, loop_ms (sum of the solver launches' own event
    durations), ms (whole timed region), results, clocks)."""
    import torch
    for _ in range(warmup):
        solver.solve(**kw)
    torch.cuda.synchronize()
    if clocks is not None:
        clocks.start()
        time.sleep(0.3)
    barrier(dist, dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters, passes, loop_ms = 0, 0, 0.0
    results = []
    for _ in range(steps):
        r = solver.solve(**kw)
        inf = solver.info()
        iters += r.iterations
        passes += inf["last_passes"]
        loop_ms += inf["last_loop_ms"]
        results.append(r)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(dist, dev)
    clk = clocks.stop() if clocks is not None else None
    return iters, passes, loop_ms, e0.elapsed_time(e1), results, clk


def roofline_block(p, info, passes, loop_ms, steps, bound, jblock=None):
    """The dominant kernel's roofline (the persistent solver launch: one per solve).
      achieved / frac : ALGORITHMIC bytes per pass (12 nnz + 7*8 n + 4 (n+1); D -> bs
                        doubles of J^-1 with block J) x passes / the launches' CUDA-event time
      layout_frac     : the bytes this layout must move (byte-coded columns: 9 B per stored entry,
                        SELL padding, no row offsets) over the same time -- what the kernel could at
                        best save on the stream
      dram_frac       : ncu dram read+write bytes per pass of the committed capture
                        (profiles/ncu_traffic.json, per workload) over this run's time per pass --
                        the L2-resident vectors make it lower than the algorithmic figure
      l2_throughput_frac / l1tex_throughput_frac : the same capture's lts / l1tex throughput (% of
                        peak / 100): the graph configs lean on the L2 (random 32-byte gather
                        sectors), the band-staged stencils on the L1/shared-memory pipe"""
    peak, peak_src = load_peaks()
    model_bytes = info["model_bytes_per_iter"]
    sec = loop_ms * 1e-3
    achieved = model_bytes * passes / sec / 1e9
    lay = layout_bytes_per_iter(info, jblock)
    tr = None if jblock else load_traffic(p.name)
    us = 1e6 * sec / passes
    rb = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
          "traffic": None if tr is None else tr["dram_bytes_per_pass"] * passes / steps,
          "traffic_basis": "ncu dram__bytes_read.sum + dram__bytes_write.sum per pass of the solver kernel "
                           "(profiles/ncu_traffic.json" + ("" if tr is None else f", capture {tr.get('capture', '?')}")
                           + ") x passes per launch",
          "peak_source": peak_src,
          "kernel": kernel_name(info),
          "achieved_basis": "algorithmic bytes nnz*12+7n*8+4(n+1) per pass (D replaced by bs doubles of J^-1 per "
                            "row with --jblock) x passes / launch duration (CUDA events on the launch stream)",
          "layout_bytes_per_iteration": lay,
          "layout_frac": lay * passes / sec / 1e9 / peak,
          "dram_frac": None if tr is None else tr["dram_bytes_per_pass"] / (us * 1e-6) / 1e9 / peak,
          # the capture's other roofs: which on-chip resource the kernel actually leans on
          "l2_throughput_frac": None if tr is None or "l2_throughput_pct" not in tr else tr["l2_throughput_pct"] / 100.0,
          "l1tex_throughput_frac": None if tr is None or "l1tex_throughput_pct" not in tr else tr["l1tex_throughput_pct"] / 100.0}
    return rb, model_bytes, achieved, us


def gather_roof(p, info, passes, loop_ms):
    """Second roof for graph layouts (sorted windows, sigma > 1): one random 8-byte x~ gather per
    stored nonzero and pass against the measured random-gather ceiling from an L2-resident array
    (tools/ubench/gather_mlp.cu).  Stencils (sigma = 1) hit L1 on most gathers, where this roof
    does not bind -- it is not reported for them."""
    if info["sigma"] <= 1:
        return None
    gps = p.Q.nnz * passes / (loop_ms * 1e-3) / 1e9
    return {"bound": "l2_random_gather", "achieved": gps, "peak": GATHER_PEAK_GPS, "unit": "G gathers/s",
            "frac": gps / GATHER_PEAK_GPS,
            "peak_source": "measured on this pool: tools/ubench/gather_mlp.cu (8-32 MB array)"}


def other_config_record(cfg, args, dev, stream):
    """One BASELINE config other than the headline one, measured the same way (device-resident
    inputs, W warm-up + K timed solves, CUDA events): it/s, us/pass and the roofline fractions."""
    import torch
    import paper_2407_03272_b200 as ajm
    W = WORKLOADS[cfg]
    t0 = time.perf_counter()
    p = make_problem(cfg)
    gen_s = time.perf_counter() - t0
    Qd = [torch.from_numpy(a).to(dev) for a in (p.Q.row_ptr, p.Q.col, p.Q.val, p.b)]
    x_out = torch.empty(p.Q.n, dtype=torch.float64, device=dev)
    with ajm.Solver(p.Q.n, *Qd[:3], Qd[3]) as solver:
        del Qd
        kw = dict(tol=W["tol"], maxit=W["maxit"], restart=True, x_out=x_out, history=False)
        steps = max(2, min(args.steps, 5))
        clocks = ClockSampler(dev.index)
        iters, passes, loop_ms, ms, results, clk = timed_solves(solver, kw, steps, 3, stream, clocks=clocks)
        info = solver.info()
    assert all(r.status == ("converged" if W["tol"] > 0 else "maxiter") for r in results)
    rb, model_bytes, achieved, us = roofline_block(p, info, passes, loop_ms, steps, "hbm")
    rec = {"config": cfg, "workload": W["workload"], "n": p.Q.n, "nnz": p.Q.nnz,
           "value": iters / (ms * 1e-3), "unit": UNIT, "steps": steps, "warmup": 3,
           "iterations_per_solve": iters / steps, "time_to_tol_ms": ms / steps, "us_per_iteration": us,
           "sigma": info["sigma"], "column_index_bytes": info["col_bytes"], "value_bytes": info["val_bytes"], "band_staged": info["band_staged"], "grid": info["grid"],
           "roofline": rb, "roofline_gather": gather_roof(p, info, passes, loop_ms), "clocks": clk,
           "generate_s": round(gen_s, 1)}
    if W["bound"] == "latency":
        rec["roofline"]["note"] = (f"{model_bytes / 1e6:.2f} MB per pass fits the L2: latency-bound "
                                   "(one grid barrier per pass), the HBM fraction is not the bound")
    del p
    return rec


def run_sharded(args, rank, world, local, dev, dist):
    """N > 1: one solve of the config sharded by contiguous row blocks over the N ranks (strong
    scaling).  value = the solve's iterations / max-over-ranks device time."""
    import numpy as np
    import torch
    import paper_2407_03272_b200 as ajm
    W = WORKLOADS[args.config]
    tol = W["tol"] if args.tol is None else args.tol
    maxit = W["maxit"] if args.maxit is None else args.maxit
    p = make_problem(args.config)
    Q = p.Q
    starts = ajm.ajm_partition_rows(Q.row_ptr, world)
    rp, cg, vv = ajm.shard_rows(Q.row_ptr, Q.col, Q.val, starts, rank)
    r0, r1 = int(starts[rank]), int(starts[rank + 1])
    bl = np.ascontiguousarray(p.b[r0:r1])
    stream = torch.cuda.current_stream()
    Qd = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (rp, cg, vv, bl)]
    solver = ajm.ShardSolver(rank, world, starts, *Qd[:3], Qd[3])
    x_out = torch.empty(r1 - r0, dtype=torch.float64, device=dev)
    kw = dict(tol=tol, maxit=maxit, restart=True, x_out=x_out, history=False)
    clocks = ClockSampler(local)
    iters, passes, loop_ms, ms, results, clk = timed_solves(solver, kw, args.steps, args.warmup, stream,
                                                            dist, dev, clocks)
    _, job_ms = reduce_job(0.0, ms, dist, dev)
    _, job_loop_ms = reduce_job(0.0, loop_ms, dist, dev)
    info = solver.info()
    assert all(r.status == ("converged" if tol > 0 else "maxiter") for r in results)
    # e2e: this rank's rows from pinned host buffers (create + connect + solve + x to host + destroy)
    host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (rp, cg, vv, bl)]
    x_host = torch.empty(r1 - r0, dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host)
    e2e_ms, e2e_iters, d2h = 0.0, 0, 0
    for k in range(1 + args.e2e_steps):
        barrier(dist, dev)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        with ajm.ShardSolver(rank, world, starts, host[0], host[1], host[2], host[3]) as s2:
            r2 = s2.solve(tol=tol, maxit=maxit, restart=True, x_out=x_host, history=True)
        a1.record(stream)
        torch.cuda.synchronize()
        if k == 0:
            continue
        e2e_iters += r2.iterations
        e2e_ms += a0.elapsed_time(a1)
        d2h = x_host.numel() * 8 + 2 * 8 * (r2.iterations + 1)
    _, e2e_ms = reduce_job(0.0, e2e_ms, dist, dev)
    solver.close()
    if rank != 0:
        return 0
    peak, peak_src = load_peaks()
    model_bytes = ajm.model_bytes_per_iter(Q.n, Q.nnz)
    achieved = model_bytes * passes / (job_loop_ms * 1e-3) / 1e9
    nz = np.diff(Q.row_ptr[starts])
    line = {
        "metric": METRIC, "value": iters / (job_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": job_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": W["workload"], "n": Q.n, "nnz": Q.nnz, "tol": tol, "maxit": maxit,
                   "parallelism": f"row-block shards x{world} (Alg. 3 lines 3-5 / §4.4 partition; halo + partials "
                                  "exchanged in-kernel over peer memory each pass: DESIGN.md §6)",
                   "row_starts": [int(v) for v in starts], "halo_entries_rank0": info["halo"],
                   "load_imbalance": float(world * nz.max() / Q.nnz), "grid": info["grid"],
                   "column_index_bytes": info["col_bytes"]},
        "iterations_per_solve": iters / args.steps, "time_to_tol_ms": job_ms / args.steps,
        "us_per_iteration": 1e3 * job_loop_ms / passes,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": world * peak, "unit": "GB/s",
                     "frac": achieved / (world * peak), "traffic": None, "peak_source": f"{world} x {peak_src}",
                     "achieved_basis": "whole-matrix algorithmic bytes nnz*12+7n*8+4(n+1) per pass x passes / "
                                       "max-over-ranks launch time"},
        "e2e": {"value": e2e_iters / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "note": "per rank: ajm_shard_create from pinned host rows + connect + solve + x rows to host + "
                        "destroy; time = max over ranks"},
        "gpu_launches": int(info["launches_per_solve"]) * args.steps,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import paper_2407_03272_b200 as ajm

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(world, "nccl")
    if world > 1 and args.parallel == "shard":
        try:
            return run_sharded(args, rank, world, local, dev, dist)
        except Exception as e:  # reported on the line of the replica run below, never hidden
            args.shard_error = f"{type(e).__name__}: {e}"[:300]
            print(f"[bench] sharded solve failed on rank {rank}: {args.shard_error}; running replicas",
                  file=sys.stderr, flush=True)
            barrier(dist, dev)
    W = WORKLOADS[args.config]
    tol = W["tol"] if args.tol is None else args.tol
    maxit = W["maxit"] if args.maxit is None else args.maxit
    p = make_problem(args.config)
    stream = torch.cuda.current_stream()
    # inputs resident in HBM before timing
    Qd = [torch.from_numpy(a).to(dev) for a in (p.Q.row_ptr, p.Q.col, p.Q.val, p.b)]
    solver = ajm.Solver(p.Q.n, *Qd[:3], Qd[3], jblock=args.jblock)
    x_out = torch.empty(p.Q.n, dtype=torch.float64, device=dev)
    kw = dict(tol=tol, maxit=maxit, restart=True, x_out=x_out, history=False)
    clocks = ClockSampler(local)
    iters, passes, loop_ms, ms, results, clk = timed_solves(solver, kw, args.steps, args.warmup, stream,
                                                            dist, dev, clocks)
    job_iters, job_ms = reduce_job(float(iters), ms, dist, dev)
    info = solver.info()
    assert all(r.status == ("converged" if tol > 0 else "maxiter") for r in results)

    # ---- e2e: the public API from pinned host buffers (create + solve + x to host + destroy) ----
    host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            for a in (p.Q.row_ptr, p.Q.col, p.Q.val, p.b)]
    x_host = torch.empty(p.Q.n, dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host)
    e2e_iters, e2e_ms, d2h = 0, 0.0, 0
    for k in range(1 + args.e2e_steps):
        barrier(dist, dev)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        with ajm.Solver(p.Q.n, host[0], host[1], host[2], host[3], jblock=args.jblock) as s2:
            r2 = s2.solve(tol=tol, maxit=maxit, restart=True, x_out=x_host, history=True)
        a1.record(stream)
        torch.cuda.synchronize()
        if k == 0:
            continue  # first e2e call warms allocator/driver paths
        e2e_iters += r2.iterations
        e2e_ms += a0.elapsed_time(a1)
        d2h = x_host.numel() * 8 + 2 * 8 * (r2.iterations + 1)
    e2e_iters, e2e_ms = reduce_job(float(e2e_iters), e2e_ms, dist, dev)
    del host, x_host, Qd
    solver.close()

    if rank != 0:
        return 0
    rb, model_bytes, achieved, us = roofline_block(p, info, passes, loop_ms, args.steps, W["bound"] if W["bound"] != "latency" else "hbm",
                                                   args.jblock)
    # the other BASELINE configs, each as a roofline fraction (north_star), same measurement
    others = []
    if world == 1 and args.config == 2 and not args.jblock and args.other_configs:
        for cfg in [int(c) for c in args.other_configs.split(",") if c]:
            others.append(other_config_record(cfg, args, dev, stream))
            torch.cuda.empty_cache()
    cpu = cpu_baseline_run(p, args.config) if (world == 1 and not args.no_cpu_baseline) else None
    # the same oracle on ONE host thread (SURVEY §8(d) oracle timing (i)), a shorter sample
    cpu1 = cpu_baseline_run(p, args.config, budget_s=4.0, nthreads=1) \
        if (world == 1 and not args.no_cpu_baseline) else None
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    l2_note = (f"inputs larger than L2: {model_bytes / 1e6:.1f} MB algorithmic traffic per pass vs "
               f"{l2_bytes / 1e6:.0f} MB L2" if model_bytes > l2_bytes else
               f"L2-resident: {model_bytes / 1e6:.2f} MB per pass fits the {l2_bytes / 1e6:.0f} MB L2, "
               "so the HBM fraction is not the bound (latency-bound: grid barrier per pass)")
    line = {
        "metric": METRIC,
        "value": job_iters / (job_ms * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": job_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": W["workload"] + (f"; block-diagonal J (eq-J-blkdiag), bs={args.jblock}"
                                                 if args.jblock else ""),
                   "n": p.Q.n, "nnz": p.Q.nnz, "tol": tol, "maxit": maxit,
                   "parallelism": f"replicas x{world} (one independent solve per GPU: DESIGN.md §6)",
                   "l2": l2_note,
                   "grid": info["grid"],
                   "column_index_bytes": info.get("col_bytes", 4),
                   "value_bytes": info.get("val_bytes", 8),
                   "band_staged": info.get("band_staged", 0),
                   "ctas_per_sm": info["ctas_per_sm"]},
        "iterations_per_solve": iters / args.steps,
        "time_to_tol_ms": ms / args.steps,
        "us_per_iteration": us,
        "model_bytes_per_iteration": model_bytes,
        "model_gbs": achieved,
        "pct_of_8tbs_nominal": 100.0 * achieved / NOMINAL_HBM_GBS,
        "roofline": rb,
        "e2e": {"value": e2e_iters / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "note": "ajm_create from pinned host CSR+b (H2D + layout build) + ajm_solve to 1e-6 "
                        "+ x and histories to host + ajm_destroy"},
        "gpu_launches": int(info["launches_per_solve"]) * args.steps,
        "paper_context": PAPER_CONTEXT,
        "clocks": clk,
        "cpu_baseline": cpu,
        "cpu_baseline_1thread": cpu1,
        "other_configs": others,
    }
    if getattr(args, "shard_error", None):
        line["shard_error"] = args.shard_error
    rg = gather_roof(p, info, passes, loop_ms)
    if rg is not None:
        line["roofline_gather"] = rg
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(WORKLOADS),
                    help="BASELINE.json configs[K-1]; default 2 = the metric's config")
    ap.add_argument("--tol", type=float, default=None, help="default: the workload's")
    ap.add_argument("--maxit", type=int, default=None, help="default: the workload's")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--jblock", type=int, default=None,
                    help="block-diagonal J of eq-J-blkdiag with this block size (default: eq-J-diag)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parallel", default="replicas", choices=["shard", "replicas"],
                    help="N > 1: N independent replicas (default, weak scaling; SURVEY §8(e)) or one "
                         "row-block sharded solve (strong scaling, DESIGN.md §6)")
    ap.add_argument("--other-configs", default="1,3,4,5",
                    help="with the default --config 2 at N=1: also measure these BASELINE configs "
                         "(comma list, '' = none) and report them under other_configs")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
