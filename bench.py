#!/usr/bin/env python
"""Benchmark: Omega sweeps/sec (SDDMM + 2x SpMM + fp64 reductions) on B200.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c2|c3|c4|c5]
prints ONE JSON line on rank 0.

A step = one Omega sweep over one instance at width k0:
R = P_Omega(W H^T) - A, R.H (CSR), R^T.W (CSC), sum r^2, ||W||^2, ||H||^2.
Default workload: BASELINE.json configs[3] (c4: 17,770 x 480,189 canonical,
|Omega| = 100,480,507, k0 = 40, fp32 values, fp64 reductions), the largest
configuration that fits one GPU and the one BASELINE.json quotes at
1/2/4/8 B200; synthetic (seeded Zipf generator,
paper_2204_14067_b200/synth.py).

Timing: W untimed warm-up steps, then K timed steps bracketed by barrier +
synchronize; each step is timed with CUDA events on the launching stream and
L2 is flushed (512 MiB write, outside the events) before every step, since
the factors of the smaller configs fit in the 126 MB L2. Multi-GPU
(torchrun): by default the ranks sweep row/column shards of ONE instance
(strong scaling: no data-path collective for the sweep,
all-gathers of W/H blocks in the BCD epoch line); ``--independent`` runs one
instance per rank instead (weak scaling). Times are the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Omega sweeps/sec (SDDMM+2×SpMM)"
UNIT = "sweeps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="bounded CPU-baseline sample (seconds of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tto", action="store_true", help="skip the time-to-objective leg")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: the ranks sweep row/column shards of ONE instance "
                         "(mfg_sweep_sharded, no data-path collective); the default for N > 1")
    ap.add_argument("--independent", action="store_true",
                    help="N > 1: one independent instance per rank (weak scaling) instead of shards")
    ap.add_argument("--no-bcd", action="store_true", help="skip the BCD-epoch leg")
    ap.add_argument("--sweep-plan", default="auto", choices=["auto", "gather", "hybrid"],
                    help="auto: time the gather-only and the hybrid panel sweep once, keep the faster")
    ap.add_argument("--flush", default="write", choices=["write", "read", "none"],
                    help="L2 flush between steps: write (zero 512 MiB), read (sum 512 MiB) or none")
    return ap.parse_args()


def instance(workload: str, seed: int):
    from paper_2204_14067_b200 import synth

    cache = os.environ.get("MFG_SYNTH_CACHE")  # optional: reuse an instance across A/B runs
    path = os.path.join(cache, f"{workload}_{seed}.npz") if cache else None
    if path and os.path.exists(path):
        z = np.load(path)
        m, n, r, c, v = int(z["m"]), int(z["n"]), z["r"], z["c"], z["v"]
    else:
        m, n, r, c, v = synth.generate(workload, seed=seed)
        if path:
            os.makedirs(cache, exist_ok=True)
            np.savez(path, m=m, n=n, r=r, c=c, v=v)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    return m, n, r, c, v, synth.CONFIGS[workload]


def kernel_bytes(nnz: int, m: int, n: int, k: int, s_v: int) -> int:
    """Compulsory DRAM bytes of one grouped sweep launch:
    CSR pass reads column ids, row ids and A and writes R; CSC pass reads row
    ids, column ids and A; 4 B of schedule mask per 32 entries per pass; W
    and H read once and RH, RtW written once (s_v bytes per value)."""
    per_nnz = (4 + 4 + s_v + s_v) + (4 + 4 + s_v) + 0.25
    return int(nnz * per_nnz + 3 * s_v * (m + n) * k)


def survey_bytes(nnz: int, m: int, n: int, k: int, s_v: int) -> int:
    """SURVEY.md §8(d) unfused algorithmic bytes: |O|(3 s_i + 4 s_v) + s_i(2m+n+3) + 3 s_v (m+n) k."""
    return int(nnz * (12 + 4 * s_v) + 4 * (2 * m + n + 3) + 3 * s_v * (m + n) * k)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index
        self.windows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for ts, line in self.samples:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm, smax = float(parts[1]), float(parts[2])
            except ValueError:
                continue
            inwin = any(a - 0.06 <= ts <= b + 0.06 for a, b in self.windows)
            rows.append((inwin, sm, smax, parts))
        if not rows:
            return None
        load = [r for r in rows if r[0]] or rows
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, _, _, p in load:
            for nm, val in zip(names, p[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[1] for r in load),
                "sm_max_mhz": max(r[2] for r in load),
                "samples": len(load), "reasons": sorted(reasons)}


def time_to_objective(target_rel: float = 1e-6):
    """Config 1 (fp64) through the drop-in solve_mf_global: wall-clock until
    the relative objective against the reference's F* (the final objective of
    the reference's own run, tests/golden/trace_c1.json) first reaches
    target_rel. Each iteration's time_s comes from the solver trace."""
    import torch

    import paper_2204_14067_b200 as P
    from paper_2204_14067_b200 import synth

    with open(os.path.join(REPO, "tests", "golden", "trace_c1.json")) as fh:
        ref = json.load(fh)
    f_star = float(ref["obj"][-1])
    m, n, r, c, v = synth.generate("c1")
    m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
    t0 = time.perf_counter()
    obs = P.ObservationSet.from_coo(m, n, r, c, v, transposed=tr)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    cfg = P.SolverConfig(**ref["cfg"])
    t0 = time.perf_counter()
    _, _, trace = P.solve_mf_global(obs, None, cfg)
    total = time.perf_counter() - t0
    hit = next(((rec.time_s, rec.iter) for rec in trace.records
                if (rec.obj - f_star) / f_star <= target_rel), (None, None))
    ref_hit = next((t for t, o in zip(ref.get("time_s", []), ref["obj"])
                    if (o - f_star) / f_star <= target_rel), None)
    return {"workload": "c1 (fp64, lam=5, k0=8, seed=0)", "target_rel_obj": target_rel,
            "f_star": f_star, "seconds": hit[0], "iterations": hit[1],
            "run_seconds": total, "omega_build_seconds": t_build,
            "final_rank": trace.final().rank,
            "reference_seconds": ref_hit, "reference_run_seconds": ref.get("elapsed_s"),
            "reference_same_box": False,
        "reference_note": "reference timings come from its own run in the build container "
                          "(8 CPU cores, tests/golden/make_golden.py --c1), NOT from this "
                          "box's host: the 560 s reference run does not fit the bench budget"}


_CPU = None  # the CpuSweep whose arrays forked pool workers inherit


def _cpu_worker_init():
    # one BLAS thread per worker process (the pool supplies the parallelism;
    # OpenBLAS's own threads would oversubscribe the cores)
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)


def _cpu_task(t):
    kind, a, b = t
    if kind == 0:
        return _CPU._csr_block(a, b)
    return _CPU._csc_block(a, b)


class CpuSweep:
    """The reference's CPU sweep (SURVEY.md §8(d) unit) restated with its own
    calls -- numpy einsum SDDMM (``pair_values``, mfg/data.py:253-263) + scipy
    CSR SpMM ``grad.csr @ H`` and CSC SpMM ``grad.csr_t @ W``
    (mfg/operators.py:108,117) -- timed on a bounded sample of the workload
    on every host core.

    A sample of fraction f is the CSR rows [0, i1) and the CSC rows (= Omega
    columns) [0, j1) that each hold ~f of the entries: SDDMM + R.H over the
    CSR rows, R^T.W over the CSC rows (their r values come from the same
    SDDMM, which the reference computes once per sweep, so they are prepared
    outside the timed region). The CSR/CSC index caches are prebuilt, as the
    survey prescribes. Row ranges are split into 4 blocks per core and run on
    a fork()ed process pool with one BLAS thread per process; the reference
    itself calls them single-threaded. Create it before CUDA is initialised."""

    def __init__(self, m, n, r, c, v, k, procs=None):
        from oracle import mfg_oracle as orc
        from paper_2204_14067_b200 import synth

        self.orc = orc
        self.om = om = orc.from_coo(m, n, r, c, v)
        w, h = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
        self.w, self.h = w.astype(np.float64), h.astype(np.float64)
        self.perm = om.csc_perm()
        self.cptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(om.cols, minlength=n), out=self.cptr[1:])
        self.crow = om.rows[self.perm]          # CSC row ids (= csr_t indices)
        self.procs = procs or len(os.sched_getaffinity(0))
        self.pool = None
        self.frac = 0.0

    def close(self):
        if self.pool is not None:
            self.pool.terminate()
            self.pool.join()
            self.pool = None

    def set_fraction(self, f: float):
        import multiprocessing as mp

        global _CPU
        om = self.om
        f = min(max(f, 0.0), 1.0)
        nnz = om.size
        self.i1 = int(np.searchsorted(om.indptr, f * nnz, side="left")) if f < 1 else om.m
        self.j1 = int(np.searchsorted(self.cptr, f * nnz, side="left")) if f < 1 else om.n
        self.i1, self.j1 = max(self.i1, 1), max(self.j1, 1)
        e1 = int(self.cptr[self.j1])
        sel = self.perm[:e1]
        # the sample's CSC-side residuals (computed once per sweep by the reference)
        self.r_csc = self.orc.pair_values(self.w, self.h, om.rows[sel], om.cols[sel]) - om.vals[sel]
        self.frac = (int(om.indptr[self.i1]) + e1) / (2.0 * max(nnz, 1))
        nb = 4 * self.procs
        ei = np.unique(np.linspace(0, self.i1, nb + 1).astype(np.int64))
        ej = np.unique(np.linspace(0, self.j1, nb + 1).astype(np.int64))
        self.tasks = ([(0, int(a), int(b)) for a, b in zip(ei[:-1], ei[1:])]
                      + [(1, int(a), int(b)) for a, b in zip(ej[:-1], ej[1:])])
        self.close()
        _CPU = self
        self.pool = mp.get_context("fork").Pool(self.procs, initializer=_cpu_worker_init)
        self.pool.map(_cpu_task, [(0, 0, 1)] * self.procs)  # workers up
        return self.frac

    def _csr_block(self, i0, i1):
        import scipy.sparse as sp

        om = self.om
        lo, hi = int(om.indptr[i0]), int(om.indptr[i1])
        r = self.orc.pair_values(self.w, self.h, om.rows[lo:hi], om.cols[lo:hi]) - om.vals[lo:hi]
        g = sp.csr_matrix((r, om.cols[lo:hi], om.indptr[i0:i1 + 1] - lo), shape=(i1 - i0, om.n))
        rh = g @ self.h
        return float(r @ r) + float(rh[0, 0] if rh.size else 0.0)

    def _csc_block(self, j0, j1):
        import scipy.sparse as sp

        lo, hi = int(self.cptr[j0]), int(self.cptr[j1])
        g = sp.csr_matrix((self.r_csc[lo:hi], self.crow[lo:hi], self.cptr[j0:j1 + 1] - lo),
                          shape=(j1 - j0, self.om.m))
        rtw = g @ self.w
        return float(rtw[0, 0] if rtw.size else 0.0)

    def step(self) -> float:
        """One timed sample; returns its wall seconds."""
        t0 = time.perf_counter()
        self.pool.map(_cpu_task, self.tasks, chunksize=1)
        return time.perf_counter() - t0

    def calibrate(self, step_seconds: float, f_min: float = 1e-3) -> float:
        """Pick the sample fraction so that one step takes ~step_seconds."""
        f = self.set_fraction(max(f_min, min(1.0, 1e6 / max(self.om.size, 1))))
        t = min(self.step() for _ in range(2))
        if f < 1.0 or t > step_seconds:
            f = self.set_fraction(min(1.0, max(f_min, f * step_seconds / max(t, 1e-6))))
        return f

    def describe(self, steps: int) -> str:
        return (f"{steps} samples of {100 * self.frac:.2f}% of the sweep each (CSR rows "
                f"[0,{self.i1}) + CSC rows [0,{self.j1}); numpy einsum SDDMM + scipy CSR/CSC "
                f"SpMM over row blocks on {self.procs} host processes); value = sampled "
                "fraction / step time, in full sweeps/s")


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle port of its own
    calls) on the host cores, rank 0 only; each step a bounded sample."""
    if rank != 0:
        return
    m, n, r, c, v, spec = instance(args.workload, seed=0)
    cs = CpuSweep(m, n, r, c, v, spec.k0)
    budget = float(os.environ.get("MFG_REF_BUDGET_S", "90"))
    cs.calibrate(budget / max(args.steps + args.warmup, 1))
    for _ in range(args.warmup):
        cs.step()
    el = sum(cs.step() for _ in range(args.steps))
    cs.close()
    value = args.steps * cs.frac / el
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": args.workload, "m": m, "n": n, "nnz": int(cs.om.size),
                   "k": spec.k0},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cs.procs, "kind": "port",
                         "sample": cs.describe(args.steps)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.shard or (world > 1 and not args.independent):
        main_shard(args, rank, world, local_rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2204_14067_b200 import _lib, synth
    from paper_2204_14067_b200.data import ObservationSet
    from paper_2204_14067_b200.mfsolver import SweepPlan

    m, n, r, c, v, spec = instance(args.workload, seed=rank)
    k = spec.k0
    # CPU baseline first: its process pool is fork()ed before CUDA initialises
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cs = CpuSweep(m, n, r, c, v, k)
        cs.calibrate(args.cpu_seconds / 4)
        el, cnt_cpu = 0.0, 0
        while el < args.cpu_seconds and cnt_cpu < 1000:
            el += cs.step()
            cnt_cpu += 1
        cpu = {"value": cnt_cpu * cs.frac / el, "unit": UNIT, "cores": cs.procs,
               "kind": "port", "sample": cs.describe(cnt_cpu)}
        cs.close()
        del cs

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    lib = _lib.lib()
    obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    w_np, h_np = synth.sweep_factors(m, n, k, seed=1 + rank, dtype=np.float32)
    t_plan = time.perf_counter()
    # the faster of the gather-only sweep and the hybrid panel sweep (timed once)
    from paper_2204_14067_b200.panel import best_sweep_plan
    plan = best_sweep_plan(obs, k, mode=args.sweep_plan)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t_plan
    hybrid = plan.kind == "hybrid"
    # resident factors in the grouped kernel layout (unpadded when k allows)
    w = plan.pad(torch.as_tensor(w_np, device=dev))
    h = plan.pad(torch.as_tensor(h_np, device=dev))
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
    flush_i = flush.view(torch.int32)
    stream = torch.cuda.current_stream()

    def do_flush():
        if args.flush == "write":
            flush.zero_()
        elif args.flush == "read":
            torch.sum(flush_i)

    # launches per sweep (our kernels), from one eager call
    c0 = lib.mfg_launch_count()
    plan.run(w, h)
    torch.cuda.synchronize()
    launches_per_step = lib.mfg_launch_count() - c0

    # capture the sweep in a CUDA graph (launch-bound at this size)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        plan.run(w, h)
    stream.wait_stream(side)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        plan.run(w, h)
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.15)

    def timed(fn, steps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        for a, b in evs:
            do_flush()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        t1 = time.time()
        if world > 1:
            dist.barrier()
        sampler.mark(t0, t1)
        return sum(a.elapsed_time(b) for a, b in evs)

    for _ in range(args.warmup):
        do_flush()
        g.replay()
    ms_total = timed(g.replay, args.steps)
    # max over ranks
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    value = world * args.steps / (ms_total / 1e3)

    # roofline leg: eager launches with per-launch CUDA events on the main kernel
    lib.mfg_profile_enable(args.steps)
    timed(lambda: plan.run(w, h), args.steps)
    tot = _lib.ctypes.c_double(0.0)
    cnt = _lib.ctypes.c_int(0)
    lib.mfg_profile_collect(_lib.ctypes.byref(tot), _lib.ctypes.byref(cnt))
    lib.mfg_profile_enable(0)
    kern_ms = tot.value / max(cnt.value, 1)
    if hybrid:
        # the sweep is a sequence of kernels (gather kernel over the cold entries,
        # panel kernel, folds, R gather): the replayed graph's device time is theirs
        kern_ms = ms_total / args.steps

    # end-to-end leg through the public API (SweepPlan.run_host) with pinned
    # host factors: H2D of the step's inputs (W, H), the sweep, and one D2H of
    # the packed results [sums | RH | RtW]
    w_host, h_host = plan.pinned_factors()
    w_host.copy_(torch.as_tensor(w_np))
    h_host.copy_(torch.as_tensor(h_np))

    def e2e_step():
        return plan.run_host(w_host, h_host)

    e2e_ms = 0.0
    for _ in range(min(args.warmup, 5)):
        e2e_step()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        do_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sums_host, _, _ = e2e_step()
        b.record(stream)
        b.synchronize()
        _ = float(sums_host[0])  # the host reads the step's result
        e2e_ms += a.elapsed_time(b)
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = world * args.steps / (float(t.item()) / 1e3)
    clocks = sampler.stop()

    # correctness spot check of the timed kernels against the fp64 sums
    sums = plan.sums.cpu().numpy()
    if not np.all(np.isfinite(sums)):
        raise RuntimeError("non-finite sweep sums")

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    kb = kernel_bytes(obs.size, m, n, k, 4)
    achieved = kb / (kern_ms * 1e-3) / 1e9
    traffic = None
    l2 = None
    tp = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            tj = json.load(fh)
        traffic = tj.get(args.workload + ("_hybrid" if hybrid else ""))
        l2b = tj.get("l2_bytes", {}).get(args.workload)
        if l2b and not hybrid:
            # bytes through L2 per launch (ncu capture) over the live kernel time,
            # against the LTS throughput cap (~6300 B/cycle at the max SM clock)
            cap = 6300 * 1.965e9 / 1e12
            l2 = {"bytes_per_launch": l2b, "achieved_TBps": l2b / (kern_ms * 1e-3) / 1e12,
                  "cap_TBps": cap, "frac": l2b / (kern_ms * 1e-3) / 1e12 / cap,
                  "source": "lts__t_sectors.sum * 32 from profiles/r1i_*_k_sweep_g8f_full.json"}

    bcd = None
    if not args.no_bcd and world == 1:
        bcd = bcd_epoch_leg(args, m, n, r, c, v, k, rank, world, dev, spec)

    tto = None
    if not args.no_tto and world == 1:
        tto = time_to_objective()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp64 reductions)",
        "data": "synthetic (seeded Zipf instance with the config's shape; no dataset records)",
        "config": {"workload": args.workload, "m": m, "n": n, "nnz": int(obs.size), "k": k,
                   "values": "fp32", "l2": {"write": "flushed before every step (512 MiB write)",
                          "read": "flushed before every step (512 MiB read)",
                          "none": "not flushed (L2-warm)"}[args.flush],
                   "timing": "per-step CUDA events, CUDA-graph replay of the sweep",
                   "parallelism": (f"{world} independent instances (one per GPU)" if world > 1
                                   else "1 GPU"),
                   "sweep_plan": (dict(kind="hybrid: hot entries from shared-memory panels (k_panel4), "
                                       "cold entries as pieces on global loads (k_cold4)"
                                       if getattr(plan, "cold", "") == "pieces" else
                                       "hybrid: hot entries from shared-memory panels, cold entries "
                                       "through the gather kernel (k_sweep_g8f)",
                                       **plan.stats) if hybrid else {"kind": "gather (k_sweep_g8f)"}),
                   "plan_trial_ms": getattr(plan, "trial_ms", None),
                   "plan_seconds": round(t_plan, 3)},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": int((m + n) * k * 4),
                "d2h_bytes_per_step": int(plan._host.numel())},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("one sweep = k_cold4 (cold entries) + k_panel4 (hot entries, the longest) "
                                "+ k_panel_fold x3-4 + k_panel_sq + k_gather4_f32 + 2 k_dot (norms)"
                                if hybrid else "k_sweep_g8f (fused CSR+CSC pass)"),
                     "bytes_per_launch": kb, "avg_launch_us": kern_ms * 1e3,
                     "peak_source": peak_src,
                     "survey_unfused_bytes": survey_bytes(obs.size, m, n, k, 4),
                     "l2": l2},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "time_to_objective": tto,
        "bcd_epoch": bcd,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bcd_epoch_leg(args, m, n, r, c, v, k, rank, world, dev, spec, shard=None):
    """One BCD epoch (mfg/mfsolver.py:78-93) over the rank's row/column shards
    of the instance, including the all-gathers of the W and H blocks
    (SURVEY.md §8(e)); fp32 factors, fp64 per-row Gram + Cholesky. Timed with
    CUDA events (max over ranks), 1 warm-up + 3 timed epochs."""
    import torch
    import torch.distributed as dist

    from paper_2204_14067_b200 import sharding, synth

    if shard is None:
        shard = sharding.make_shard(m, n, r, c, v, rank, world)
    mf = sharding.ShardedMF(shard, sharding.DeviceOps(torch.float32), sharding.Comm(), dev)
    w_np, h_np = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
    w = torch.as_tensor(w_np, device=dev)
    h = torch.as_tensor(h_np, device=dev)
    lam = float(spec.lam)
    mf.bcd_epoch(w, h, lam)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ms = []
    for _ in range(3):
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        w2, h2 = mf.bcd_epoch(w, h, lam)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = torch.tensor([min(ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_epoch = float(t.item())
    if not (torch.isfinite(w2).all() and torch.isfinite(h2).all()):
        raise RuntimeError("non-finite BCD epoch")
    nnz = len(v)
    flops = 2.0 * nnz * k * (k + 1)   # row-Gram assembly per epoch
    del mf
    torch.cuda.empty_cache()
    return {"ms_per_epoch": ms_epoch, "epochs_per_s": 1e3 / ms_epoch, "lam": lam, "k": k,
            "gram_flops": flops, "gram_tflops": flops / (ms_epoch * 1e-3) / 1e12,
            "timing": "best of 3 epochs (after 1 warm-up), CUDA events, max over ranks",
            "parallelism": (f"{world} row/column shards, W and H blocks all-gathered (NCCL)"
                            if world > 1 else "1 GPU")}


def main_shard(args, rank, world, local_rank):
    """Strong scaling of one instance: rank p sweeps its row block R_p (CSR)
    and column block C_p (CSC) with full W/H replicas;
    R.H rows R_p and R^T.W rows C_p are final on their rank, so the data
    path has no collective. value = whole-instance sweeps per second."""
    import torch
    import torch.distributed as dist

    from paper_2204_14067_b200 import _lib, sharding, synth

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    lib = _lib.lib()
    m, n, r, c, v, spec = instance(args.workload, seed=0)
    k = spec.k0
    shard = sharding.make_shard(m, n, r, c, v, rank, world)
    r0, r1 = shard.row_block
    c0, c1 = shard.col_block
    ops = sharding.DeviceOps(torch.float32)
    obs_r = ops.prepare(r1 - r0, n, shard.r_rows, shard.r_cols, shard.r_vals)
    obs_c = ops.prepare(c1 - c0, m, shard.c_rows, shard.c_cols, shard.c_vals)
    plan = sharding.ShardSweepPlan(shard, obs_r, obs_c, k)
    w_np, h_np = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
    w = plan.pad(torch.as_tensor(w_np, device=dev))
    h = plan.pad(torch.as_tensor(h_np, device=dev))
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    c_0 = lib.mfg_launch_count()
    plan.run(w, h)
    torch.cuda.synchronize()
    launches_per_step = lib.mfg_launch_count() - c_0
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        plan.run(w, h)
    stream.wait_stream(side)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        plan.run(w, h)
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.15)

    def timed(fn, steps, pre=None):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        t1 = time.time()
        if world > 1:
            dist.barrier()
        sampler.mark(t0, t1)
        return sum(a.elapsed_time(b) for a, b in evs)

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        flush.zero_()
        g.replay()
    ms_total = max_over_ranks(timed(g.replay, args.steps))
    value = args.steps / (ms_total / 1e3)
    lib.mfg_profile_enable(args.steps)
    timed(lambda: plan.run(w, h), args.steps)
    tot = _lib.ctypes.c_double(0.0)
    cnt = _lib.ctypes.c_int(0)
    lib.mfg_profile_collect(_lib.ctypes.byref(tot), _lib.ctypes.byref(cnt))
    lib.mfg_profile_enable(0)
    kern_ms = tot.value / max(cnt.value, 1)
    # end to end: H2D of the full factor replicas from pinned host memory,
    # the shard sweep, D2H of this rank's [sums | R.H rows | R^T.W rows]
    w_host = torch.as_tensor(w_np).pin_memory()
    h_host = torch.as_tensor(h_np).pin_memory()
    sums_host = torch.empty(3, dtype=torch.float64).pin_memory()
    rh_host = torch.empty(plan.RH.shape, dtype=plan.RH.dtype).pin_memory()
    rtw_host = torch.empty(plan.RtW.shape, dtype=plan.RtW.dtype).pin_memory()

    def e2e_step():
        w[:, :k].copy_(w_host, non_blocking=True)
        h[:, :k].copy_(h_host, non_blocking=True)
        plan.run(w, h)
        sums_host.copy_(plan.sums, non_blocking=True)
        rh_host.copy_(plan.RH, non_blocking=True)
        rtw_host.copy_(plan.RtW, non_blocking=True)

    for _ in range(min(args.warmup, 5)):
        e2e_step()
    e2e_ms = max_over_ranks(timed(e2e_step, args.steps))
    e2e_value = args.steps / (e2e_ms / 1e3)
    clocks = sampler.stop()
    sums = plan.sums.cpu().numpy()
    if not np.all(np.isfinite(sums)):
        raise RuntimeError("non-finite sweep sums")
    bcd = None
    if not args.no_bcd:
        bcd = bcd_epoch_leg(args, m, n, r, c, v, k, rank, world, dev, spec, shard=shard)
    if rank == 0:
        nnz_r, nnz_c = obs_r.size, obs_c.size
        kb = int(nnz_r * 16 + nnz_c * 12 + 0.125 * (nnz_r + nnz_c)
                 + 12 * ((r1 - r0) + (c1 - c0)) * k)
        peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        if os.path.exists(peaks_path):
            with open(peaks_path) as fh:
                peak = float(json.load(fh)["hbm_gbs"])
            peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
        achieved = kb / (kern_ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (fp64 reductions)",
            "data": "synthetic (seeded Zipf instance with the config's shape; no dataset records)",
            "config": {"workload": args.workload, "m": m, "n": n, "nnz": len(v), "k": k,
                       "values": "fp32", "l2": "flushed before every step (512 MiB write)",
                       "timing": "per-step CUDA events, CUDA-graph replay, max over ranks",
                       "parallelism": f"{world} row/column shards of one instance "
                                      "(mfg_sweep_sharded; no data-path collective)",
                       "rank0_shard": {"rows": r1 - r0, "cols": c1 - c0, "nnz_rows": nnz_r,
                                       "nnz_cols": nnz_c}},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int((m + n) * k * 4),
                    "d2h_bytes_per_step": int(24 + (plan.RH.numel() + plan.RtW.numel()) * 4)},
            "gpu_launches": int(launches_per_step * args.steps),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "k_sweep_g8f on rank 0's shards",
                         "bytes_per_launch": kb, "avg_launch_us": kern_ms * 1e3,
                         "peak_source": peak_src},
            "cpu_baseline": None,
            "clocks": clocks,
            "bcd_epoch": bcd,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
