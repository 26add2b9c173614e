#!/usr/bin/env python
"""Benchmark: Omega sweeps/sec (SDDMM + 2x SpMM + fp64 reductions) on B200.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c2|c3|c4|c5]
prints ONE JSON line on rank 0.

A step = one Omega sweep over one instance at width k0:
R = P_Omega(W H^T) - A, R.H (CSR), R^T.W (CSC), sum r^2, ||W||^2, ||H||^2.
Default workload: BASELINE.json configs[1] (c2: 3706 x 6040 canonical,
|Omega| = 1,000,209, k0 = 20, fp32 values, fp64 reductions), synthetic
(seeded Zipf generator, paper_2204_14067_b200/synth.py).

Timing: W untimed warm-up steps, then K timed steps bracketed by barrier +
synchronize; each step is timed with CUDA events on the launching stream and
L2 is flushed (512 MiB write, outside the events) before every step, since
the c2 working set (~30 MB) fits in the 126 MB L2. Multi-GPU (torchrun): each
rank sweeps its own instance (independent partitions, weak scaling, no
collective on the data path); the reported time is the max over ranks.
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
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="bounded CPU-baseline sample (seconds of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tto", action="store_true", help="skip the time-to-objective leg")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: the ranks sweep row/column shards of ONE instance "
                         "(mfg_sweep_sharded, no data-path collective) instead of one instance each")
    ap.add_argument("--sweep", default="grouped", choices=["grouped", "staged"],
                    help="sweep kernel: all-gather grouped (k_sweep_g8f) or shared-memory staged")
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
            "reference_note": "reference timings from its own run in the build container "
                              "(8 CPU cores, tests/golden/make_golden.py --c1)"}


def cpu_sweep_setup(m, n, r, c, v, k):
    from oracle import mfg_oracle as orc
    from paper_2204_14067_b200 import synth

    om = orc.from_coo(m, n, r, c, v)
    w, h = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
    w, h = w.astype(np.float64), h.astype(np.float64)
    return orc, om, w, h


def cpu_sweep_port(orc, om, w, h, perm, csc):
    """The reference's sweep (pair_values einsum + scipy CSR/CSC SpMM) with the
    CSR/CSC index caches prebuilt, as SURVEY.md §8(d) prescribes."""
    import scipy.sparse as sp

    r = orc.pair_values(w, h, om.rows, om.cols) - om.vals
    rh = sp.csr_matrix((r, om.cols, om.indptr), shape=(om.m, om.n)) @ h
    rt = sp.csr_matrix((r[perm], csc.indices, csc.indptr), shape=(om.n, om.m))
    rtw = rt @ w
    return r, rh, rtw, float(r @ r), float(np.sum(w * w)), float(np.sum(h * h))


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle port), rank 0 only."""
    if rank != 0:
        return
    m, n, r, c, v, spec = instance(args.workload, seed=0)
    orc, om, w, h = cpu_sweep_setup(m, n, r, c, v, spec.k0)
    perm = om.csc_perm()
    csc = om.a_csr_t
    for _ in range(args.warmup):
        cpu_sweep_port(orc, om, w, h, perm, csc)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_sweep_port(orc, om, w, h, perm, csc)
    el = time.perf_counter() - t0
    value = args.steps / el
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": args.workload, "m": m, "n": n, "nnz": int(om.size), "k": spec.k0},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{args.steps} full {args.workload} sweeps (numpy einsum "
                                   "SDDMM + scipy CSR/CSC SpMM; single-threaded like the "
                                   "reference's sparse calls)"},
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
    if args.shard:
        main_shard(args, rank, world, local_rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2204_14067_b200 import _lib, synth
    from paper_2204_14067_b200.data import ObservationSet
    from paper_2204_14067_b200.mfsolver import SweepPlan

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    lib = _lib.lib()

    m, n, r, c, v, spec = instance(args.workload, seed=rank)
    k = spec.k0
    obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    w_np, h_np = synth.sweep_factors(m, n, k, seed=1 + rank, dtype=np.float32)
    t_plan = time.perf_counter()
    plan = SweepPlan(obs, k, compute_f64=False, staged=args.sweep == "staged")
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t_plan
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
        traffic = tj.get(args.workload)
        l2b = tj.get("l2_bytes", {}).get(args.workload)
        if l2b and plan.staged is None:
            # bytes through L2 per launch (ncu capture) over the live kernel time,
            # against the LTS throughput cap (~6300 B/cycle at the max SM clock)
            cap = 6300 * 1.965e9 / 1e12
            l2 = {"bytes_per_launch": l2b, "achieved_TBps": l2b / (kern_ms * 1e-3) / 1e12,
                  "cap_TBps": cap, "frac": l2b / (kern_ms * 1e-3) / 1e12 / cap,
                  "source": "lts__t_sectors.sum * 32 from profiles/r1i_*_k_sweep_g8f_full.json"}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        orc, om, wc, hc = cpu_sweep_setup(m, n, r, c, v, k)
        perm = om.csc_perm()
        csc = om.a_csr_t
        t0 = time.perf_counter()
        cnt_cpu = 0
        while True:
            cpu_sweep_port(orc, om, wc, hc, perm, csc)
            cnt_cpu += 1
            el = time.perf_counter() - t0
            if el >= args.cpu_seconds or cnt_cpu >= 1000:
                break
        cpu = {"value": cnt_cpu / el, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{cnt_cpu} full {args.workload} sweeps on the host "
                         f"({os.cpu_count()} cores visible; the reference's einsum/scipy "
                         "sparse calls are single-threaded)"}

    tto = None
    if not args.no_tto and world == 1:
        tto = time_to_objective()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp64 reductions)",
        "data": "synthetic",
        "config": {"workload": args.workload, "m": m, "n": n, "nnz": int(obs.size), "k": k,
                   "values": "fp32", "l2": {"write": "flushed before every step (512 MiB write)",
                          "read": "flushed before every step (512 MiB read)",
                          "none": "not flushed (L2-warm)"}[args.flush],
                   "timing": "per-step CUDA events, CUDA-graph replay of the sweep",
                   "parallelism": f"{world} independent partitions (one per GPU)",
                   "sweep": args.sweep, "plan_seconds": round(t_plan, 3),
                   **({"staged": plan.staged.stats()} if plan.staged is not None else {})},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": int((m + n) * k * 4),
                "d2h_bytes_per_step": int(plan._host.numel())},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("k_sweep_g8f (fused CSR+CSC pass)" if plan.staged is None else
                                "k_sweep_staged + k_staged_fold (timed together)"),
                     "bytes_per_launch": kb, "avg_launch_us": kern_ms * 1e3,
                     "peak_source": peak_src,
                     "survey_unfused_bytes": survey_bytes(obs.size, m, n, k, 4),
                     "l2": l2},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "time_to_objective": tto,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
            "data": "synthetic",
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
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
