"""Kernel-time breakdown of solve_mf_global (diagnostics): torch.profiler
(CUPTI) over a run, CUDA kernel time aggregated by name, GPU-busy fraction
against wall clock. Usage: python tools/kernel_breakdown.py c1 [iters]"""
import sys, os, time, collections, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_14067_b200 as P
from paper_2204_14067_b200 import synth

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dt = torch.float64 if wl == "c1" else torch.float32
m, n, r, c, v = synth.generate(wl)
m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
obs = P.ObservationSet.from_coo(m, n, r, c, v, transposed=tr, dtype=dt)
cfg = P.SolverConfig(lam=synth.CONFIGS[wl].lam, k0=synth.CONFIGS[wl].k0, max_outer_iters=iters, seed=0)
P.solve_mf_global(obs, None, P.SolverConfig(lam=cfg.lam, k0=cfg.k0, max_outer_iters=1, seed=0))  # warm-up
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    t0 = time.perf_counter()
    x, _, trace = P.solve_mf_global(obs, None, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
T = collections.Counter(); N = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        T[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        N[e.name] += 1
tot = sum(T.values()) / 1e6
out = {"workload": wl, "iters": len(trace) - 1, "rank": x.rank, "wall_s": wall, "gpu_kernel_s": tot,
       "gpu_busy_frac": tot / wall, "launches": sum(N.values()), "top": []}
for name, t in T.most_common(25):
    out["top"].append({"kernel": name[:110], "s": t / 1e6, "n": N[name], "share": t / 1e6 / tot})
print(json.dumps(out, indent=1))
