"""solve_mf_global on a BASELINE config (fp32 storage for c2-c5), a few outer
iterations, with per-iteration wall times: python tools/solve_cfg.py c4 4"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_14067_b200 as P
from paper_2204_14067_b200 import synth

wl = sys.argv[1]; iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = synth.CONFIGS[wl]
t0 = time.perf_counter()
m, n, r, c, v = synth.generate(wl)
m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
t_gen = time.perf_counter() - t0
dt = torch.float64 if spec.dtype == "f64" else torch.float32
t0 = time.perf_counter()
obs = P.ObservationSet.from_coo(m, n, r, c, v, transposed=tr, dtype=dt)
torch.cuda.synchronize()
t_build = time.perf_counter() - t0
cfg = P.SolverConfig(lam=spec.lam, k0=spec.k0, seed=0, max_outer_iters=iters)
t0 = time.perf_counter()
x, wf, trace = P.solve_mf_global(obs, None, cfg)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print(f"{wl}: gen {t_gen:.1f}s build {t_build:.2f}s solve {el:.1f}s for {len(trace)-1} outer iterations")
for rec in trace.records:
    print(f"  it {rec.iter} rank {rec.rank} obj {rec.obj:.10g} time {rec.time_s:.2f}s k_t {rec.k_t} sweeps {rec.eig_sweeps} bt {rec.backtracks}")
