# Analysis tool (build container only): runs the REFERENCE twice on config 1,
# the second time with its input perturbed by 1e-15 relative, and prints the
# per-iteration relative change of its own objective. Not product, not a test.
# Usage: PYTHONPATH=/root/reference/pkg/src python tools/ref_sensitivity.py
import sys, numpy as np, time
sys.path.insert(0, "/root/repo")
import mfglobal as R
from mfglobal import data as rd, driver as rdrv
from paper_2204_14067_b200 import synth
m, n, r, c, v = synth.generate("c1"); m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
out = {}
for name, eps in [("base", 0.0), ("pert", 1e-15)]:
    rng = np.random.default_rng(5)
    vv = v * (1 + eps * rng.standard_normal(v.size))
    obs = rd.ObservationSet.from_coo(m, n, r, c, vv, transposed=tr)
    cfg = rdrv.SolverConfig(lam=5.0, k0=8, seed=0, max_outer_iters=4)
    t0 = time.time()
    x, _, trace = rdrv.solve_mf_global(obs, None, cfg)
    out[name] = [rec.obj for rec in trace.records]
    print(name, time.time() - t0, out[name], flush=True)
a, b = np.array(out["base"]), np.array(out["pert"])
print("relative change per iteration under 1e-15 input perturbation:", np.abs(a - b) / a)
