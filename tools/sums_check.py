"""Print the fused sweep's fp64 sums (repr) for a workload: run under two
MFG_LIB_PATH builds to check that a change keeps them bitwise identical."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.mfsolver import SweepPlan
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
m, n, r, c, v = synth.generate(wl); m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
k = synth.CONFIGS[wl].k0
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
w, h = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
plan = SweepPlan(obs, k, want_rh=True, want_rtw=True)
W = plan.pad(torch.as_tensor(w).cuda()); H = plan.pad(torch.as_tensor(h).cuda())
plan.run(W, H); torch.cuda.synchronize()
print(wl, [repr(float(x)) for x in plan.sums.cpu().numpy()[:3]],
      float(plan.RH.double().abs().sum()), float(plan.RtW.double().abs().sum()))
