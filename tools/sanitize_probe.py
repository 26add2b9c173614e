"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
the grouped sweep with chunk-crossing rows (lock-free row finisher + last-
arriver fold) and both BCD paths (DMMA warp-per-row with split heavy rows,
and the SIMT kernel) on a c2-shaped instance scaled down, fp32 and fp64."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth  # noqa: E402
from paper_2204_14067_b200.data import ObservationSet  # noqa: E402
from paper_2204_14067_b200.mfsolver import SweepPlan, _half_sweep, check_bcd_status  # noqa: E402

m, n, r, c, v = synth.generate("c2", scale=0.1, seed=3)
m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
for dt in (torch.float32, torch.float64):
    obs = ObservationSet.from_coo(m, n, r, c, v, dtype=dt)
    for k in (20, 40):
        w, h = synth.sweep_factors(m, n, k, seed=k)
        plan = SweepPlan(obs, k)
        wt = plan.pad(torch.as_tensor(w, device="cuda"))
        ht = plan.pad(torch.as_tensor(h, device="cuda"))
        plan.run(wt, ht)
        plan.run(wt, ht)
        for tr, other in ((False, torch.as_tensor(h, device="cuda")), (True, torch.as_tensor(w, device="cuda"))):
            _half_sweep(obs, tr, other.to(dt), 5.0)
        check_bcd_status()
torch.cuda.synchronize()
print("sanitize probe ok", m, n, len(v))
