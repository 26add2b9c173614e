import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.mfsolver import SweepPlan
for dt in (torch.float32, torch.float64):
    for k in (8, 20, 32, 40, 64):
        m, n, r, c, v = synth.generate("c3", scale=0.03, seed=100 + k)
        m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
        obs = ObservationSet.from_coo(m, n, r, c, v, dtype=dt)
        plan = SweepPlan(obs, k)
        w, h = synth.sweep_factors(m, n, k, seed=k)
        W = plan.pad(torch.as_tensor(w).to(dt).cuda()); H = plan.pad(torch.as_tensor(h).to(dt).cuda())
        try:
            plan.run(W, H); torch.cuda.synchronize()
            print(dt, k, "kp", plan.kp, "ok", plan.sums.cpu().numpy()[0], flush=True)
        except Exception as e:
            print(dt, k, "kp", plan.kp, "FAIL", str(e)[:80], flush=True)
            raise
