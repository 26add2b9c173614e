import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth, mfsolver as MF
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.operators import FactorPair
k = 64
m, n, r, c, v = synth.generate("c3", scale=0.03, seed=k)
m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
w, h = synth.sweep_factors(m, n, k, seed=k)
print(m, n, len(v), flush=True)
for dtype in (torch.float64, torch.float32):
    obs = ObservationSet.from_coo(m, n, r, c, v, dtype=dtype)
    wf = FactorPair(torch.as_tensor(w).to(dtype), torch.as_tensor(h).to(dtype))
    print("run", dtype, flush=True)
    out = MF.sweep(obs, wf, want_r=True, want_rh=True, want_rtw=True, compute_f64=False)
    torch.cuda.synchronize(); print("ok", out[3], flush=True)
