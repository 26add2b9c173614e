"""Diagnostics: per-worker phase timing of the grouped sweep (clock64 stamps)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2204_14067_b200 import _lib, synth
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.mfsolver import SweepPlan
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
m, n, r, c, v = synth.generate(wl); m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
k = synth.CONFIGS[wl].k0
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
w, h = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
plan = SweepPlan(obs, k)
W = plan.pad(torch.as_tensor(w).cuda()); H = plan.pad(torch.as_tensor(h).cuda())
probe = torch.zeros(10 * 4_000_000, dtype=torch.int64, device="cuda")
lib = _lib.lib()
for it in range(3):
    plan.run(W, H)
torch.cuda.synchronize()
flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda"); flush.zero_()
lib.mfg_set_probe(probe.data_ptr())
plan.run(W, H); torch.cuda.synchronize()
lib.mfg_set_probe(None)
p = probe.view(-1, 10).cpu().numpy()
p = p[p[:, 0] != 0]
t0 = p[:, 0].min()
init = p[:, 1] - p[:, 0]; loop = p[:, 2] - p[:, 1]; fin = p[:, 3] - p[:, 2]; tot = p[:, 3] - p[:, 0]
print(wl, "workers", len(p), "span cycles", p[:, 3].max() - t0)
for name, a in [("init", init), ("loop", loop), ("finish", fin), ("total", tot), ("issue", p[:, 4]), ("wait", p[:, 5]), ("fetch+bits", p[:, 6]), ("lds+dot", p[:, 7]), ("reduce", p[:, 8]), ("r+acc", p[:, 9])]:
    print(f"{name:7s} mean {a.mean():9.0f} p50 {np.median(a):9.0f} p90 {np.percentile(a, 90):9.0f} max {a.max():9.0f}")
st = p[:, 0] - t0
print("start offsets (ns): p10", np.percentile(st, 10), "p50", np.median(st), "p90", np.percentile(st, 90), "max", st.max())
en = p[:, 3] - t0
print("end offsets (ns): p10", np.percentile(en, 10), "p50", np.median(en), "p90", np.percentile(en, 90), "max", en.max())
print("units: ns (globaltimer)")
# clocks differ per SM; use relative numbers only
