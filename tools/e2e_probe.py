"""Break the bench e2e step (c2) into stages with CUDA events."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.mfsolver import SweepPlan

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
m, n, r, c, v = synth.generate(wl); m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
k = synth.CONFIGS[wl].k0
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
w_np, h_np = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
plan = SweepPlan(obs, k)
w = plan.pad(torch.as_tensor(w_np).cuda()); h = plan.pad(torch.as_tensor(h_np).cuda())
w_host = torch.as_tensor(w_np).pin_memory(); h_host = torch.as_tensor(h_np).pin_memory()
s = torch.cuda.current_stream()
tot = 0.0
host = 0.0
N = 200
flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
for it in range(N + 10):
    if len(sys.argv) > 2:
        flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    t0 = time.perf_counter()
    sums, _, _ = plan.run_host(w_host, h_host)
    host += time.perf_counter() - t0
    b.record(s)
    b.synchronize()
    if it >= 10:
        tot += a.elapsed_time(b)
print(f"run_host total {1e3 * tot / N:8.1f} us  host enqueue {1e6 * host / (N + 10):6.1f} us (ld={plan.ld}, k={k})")
