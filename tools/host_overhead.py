"""Host-side enqueue cost of the sweep entry points (c2)."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth, _lib
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.mfsolver import SweepPlan

m, n, r, c, v = synth.generate("c2"); m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
k = 20
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
w_np, h_np = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
plan = SweepPlan(obs, k)
w = plan.pad(torch.as_tensor(w_np).cuda()); h = plan.pad(torch.as_tensor(h_np).cuda())
wh = torch.as_tensor(w_np).pin_memory(); hh = torch.as_tensor(h_np).pin_memory()
lib = _lib.lib()
args = plan._args(w, h, torch.cuda.current_stream().cuda_stream)
dst = torch.empty_like(w); hostbuf = torch.empty(w.numel() * 4, dtype=torch.uint8).pin_memory()

def bench(name, fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t = 0.0
    for _ in range(n):
        t0 = time.perf_counter(); fn(); t += time.perf_counter() - t0
        torch.cuda.synchronize()
    print(f"{name:28s} {1e6 * t / n:7.1f} us/call (host)")

bench("mfg_sweep (cached args)", lambda: lib.mfg_sweep(*args))
bench("plan.run", lambda: plan.run(w, h))
bench("plan.run_host", lambda: plan.run_host(wh, hh))
bench("torch H2D copy_ 483KB", lambda: dst.copy_(wh, non_blocking=True))
bench("torch D2H copy_ 483KB", lambda: hostbuf.copy_(dst.view(torch.uint8).view(-1), non_blocking=True))
bench("empty sync", lambda: None)
