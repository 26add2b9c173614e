"""A/B of the end-to-end sweep: results copied back by a D2H node after the
kernel (current run_host) vs written by the kernel straight into the pinned
host buffer (mapped, UVA), so the output rows cross PCIe while the sweep
still runs. Usage: python tools/e2e_mapped.py c2 [steps]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import _lib, synth
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.mfsolver import SweepPlan

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
m, n, r, c, v = synth.generate(wl)
m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
k = synth.CONFIGS[wl].k0
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
w_np, h_np = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
plan = SweepPlan(obs, k, want_rh=True, want_rtw=True)
w_host, h_host = plan.pinned_factors()
w_host.copy_(torch.as_tensor(w_np)); h_host.copy_(torch.as_tensor(h_np))
stream = torch.cuda.current_stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

sums_a, rh_a, rtw_a = [x.clone() for x in plan.run_host(w_host, h_host)]
torch.cuda.synchronize()
ref = [x.clone() for x in plan.run_host(w_host, h_host)]
torch.cuda.synchronize()

lib = _lib.lib()
mapped = torch.empty_like(plan._host).pin_memory()
tail = list(plan._host_tail)
tail[5] = mapped.data_ptr()   # out -> pinned host memory (UVA device pointer)
tail[6] = None                # no D2H node
nb_rh = plan.RH.numel() * plan.RH.element_size()
views = (mapped[:24].view(torch.float64), mapped[32:32 + nb_rh].view(torch.float32).view(m, k),
         mapped[32 + nb_rh:].view(torch.float32).view(n, k))


def call(st):
    _lib.check(lib.mfg_sweep_host(*plan._host_args, w_host.data_ptr(), h_host.data_ptr(), *tail, st),
               "sweep_host mapped")


call(stream.cuda_stream); torch.cuda.synchronize()
side = torch.cuda.Stream(); side.wait_stream(stream)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
    call(side.cuda_stream)
stream.wait_stream(side)
g.replay(); torch.cuda.synchronize()
for a_, b_ in zip(ref, views):
    assert torch.equal(a_, b_), "mapped output differs"
print("mapped output bitwise equal to the D2H path")


def timeit(fn, read):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        _ = float(read()[0])
        tot += a.elapsed_time(b)
    return tot / steps * 1e3


for rep in range(2):
    t_d2h = timeit(lambda: plan.run_host(w_host, h_host), lambda: plan._host_views[0])
    t_map = timeit(lambda: g.replay(), lambda: views[0])
    print(f"{wl} rep{rep}: D2H node {t_d2h:.1f} us/step ({1e6 / t_d2h:.0f}/s)  "
          f"mapped output {t_map:.1f} us/step ({1e6 / t_map:.0f}/s)")
