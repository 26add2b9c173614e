"""Time the BCD half-sweeps at a given workload and rank (diagnostics):
    python tools/bcd_probe.py c3 480"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth  # noqa: E402
from paper_2204_14067_b200.data import ObservationSet  # noqa: E402
from paper_2204_14067_b200.mfsolver import _half_sweep  # noqa: E402

wl, k = sys.argv[1], int(sys.argv[2])
m, n, r, c, v = synth.generate(wl)
m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
g = torch.Generator(device="cuda").manual_seed(0)
H = (0.1 * torch.randn((n, k), device="cuda", generator=g)).float()
W = (0.1 * torch.randn((m, k), device="cuda", generator=g)).float()
for name, tr, other in (("rows (CSR)", False, H), ("cols (CSC)", True, W)):
    _half_sweep(obs, tr, other, 50.0)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5 if k <= 200 else 2):   # best of n (clock ramp, first-touch)
        t = time.perf_counter()
        out = _half_sweep(obs, tr, other, 50.0)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    chk = repr(float(out.double().abs().sum())) if torch.is_tensor(out) else "-"
    deg = np.diff(obs.dev.csc.ptr.cpu().numpy() if tr else obs.dev.csr.ptr.cpu().numpy())
    print(f"{wl} k={k} {name}: {1e3 * best:.2f} ms; rows {deg.size}, "
          f"d mean {deg.mean():.0f} max {deg.max()}, rows with d > 150: {(deg > 150).sum()}; checksum {chk}")
