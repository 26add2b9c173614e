"""Run one BCD half-sweep twice (warm-up + profiled) for ncu:
    python tools/bcd_one.py c4 40 csc"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth  # noqa: E402
from paper_2204_14067_b200.data import ObservationSet  # noqa: E402
from paper_2204_14067_b200.mfsolver import _half_sweep  # noqa: E402

wl, k, side = sys.argv[1], int(sys.argv[2]), sys.argv[3]
m, n, r, c, v = synth.generate(wl)
m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
g = torch.Generator(device="cuda").manual_seed(0)
other = (0.1 * torch.randn((m if side == "csc" else n, k), device="cuda", generator=g)).float()
for _ in range(2):
    _half_sweep(obs, side == "csc", other, 50.0)
torch.cuda.synchronize()
print("done")
