"""One dense.qr call at a given shape (for ncu launch lists): python tools/qr_one.py 2000 300"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import dense
m, p = int(sys.argv[1]), int(sys.argv[2])
b = torch.randn(m, p, dtype=torch.float64, device="cuda")
for _ in range(2):
    q, d = dense.qr(b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    q, d = dense.qr(b)
e1.record(); torch.cuda.synchronize()
print(m, p, "ms per qr (events)", e0.elapsed_time(e1) / 20)
