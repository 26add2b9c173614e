"""One Gram (k_gemm_tn) and one tall-times-small product (k_gemm_nn) at a given
shape, for ncu captures: python tools/gemm_one.py 480189 120"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import dense
m, p = int(sys.argv[1]), int(sys.argv[2])
a = torch.randn(m, p, dtype=torch.float64, device="cuda")
s = torch.randn(p, p, dtype=torch.float64, device="cuda")
for _ in range(3):
    g = dense.gram(a)
    c = dense.matmul(a, s)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
for _ in range(20):
    g = dense.gram(a)
e[1].record()
for _ in range(20):
    c = dense.matmul(a, s)
e[2].record(); torch.cuda.synchronize()
tg, tm = e[0].elapsed_time(e[1]) / 20, e[1].elapsed_time(e[2]) / 20
fl = 2.0 * m * p * p
print(f"{m} x {p}: gram {tg:.3f} ms ({fl / tg / 1e9:.1f} TF/s, {m * p * 8 / tg / 1e6:.0f} GB/s of A), "
      f"matmul {tm:.3f} ms ({fl / tm / 1e9:.1f} TF/s)")
