"""dense.qr (csrc/qr.cu) against torch.linalg.qr (cuSOLVER geqrf + orgqr) at the
block shapes of configs 1-4: milliseconds per factorisation, max |Q^T Q - I|.
Usage: python tools/qr_bench.py"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import dense, kernels as K

def t_ms(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, out

import sys
SHAPES = [(2000, 24), (2000, 96), (2000, 300), (1500, 300), (3706, 80), (6040, 320), (6040, 1600),
             (10677, 240), (71567, 240), (17770, 160), (480189, 120)]
if len(sys.argv) > 1 and sys.argv[1] == "wide":
    SHAPES = [(10677, 480), (10677, 960), (71567, 480), (71567, 960), (17770, 640), (6040, 800), (3706, 800), (2000, 600)]
for m, p in SHAPES:
    b = torch.randn(m, p, dtype=torch.float64, device="cuda")
    b[:, : p // 4] *= 1e4
    ours, (q, d) = t_ms(lambda: dense.qr(b))
    lib, (q0, r0) = t_ms(lambda: torch.linalg.qr(b))
    scale = float(torch.linalg.norm(b))
    chol, qc = t_ms(lambda: K._cholqr2(b, scale, 1e-10))
    eye = torch.eye(p, dtype=torch.float64, device="cuda")
    err = float((dense.gram(q) - eye).abs().max())
    derr = float(((d - r0.diagonal().abs()) / r0.diagonal().abs()).abs().max())
    print(f"{m:7d} x {p:5d}  ours {ours:8.2f} ms  cusolver {lib:8.2f} ms  x{lib / ours:5.2f}  "
          f"cholqr2 {chol:8.2f} ms ({'ok' if qc is not None else 'declined'})  orth {err:.1e}  diag rel {derr:.1e}", flush=True)
