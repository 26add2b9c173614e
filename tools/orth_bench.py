import sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import kernels as K
for m, p in [(3706, 80), (3706, 320), (3706, 1600), (17770, 160)]:
    b = torch.randn(m, p, dtype=torch.float64, device="cuda")
    b[:, : p // 4] *= 1e4  # Krylov-like column scale spread
    scale = float(torch.linalg.norm(b))
    for name, fn in [("cholqr2", lambda: K._cholqr2(b, scale, 1e-10)), ("householder", lambda: torch.linalg.qr(b)),
                     ("orthonormalize", lambda: K.orthonormalize(b))]:
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5): out = fn()
        torch.cuda.synchronize()
        ok = "" if name != "cholqr2" else ("fast" if out is not None else "fallback")
        print(m, p, name, round((time.perf_counter() - t) / 5 * 1e3, 2), "ms", ok)
