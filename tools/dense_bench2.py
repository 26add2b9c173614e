"""eigh / qr backends at c1 sizes (fp64): cusolver vs magma preference."""
import time, torch
dev = "cuda"
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / n
m = 1500
for lib in ("cusolver", "magma"):
    try:
        torch.backends.cuda.preferred_linalg_library(lib)
    except Exception as e:
        print(lib, "unavailable", e); continue
    for p in (512, 1024, 1400):
        b = torch.randn(m, p, dtype=torch.float64, device=dev)
        s = torch.randn(p, p, dtype=torch.float64, device=dev); s = s + s.T
        try:
            r = {"qr": t(lambda: torch.linalg.qr(b, mode="reduced")), "eigh": t(lambda: torch.linalg.eigh(s))}
        except Exception as e:
            r = {"err": str(e)[:80]}
        print(lib, p, r, flush=True)
