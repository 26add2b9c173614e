"""Dense lifting-step pieces at c1 sizes (fp64): QR, CholQR2, eigh, GEMMs."""
import time, torch
torch.manual_seed(0)
dev = "cuda"

def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / n

m = 1500
for p in (128, 256, 512, 1024, 1400):
    b = torch.randn(m, p, dtype=torch.float64, device=dev)
    s = torch.randn(p, p, dtype=torch.float64, device=dev); s = s + s.T
    g = b.T @ b
    r = {}
    r["qr"] = t(lambda: torch.linalg.qr(b, mode="reduced"))
    r["geqrf"] = t(lambda: torch.geqrf(b))
    r["gram"] = t(lambda: b.T @ b)
    r["chol"] = t(lambda: torch.linalg.cholesky_ex(g))
    L = torch.linalg.cholesky(g)
    r["trsm"] = t(lambda: torch.linalg.solve_triangular(L.T, b, upper=True, left=False))
    r["eigh"] = t(lambda: torch.linalg.eigh(s))
    r["eigvalsh"] = t(lambda: torch.linalg.eigvalsh(s))
    r["svd"] = t(lambda: torch.linalg.svd(b, full_matrices=False))
    print(f"p={p:5d} " + " ".join(f"{k} {v:7.2f}ms" for k, v in r.items()), flush=True)
