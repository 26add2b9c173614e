"""Time the lifting-step SpMMs (G_csr @ V, G_csc^T @ U, fp64) at a workload
and block width p (diagnostics): python tools/spmm_probe.py c3 480"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth, operators
from paper_2204_14067_b200.data import ObservationSet
wl, p = sys.argv[1], int(sys.argv[2])
m, n, r, c, v = synth.generate(wl); m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
g = torch.Generator(device="cuda").manual_seed(0)
G = torch.randn(len(v), dtype=torch.float64, device="cuda", generator=g)
V = torch.randn((n, p), dtype=torch.float64, device="cuda", generator=g)
U = torch.randn((m, p), dtype=torch.float64, device="cuda", generator=g)
from paper_2204_14067_b200 import _lib
lib = _lib.lib()
dev = obs.dev
for name, lay, X, rows in (("G @ V (CSR)", dev.csr, V, m), ("G^T @ U (CSC)", dev.csc, U, n)):
    out = torch.empty((rows, p), dtype=torch.float64, device="cuda")
    wsb = lib.mfg_spmm_workspace(lay.ref, p)
    ws = dev.workspace(wsb)
    call = lambda: _lib.check(lib.mfg_spmm(_lib.MFG_F64, lay.ref, p, G.data_ptr(), X.data_ptr(), p, 1.0, 0.0,
                                           out.data_ptr(), p, ws.data_ptr(), wsb, _lib.stream_ptr()), "spmm")
    call(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); reps = 5
    for _ in range(reps):
        call()
    b.record(); b.synchronize()
    t = a.elapsed_time(b) / reps * 1e-3
    nnz = len(v)
    gathered = nnz * p * 8
    alg = nnz * 12 + 4 * (rows + 1) + 8 * (m + n) * p
    print(f"{wl} p={p} {name}: {t * 1e3:.2f} ms; algorithmic {alg / t / 1e9:.0f} GB/s, "
          f"gathered rows {gathered / t / 1e12:.2f} TB/s through L2, {2 * nnz * p / t / 1e12:.2f} TFLOP/s")
