"""The lifting-step SpMMs at a workload and block width p, whole and in
column slabs of width w (the gathered slab of the dense block then fits L2):
python tools/spmm_slab_probe.py c4 160"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import _lib, synth
from paper_2204_14067_b200.data import ObservationSet
wl, p = sys.argv[1], int(sys.argv[2])
m, n, r, c, v = synth.generate(wl); m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
g = torch.Generator(device="cuda").manual_seed(0)
G = torch.randn(len(v), dtype=torch.float64, device="cuda", generator=g)
V = torch.randn((n, p), dtype=torch.float64, device="cuda", generator=g)
U = torch.randn((m, p), dtype=torch.float64, device="cuda", generator=g)
lib = _lib.lib()
dev = obs.dev
flush = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
for name, lay, X, rows in (("G @ V (CSR, gathers n-side rows)", dev.csr, V, m),
                           ("G^T @ U (CSC, gathers m-side rows)", dev.csc, U, n)):
    ref = None
    for w in (p, 80, 64, 48, 40, 32, 24, 16):
        if w > p:
            continue
        out = torch.zeros((rows, p), dtype=torch.float64, device="cuda")
        wsb = lib.mfg_spmm_workspace(lay.ref, w)
        ws = dev.workspace(wsb)

        def call():
            for s in range(0, p, w):
                ww = min(w, p - s)
                _lib.check(lib.mfg_spmm(_lib.MFG_F64, lay.ref, ww, G.data_ptr(), X.data_ptr() + 8 * s, p,
                                        1.0, 0.0, out.data_ptr() + 8 * s, p, ws.data_ptr(), wsb,
                                        _lib.stream_ptr()), "spmm")
        call(); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); call(); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        if ref is None:
            ref = out.clone()
        err = float((out - ref).abs().max() / ref.abs().max())
        print(f"{wl} p={p} {name}: slab {w:4d}: {min(ts):8.2f} ms  (rel diff to whole {err:.1e}, "
              f"bitwise {bool(torch.equal(out, ref))})", flush=True)
