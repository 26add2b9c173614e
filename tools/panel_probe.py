"""Hybrid (panel + gather) sweep against the gather-only sweep: parity, bitwise
repeatability and kernel time (CUDA events, L2 flushed between runs).
usage: python tools/panel_probe.py c4 [k] [scale]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_14067_b200 as P
from paper_2204_14067_b200 import _lib, mfsolver, panel, synth

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else synth.CONFIGS[wl].k0
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
t0 = time.time()
m, n, r, c, v = synth.generate(wl, scale=scale, seed=0)
m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
obs = P.ObservationSet.from_coo(m, n, r, c, v).with_dtype(torch.float32)
print(f"{wl}: {m} x {n}, nnz {len(r)}, k {k}; instance {time.time() - t0:.1f}s", flush=True)
w, h = synth.sweep_factors(m, n, k, seed=1)
base = mfsolver.SweepPlan(obs, k)
wd = base.pad(torch.as_tensor(w, dtype=torch.float32, device="cuda"))
hd = base.pad(torch.as_tensor(h, dtype=torch.float32, device="cuda"))
t0 = time.time()
hyb = panel.HybridSweepPlan(obs, k)
torch.cuda.synchronize()
print(f"hybrid plan build {time.time() - t0:.1f}s", json.dumps(hyb.stats), flush=True)
assert hyb.ld == base.ld, (hyb.ld, base.ld)

base.run(wd, hd)
hyb.run(wd, hd)
torch.cuda.synchronize()
if os.environ.get("MFG_PROBE_QUICK"):
    sys.exit(0)


def rel(a, b):
    a = a.double(); b = b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


out = {"R": rel(hyb.R, base.R), "RH": rel(hyb.RH, base.RH), "RtW": rel(hyb.RtW, base.RtW),
       "sums": [float(x) for x in ((hyb.sums - base.sums).abs() / base.sums.abs()).cpu()]}
print("hybrid vs gather sweep (max abs diff / max abs):", json.dumps(out), flush=True)
g = torch.Generator(device="cpu").manual_seed(0)
dev = obs.dev
nnz = obs.size
samp = torch.randint(0, nnz, (4096,), generator=g).cuda()
rows = dev.csr.row_of[:nnz][samp].long(); cols = dev.csr.idx[:nnz][samp].long()
w64 = wd[:, :k].double(); h64 = hd[:, :k].double()
r64 = (w64[rows] * h64[cols]).sum(1) - dev.vals[:nnz][samp].double()
print("sampled R vs fp64: max abs err", float((hyb.R[samp].double() - r64).abs().max()),
      "(gather kernel:", float((base.R[samp].double() - r64).abs().max()), ")", flush=True)
keep = [hyb.R.clone(), hyb.RH.clone(), hyb.RtW.clone(), hyb.sums.clone()]
hyb.run(wd, hd)
torch.cuda.synchronize()
same = all(torch.equal(a, b) for a, b in zip(keep, [hyb.R, hyb.RH, hyb.RtW, hyb.sums]))
print("bitwise repeatable:", same, flush=True)

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=8):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return round(float(np.median(ts)), 4)


res = {"workload": wl, "k": k, "gather_ms": t(lambda: base.run(wd, hd)),
       "hybrid_ms": t(lambda: hyb.run(wd, hd)), "stats": hyb.stats}
print(json.dumps(res), flush=True)
lib = _lib.lib()
st = _lib.stream_ptr()


def cold():
    if hyb.cold == "pieces":
        _lib.check(lib.mfg_cold_sweep(hyb.ld, hyb.p0.cold_ref, hyb.p1.cold_ref, wd.data_ptr(), hd.data_ptr(),
                                      hyb.RH.data_ptr(), hyb.RtW.data_ptr(), 1.0,
                                      hyb.cold_counters.data_ptr(), st), "cold")
        return
    _lib.check(lib.mfg_sweep_sharded(_lib.MFG_F32, 0, hyb.cold_csr.ref, hyb.cold_csc.ref, k,
               hyb.cold_vals.data_ptr(), hyb.cold_vals_csc.data_ptr(), wd.data_ptr(), wd.data_ptr(),
               hyb.ld, hd.data_ptr(), hd.data_ptr(), hyb.ld, hyb._rcold.data_ptr(), hyb.RH.data_ptr(),
               hyb.RtW.data_ptr(), 1.0, hyb.sums.data_ptr(), hyb.ws.data_ptr(), hyb.wsb, st), "cold")


def pan_list(plist):
    n = int(plist.shape[0])
    if n:
        cs = (torch.arange(148, device="cuda") * n // 148).to(torch.int32)
        cnt = torch.zeros(n + 2, dtype=torch.int32, device="cuda")
        return lambda: _lib.check(lib.mfg_panel_sweep(hyb.ld, n, plist.data_ptr(), cs.data_ptr(), hyb.p0.ref,
                                  hyb.p1.ref, wd.data_ptr(), hd.data_ptr(), cnt.data_ptr(), st), "panel")
    return lambda: None


def pan():
    _lib.check(lib.mfg_panel_sweep(hyb.ld, hyb.n_list, hyb.plist.data_ptr(), hyb.cta_start.data_ptr(), hyb.p0.ref,
               hyb.p1.ref, wd.data_ptr(), hd.data_ptr(), hyb.counters.data_ptr(), st), "panel")


def fold():
    _lib.check(lib.mfg_panel_fold(hyb.ld, k, hyb.p0.ref, hyb.RH.data_ptr(), k, 1.0, 0, hyb.sums.data_ptr(), hyb.sq_ws.data_ptr(), st), "f")
    _lib.check(lib.mfg_panel_fold(hyb.ld, k, hyb.p1.ref, hyb.RtW.data_ptr(), k, 1.0, 0, None, None, st), "f")


def rg():
    _lib.check(lib.mfg_gather(_lib.MFG_F32, nnz, hyb._rsrc.data_ptr(), hyb._rcat.data_ptr(),
                              hyb.R.data_ptr(), st), "g")


print(json.dumps({"cold_ms": t(cold), "panel_ms": t(pan), "panel_csr_ms": t(pan_list(hyb.p0.plist)),
                  "panel_csc_ms": t(pan_list(hyb.p1.plist)), "fold_ms": t(fold), "rgather_ms": t(rg)}), flush=True)
