"""Diagnostics: per-worker phase timing of the grouped sweep (globaltimer stamps)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import _lib, synth
from paper_2204_14067_b200.data import ObservationSet
from paper_2204_14067_b200.mfsolver import SweepPlan


def chunks(nnz, wps=32):
    cb = max(4, min(512, -(-nnz // (8 * 148 * wps))))
    cb = (cb + 3) & ~3
    return -(-nnz // (cb * 8))


wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
m, n, r, c, v = synth.generate(wl); m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
k = synth.CONFIGS[wl].k0
obs = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
w, h = synth.sweep_factors(m, n, k, seed=1, dtype=np.float32)
plan = SweepPlan(obs, k)
W = plan.pad(torch.as_tensor(w).cuda()); H = plan.pad(torch.as_tensor(h).cuda())
n0 = n1 = chunks(len(v))
grid = -(-(((n0 + 3) & ~3) + ((n1 + 3) & ~3)) // 32)
probe = torch.zeros(10 * (n0 + n1) + 2 * grid + 16, dtype=torch.int64, device="cuda")
lib = _lib.lib()
for it in range(3):
    plan.run(W, H)
torch.cuda.synchronize()
flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda"); flush.zero_()
lib.mfg_set_probe(probe.data_ptr())
plan.run(W, H); torch.cuda.synchronize()
lib.mfg_set_probe(None)
allp = probe.cpu().numpy()
p = allp[: 10 * (n0 + n1)].reshape(-1, 10)
p = p[p[:, 0] != 0]
blk = allp[10 * (n0 + n1): 10 * (n0 + n1) + 2 * grid].reshape(-1, 2)
t0 = blk[:, 0].min()
print(wl, "workers", len(p), "blocks", grid)
for name, a in [("init", p[:, 1] - p[:, 0]), ("loop", p[:, 2] - p[:, 1]), ("finish", p[:, 3] - p[:, 2]),
                ("total", p[:, 3] - p[:, 0])]:
    print(f"{name:7s} mean {a.mean():9.0f} p50 {np.median(a):9.0f} p90 {np.percentile(a, 90):9.0f} max {a.max():9.0f}")
print("block entry offsets: p50 %.0f max %.0f" % (np.median(blk[:, 0] - t0), (blk[:, 0] - t0).max()))
print("worker start: min %.0f p50 %.0f; worker end: p50 %.0f p90 %.0f max %.0f" % (
    (p[:, 0] - t0).min(), np.median(p[:, 0] - t0), np.median(p[:, 3] - t0), np.percentile(p[:, 3] - t0, 90), (p[:, 3] - t0).max()))
print("final fold done at %.0f" % (blk[:, 1].max() - t0))
print("units: ns (globaltimer)")

# correlates of the loop time: pass, row starts per chunk, warp slot in the CTA
cb = max(4, min(512, -(-len(v) // (8 * 148 * 32)))); cb = (cb + 3) & ~3; CB = cb * 8
pp = allp[: 10 * (n0 + n1)].reshape(-1, 10)
loop = (pp[:, 2] - pp[:, 1]).astype(float)
ok = pp[:, 0] != 0
indptr_r = np.asarray(obs.indptr)
cnt_c = np.bincount(np.asarray(obs.cols), minlength=n)
indptr_c = np.concatenate([[0], np.cumsum(cnt_c)])
def starts(ptr, nch):
    s = np.zeros(nch)
    st = ptr[:-1][np.diff(ptr) > 0]
    np.add.at(s, np.minimum(st // CB, nch - 1), 1)
    return s
rs = np.concatenate([starts(indptr_r, n0), starts(indptr_c, n1)])
pas = np.concatenate([np.zeros(n0), np.ones(n1)])
for ps in (0, 1):
    sel = ok & (pas == ps)
    print(f"pass {ps}: loop mean {loop[sel].mean():.0f} p90 {np.percentile(loop[sel], 90):.0f} max {loop[sel].max():.0f}")
for lo, hi in ((0, 1), (1, 3), (3, 6), (6, 12), (12, 1000)):
    sel = ok & (rs >= lo) & (rs < hi)
    if sel.any():
        print(f"row starts [{lo},{hi}): n={sel.sum():5d} loop mean {loop[sel].mean():.0f} max {loop[sel].max():.0f}")
gid = np.concatenate([np.arange(n0), ((n0 + 3) & ~3) + np.arange(n1)])
slot = (gid % 32) // 4   # warp within the CTA
for w_ in range(8):
    sel = ok & (slot == w_)
    print(f"warp slot {w_}: loop mean {loop[sel].mean():.0f}")
blkid = gid // 32
bm = np.array([loop[ok & (blkid == b_)].mean() if (ok & (blkid == b_)).any() else np.nan for b_ in range(grid)])
print("per-block loop mean: min %.0f p50 %.0f max %.0f" % (np.nanmin(bm), np.nanmedian(bm), np.nanmax(bm)))
# warp-level: row starts summed over the warp's 4 workers
rsw = np.zeros_like(rs)
for base in (0, n0):
    nn = n0 if base == 0 else n1
    for g0 in range(0, nn, 4):
        rsw[base + g0: base + min(g0 + 4, nn)] = rs[base + g0: base + min(g0 + 4, nn)].sum()
for lo, hi in ((0, 3), (3, 6), (6, 10), (10, 15), (15, 1000)):
    sel = ok & (rsw >= lo) & (rsw < hi)
    if sel.any():
        print(f"warp row starts [{lo},{hi}): n={sel.sum():5d} loop mean {loop[sel].mean():.0f} max {loop[sel].max():.0f}")
