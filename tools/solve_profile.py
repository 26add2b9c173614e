"""Time solve_mf_global on a config and attribute time to phases (diagnostics)."""
import sys, os, time, json, collections, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_14067_b200 as P
from paper_2204_14067_b200 import synth, mfsolver, proxlift, eigensolver, kernels, operators, data, driver
wl = sys.argv[1]; iters = int(sys.argv[2]); dt = torch.float32 if wl != "c1" else torch.float64
m, n, r, c, v = synth.generate(wl); m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
obs = P.ObservationSet.from_coo(m, n, r, c, v, transposed=tr, dtype=dt)
T = collections.Counter(); N = collections.Counter()
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        out = f(*a, **k)
        torch.cuda.synchronize(); T[name] += time.perf_counter() - t; N[name] += 1
        return out
    setattr(mod, name, g)
for mod, name in [(operators, "spmm"), (driver, "mf_phase"), (driver, "mf_objective"), (driver, "inexact_prox_step"), (proxlift, "solve_topk"),
                  (proxlift, "certify_epsilon"), (proxlift, "exact_svd_short_fat"), (eigensolver, "orthonormalize"),
                  (eigensolver, "_ritz"), (driver, "build_warmstart"), (driver, "residual_on_omega_svd"),
                  (mfsolver, "bcd_epoch")]:
    wrap(mod, name)
CQ = collections.Counter()
_orig_cq = kernels._cholqr2
def _cq(b, scale, tol):
    t = time.perf_counter()
    out = _orig_cq(b, scale, tol)
    torch.cuda.synchronize()
    key = ("ok" if out is not None else "fail", (b.shape[1] // 64) * 64)
    CQ[key] += 1
    T["cholqr2_" + key[0]] += time.perf_counter() - t
    return out
kernels._cholqr2 = _cq
_orig_qr = torch.linalg.qr
QRN = collections.Counter()
def _qr(a, mode="reduced"):
    QRN[(a.shape[1] // 128) * 128] += 1
    torch.cuda.synchronize(); t = time.perf_counter()
    out = _orig_qr(a, mode=mode)
    torch.cuda.synchronize(); T["householder_qr"] += time.perf_counter() - t
    return out
kernels.torch.linalg.qr = _qr
cfg = P.SolverConfig(lam=synth.CONFIGS[wl].lam, k0=synth.CONFIGS[wl].k0, max_outer_iters=iters, seed=0)
t0 = time.perf_counter()
x, _, trace = P.solve_mf_global(obs, None, cfg)
el = time.perf_counter() - t0
print(wl, "iters", len(trace) - 1, "time", round(el, 2), "s; rank", x.rank, "F", trace.final().obj)
for rec in trace.records: print("  it", rec.iter, "t=%.2f" % rec.time_s, "obj %.8g" % rec.obj, "rank", rec.rank, "k_t", rec.k_t, "sweeps", rec.eig_sweeps, "bt", rec.backtracks)
for k_, t_ in T.most_common(): print(f"{k_:24s} {t_:8.2f}s  n={N[k_]}")
for k_, c_ in sorted(CQ.items(), key=lambda kv: (kv[0][1], kv[0][0])): print("cholqr2", k_, c_)
print("householder qr calls by width:", sorted(QRN.items()))
