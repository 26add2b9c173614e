"""Where solve_mf_global's time goes at config 1 (or another config), with
synchronised timers around the dense lifting pieces: the Householder QR of
orthonormalize (with its block shapes), CholeskyQR2, shifted CholeskyQR3,
eigh, svd, the Rayleigh-Ritz step, apply_gram and the BCD epochs.
Usage: python tools/c1_phase_times.py [c1] [iters]   (MFG_QR selects the QR)"""
import collections, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_14067_b200 as P
from paper_2204_14067_b200 import eigensolver, kernels as K, mfsolver, operators, proxlift, synth

T = collections.Counter(); N = collections.Counter(); SH = collections.Counter()

def timed(mod, name, label=None, shape_of=None):
    fn = getattr(mod, name)
    label = label or name
    def wrap(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize(); T[label] += time.perf_counter() - t; N[label] += 1
        if shape_of is not None:
            SH[(label, tuple(shape_of(*a, **k)))] += 1
        return out
    setattr(mod, name, wrap)

timed(K, "_householder", shape_of=lambda c: c.shape)
timed(K, "_cholqr2", shape_of=lambda b, *r: b.shape)
timed(K, "_scholqr3")
timed(K, "_refactor_r", shape_of=lambda q, r, idx, j0: (r.shape[0], int(idx.numel()), j0))
timed(torch.linalg, "eigh", "eigh", shape_of=lambda t, *r, **k: t.shape)
timed(torch.linalg, "svd", "svd")
timed(eigensolver, "_ritz")
timed(eigensolver, "orthonormalize", "orthonormalize(eig)")
timed(proxlift, "orthonormalize", "orthonormalize(prox)")
timed(operators.ShiftedOperator, "apply_gram")
timed(mfsolver, "bcd_epoch")
timed(proxlift, "certify_epsilon")
timed(proxlift, "exact_svd_short_fat")

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 19
spec = synth.CONFIGS[wl]
m, n, r, c, v = synth.generate(wl)
m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
dt = torch.float64 if spec.dtype == "f64" else torch.float32
obs = P.ObservationSet.from_coo(m, n, r, c, v, transposed=tr, dtype=dt)
cfg = P.SolverConfig(lam=spec.lam, k0=spec.k0, seed=0, max_outer_iters=iters)
P.solve_mf_global(obs, None, P.SolverConfig(lam=spec.lam, k0=spec.k0, seed=0, max_outer_iters=1))
T.clear(); N.clear(); SH.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
x, wf, trace = P.solve_mf_global(obs, None, cfg)
torch.cuda.synchronize(); el = time.perf_counter() - t0
print(f"{wl}: {len(trace) - 1} outer iterations, rank {x.rank}, {el:.2f} s (timers synchronise, so this is an upper bound)")
for k_, t in T.most_common():
    print(f"  {k_:24s} {t:8.3f} s  {N[k_]:6d} calls  {1e3 * t / max(N[k_], 1):8.3f} ms/call")
for lab in ("_householder", "_cholqr2", "_refactor_r", "eigh"):
    tops = sorted(((cnt, sh) for (l, sh), cnt in SH.items() if l == lab), reverse=True)[:8]
    print(f"  {lab} shapes (count, shape):", tops)
