"""Share of entries whose gathered row is among the H most frequent (per pass)."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth
for wl in sys.argv[1:]:
    cache = os.environ.get("MFG_SYNTH_CACHE")
    path = os.path.join(cache, f"{wl}_0.npz") if cache else None
    if path and os.path.exists(path):
        z = np.load(path); m, n, r, c, v = int(z["m"]), int(z["n"]), z["r"], z["c"], z["v"]
    else:
        m, n, r, c, v = synth.generate(wl)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    k = synth.CONFIGS[wl].k0
    for name, ids, N in (("CSR pass gathers H (cols)", c, n), ("CSC pass gathers W (rows)", r, m)):
        deg = np.sort(np.bincount(ids, minlength=N))[::-1]
        cs = np.cumsum(deg) / deg.sum()
        rowb = k * 4
        out = []
        for kb in (48, 96, 160):
            H = (kb * 1024) // rowb
            out.append(f"{kb}KB->{H} rows: {cs[min(H, N) - 1]:.3f}")
        print(wl, name, "N", N, "; ".join(out), flush=True)
