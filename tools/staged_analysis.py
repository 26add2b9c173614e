"""Sizing of the shared-memory staged sweep per workload (design tool).

For each pass (CSR: rows gather H; CSC: rows gather W), the gathered rows are
ranked by degree and cut into blocks of S rows (S = smem budget / row bytes).
A block is staged when its entries per nonempty (row, block) pair (L) reach
a threshold; the rest is the cold stream. Prints entries covered, pieces
(partial row vectors the fold adds) and the L2 traffic model against the
current all-gather design.

    python tools/staged_analysis.py c2 [c3 c4]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_14067_b200 import synth  # noqa: E402

K = {"c1": 8, "c2": 20, "c3": 30, "c4": 40, "c5": 64}
BUDGET = int(os.environ.get("BUDGET", 190 * 1024))
LMIN = float(os.environ.get("LMIN", 4.0))


def analyse(rows, cols, nrows, ng, k):
    rb = ((k * 4 + 15) // 16) * 16
    S = BUDGET // rb
    deg = np.bincount(cols, minlength=ng)
    order = np.argsort(-deg, kind="stable")
    rank = np.empty(ng, np.int64)
    rank[order] = np.arange(ng)
    blk = rank // S
    nb = int(blk.max()) + 1
    eb = blk[cols]
    ent = np.bincount(eb, minlength=nb)
    key = np.unique(eb * nrows + rows)
    pairs = np.bincount(key // nrows, minlength=nb)
    L = ent / np.maximum(pairs, 1)
    staged = 0
    while staged < nb and L[staged] >= LMIN:
        staged += 1
    nnz = len(rows)
    e_st = int(ent[:staged].sum())
    p_st = int(pairs[:staged].sum())
    cold = nnz - e_st
    cold_rows = len(np.unique(rows[eb >= staged])) if cold else 0
    gb_now = nnz * rb
    gb_new = cold * rb + 2 * (p_st + cold_rows) * rb + 148 * min(staged, 3) * S * rb
    print(f"   rb={rb} S={S} blocks={nb} staged={staged} entries staged {e_st/nnz:.1%} "
          f"pieces={p_st + cold_rows} (L first/last staged {L[0]:.1f}/{L[staged-1] if staged else 0:.1f})"
          f"  gather L2 bytes now {gb_now/1e6:.1f} MB -> ~{gb_new/1e6:.1f} MB")


for name in sys.argv[1:] or ["c2"]:
    t = time.time()
    m, n, r, c, v = synth.generate(name)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    r = np.asarray(r, np.int64)
    c = np.asarray(c, np.int64)
    print(f"{name}: {m} x {n}, nnz {len(r)}, k {K[name]} (gen {time.time()-t:.0f}s)")
    print("  CSR pass (rows gather H):")
    analyse(r, c, m, n, K[name])
    print("  CSC pass (cols gather W):")
    analyse(c, r, n, m, K[name])
