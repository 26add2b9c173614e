"""Seeded synthetic Omega instances for the BASELINE.json configs c1..c5.

The paper's recommender datasets are not available (no network, and their
records must not be reproduced), so every benchmark and large parity case runs
on synthetic instances with the shapes, degree distributions and value
distributions that ``BASELINE.json:configs`` describes. The recipe follows
SURVEY.md §8(d):

* c1: |Omega| positions uniformly without replacement; values
  clip(rint(3 + W* H*^T + N(0, 0.5^2)), 1, 5) with W*, H* of rank 5.
* c2..c5: capped Zipf row degrees d_i = clip(floor(C * pi_i^-s_r), d_min, n)
  with C bisected so sum(d) hits |Omega| exactly; per row, d_i distinct
  columns drawn without replacement with weight rho_j^-s_c (successive
  sampling = draw with replacement, keep first occurrences; Efraimidis-
  Spirakis keys for heavy rows). Values offset + rank-r Gaussian signal +
  Gaussian noise, then quantised.

"N(0, v)" in the config text is read as variance v (so a rank-r signal with
factor entries of variance 1/sqrt(r) has unit entry variance); this choice is
recorded in DESIGN.md. All values are exactly representable in fp32.

Instances are returned in *raw* (user x item) orientation as COO arrays; the
canonical m <= n orientation is applied by :func:`canonical` exactly as the
reference's loader does (``mfg/data.py:229-236``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    m: int            # raw rows (users)
    n: int            # raw cols (items)
    nnz: int
    k0: int
    dtype: str        # "f64" or "f32"
    rank: int
    offset: float
    signal_std: float
    noise_std: float
    quant: tuple      # (step, lo, hi)
    s_row: float = 0.0
    s_col: float = 0.0
    d_min: int = 1
    uniform: bool = False
    lam: float = 5.0  # lambda; unspecified for c2..c5 (recorded in DESIGN.md)


CONFIGS = {
    "c1": ConfigSpec("c1", 2000, 1500, 100_000, 8, "f64", 5, 3.0, 1.0, 0.5,
                     (1.0, 1.0, 5.0), uniform=True, lam=5.0),
    "c2": ConfigSpec("c2", 6040, 3706, 1_000_209, 20, "f32", 10, 3.0, 1.0, 0.6,
                     (1.0, 1.0, 5.0), s_row=1.0, s_col=1.0, d_min=20, lam=50.0),
    "c3": ConfigSpec("c3", 71_567, 10_677, 10_000_054, 30, "f32", 15, 3.5, 1.0, 0.7,
                     (0.5, 0.5, 5.0), s_row=1.1, s_col=1.1, lam=100.0),
    "c4": ConfigSpec("c4", 480_189, 17_770, 100_480_507, 40, "f32", 20, 3.6, 1.0, 0.8,
                     (1.0, 1.0, 5.0), s_row=1.2, s_col=0.9, lam=500.0),
    "c5": ConfigSpec("c5", 1_000_990, 624_961, 252_800_275, 64, "f32", 32, 50.0, 20.0, 10.0,
                     (1.0, 0.0, 100.0), s_row=1.3, s_col=1.3, lam=2000.0),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def zipf_degrees(rng, m: int, n: int, nnz: int, s: float, d_min: int) -> np.ndarray:
    """Capped Zipf degree sequence with sum exactly ``nnz``."""
    if m * d_min > nnz or m * n < nnz:
        raise ValueError("infeasible degree sequence")
    ranks = rng.permutation(m).astype(np.float64) + 1.0
    base = ranks ** (-s)

    def total(c):
        return int(np.clip(np.floor(c * base), d_min, n).sum())

    lo, hi = 0.0, 1.0
    while total(hi) < nnz:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if total(mid) <= nnz:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-12 * hi:
            break
    d = np.clip(np.floor(lo * base), d_min, n).astype(np.int64)
    deficit = nnz - int(d.sum())
    # shave the remainder deterministically: +1 on the highest-weight rows
    # that are below the cap
    order = np.argsort(ranks, kind="stable")
    for i in order:
        if deficit == 0:
            break
        if d[i] < n:
            d[i] += 1
            deficit -= 1
    assert int(d.sum()) == nnz
    return d


def _sample_rows(rng, degs: np.ndarray, row_ids: np.ndarray, n: int,
                 cumw: np.ndarray, logw: np.ndarray, heavy_frac: float = 1.0 / 16):
    """Columns for the given rows: returns (rows, cols) int64 arrays."""
    out_r, out_c = [], []
    heavy = degs > max(64, int(heavy_frac * n))
    # Efraimidis-Spirakis for heavy rows: top-d of log(U)/w
    for i, d in zip(row_ids[heavy], degs[heavy]):
        if d >= n:
            cols = np.arange(n, dtype=np.int64)
        else:
            # Efraimidis-Spirakis: the d largest U^(1/w), i.e. log(U)/w
            keys = np.log(rng.random(n)) / np.exp(logw)
            cols = np.sort(np.argpartition(-keys, d - 1)[:d]).astype(np.int64)
        out_r.append(np.full(cols.size, i, dtype=np.int64))
        out_c.append(cols)
    light_ids = row_ids[~heavy]
    light_d = degs[~heavy]
    pending_ids, pending_d = light_ids, light_d
    factor = 1.5
    total_w = cumw[-1]
    while pending_ids.size:
        draws = np.ceil(pending_d * factor).astype(np.int64) + 4
        rep_rows = np.repeat(np.arange(pending_ids.size, dtype=np.int64), draws)
        u = rng.random(rep_rows.size) * total_w
        cols = np.minimum(np.searchsorted(cumw, u, side="right"), n - 1).astype(np.int64)
        keys = rep_rows * n + cols
        uniq, first = np.unique(keys, return_index=True)
        urow = uniq // n
        # order distinct draws within each row by their first draw position
        o = np.lexsort((first, urow))
        urow, ucol = urow[o], (uniq % n)[o]
        counts = np.bincount(urow, minlength=pending_ids.size)
        starts = np.zeros(pending_ids.size + 1, dtype=np.int64)
        np.cumsum(counts, out=starts[1:])
        ok = counts >= pending_d
        # keep the first d distinct per satisfied row
        pos_in_row = np.arange(urow.size, dtype=np.int64) - starts[urow]
        keep = ok[urow] & (pos_in_row < pending_d[urow])
        out_r.append(pending_ids[urow[keep]])
        out_c.append(ucol[keep])
        pending_ids, pending_d = pending_ids[~ok], pending_d[~ok]
        factor *= 2.0
    if not out_r:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(out_r), np.concatenate(out_c)


def _values(rng, spec: ConfigSpec, rows, cols, m, n) -> np.ndarray:
    sd = spec.rank ** -0.25
    u = rng.normal(0.0, sd, (m, spec.rank))
    v = rng.normal(0.0, sd, (n, spec.rank))
    sig = np.empty(rows.size)
    ch = 1 << 22
    for s in range(0, rows.size, ch):
        e = min(rows.size, s + ch)
        sig[s:e] = np.einsum("ij,ij->i", u[rows[s:e]], v[cols[s:e]])
    noise = rng.normal(0.0, spec.noise_std, rows.size)
    x = spec.offset + spec.signal_std * sig + noise
    step, lo, hi = spec.quant
    return np.clip(np.rint(x / step) * step, lo, hi)


def generate(name: str, seed: int = 0, scale: float = 1.0):
    """Raw (user x item) COO instance for config ``name``.

    ``scale`` < 1 shrinks m, n and |Omega| proportionally (same distributions)
    for quick tests. Returns (m, n, rows, cols, vals) with int64/float64 arrays.
    """
    spec = CONFIGS[name]
    m = max(2, int(round(spec.m * scale)))
    n = max(2, int(round(spec.n * scale)))
    nnz = max(1, int(round(spec.nnz * scale * scale))) if scale != 1.0 else spec.nnz
    nnz = min(nnz, m * n)
    rng = _rng(seed)
    if spec.uniform:
        pos = rng.choice(m * n, size=nnz, replace=False)
        rows, cols = pos // n, pos % n
    else:
        d_min = min(spec.d_min, max(1, nnz // m))
        degs = zipf_degrees(rng, m, n, nnz, spec.s_row, d_min)
        crank = rng.permutation(n).astype(np.float64) + 1.0
        w = crank ** (-spec.s_col)
        cumw = np.cumsum(w)
        logw = np.log(w)
        rows_l, cols_l = [], []
        ids = np.arange(m, dtype=np.int64)
        budget = 1 << 24
        cs = np.cumsum(degs)
        start = 0
        while start < m:
            base = cs[start - 1] if start else 0
            stop = int(np.searchsorted(cs, base + budget, side="right"))
            stop = max(stop, start + 1)
            r, c = _sample_rows(rng, degs[start:stop], ids[start:stop], n, cumw, logw)
            rows_l.append(r)
            cols_l.append(c)
            start = stop
        rows, cols = np.concatenate(rows_l), np.concatenate(cols_l)
    vals = _values(rng, spec, rows, cols, m, n)
    return m, n, rows.astype(np.int64), cols.astype(np.int64), vals


def canonical(m, n, rows, cols, vals):
    """Apply the reference loader's m <= n rule (``mfg/data.py:229-236``)."""
    if m > n:
        return n, m, cols, rows, vals, True
    return m, n, rows, cols, vals, False


def sweep_factors(m: int, n: int, k: int, seed: int = 1, dtype=np.float64):
    """Fixed seeded W (m x k), H (n x k) with entries N(0, 1/sqrt(k)) (variance)."""
    rng = _rng(seed)
    sd = k ** -0.25
    w = rng.normal(0.0, sd, (m, k)).astype(dtype)
    h = rng.normal(0.0, sd, (n, k)).astype(dtype)
    return w, h
