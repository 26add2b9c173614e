"""CPU ORACLE for the Omega-sweep hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy/scipy, the reference's (mfglobal 0.1.0,
/root/reference/pkg/src/mfglobal) arithmetic for the functions on the hot
path. It is the checker for the CUDA path and the CPU baseline leg of
``bench.py``; it is NEVER imported by the product package
``paper_2204_14067_b200`` (which fails loudly without its CUDA library).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline
and ``--impl reference``) may import it.

Pinning: every function here is checked in ``tests/test_oracle_golden.py``
against fixtures produced by running the reference itself in the build
container (``tests/golden/make_golden.py``, which imports
``/root/reference/pkg/src``). The arithmetic of the reference lives in
numpy 2.3.5 / scipy 1.18.1 (OpenBLAS 0.3.30); the reference pins only lower
bounds (``pkg/pyproject.toml:10-14``), so these installed versions are the
effective pin.

Citations are ``mfg/<file>:<line>`` with ``mfg = pkg/src/mfglobal``.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

EVAL_CHUNK = 1 << 18       # mfg/data.py:29
PAIR_CHUNK = 1 << 25       # mfg/mfsolver.py:18
ORTH_TOL = 1e-10           # mfg/kernels.py:14
SIGMA_FLOOR = 1e-12        # mfg/kernels.py:17
GRAM_MAX_K = 64            # mfg/kernels.py:19
GRAM_MIN_RATIO = 1e-6      # mfg/kernels.py:22


class OracleDatasetError(ValueError):
    pass


class Omega:
    """Sorted Omega with CSR + CSC views (mfg/data.py:46-119)."""

    def __init__(self, m, n, rows, cols, vals, indptr):
        self.m, self.n = m, n
        self.rows, self.cols, self.vals, self.indptr = rows, cols, vals, indptr
        self.a_csr = sp.csr_matrix((vals, cols, indptr), shape=(m, n))
        # mfg/data.py:113-115: CSC view as the transpose converted to CSR
        self.a_csr_t = self.a_csr.T.tocsr()
        ones = np.ones_like(vals)
        self.pattern_csr = sp.csr_matrix((ones, cols, indptr), shape=(m, n))
        self.pattern_csr_t = self.pattern_csr.T.tocsr()

    @property
    def size(self):
        return int(self.vals.size)

    def csc_perm(self) -> np.ndarray:
        """CSC position -> CSR position, i.e. the stable argsort of cols."""
        return np.argsort(self.cols, kind="stable")


def from_coo(m, n, rows, cols, vals) -> Omega:
    """mfg/data.py:70-102 (range checks, lexsort, duplicate rejection, indptr)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size != cols.size or rows.size != vals.size:
        raise OracleDatasetError("index/value arrays disagree in length")
    if rows.size:
        if rows.min() < 0 or rows.max() >= m:
            raise OracleDatasetError("row index out of range")
        if cols.min() < 0 or cols.max() >= n:
            raise OracleDatasetError("column index out of range")
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size > 1:
        dup = (np.diff(rows) == 0) & (np.diff(cols) == 0)
        if dup.any():
            i = int(np.flatnonzero(dup)[0])
            raise OracleDatasetError(
                f"duplicate entry at ({rows[i]}, {cols[i]}); refusing to aggregate")
    indptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=m), out=indptr[1:])
    return Omega(m, n, rows, cols, vals, indptr)


def pair_values(left, right, rows, cols):
    """mfg/data.py:253-263: chunked per-entry row inner products (SDDMM core)."""
    out = np.empty(rows.size)
    for s in range(0, rows.size, EVAL_CHUNK):
        e = min(s + EVAL_CHUNK, rows.size)
        out[s:e] = np.einsum("ij,ij->i", left[rows[s:e]], right[cols[s:e]], optimize=False)
    return out


def residual(om: Omega, w, h):
    """mfg/data.py:272-280: r = (W H^T)_Omega - A."""
    return pair_values(w, h, om.rows, om.cols) - om.vals


def triplet_values(u, sigma, v, rows, cols):
    """mfg/data.py:266-269."""
    if sigma.size == 0:
        return np.zeros(rows.size)
    return pair_values(u * sigma, v, rows, cols)


def loss_quad(r):
    """mfg/data.py:291-293 (no 1/2)."""
    return float(r @ r)


def csr_of(om: Omega, vals):
    return sp.csr_matrix((vals, om.cols, om.indptr), shape=(om.m, om.n))


def sweep(om: Omega, w, h):
    """The metric's unit of work: SDDMM, R.H (CSR), R^T.W
    (CSC), sum r^2, ||W||^2, ||H||^2 — each via the reference's own calls
    (mfg/data.py:279 / mfg/data.py:153-158 / mfg/operators.py:108,117)."""
    r = residual(om, w, h)
    rc = csr_of(om, r)
    rh = rc @ h
    rtw = rc.T.tocsr() @ w
    return r, rh, rtw, float(r @ r), float(np.sum(w * w)), float(np.sum(h * h))


def spmm_csr(om: Omega, vals, block):
    """grad.csr @ block (mfg/operators.py:108)."""
    return csr_of(om, vals) @ block


def spmm_csc(om: Omega, vals, block):
    """grad.csr_t @ block (mfg/operators.py:117,135)."""
    return csr_of(om, vals).T.tocsr() @ block


def half_sweep(a_csr, pattern_csr, other, lam):
    """mfg/mfsolver.py:53-75: exact row minimisers via pair-product SpMM and
    a batched LU solve."""
    m = a_csr.shape[0]
    k = other.shape[1]
    iu, ju = np.triu_indices(k)
    npairs = iu.size
    g_tri = np.empty((m, npairs))
    step = max(1, PAIR_CHUNK // max(1, other.shape[0]))
    for s in range(0, npairs, step):
        e = min(npairs, s + step)
        g_tri[:, s:e] = pattern_csr @ (other[:, iu[s:e]] * other[:, ju[s:e]])
    normal = np.empty((m, k, k))
    normal[:, iu, ju] = g_tri
    normal[:, ju, iu] = g_tri
    normal *= 2.0
    normal[:, np.arange(k), np.arange(k)] += lam
    rhs = 2.0 * (a_csr @ other)
    return np.linalg.solve(normal, rhs[:, :, None])[:, :, 0]


def bcd_epoch(om: Omega, w, h, lam):
    """mfg/mfsolver.py:78-93."""
    if lam <= 0:
        raise ValueError("lam must be positive")
    if w.shape[1] == 0:
        return w, h
    w_new = half_sweep(om.a_csr, om.pattern_csr, h, lam)
    h_new = half_sweep(om.a_csr_t, om.pattern_csr_t, w_new, lam)
    return w_new, h_new


def mf_objective(om: Omega, w, h, lam):
    """mfg/mfsolver.py:48-50 with FactorPair.frob_sq (mfg/operators.py:53-55)."""
    r = residual(om, w, h)
    return float(r @ r) + 0.5 * lam * float(np.sum(w * w) + np.sum(h * h))


def shifted_apply(om, w, h, gvals, alpha, block):
    """mfg/operators.py:102-109."""
    out = w @ (h.T @ block)
    if alpha != 0.0:
        out -= alpha * spmm_csr(om, gvals, block)
    return out


def shifted_apply_t(om, w, h, gvals, alpha, block):
    """mfg/operators.py:111-118."""
    out = h @ (w.T @ block)
    if alpha != 0.0:
        out -= alpha * spmm_csc(om, gvals, block)
    return out


def shifted_project_rows(om, w, h, gvals, alpha, basis):
    """mfg/operators.py:124-136 (without the capacity cap)."""
    out = (basis.T @ w) @ h.T
    if alpha != 0.0:
        out -= alpha * spmm_csc(om, gvals, basis).T
    return out


def shifted_frob_sq(om, w, h, gvals, alpha):
    """mfg/operators.py:142-152."""
    ww = float(np.sum((w.T @ w) * (h.T @ h)))
    gg = float(gvals @ gvals)
    xg = float(gvals @ pair_values(w, h, om.rows, om.cols))
    return ww - 2.0 * alpha * xg + alpha ** 2 * gg


def orthonormalize(b, tol=ORTH_TOL):
    """mfg/kernels.py:76-105 (Householder QR + repeated column screening)."""
    b = np.asarray(b, dtype=np.float64)
    m = b.shape[0]
    if b.shape[1] == 0:
        return np.zeros((m, 0)), 0
    scale = np.linalg.norm(b)
    if scale == 0.0:
        return np.zeros((m, 0)), 0
    cols = b
    while True:
        q, r = np.linalg.qr(cols)
        diag = np.abs(np.diag(r))
        keep = np.zeros(cols.shape[1], dtype=bool)
        keep[: diag.size] = diag > tol * scale
        if keep.all():
            return q[:, : cols.shape[1]], cols.shape[1]
        cols = cols[:, keep]
        if cols.shape[1] == 0:
            return np.zeros((m, 0)), 0


def soft_threshold(sigma_hat, beta):
    """mfg/kernels.py:138-163."""
    sigma_hat = np.asarray(sigma_hat, dtype=np.float64)
    if sigma_hat.size == 0:
        return np.zeros(0), np.zeros(0, dtype=np.intp), None
    floor = SIGMA_FLOOR * sigma_hat[0]
    alive = (sigma_hat - beta > 0.0) & (sigma_hat > floor)
    kept = np.flatnonzero(alive)
    sigma = sigma_hat[kept] - beta
    r = kept.size
    largest = float(sigma_hat[r]) if r < sigma_hat.size else None
    return sigma, kept, largest


def exact_svd_short_fat(mat):
    """mfg/kernels.py:108-135."""
    mat = np.asarray(mat, dtype=np.float64)
    k, n = mat.shape
    if k == 0:
        return np.zeros((0, 0)), np.zeros(0), np.zeros((n, 0))
    scale = np.linalg.norm(mat)
    if scale == 0.0:
        return np.eye(k), np.zeros(k), np.eye(n, k)
    if k <= GRAM_MAX_K:
        gram = mat @ mat.T
        wv, u_small = np.linalg.eigh(gram)
        wv = np.clip(wv[::-1], 0.0, None)
        u_small = u_small[:, ::-1]
        if wv[-1] > GRAM_MIN_RATIO * wv[0]:
            sigma = np.sqrt(wv)
            v = mat.T @ (u_small / sigma)
            return u_small, sigma, v
    u, sigma, vt = np.linalg.svd(mat, full_matrices=False)
    return u, sigma, vt.T
