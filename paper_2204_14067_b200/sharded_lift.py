"""Sharded lifting step (SURVEY.md §8(e) "Lifting"): the partial SVD of
Z = L R^T - alpha * G by warm-started block Krylov / power iterations,
tall-skinny QR, Rayleigh-Ritz and soft-thresholding, over an Omega that is
row-sharded (CSR) and column-sharded (CSC) across ranks.

Layout (as ``sharding.ShardedMF``): rank p owns the rows R_p = [r0, r1) of
the m side and the columns C_p = [c0, c1) of the n side; the low-rank
factors L (m x r) and R (n x r) are replicated. Blocks on the m side
("U blocks", m x q) are row-sharded: each rank holds its R_p rows. Blocks on
the n side ("V blocks", n x q) are sharded by C_p.

Exchanges per operation (mfg/operators.py:102-136, mfg/eigensolver.py:81-179,
mfg/kernels.py:76-135 sharded):
  apply(V)      Z V = L (R^T V) - alpha G V: R^T V is a summed r x q Gram;
                G V on the row shard needs all of V -> all-gather of V blocks.
  apply_t(U)    the transpose, with an all-gather of U blocks.
  Ritz          q^T S q and the residual norms are summed Grams; the p x p
                eigenproblem is solved redundantly on every rank.
  QR            CholeskyQR2 with summed Grams when well conditioned, else TSQR
                (local Householder QR, all-gather of the R factors, QR of the
                stacked R factors on every rank); rank screening on the
                |R_jj| of that R, identical bits on every rank.
  short-fat SVD of B^T Z: summed k x k Gram + redundant eigh, or TSQR of
                (B^T Z)^T when the Gram route is not accurate enough.

Every sum over ranks is an all-gather followed by an addition in rank order
(``ShardComm.sum_ordered``), so all ranks hold identical bits and take
identical host decisions (ranks, stopping, soft-threshold), whatever the
collective's algorithm. Local arithmetic on the shard is injected through
``ops`` (``DeviceOps`` on the GPU; the CPU tests inject the oracle).
"""

from __future__ import annotations

import numpy as np
import torch

from .eigensolver import EigConfig, EigResult, _FLOOR
from .kernels import GRAM_MAX_K, GRAM_MIN_RATIO, ORTH_TOL, soft_threshold
from .sharding import Comm

_CHOLQR_MIN_RATIO = 1e-5   # as kernels._cholqr2
_CHOLQR_MARGIN = 1e3


class ShardComm(Comm):
    """Comm plus an order-deterministic elementwise sum of tensors."""

    def sum_ordered(self, t: torch.Tensor) -> torch.Tensor:
        """Sum of ``t`` over ranks, added in rank order (identical bits on
        every rank)."""
        if self.world == 1:
            return t
        out = self.gather_flat(t)
        s = out[0].clone()
        for p in range(1, self.world):
            s += out[p]
        return s

    def all_gather_list(self, t: torch.Tensor) -> list:
        if self.world == 1:
            return [t]
        return list(self.gather_flat(t).unbind(0))


class ShardedOperator:
    """Z = L R^T - alpha * G on the sharded Omega (mfg/operators.py:84-152).

    ``mf`` is the rank's ``sharding.ShardedMF`` (shard, ops, handles);
    ``left`` (m x r) and ``right`` (n x r) are the replicated factors;
    ``g_row`` / ``g_col`` are G's values on the row / column shard in the
    ops' handle order (e.g. 2 * ops.residual(...))."""

    def __init__(self, mf, comm: ShardComm, left: torch.Tensor, right: torch.Tensor,
                 g_row, g_col, alpha: float):
        self.mf = mf
        self.comm = comm
        self.s = mf.s
        self.ops = mf.ops
        self.alpha = float(alpha)
        r0, r1 = self.s.row_block
        c0, c1 = self.s.col_block
        self._l_loc = left[r0:r1].double()
        self._r_loc = right[c0:c1].double()
        self.g_row = g_row
        self.g_col = g_col

    @property
    def shape(self) -> tuple[int, int]:
        return self.s.m, self.s.n

    def apply(self, v_loc: torch.Tensor) -> torch.Tensor:
        """(Z V) rows R_p from the V block rows C_p."""
        rtv = self.comm.sum_ordered(self._r_loc.T @ v_loc)
        out = self._l_loc @ rtv
        if self.alpha != 0.0:
            v_full = self.comm.allgather_blocks(v_loc, self.s.col_blocks)
            out = out - self.alpha * self.ops.spmm(self.mf.hr, self.g_row, v_full)
        return out

    def apply_t(self, u_loc: torch.Tensor) -> torch.Tensor:
        """(Z^T U) rows C_p from the U block rows R_p."""
        ltu = self.comm.sum_ordered(self._l_loc.T @ u_loc)
        out = self._r_loc @ ltu
        if self.alpha != 0.0:
            u_full = self.comm.allgather_blocks(u_loc, self.s.row_blocks)
            out = out - self.alpha * self.ops.spmm(self.mf.hc, self.g_col, u_full)
        return out

    def apply_gram(self, u_loc: torch.Tensor) -> torch.Tensor:
        return self.apply(self.apply_t(u_loc))


# ---------------------------------------------------------------------------
# tall-skinny QR on row-sharded blocks


def _frob(comm: ShardComm, b_loc: torch.Tensor) -> float:
    return float(torch.sqrt(comm.sum_ordered(torch.sum(b_loc * b_loc).reshape(1)))[0])


def _tsqr(comm: ShardComm, b_loc: torch.Tensor):
    """Householder TSQR: (Q rows of this rank, R) with B = Q R; R identical
    on every rank."""
    p = b_loc.shape[1]
    q_l, r_l = torch.linalg.qr(b_loc, mode="reduced")     # r_l: min(m_p, p) x p
    rows = r_l.shape[0]
    if comm.world == 1 and rows == p:
        return q_l, r_l                                     # one block: its QR is the TSQR
    r_pad = torch.zeros((p, p), dtype=b_loc.dtype, device=b_loc.device)
    r_pad[:rows] = r_l
    stack = torch.cat(comm.all_gather_list(r_pad), dim=0)   # (world * p) x p
    q_s, r = torch.linalg.qr(stack, mode="reduced")
    blk = q_s[comm.rank * p: comm.rank * p + rows]
    return q_l @ blk, r


def _cholqr2(comm: ShardComm, b_loc: torch.Tensor, scale: float, tol: float):
    """CholeskyQR2 with summed Grams on the column-equilibrated block, or None
    when it cannot certify the screening decision (as kernels._cholqr2)."""
    cn = torch.sqrt(comm.sum_ordered(torch.sum(b_loc * b_loc, dim=0)))
    if bool((cn == 0).any()):
        return None
    bt = b_loc / cn
    r1, info = torch.linalg.cholesky_ex(comm.sum_ordered(bt.T @ bt), upper=True)
    d = torch.abs(torch.diagonal(r1))
    stats = torch.stack([info.double(), d.min(), d.max(), (d * cn).min()]).cpu().numpy()
    if (stats[0] != 0 or not (stats[1] >= _CHOLQR_MIN_RATIO * stats[2])
            or not (stats[3] > _CHOLQR_MARGIN * tol * scale)):
        return None
    q1 = torch.linalg.solve_triangular(r1, bt, upper=True, left=False)
    r2, info2 = torch.linalg.cholesky_ex(comm.sum_ordered(q1.T @ q1), upper=True)
    if int(info2.item()) != 0:
        return None
    return torch.linalg.solve_triangular(r2, q1, upper=True, left=False)


def orthonormalize(comm: ShardComm, b_loc: torch.Tensor, m: int, tol: float = ORTH_TOL,
                   fast: list | None = None):
    """Sharded mfg/kernels.py:76-105: orthonormal basis of range(B) (this
    rank's rows of the m x p block) and its rank, screening |R_jj| <= tol *
    ||B||_F on the R of a TSQR and repeating until stable; CholeskyQR2 fast
    path as in kernels.orthonormalize."""
    m_loc, p = b_loc.shape
    if p == 0:
        return b_loc.new_zeros((m_loc, 0)), 0
    scale = _frob(comm, b_loc)
    if scale == 0.0:
        return b_loc.new_zeros((m_loc, 0)), 0
    # ``fast``: a caller-held switch for the CholeskyQR2 path, cleared by its
    # first failure (as kernels.orthonormalize: the LM-Krylov candidate
    # blocks stay ill conditioned once they fail)
    if 8 <= p <= m and (fast is None or fast[0]):
        q = _cholqr2(comm, b_loc, scale, tol)
        if q is not None:
            return q, p
        if fast is not None:
            fast[0] = False
    cols = b_loc
    while True:
        q, r = _tsqr(comm, cols)
        diag = torch.abs(torch.diagonal(r)).cpu().numpy()
        keep = np.zeros(cols.shape[1], dtype=bool)
        keep[: diag.size] = diag > tol * scale
        if keep.all():
            return q.contiguous(), int(cols.shape[1])
        idx = torch.as_tensor(np.flatnonzero(keep), device=b_loc.device)
        cols = cols.index_select(1, idx)
        if cols.shape[1] == 0:
            return b_loc.new_zeros((m_loc, 0)), 0


# ---------------------------------------------------------------------------
# eigensolvers (mfg/eigensolver.py:53-193 sharded)


def _complete_basis(comm: ShardComm, q_loc: torch.Tensor, k: int, r0: int, m: int) -> torch.Tensor:
    """Pad with deterministic e_j columns (53-71); row j lives on the rank
    whose block holds it."""
    m_loc = q_loc.shape[0]
    cols = [q_loc]
    width = q_loc.shape[1]
    j = 0
    while width < k and j < m:
        e = torch.zeros(m_loc, dtype=torch.float64, device=q_loc.device)
        if r0 <= j < r0 + m_loc:
            e[j - r0] = 1.0
        for block in cols:
            e = e - block @ comm.sum_ordered(block.T @ e)
        nrm = float(torch.sqrt(comm.sum_ordered(torch.sum(e * e).reshape(1)))[0])
        if nrm > 1e-8:
            cols.append((e / nrm)[:, None])
            width += 1
        j += 1
    if width < k:
        raise ValueError(f"cannot build a rank-{k} basis in dimension {m}")
    return torch.cat(cols, dim=1) if len(cols) > 1 else q_loc


def _ritz(op: ShardedOperator, q_loc: torch.Tensor):
    """Rayleigh-Ritz on span(q): (vectors, values[host], S vectors, residuals[host])."""
    comm = op.comm
    sq = op.apply_gram(q_loc)
    t = comm.sum_ordered(q_loc.T @ sq)
    t = 0.5 * (t + t.T)
    w, p = torch.linalg.eigh(t)
    w = torch.clamp(torch.flip(w, (0,)), min=0.0)
    p = torch.flip(p, (1,))
    vecs = q_loc @ p
    svecs = sq @ p
    d = svecs - vecs * w
    res = torch.sqrt(comm.sum_ordered(torch.sum(d * d, dim=0)))
    return vecs, w.cpu().numpy(), svecs, res.cpu().numpy()


def _prepare(op: ShardedOperator, r0_loc: torch.Tensor, k: int) -> torch.Tensor:
    q, rank = orthonormalize(op.comm, r0_loc, op.shape[0])
    if rank < k:
        q = _complete_basis(op.comm, q, k, op.s.row_block[0], op.s.m)
    return q


def lmkrylov_topk(op: ShardedOperator, r0_loc: torch.Tensor, cfg: EigConfig) -> EigResult:
    """Limited-memory block Krylov (mfg/eigensolver.py:130-179) on row-sharded
    blocks; ``basis`` holds this rank's rows."""
    comm = op.comm
    m = op.shape[0]
    k = r0_loc.shape[1]
    if k > m:
        raise ValueError(f"requested k={k} exceeds dimension m={m}")
    if k == 0:
        return EigResult(r0_loc.new_zeros((r0_loc.shape[0], 0)), np.zeros(0), np.zeros(0), 0, True)
    u = _prepare(op, r0_loc.double(), k)
    hist: list = []
    history: list = []
    basis, w, res = u, np.zeros(k), np.full(k, np.inf)
    converged = False
    it = 0
    fast_cand, fast_comp = [True], [True]   # CholeskyQR2 fast path per call site
    for it in range(1, cfg.max_iters + 1):
        p_blk = op.apply_gram(u)
        cand = p_blk if cfg.memory == 0 else torch.cat([p_blk, u] + hist, dim=1)
        q, rank = orthonormalize(comm, cand, m, fast=fast_cand)
        if rank < k:
            q = _complete_basis(comm, q, k, op.s.row_block[0], m)
        ritz_vecs, w_all, _, res_all = _ritz(op, q)
        basis = ritz_vecs[:, :k]
        w = w_all[:k]
        res = res_all[:k]
        history.append(w.copy())
        rmax = float(res.max())
        done = rmax <= cfg.residual_tol
        stalled = not done and rmax <= _FLOOR * max(w[0], 1e-300)
        if cfg.memory >= 2 and not (done or stalled):
            comp = u - basis @ comm.sum_ordered(basis.T @ u)
            cq, crank = orthonormalize(comm, comp, m, fast=fast_comp)
            if crank:
                hist = [cq] + hist
            hist = hist[: cfg.memory - 1]
        u = basis
        if done:
            converged = True
            break
        if stalled:
            break
    return EigResult(basis, w, res, it, converged, history)


def power_topk(op: ShardedOperator, r0_loc: torch.Tensor, cfg: EigConfig) -> EigResult:
    """Block power iteration with per-sweep Ritz extraction (95-127), sharded."""
    comm = op.comm
    m = op.shape[0]
    k = r0_loc.shape[1]
    if k > m:
        raise ValueError(f"requested k={k} exceeds dimension m={m}")
    if k == 0:
        return EigResult(r0_loc.new_zeros((r0_loc.shape[0], 0)), np.zeros(0), np.zeros(0), 0, True)
    u = _prepare(op, r0_loc.double(), k)
    y = op.apply_gram(u)
    history: list = []
    basis, w, res = u, np.zeros(k), np.full(k, np.inf)
    converged = False
    it = 0
    for it in range(1, cfg.max_iters + 1):
        q, rank = orthonormalize(comm, y, m)
        if rank < k:
            q = _complete_basis(comm, q, k, op.s.row_block[0], m)
        basis, w, svecs, res = _ritz(op, q)
        history.append(w.copy())
        rmax = float(res.max())
        if rmax <= cfg.residual_tol:
            converged = True
            break
        if rmax <= _FLOOR * max(w[0], 1e-300):
            break
        y = svecs
    return EigResult(basis, w, res, it, converged, history)


def solve_topk(op: ShardedOperator, r0_loc: torch.Tensor, cfg: EigConfig) -> EigResult:
    if cfg.method == "power":
        return power_topk(op, r0_loc, cfg)
    return lmkrylov_topk(op, r0_loc, cfg)


# ---------------------------------------------------------------------------
# projection, short-fat SVD and soft-threshold (mfg/proxlift.py:356-372)


def exact_svd_short_fat(comm: ShardComm, mt_loc: torch.Tensor, c0: int = 0):
    """SVD of the short-fat M (k x n) given M^T's column-shard rows
    (mfg/kernels.py:108-135): returns (u k x k, sigma[host], V rows of C_p).

    Gram route (k <= 64, Gram spectrum within 1e-6) from the summed M M^T;
    otherwise TSQR of M^T and an SVD of its k x k R factor (redundant)."""
    k = mt_loc.shape[1]
    if k == 0:
        return mt_loc.new_zeros((0, 0)), np.zeros(0), mt_loc.new_zeros((mt_loc.shape[0], 0))
    scale = _frob(comm, mt_loc)
    if scale == 0.0:   # identity factors, zero values (as kernels.exact_svd_short_fat)
        eye_rows = torch.zeros_like(mt_loc)
        j = torch.arange(mt_loc.shape[0], device=mt_loc.device) + c0
        sel = j < k
        eye_rows[sel, j[sel]] = 1.0
        return torch.eye(k, dtype=mt_loc.dtype, device=mt_loc.device), np.zeros(k), eye_rows
    if k <= GRAM_MAX_K:
        gram = comm.sum_ordered(mt_loc.T @ mt_loc)
        w, u_small = torch.linalg.eigh(gram)
        w = torch.clamp(torch.flip(w, (0,)), min=0.0)
        u_small = torch.flip(u_small, (1,))
        wh = w.cpu().numpy()
        if wh[-1] > GRAM_MIN_RATIO * wh[0]:
            sigma = torch.sqrt(w)
            return u_small, np.sqrt(wh), mt_loc @ (u_small / sigma)
    # M^T = Q R (TSQR over the column shards); M = R^T Q^T; R^T = U S Vr^T
    q_loc, r = _tsqr(comm, mt_loc)
    u_r, s, vt = torch.linalg.svd(r.T, full_matrices=False)
    return u_r, s.cpu().numpy(), q_loc @ vt.T


def partial_svd_step(op: ShardedOperator, r0_loc: torch.Tensor, cfg: EigConfig, beta: float):
    """The lifting step's spectral part, sharded: top-k eigenbasis B of Z Z^T
    (warm start r0), the projection B^T Z, its exact short-fat SVD and the
    soft-threshold at beta. Returns (U rows of R_p, sigma[host], V rows of
    C_p, eig result, largest truncated value)."""
    eig = solve_topk(op, r0_loc, cfg)
    basis = eig.basis
    mt_loc = op.apply_t(basis)                       # (B^T Z)^T rows of C_p
    u_s, sig_hat, v_loc = exact_svd_short_fat(op.comm, mt_loc, op.s.col_block[0])
    sigma, kept, largest = soft_threshold(sig_hat, beta)
    idx = torch.as_tensor(kept, device=basis.device, dtype=torch.long)
    u_loc = basis @ u_s.index_select(1, idx)
    return u_loc, sigma, v_loc.index_select(1, idx), eig, largest
