"""Row/column sharding of Omega across ranks.

One process per GPU. Rank p owns
  * a row block R_p = [r0, r1) of the CSR side (contiguous rows with ~equal
    nnz, so Zipf-heavy rows do not unbalance ranks), and
  * a column block C_p = [c0, c1) of the CSC side (equal-nnz columns),
and keeps full replicas of W (m x k) and H (n x k).

  sweep       : R.H rows of R_p from the row shard, R^T.W rows of C_p from the
                column shard; sum r^2 from the row shard only. No data-path
                exchange; the fp64 partial sums are all-gathered and added in
                rank order, so every rank holds the same bits.
  BCD epoch   : W rows of R_p from the row shard -> all-gather W blocks; then
                H rows of C_p from the column shard with the new W ->
                all-gather H blocks (mfg/mfsolver.py:78-93 sharded).
  objective   : sum r^2 (ordered all-gather) + lam/2 (||W||^2 + ||H||^2) from
                the replicas.

Local arithmetic is injected (``ops``): ``DeviceOps`` runs libmfg_b200 on the
rank's GPU (NCCL collectives); the CPU tests inject the oracle under gloo.
Per-row results do not depend on the sharding (each row's reduction order is
the same as single-process), which the tests check bitwise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def balanced_blocks(counts: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Contiguous blocks of indices with ~equal sum(counts) (equal nnz)."""
    counts = np.asarray(counts, dtype=np.int64)
    n = counts.size
    csum = np.concatenate([[0], np.cumsum(counts)])
    total = int(csum[-1])
    bounds = [0]
    for p in range(1, parts):
        target = total * p / parts
        b = int(np.searchsorted(csum, target, side="left"))
        b = min(max(b, bounds[-1]), n)
        bounds.append(b)
    bounds.append(n)
    return [(bounds[p], bounds[p + 1]) for p in range(parts)]


@dataclass
class Shard:
    """The entries a rank owns, in both orientations (local COO)."""

    rank: int
    world: int
    m: int
    n: int
    row_block: tuple[int, int]
    col_block: tuple[int, int]
    row_blocks: list
    col_blocks: list
    # row shard: local row id (i - r0), global column id, value
    r_rows: np.ndarray
    r_cols: np.ndarray
    r_vals: np.ndarray
    # column shard, transposed: local column id (j - c0) as the row, global row id
    c_rows: np.ndarray
    c_cols: np.ndarray
    c_vals: np.ndarray


def make_shard(m: int, n: int, rows, cols, vals, rank: int, world: int) -> Shard:
    """Cut a global COO Omega into the rank's row and column shards."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    rb = balanced_blocks(np.bincount(rows, minlength=m), world)
    cb = balanced_blocks(np.bincount(cols, minlength=n), world)
    r0, r1 = rb[rank]
    c0, c1 = cb[rank]
    rs = (rows >= r0) & (rows < r1)
    cs = (cols >= c0) & (cols < c1)
    return Shard(rank, world, m, n, (r0, r1), (c0, c1), rb, cb,
                 rows[rs] - r0, cols[rs], vals[rs],
                 cols[cs] - c0, rows[cs], vals[cs])


class Comm:
    """torch.distributed wrapper: padded all-gather of row blocks and
    order-deterministic fp64 sums. Every collective is one all-gather into a
    single tensor (``ncoll`` counts them); scalar sums are batched and read
    back with one device-to-host copy."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.ncoll = 0

    def gather_flat(self, t: torch.Tensor) -> torch.Tensor:
        """All-gather of equal-shape tensors into one (world, *t.shape) tensor."""
        t = t.contiguous()
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.ncoll += 1
        try:
            dist.all_gather_into_tensor(out, t, group=self.group)
        except (RuntimeError, NotImplementedError, AttributeError):
            parts = list(out.unbind(0))
            dist.all_gather(parts, t, group=self.group)
        return out

    def allgather_blocks(self, local: torch.Tensor, blocks: list) -> torch.Tensor:
        """Concatenate every rank's row block (sizes from ``blocks``)."""
        if self.world == 1:
            return local
        width = local.shape[1]
        maxr = max(b - a for a, b in blocks)
        pad = torch.zeros((maxr, width), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        out = self.gather_flat(pad)
        return torch.cat([out[p, : b - a] for p, (a, b) in enumerate(blocks)], dim=0)

    def ordered_sums(self, xs, device) -> list:
        """Rank-ordered sums of a batch of fp64 scalars (one all-gather, one
        8*world*len(xs)-byte read-back; identical bits on every rank)."""
        xs = [float(x) for x in xs]
        if self.world == 1:
            return xs
        t = torch.tensor(xs, dtype=torch.float64, device=device)
        g = self.gather_flat(t).cpu().numpy()
        out = []
        for j in range(len(xs)):
            s = 0.0
            for p in range(self.world):
                s += float(g[p, j])
            out.append(s)
        return out

    def ordered_sum(self, x: float, device) -> float:
        """Sum of one fp64 scalar per rank, added in rank order (identical
        bits on every rank, independent of the collective's algorithm)."""
        return self.ordered_sums([x], device)[0]


class ShardedMF:
    """MF-phase building blocks over a sharded Omega.

    ``ops`` provides the local arithmetic on one orientation's shard:
      ops.prepare(n_local_rows, n_cols, rows, cols, vals) -> handle
      ops.sweep(handle, self_rows, other_full) -> (acc_rows, sumsq)
          acc_rows[i] = sum_j r_ij other_j with r_ij = self_i . other_j - a_ij
      ops.half_sweep(handle, other_full, lam) -> new self rows
      ops.residual(handle, self_rows, other_full) -> r values (handle order)
      ops.spmm(handle, vals, block_full) -> rows sum_j vals_ij block_j
      ops.sddmm_sums(handle, left_rows, right_full, scale, g, with_a) -> fp64
          (sum r^2, sum g (r - g/2), sum g p)
    (the last three serve the sharded lifting step and driver,
    ``sharded_lift`` / ``sharded_solver``).
    """

    def __init__(self, shard: Shard, ops, comm: Comm, device):
        self.s = shard
        self.ops = ops
        self.comm = comm
        self.device = device
        r0, r1 = shard.row_block
        c0, c1 = shard.col_block
        self.hr = ops.prepare(r1 - r0, shard.n, shard.r_rows, shard.r_cols, shard.r_vals)
        self.hc = ops.prepare(c1 - c0, shard.m, shard.c_rows, shard.c_cols, shard.c_vals)

    def sweep(self, w: torch.Tensor, h: torch.Tensor):
        """(R.H full, R^T.W full, sum r^2) with one all-gather per orientation."""
        r0, r1 = self.s.row_block
        c0, c1 = self.s.col_block
        rh, sq = self.ops.sweep(self.hr, w[r0:r1], h)
        rtw, _ = self.ops.sweep(self.hc, h[c0:c1], w)
        rh_full = self.comm.allgather_blocks(rh, self.s.row_blocks)
        rtw_full = self.comm.allgather_blocks(rtw, self.s.col_blocks)
        return rh_full, rtw_full, self.comm.ordered_sum(sq, self.device)

    def loss(self, w: torch.Tensor, h: torch.Tensor) -> float:
        r0, r1 = self.s.row_block
        _, sq = self.ops.sweep(self.hr, w[r0:r1], h)
        return self.comm.ordered_sum(sq, self.device)

    def objective(self, w: torch.Tensor, h: torch.Tensor, lam: float) -> float:
        """mf_objective (mfg/mfsolver.py:48-50) on the sharded Omega."""
        frob = float(torch.sum(w.double() * w.double()) + torch.sum(h.double() * h.double()))
        return self.loss(w, h) + 0.5 * lam * frob

    def bcd_epoch(self, w: torch.Tensor, h: torch.Tensor, lam: float):
        """mfg/mfsolver.py:78-93 with an all-gather after each half-sweep."""
        if lam <= 0:
            raise ValueError("lam must be positive")
        w_loc = self.ops.half_sweep(self.hr, h, lam)
        w_new = self.comm.allgather_blocks(w_loc, self.s.row_blocks)
        h_loc = self.ops.half_sweep(self.hc, w_new, lam)
        h_new = self.comm.allgather_blocks(h_loc, self.s.col_blocks)
        if hasattr(self.ops, "check"):
            self.ops.check()
        return w_new, h_new


class DeviceOps:
    """Local arithmetic on the rank's GPU through libmfg_b200."""

    def __init__(self, dtype=torch.float64):
        self.dtype = dtype

    def prepare(self, nrows, ncols, rows, cols, vals):
        from .data import ObservationSet

        return ObservationSet.from_coo(nrows, ncols, rows, cols, vals, dtype=self.dtype)

    def sweep(self, obs, self_rows, other_full):
        from .mfsolver import SweepPlan

        k = int(self_rows.shape[1])
        plan = SweepPlan(obs, k, want_r=False, want_rh=True, want_rtw=False,
                         compute_f64=self.dtype == torch.float32)
        plan.run(self_rows.to(self.dtype).contiguous(), other_full.to(self.dtype).contiguous())
        return plan.RH, float(plan.sums[0].item())

    def half_sweep(self, obs, other_full, lam):
        from .mfsolver import _half_sweep

        return _half_sweep(obs, False, other_full, lam)

    def check(self):
        """NumericalError if a half-sweep since the last check was non-SPD."""
        from .mfsolver import check_bcd_status

        check_bcd_status()

    def residual(self, obs, self_rows, other_full):
        """r on the shard (fp64, the handle's CSR order): self_i . other_j - a_ij.
        Factors stored in fp32 convert to fp64 exactly; fp64 blocks (SVD
        triplets of the lifting step) are used at full precision."""
        from .data import sddmm

        vals, _ = sddmm(obs, self_rows.double(), other_full.double(), dtype=torch.float64)
        return vals

    def sddmm_sums(self, obs, left_rows, right_full, scale, g_vals, with_a=True):
        """fp64 (sum r^2, sum g (r - g/2), sum g p) with p_ij = left_i diag(scale)
        right_j and r = p - a (r = p without a) over the shard (mfg_sddmm)."""
        from .data import sddmm

        sc = None if scale is None else torch.as_tensor(scale).double().cpu().numpy()
        _, sums = sddmm(obs, left_rows.double(), right_full.double(), scale=sc, a=with_a,
                        g=g_vals.double(), want_out=False, dtype=torch.float64)
        return float(sums[0]), float(sums[1]), float(sums[2])

    def spmm(self, obs, vals, block_full):
        """sum_j vals_ij block_j for the shard's rows (fp64, libmfg_b200 mfg_spmm)."""
        from .data import SparseResidual
        from .operators import spmm

        out = torch.zeros((obs.m, block_full.shape[1]), dtype=torch.float64, device=block_full.device)
        return spmm(SparseResidual(obs.m, obs.n, obs, vals), block_full.double(), False, 1.0, 0.0, out)


class ShardSweepPlan:
    """One rank's part of the Omega sweep with the grouped kernel
    (``mfg_sweep_sharded``): R over the row shard, the rows R_p of R.H, the
    rows C_p of R^T.W (final: no exchange on the data path) and the local
    fp64 sums [sum r^2 over the row shard, ||W_{R_p}||^2, ||H_{C_p}||^2].

    ``obs_rows`` / ``obs_cols`` are the ObservationSets of the rank's row
    shard (local rows x n) and transposed column shard (local columns x m),
    as ``DeviceOps.prepare`` builds them from a ``Shard``. Factors passed to
    ``run`` are the full replicas in the grouped kernel's layout (``ld``)."""

    def __init__(self, shard: Shard, obs_rows, obs_cols, k: int, *, want_r: bool = True,
                 out_scale: float = 1.0):
        from . import _lib
        from .mfsolver import grouped_ld

        self.s, self.k = shard, int(k)
        self.obs_r, self.obs_c = obs_rows, obs_cols
        dt = obs_rows.dtype
        if obs_cols.dtype != dt:
            raise ValueError("row and column shards must share a dtype")
        self.dt = dt
        dev = obs_rows.dev.device
        self.ld = grouped_ld(self.k, dt) or self.k
        self.out_scale = float(out_scale)
        r0, r1 = shard.row_block
        c0, c1 = shard.col_block
        self.R = torch.empty(obs_rows.size, dtype=dt, device=dev) if want_r else None
        self.RH = torch.zeros((r1 - r0, self.k), dtype=dt, device=dev)
        self.RtW = torch.zeros((c1 - c0, self.k), dtype=dt, device=dev)
        self.sums = torch.zeros(3, dtype=torch.float64, device=dev)
        lib = _lib.lib()
        self.wsb = lib.mfg_sweep_workspace(obs_rows.dev.csr.ref, obs_cols.dev.csr.ref, self.k)
        self.ws = torch.zeros(self.wsb, dtype=torch.uint8, device=dev)

    def pad(self, f: torch.Tensor) -> torch.Tensor:
        if self.ld == self.k:
            return f.to(self.dt).contiguous()
        out = torch.zeros((f.shape[0], self.ld), dtype=self.dt, device=f.device)
        out[:, : f.shape[1]] = f
        return out

    def run(self, w_full: torch.Tensor, h_full: torch.Tensor) -> None:
        from . import _lib

        r0, _ = self.s.row_block
        c0, _ = self.s.col_block
        lib = _lib.lib()
        es = w_full.element_size()
        _lib.check(lib.mfg_sweep_sharded(
            _lib.dtype_code(self.dt), 0, self.obs_r.dev.csr.ref, self.obs_c.dev.csr.ref, self.k,
            self.obs_r.dev.vals.data_ptr(), self.obs_c.dev.vals.data_ptr(),
            w_full.data_ptr() + r0 * self.ld * es, w_full.data_ptr(), self.ld,
            h_full.data_ptr() + c0 * self.ld * es, h_full.data_ptr(), self.ld,
            _lib.ptr(self.R), self.RH.data_ptr(), self.RtW.data_ptr(), self.out_scale,
            self.sums.data_ptr(), self.ws.data_ptr(), self.wsb, _lib.stream_ptr()), "sharded sweep")
