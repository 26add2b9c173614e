"""Sharded MF-Global driver: ``solve_mf_global`` over a
row/column-sharded Omega, one process per GPU.

The outer loop is mfg/driver.py:264-344 (`_run_lifted`) with every piece
that touches Omega or an m- / n-sized block replaced by its sharded form:

  MF phase      sharded BCD epochs with the monotone guard (``ShardedMF``,
                mfg/mfsolver.py:96-112)
  gradient      G = 2 R on the row shard and on the column shard
  BB stepsize   0.5 ||dG||^2 as an ordered sum over the row shards, the
                factored distance from summed Grams (mfg/proxlift.py:96-124)
  warm start    orthonormalisation of [U, W] by TSQR / CholQR2 over row
                blocks; the host Philox stream is drawn at full length m on
                every rank and each rank keeps its rows (127-181)
  prox step     backtracking over alpha; sharded LM-Krylov / power
                eigensolver, (B^T Z)^T on the column shard, short-fat SVD
                from summed Grams, soft-threshold on identical host bits,
                Eq. 5 terms by an SDDMM over the row shard (317-410)
  certificate   the estimated mode of certify_epsilon (194-314): the
                low-rank-plus-G operator applied shard-wise with all-gathered
                inputs, power iterations on vectors drawn from the fixed
                Philox(0x5EEDCE27) at full length n (each rank keeps its
                columns), the ||Z||_F bound from Grams and an SDDMM.

Layout: U (m x r) blocks are row-sharded (rows R_p), V (n x r) blocks are
column-sharded (rows C_p); W, H, sigma are replicated. Every sum over ranks
is an all-gather added in rank order (``ShardComm.sum_ordered`` /
``Comm.ordered_sum``), so all ranks take identical host decisions (ranks,
backtracks, eigensolver stops, certification retries).

Local arithmetic is injected through ``ops`` (``sharding.DeviceOps`` on the
GPU; tests inject the oracle). The exact-dense certification mode, a
test-scale mode of the reference (m * n <= 1e6), is not sharded: ``auto``
resolves to ``estimated`` here.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import sharded_lift as sl
from .data import LIPSCHITZ
from .driver import IterationRecord, IterationTrace, NumericalError, SolverConfig, _window_converged
from .eigensolver import EigResult
from .kernels import SIGMA_FLOOR, soft_threshold
from .proxlift import (
    CERT_MAX_VECTORS,
    CERT_POWER_ITERS,
    CERT_SEED,
    BacktrackingError,
    StepParams,
    _BACKTRACK_SAFETY,
    _EQ5_SLACK,
)

# fp32-mode MF guard slack (as mfsolver.guard_slack)
_GUARD = {torch.float64: 1e-9, torch.float32: 1e-6}


@dataclass
class ShardedTriplet:
    """Compact SVD X = U diag(sigma) V^T with U rows R_p, V rows C_p."""

    u_loc: torch.Tensor
    sigma: np.ndarray
    v_loc: torch.Tensor

    @property
    def rank(self) -> int:
        return int(self.sigma.size)

    def sigma_dev(self) -> torch.Tensor:
        return torch.as_tensor(self.sigma, dtype=torch.float64, device=self.u_loc.device)

    def nuclear_norm(self) -> float:
        return float(np.sum(self.sigma))


class _Ctx:
    """Rank context: shard, ops, communicator, block bounds."""

    def __init__(self, mf, comm: sl.ShardComm):
        self.mf, self.comm, self.ops, self.s = mf, comm, mf.ops, mf.s
        self.r0, self.r1 = self.s.row_block
        self.c0, self.c1 = self.s.col_block
        self.m, self.n = self.s.m, self.s.n
        self.device = mf.device

    def osum(self, x: float) -> float:
        return self.comm.ordered_sum(float(x), self.device)

    def tsum(self, t: torch.Tensor) -> torch.Tensor:
        return self.comm.sum_ordered(t)

    def dot(self, a: torch.Tensor, b: torch.Tensor) -> float:
        return self.osum(float(torch.dot(a, b)))

    def norm(self, a: torch.Tensor) -> float:
        return math.sqrt(max(self.dot(a, a), 0.0))

    def full_v(self, v_loc: torch.Tensor) -> torch.Tensor:
        return self.comm.allgather_blocks(v_loc.contiguous(), self.s.col_blocks)

    def full_u(self, u_loc: torch.Tensor) -> torch.Tensor:
        return self.comm.allgather_blocks(u_loc.contiguous(), self.s.row_blocks)


# ---------------------------------------------------------------------------
# factored products (mfg/operators.py:67-81)


def _views(ctx: _Ctx, a):
    if isinstance(a, ShardedTriplet):
        return a.u_loc * a.sigma_dev(), a.v_loc
    w, h = a
    return w[ctx.r0:ctx.r1].double(), h[ctx.c0:ctx.c1].double()


def inner_product(ctx: _Ctx, a, b) -> float:
    la, ra = _views(ctx, a)
    lb, rb = _views(ctx, b)
    if la.shape[1] == 0 or lb.shape[1] == 0:
        return 0.0
    gl, gr = la.T @ lb, ra.T @ rb
    both = ctx.tsum(torch.cat([gl.reshape(-1), gr.reshape(-1)]))   # one collective
    return float(torch.sum(both[: gl.numel()] * both[gl.numel():]))


def frob_dist_sq(ctx: _Ctx, a, b) -> float:
    d = inner_product(ctx, a, a) - 2.0 * inner_product(ctx, a, b) + inner_product(ctx, b, b)
    return max(d, 0.0)


# ---------------------------------------------------------------------------
# SVD <-> factors (mfg/mfsolver.py:25-45)


def svd_from_full_factors(ctx: _Ctx, w: torch.Tensor, h: torch.Tensor) -> ShardedTriplet:
    """The initial iterate's SVD, computed redundantly from the replicated
    factors on every rank (identical bits), then sliced to the local rows."""
    dev = ctx.device
    if w.shape[1] == 0:
        return ShardedTriplet(torch.zeros((ctx.r1 - ctx.r0, 0), dtype=torch.float64, device=dev),
                              np.zeros(0), torch.zeros((ctx.c1 - ctx.c0, 0), dtype=torch.float64,
                                                       device=dev))
    qw, rw = torch.linalg.qr(w.double())
    qh, rh = torch.linalg.qr(h.double())
    u_mid, s, vt_mid = torch.linalg.svd(rw @ rh.T)
    sh = s.cpu().numpy()
    kept = np.flatnonzero(sh > SIGMA_FLOOR * sh[0]) if sh.size and sh[0] > 0 else np.zeros(0, int)
    idx = torch.as_tensor(kept, device=qw.device, dtype=torch.long)
    u = qw @ u_mid.index_select(1, idx)
    v = qh @ vt_mid.T.index_select(1, idx)
    return ShardedTriplet(u[ctx.r0:ctx.r1].contiguous(), sh[kept], v[ctx.c0:ctx.c1].contiguous())


def factors_from_svd(ctx: _Ctx, x: ShardedTriplet, dtype):
    """Replicated W = U sqrt(s), H = V sqrt(s) (all-gather of the blocks)."""
    root = torch.as_tensor(np.sqrt(x.sigma), dtype=torch.float64, device=ctx.device)
    w = ctx.full_u(x.u_loc * root)
    h = ctx.full_v(x.v_loc * root)
    return w.to(dtype), h.to(dtype)


# ---------------------------------------------------------------------------
# residuals on the shards


@dataclass
class ShardGrad:
    """G = 2 R on the row shard and on the column shard (handle order), and
    sum r^2 over all of Omega (identical on every rank)."""

    g_row: torch.Tensor
    g_col: torch.Tensor
    loss: float

    @property
    def gss(self) -> float:
        return LIPSCHITZ * LIPSCHITZ * self.loss


def grad_factors(ctx: _Ctx, w: torch.Tensor, h: torch.Tensor) -> ShardGrad:
    r_row = ctx.ops.residual(ctx.mf.hr, w[ctx.r0:ctx.r1], h)
    r_col = ctx.ops.residual(ctx.mf.hc, h[ctx.c0:ctx.c1], w)
    loss = ctx.osum(float(torch.dot(r_row, r_row)))
    return ShardGrad(LIPSCHITZ * r_row, LIPSCHITZ * r_col, loss)


def grad_triplet(ctx: _Ctx, x: ShardedTriplet) -> ShardGrad:
    """residual_on_omega_svd + gradient (mfg/data.py:283-298) on both shards."""
    if x.rank == 0:
        z_r = torch.zeros((ctx.r1 - ctx.r0, 1), dtype=torch.float64, device=ctx.device)
        z_c = torch.zeros((ctx.c1 - ctx.c0, 1), dtype=torch.float64, device=ctx.device)
        zf_n = torch.zeros((ctx.n, 1), dtype=torch.float64, device=ctx.device)
        zf_m = torch.zeros((ctx.m, 1), dtype=torch.float64, device=ctx.device)
        return grad_factors_raw(ctx, z_r, zf_n, z_c, zf_m)
    us = x.u_loc * x.sigma_dev()
    v_full = ctx.full_v(x.v_loc)
    u_full_s = ctx.full_u(us)
    return grad_factors_raw(ctx, us, v_full, x.v_loc, u_full_s)


def grad_factors_raw(ctx, left_row, right_full, self_col, other_full) -> ShardGrad:
    r_row = ctx.ops.residual(ctx.mf.hr, left_row, right_full)
    r_col = ctx.ops.residual(ctx.mf.hc, self_col, other_full)
    loss = ctx.osum(float(torch.dot(r_row, r_row)))
    return ShardGrad(LIPSCHITZ * r_row, LIPSCHITZ * r_col, loss)


# ---------------------------------------------------------------------------
# lifting step pieces


def bb_stepsize(ctx: _Ctx, x_t, x_prev, g_t: ShardGrad, g_prev: ShardGrad, p: StepParams,
                fallback: float) -> float:
    """Clamped BB initialisation (mfg/proxlift.py:96-124)."""
    diff = g_t.g_row - g_prev.g_row
    num = 0.5 * ctx.osum(float(torch.dot(diff, diff)))
    den = frob_dist_sq(ctx, x_t, x_prev)
    if den <= 0.0:
        return fallback
    if p.bb_reciprocal:
        if num <= 0.0:
            return p.alpha_max
        ratio = den / num
    else:
        ratio = num / den
    return float(min(max(ratio, p.alpha_min), p.alpha_max))


def build_warmstart(ctx: _Ctx, u_loc, w_loc, ws, cur_rank: int) -> torch.Tensor:
    """Warm-start basis R_t (mfg/proxlift.py:127-169), row-sharded."""
    r_hat, _ = sl.orthonormalize(ctx.comm, torch.cat([u_loc, w_loc.double()], dim=1), ctx.m)
    trigger = cur_rank == ws.prev_rank and ws.last_trunc_count <= 1
    r = r_hat
    appended = False
    if trigger:
        if ws.retained is not None:
            u = ws.retained
        else:
            u = torch.as_tensor(ws.rng.standard_normal(ctx.m)[ctx.r0:ctx.r1], device=ctx.device)
        u_t = u - r_hat @ ctx.tsum(r_hat.T @ u)
        g = torch.as_tensor(ws.rng.standard_normal(ctx.m)[ctx.r0:ctx.r1], device=ctx.device)
        g = g - r_hat @ ctx.tsum(r_hat.T @ g)
        nu = ctx.norm(u_t)
        if nu > 0.0:
            un = u_t / nu
            g = g - un * ctx.dot(un, g)
        gn = ctx.norm(g)
        xi = (ws.psi / gn) * g if gn > 0.0 else torch.zeros_like(g)
        col = (u_t + xi)[:, None]
        r, rank = sl.orthonormalize(ctx.comm, torch.cat([r_hat, col], dim=1), ctx.m)
        appended = rank > r_hat.shape[1]
    if cur_rank == ws.prev_rank and r.shape[1] > cur_rank + 1:
        probe = r[:, -1:] if appended else r[:, cur_rank: cur_rank + 1]
        r = torch.cat([r[:, :cur_rank], probe], dim=1)
    ws.pending_rank = cur_rank
    return r.contiguous()


class _LowRankPlusG:
    """Y = L R^T B + s * G B on the shards (L rows R_p, R rows C_p)."""

    def __init__(self, ctx: _Ctx, l_loc, r_loc, g: ShardGrad, s: float):
        self.ctx, self.l_loc, self.r_loc, self.g, self.s = ctx, l_loc, r_loc, g, s

    def apply(self, v_loc):     # n-side block (rows C_p) -> m-side rows R_p
        ctx = self.ctx
        out = self.l_loc @ ctx.tsum(self.r_loc.T @ v_loc)
        if self.s != 0.0:
            out = out + self.s * ctx.ops.spmm(ctx.mf.hr, self.g.g_row, ctx.full_v(v_loc))
        return out

    def apply_t(self, u_loc):   # m-side rows R_p -> n-side rows C_p
        ctx = self.ctx
        out = self.r_loc @ ctx.tsum(self.l_loc.T @ u_loc)
        if self.s != 0.0:
            out = out + self.s * ctx.ops.spmm(ctx.mf.hc, self.g.g_col, ctx.full_u(u_loc))
        return out


def _frob_sq_z(ctx: _Ctx, w, h, g: ShardGrad, alpha: float) -> float:
    """||W H^T - alpha G||_F^2 (mfg/operators.py:142-152)."""
    ww = inner_product(ctx, (w, h), (w, h))
    xg = ctx.osum(ctx.ops.sddmm_sums(ctx.mf.hr, w[ctx.r0:ctx.r1].double(), h.double(), None,
                                     g.g_row, with_a=False)[2])
    return ww - 2.0 * alpha * xg + alpha ** 2 * g.gss


def certify_epsilon(ctx: _Ctx, x_next: ShardedTriplet, w, h, g: ShardGrad, alpha: float,
                    lam: float, sigma_hat) -> float:
    """Estimated mode of mfg/proxlift.py:194-314 on the shards."""
    dev = ctx.device
    u, v = x_next.u_loc, x_next.v_loc
    scale = torch.as_tensor(x_next.sigma / alpha + lam, dtype=torch.float64, device=dev)
    left = torch.cat([u * scale, -w[ctx.r0:ctx.r1].double() / alpha], dim=1)
    right = torch.cat([v, h[ctx.c0:ctx.c1].double()], dim=1)
    op = _LowRankPlusG(ctx, left, right, g, 1.0)
    rest_sq = 0.0
    if x_next.rank:
        gtu = op.apply_t(u)
        gv = op.apply(v)
        gv_perp = gv - u @ ctx.tsum(u.T @ gv)
        rest_sq = ctx.osum(float(torch.sum(gtu * gtu) + torch.sum(gv_perp * gv_perp)))

    def gc_apply(vec):
        if x_next.rank:
            vec = vec - v @ ctx.tsum(v.T @ vec)
        out = op.apply(vec[:, None].contiguous())[:, 0]
        if x_next.rank:
            out = out - u @ ctx.tsum(u.T @ out)
        return out

    def gc_apply_t(vec):
        if x_next.rank:
            vec = vec - u @ ctx.tsum(u.T @ vec)
        out = op.apply_t(vec[:, None].contiguous())[:, 0]
        if x_next.rank:
            out = out - v @ ctx.tsum(v.T @ out)
        return out

    rng = np.random.Generator(np.random.Philox(CERT_SEED))
    found: list = []
    excess_sq = 0.0
    for _ in range(CERT_MAX_VECTORS):
        vec = torch.as_tensor(rng.standard_normal(ctx.n)[ctx.c0:ctx.c1], device=dev)
        if x_next.rank:
            vec = vec - v @ ctx.tsum(v.T @ vec)
        for _, _, qv in found:
            vec = vec - qv * ctx.dot(qv, vec)
        nrm = ctx.norm(vec)
        if nrm < 1e-300:
            break
        vec = vec / nrm
        s_est = 0.0
        uvec = torch.zeros(ctx.r1 - ctx.r0, dtype=torch.float64, device=dev)
        for _ in range(CERT_POWER_ITERS):
            uvec = gc_apply(vec)
            for s_i, pu, qv in found:
                uvec = uvec - pu * (s_i * ctx.dot(qv, vec))
            un = ctx.norm(uvec)
            if un < 1e-300:
                s_est = 0.0
                break
            uvec = uvec / un
            vec_new = gc_apply_t(uvec)
            for s_i, pu, qv in found:
                vec_new = vec_new - qv * (s_i * ctx.dot(pu, uvec))
            s_est = ctx.norm(vec_new)
            if s_est < 1e-300:
                break
            vec = vec_new / s_est
        found.append((s_est, uvec, vec))
        if s_est <= lam:
            break
        excess_sq += (s_est - lam) ** 2
    estimate = math.sqrt(rest_sq + excess_sq)
    z_sq = _frob_sq_z(ctx, w, h, g, alpha)
    sh = np.asarray(sigma_hat, dtype=np.float64)
    bound = math.sqrt(max(z_sq - float(sh @ sh), 0.0)) / alpha
    return min(estimate, bound)


@dataclass
class ShardedLiftOutcome:
    x_next: ShardedTriplet
    alpha_used: float
    backtracks: int
    eps_achieved: float
    eps_warning: bool
    largest_truncated: float | None
    truncated_vector: torch.Tensor | None
    trunc_count: int
    k_t: int
    f_next: float
    grad_inner: float
    dist_sq: float
    eig_sweeps: int


def inexact_prox_step(ctx: _Ctx, w, h, g: ShardGrad, alpha_bb: float, params: StepParams,
                      r_t_loc, eig_cfg, eps_target: float, cert_retries: int = 2):
    """Backtracking inexact proximal-gradient step (mfg/proxlift.py:317-410),
    sharded; X~ = W H^T with W, H replicated."""
    if eps_target <= 0:
        raise ValueError("eps_target must be positive")
    k_t = r_t_loc.shape[1]
    f_base = 0.25 * g.gss
    i_max = (int(math.ceil(math.log(params.alpha_min / params.alpha_max) / math.log(params.beta)))
             + _BACKTRACK_SAFETY)
    warm = r_t_loc
    sweeps = 0
    w_loc = w[ctx.r0:ctx.r1].double()
    for i in range(i_max + 1):
        alpha = alpha_bb * params.beta ** i
        op = sl.ShardedOperator(ctx.mf, ctx.comm, w, h, g.g_row, g.g_col, alpha)
        tol = eps_target / (params.alpha_max * max(k_t, 1))
        for retry in range(cert_retries + 1):
            if k_t == 0:
                eig = EigResult(r_t_loc.new_zeros((r_t_loc.shape[0], 0)), np.zeros(0), np.zeros(0),
                                0, True)
            else:
                eig = sl.solve_topk(op, warm, replace(eig_cfg, residual_tol=tol))
                warm = eig.basis
            sweeps += eig.iters_used
            mt_loc = op.apply_t(eig.basis)
            u_small, sigma_hat, v_loc = sl.exact_svd_short_fat(ctx.comm, mt_loc, ctx.c0)
            u_full = eig.basis @ u_small
            sigma, kept, largest = soft_threshold(sigma_hat, alpha * params.lam)
            idx = torch.as_tensor(kept, device=u_full.device, dtype=torch.long)
            x_next = ShardedTriplet(u_full.index_select(1, idx).contiguous(), sigma,
                                    v_loc.index_select(1, idx).contiguous())
            if x_next.rank:
                left = x_next.u_loc
                right = ctx.full_v(x_next.v_loc)
                scale = x_next.sigma_dev()
            else:
                left = torch.zeros((ctx.r1 - ctx.r0, 1), dtype=torch.float64, device=ctx.device)
                right = torch.zeros((ctx.n, 1), dtype=torch.float64, device=ctx.device)
                scale = None
            s0, s1, _ = ctx.ops.sddmm_sums(ctx.mf.hr, left, right, scale, g.g_row, with_a=True)
            f_next, g_inner = ctx.osum(s0), ctx.osum(s1)
            dist_sq = frob_dist_sq(ctx, x_next, (w, h))
            rhs = f_base + g_inner + (params.delta / alpha) * dist_sq
            slack = _EQ5_SLACK * (abs(f_base) + abs(g_inner) + (params.delta / alpha) * dist_sq + 1.0)
            if f_next > rhs + slack:
                break
            eps = certify_epsilon(ctx, x_next, w, h, g, alpha, params.lam, sigma_hat)
            if eps <= eps_target or retry == cert_retries:
                trunc_count = k_t - kept.size
                vec = u_full[:, kept.size].clone() if trunc_count > 0 else None
                return ShardedLiftOutcome(
                    x_next=x_next, alpha_used=alpha, backtracks=i, eps_achieved=eps,
                    eps_warning=eps > eps_target, largest_truncated=largest, truncated_vector=vec,
                    trunc_count=trunc_count, k_t=k_t, f_next=f_next, grad_inner=g_inner,
                    dist_sq=dist_sq, eig_sweeps=sweeps)
            tol *= 0.1
    raise BacktrackingError(
        f"no stepsize accepted after {i_max + 1} trials from alpha_bb={alpha_bb!r}")


# ---------------------------------------------------------------------------
# the outer loop (mfg/driver.py:247-354)


def _update_warmstart(ws, out: ShardedLiftOutcome) -> None:
    """mfg/proxlift.py:172-181 (the retained vector keeps this rank's rows)."""
    if out.truncated_vector is not None:
        ws.retained = out.truncated_vector.clone()
    ws.last_trunc_count = out.trunc_count
    ws.prev_rank = ws.pending_rank
    ws.psi *= ws.psi_decay


def _mf_phase(ctx: _Ctx, w, h, lam: float, epochs: int, slack: float):
    if epochs <= 0:
        return w, h
    prev = ctx.mf.objective(w, h, lam)
    for _ in range(epochs):
        w, h = ctx.mf.bcd_epoch(w, h, lam)
        cur = ctx.mf.objective(w, h, lam)
        if cur > prev + slack * (1.0 + abs(prev)):
            raise NumericalError(f"BCD sweep increased the objective: {prev!r} -> {cur!r}")
        prev = cur
    return w, h


def solve_mf_global_sharded(mf, comm: sl.ShardComm, cfg: SolverConfig, *, dtype=torch.float64,
                            mf_epochs: int | None = None, f_star: float | None = None):
    """MF-Global on this rank's shard of Omega (same SolverConfig, same trace
    schema as ``solve_mf_global``; collective calls must be made by every
    rank). ``dtype`` is the storage type of the MF factors (fp32 mode: the
    lifting step and all reductions stay fp64). Returns (X as a
    ShardedTriplet of local blocks, (W, H) replicated, trace)."""
    from .proxlift import WarmStartState

    if cfg.cert_mode not in ("auto", "estimated"):
        raise ValueError("the sharded solver certifies in the estimated mode only")
    ctx = _Ctx(mf, comm)
    epochs = cfg.mf_epochs if mf_epochs is None else mf_epochs
    rng = np.random.Generator(np.random.Philox(cfg.seed))
    params = cfg.step_params()
    eig_cfg = cfg.eig_config()
    trace = IterationTrace()
    slack = _GUARD[dtype]
    t_start = time.perf_counter()
    w0 = cfg.init_scale * (2.0 * rng.random((ctx.m, cfg.k0)) - 1.0)
    h0 = cfg.init_scale * (2.0 * rng.random((ctx.n, cfg.k0)) - 1.0)
    x = svd_from_full_factors(ctx, torch.as_tensor(w0, device=ctx.device),
                              torch.as_tensor(h0, device=ctx.device))
    w_t, h_t = factors_from_svd(ctx, x, dtype)
    g_x = grad_triplet(ctx, x)
    f_x = g_x.loss + cfg.lam * x.nuclear_norm()
    eps0 = cfg.eps0_scale * LIPSCHITZ * np.sqrt(g_x.loss)
    ws = WarmStartState(rng=rng, psi=cfg.psi0_scale * (x.sigma[0] if x.rank else 1.0),
                        psi_decay=cfg.psi_rho)

    def rel(f):
        return (f - f_star) / abs(f_star) if f_star else float("nan")

    trace.append(IterationRecord(0, time.perf_counter() - t_start, f_x, rel(f_x), x.rank,
                                 float("nan"), float("nan"), float("nan"), 0, float("nan"),
                                 float("nan"), 0, x.rank))
    objs = [f_x]
    x_prev = g_prev = None
    alpha_prev = 1.0 / LIPSCHITZ
    for t in range(cfg.max_outer_iters):
        w, h = _mf_phase(ctx, w_t, h_t, cfg.lam, epochs, slack)
        f_mf = ctx.mf.objective(w, h, cfg.lam)
        if f_mf > f_x + slack * (1.0 + abs(f_x)):
            raise NumericalError(
                f"MF phase guard violated at t={t}: F(W,H)={f_mf!r} > F(X)={f_x!r}", trace)
        g_tilde = grad_factors(ctx, w, h)
        if x_prev is None:
            alpha_bb = 1.0 / LIPSCHITZ
        else:
            alpha_bb = bb_stepsize(ctx, x, x_prev, g_x, g_prev, params, alpha_prev)
        r_t = build_warmstart(ctx, x.u_loc, w[ctx.r0:ctx.r1], ws, x.rank)
        eps_t = eps0 * cfg.eps_rho ** t
        out = inexact_prox_step(ctx, w, h, g_tilde, alpha_bb, params, r_t, eig_cfg, eps_t,
                                cfg.cert_retries)
        x_prev, g_prev = x, g_x
        x = out.x_next
        _update_warmstart(ws, out)
        g_x = grad_triplet(ctx, x)
        f_prev = f_x
        f_x = g_x.loss + cfg.lam * x.nuclear_norm()
        if not np.isfinite(f_x):
            raise NumericalError(f"non-finite objective at t={t}", trace)
        w_t, h_t = factors_from_svd(ctx, x, dtype)
        alpha_prev = out.alpha_used
        trace.append(IterationRecord(
            t + 1, time.perf_counter() - t_start, f_x, rel(f_x), x.rank, float("nan"),
            float("nan"), out.alpha_used, out.backtracks, eps_t, out.eps_achieved, out.eig_sweeps,
            out.k_t, f_prev=f_prev, f_mf=f_mf, dist=float(np.sqrt(out.dist_sq)),
            eps_warning=out.eps_warning))
        objs.append(f_x)
        if _window_converged(objs, cfg):
            break
    return x, (w_t, h_t), trace
