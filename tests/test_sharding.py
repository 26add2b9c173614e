"""Multi-rank path on CPU: world_size 2 over gloo with the
oracle as local arithmetic, checked against the single-process oracle; plus
a 1-GPU emulation of the 2-shard decomposition on the CUDA kernels."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mfg_oracle as orc
from paper_2204_14067_b200 import sharding, synth


class OracleOps:
    """Local arithmetic of ShardedMF restated on the CPU oracle (test only)."""

    def prepare(self, nrows, ncols, rows, cols, vals):
        return orc.from_coo(nrows, ncols, rows, cols, vals)

    def sweep(self, om, self_rows, other_full):
        w, h = self_rows.numpy(), other_full.numpy()
        r = orc.residual(om, w, h)
        return torch.as_tensor(orc.spmm_csr(om, r, h)), float(r @ r)

    def half_sweep(self, om, other_full, lam):
        o = other_full.numpy()
        return torch.as_tensor(orc.half_sweep(om.a_csr, om.pattern_csr, o, lam))

    def residual(self, om, self_rows, other_full):
        return torch.as_tensor(orc.residual(om, self_rows.numpy(), other_full.numpy()))

    def spmm(self, om, vals, block_full):
        return torch.as_tensor(orc.spmm_csr(om, vals.numpy(), block_full.numpy()))


def _instance():
    m, n, r, c, v = synth.generate("c2", scale=0.05, seed=11)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    w, h = synth.sweep_factors(m, n, 6, seed=3)
    return m, n, r, c, v, w, h


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, r, c, v, w, h = _instance()
        shard = sharding.make_shard(m, n, r, c, v, rank, world)
        comm = sharding.Comm()
        mf = sharding.ShardedMF(shard, OracleOps(), comm, torch.device("cpu"))
        W, H = torch.as_tensor(w), torch.as_tensor(h)
        rh, rtw, sq = mf.sweep(W, H)
        obj = mf.objective(W, H, 3.0)
        c0 = comm.ncoll
        w1, h1 = mf.bcd_epoch(W, H, 3.0)     # one MF-phase epoch: W / H all-gathers
        obj1 = mf.objective(w1, h1, 3.0)     # + the guard's objective (one batched sum)
        ncoll_epoch = comm.ncoll - c0
        c0 = comm.ncoll
        sums = comm.ordered_sums([rank + 0.5, 2.0 ** -rank, 1e16 * (rank + 1)], torch.device("cpu"))
        ncoll_sums = comm.ncoll - c0
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), rh=rh.numpy(), rtw=rtw.numpy(), sq=sq,
                 obj=obj, w1=w1.numpy(), h1=h1.numpy(), obj1=obj1, ncoll_epoch=ncoll_epoch,
                 sums=np.array(sums), ncoll_sums=ncoll_sums,
                 rb=np.array(shard.row_block), cb=np.array(shard.col_block))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_balanced_blocks_cover_and_balance():
    counts = np.array([100, 1, 1, 1, 50, 50, 0, 0, 3, 200, 1, 1])
    for parts in (1, 2, 3, 5):
        b = sharding.balanced_blocks(counts, parts)
        assert b[0][0] == 0 and b[-1][1] == counts.size
        assert all(b[i][1] == b[i + 1][0] for i in range(parts - 1))
    b = sharding.balanced_blocks(np.ones(1000, dtype=int), 4)
    assert [y - x for x, y in b] == [250, 250, 250, 250]


def test_make_shard_partitions_omega():
    m, n, r, c, v, _, _ = _instance()
    seen_r, seen_c = 0, 0
    for rank in range(3):
        s = sharding.make_shard(m, n, r, c, v, rank, 3)
        seen_r += s.r_vals.size
        seen_c += s.c_vals.size
        assert np.all(s.r_rows >= 0) and np.all(s.r_rows < s.row_block[1] - s.row_block[0])
        assert np.all(s.c_rows >= 0) and np.all(s.c_rows < s.col_block[1] - s.col_block[0])
    assert seen_r == v.size and seen_c == v.size


def test_two_ranks_gloo_match_single_process():
    m, n, r, c, v, w, h = _instance()
    om = orc.from_coo(m, n, r, c, v)
    rr, rh, rtw, sq, w2, h2 = orc.sweep(om, w, h)
    w1, h1 = orc.bcd_epoch(om, w, h, 3.0)
    obj = orc.mf_objective(om, w, h, 3.0)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"r{p}.npz")) for p in range(2)]
    for x in res:
        # CSR/CSC SpMM rows: each row's sum is computed exactly as unsharded
        assert np.array_equal(x["rh"], rh)
        assert np.array_equal(x["rtw"], rtw)
        assert float(x["sq"]) == pytest.approx(sq, rel=1e-13)
        assert float(x["obj"]) == pytest.approx(obj, rel=1e-13)
        # BCD rows are independent exact minimisers: bitwise identical
        assert np.array_equal(x["w1"], w1)
        assert np.array_equal(x["h1"], h1)
    # both ranks hold identical replicas and identical fp64 sums
    assert float(res[0]["sq"]) == float(res[1]["sq"])
    assert np.array_equal(res[0]["w1"], res[1]["w1"])
    # data plane: an MF-phase epoch (BCD + objective guard) is 3 collectives,
    # and a batch of scalars is one collective, summed in rank order
    obj1 = orc.mf_objective(om, w1, h1, 3.0)
    for x in res:
        assert int(x["ncoll_epoch"]) <= 3
        assert float(x["obj1"]) == pytest.approx(obj1, rel=1e-13)
        assert int(x["ncoll_sums"]) == 1
        assert list(x["sums"]) == [(0.5 + 1.5), 1.0 + 0.5, 1e16 + 2e16]


@pytest.mark.gpu
def test_two_shard_decomposition_on_gpu():
    """The 2-rank decomposition evaluated on one GPU (ranks emulated in turn,
    collectives replaced by concatenation): equals the unsharded kernels."""
    from paper_2204_14067_b200 import mfsolver as MF
    from paper_2204_14067_b200.data import ObservationSet
    from paper_2204_14067_b200.operators import FactorPair

    m, n, r, c, v, w, h = _instance()
    W, H = torch.as_tensor(w).cuda(), torch.as_tensor(h).cuda()
    ops = sharding.DeviceOps(torch.float64)
    rh_parts, rtw_parts, sqs, w1_parts = [], [], [], []
    shards = [sharding.make_shard(m, n, r, c, v, p, 2) for p in range(2)]
    for s in shards:
        hr = ops.prepare(s.row_block[1] - s.row_block[0], n, s.r_rows, s.r_cols, s.r_vals)
        hc = ops.prepare(s.col_block[1] - s.col_block[0], m, s.c_rows, s.c_cols, s.c_vals)
        a, sq = ops.sweep(hr, W[s.row_block[0]:s.row_block[1]], H)
        b, _ = ops.sweep(hc, H[s.col_block[0]:s.col_block[1]], W)
        rh_parts.append(a)
        rtw_parts.append(b)
        sqs.append(sq)
        w1_parts.append(ops.half_sweep(hr, H, 3.0))
    obs = ObservationSet.from_coo(m, n, r, c, v)
    _, RH, RtW, sums = MF.sweep(obs, FactorPair(W, H), want_rh=True, want_rtw=True)
    assert torch.allclose(torch.cat(rh_parts), RH, rtol=0, atol=1e-12)
    assert torch.allclose(torch.cat(rtw_parts), RtW, rtol=0, atol=1e-12)
    assert sum(sqs) == pytest.approx(float(sums[0]), rel=1e-12)
    w1 = MF.bcd_epoch(obs, FactorPair(W, H), 3.0).w
    assert torch.equal(torch.cat(w1_parts), w1)


# ---------------------------------------------------------------------------
# sharded lifting step (sharded_lift): partial SVD of Z = W H^T - alpha G


LIFT_ALPHA = 0.35
LIFT_K = 5


def _lift_run(world_rank, world, ops, device):
    """Shared body: sharded operator, LM-Krylov top-k, projection, SVD and
    soft-threshold; returns gathered results (identical on every rank)."""
    from paper_2204_14067_b200 import sharded_lift as SL
    from paper_2204_14067_b200.eigensolver import EigConfig

    m, n, r, c, v, w, h = _instance()
    shard = sharding.make_shard(m, n, r, c, v, world_rank, world)
    comm = SL.ShardComm()
    mf = sharding.ShardedMF(shard, ops, comm, device)
    W, H = torch.as_tensor(w).to(device), torch.as_tensor(h).to(device)
    r0_, r1_ = shard.row_block
    c0_, c1_ = shard.col_block
    g_row = 2.0 * ops.residual(mf.hr, W[r0_:r1_], H)
    g_col = 2.0 * ops.residual(mf.hc, H[c0_:c1_], W)
    op = SL.ShardedOperator(mf, comm, W, H, g_row, g_col, LIFT_ALPHA)
    rng = np.random.default_rng(7)
    r0 = torch.as_tensor(rng.standard_normal((m, LIFT_K))).to(device)
    cfg = EigConfig(memory=3, max_iters=40, residual_tol=1e-9)
    u_loc, sigma, v_loc, eig, largest = SL.partial_svd_step(op, r0[r0_:r1_], cfg, beta=0.05)
    u = comm.allgather_blocks(u_loc, shard.row_blocks)
    vv = comm.allgather_blocks(v_loc, shard.col_blocks)
    basis = comm.allgather_blocks(eig.basis, shard.row_blocks)
    return dict(eigvals=eig.eigvals, iters=eig.iters_used, res=eig.residuals, sigma=sigma,
                x=(u.double() * torch.as_tensor(sigma).to(device)) @ vv.double().T,
                proj=basis @ basis.T)


def _lift_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = _lift_run(rank, world, OracleOps(), torch.device("cpu"))
        np.savez(os.path.join(out_dir, f"l{rank}.npz"), eigvals=out["eigvals"], iters=out["iters"],
                 sigma=out["sigma"], x=out["x"].numpy(), proj=out["proj"].numpy())
    finally:
        dist.destroy_process_group()


def _dense_z():
    m, n, r, c, v, w, h = _instance()
    om = orc.from_coo(m, n, r, c, v)
    g = 2.0 * orc.residual(om, w, h)
    gd = orc.csr_of(om, g).toarray()
    return w @ h.T - LIFT_ALPHA * gd


def test_sharded_lifting_two_ranks_gloo():
    """2 ranks over gloo (oracle SpMMs) vs 1 rank vs a dense eigendecomposition:
    same iteration count and identified rank; Ritz values, soft-thresholded
    spectrum and the new iterate X agree to rounding."""
    one = _lift_run(0, 1, OracleOps(), torch.device("cpu"))
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_lift_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"l{p}.npz")) for p in range(2)]
    for x in res:
        assert int(x["iters"]) == one["iters"]
        assert x["sigma"].size == one["sigma"].size
        np.testing.assert_allclose(x["eigvals"], one["eigvals"], rtol=1e-11)
        np.testing.assert_allclose(x["sigma"], one["sigma"], rtol=1e-11)
        np.testing.assert_allclose(x["x"], one["x"].numpy(), rtol=0, atol=1e-10 * np.abs(x["x"]).max())
    # every rank holds identical bits
    assert np.array_equal(res[0]["sigma"], res[1]["sigma"])
    assert np.array_equal(res[0]["x"], res[1]["x"])
    # against a dense eigendecomposition of Z Z^T
    z = _dense_z()
    ev = np.sort(np.linalg.eigvalsh(z @ z.T))[::-1][:LIFT_K]
    np.testing.assert_allclose(one["eigvals"], ev, rtol=1e-8)
    s_hat = np.sqrt(ev)
    kept = s_hat[s_hat > 0.05] - 0.05
    np.testing.assert_allclose(one["sigma"], kept, rtol=1e-8)


@pytest.mark.gpu
def test_sharded_lifting_one_rank_on_gpu_matches_product():
    """The sharded lifting code with DeviceOps (libmfg_b200 SpMMs) at world 1
    against the product eigensolver on the same operator."""
    from paper_2204_14067_b200 import eigensolver as E
    from paper_2204_14067_b200.data import ObservationSet, residual_on_omega
    from paper_2204_14067_b200.operators import FactorPair, ShiftedOperator

    got = _lift_run(0, 1, sharding.DeviceOps(torch.float64), torch.device("cuda"))
    m, n, r, c, v, w, h = _instance()
    obs = ObservationSet.from_coo(m, n, r, c, v)
    wf = FactorPair(torch.as_tensor(w).cuda(), torch.as_tensor(h).cuda())
    grad = residual_on_omega(obs, wf).scaled(2.0)
    op = ShiftedOperator(wf, grad, LIFT_ALPHA)
    r0 = torch.as_tensor(np.random.default_rng(7).standard_normal((m, LIFT_K))).cuda()
    ref = E.lmkrylov_topk(op, r0, E.EigConfig(memory=3, max_iters=40, residual_tol=1e-9))
    assert got["iters"] == ref.iters_used
    np.testing.assert_allclose(got["eigvals"], ref.eigvals, rtol=1e-11)
    z = _dense_z()
    ev = np.sort(np.linalg.eigvalsh(z @ z.T))[::-1][:LIFT_K]
    np.testing.assert_allclose(got["eigvals"], ev, rtol=1e-8)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 3])
def test_shard_sweep_plans_reassemble_the_full_sweep(world):
    """mfg_sweep_sharded on every rank's shards (run one after another on one
    GPU): R, R.H and R^T.W blocks reassemble the single-GPU grouped sweep,
    and the rank-ordered sums of the local sums are the full sums."""
    from paper_2204_14067_b200.data import ObservationSet
    from paper_2204_14067_b200.mfsolver import SweepPlan
    m, n, r, c, v = synth.generate("c2", scale=0.2, seed=4)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    k = 20
    w, h = synth.sweep_factors(m, n, k, seed=6, dtype=np.float32)
    full = ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    ref = SweepPlan(full, k)
    W, H = ref.pad(torch.as_tensor(w).cuda()), ref.pad(torch.as_tensor(h).cuda())
    ref.run(W, H)
    ops = sharding.DeviceOps(torch.float32)
    Rs, RHs, RtWs, sums = [], [None] * world, [None] * world, np.zeros(3)
    for rank in range(world):
        s = sharding.make_shard(m, n, r, c, v, rank, world)
        r0, r1 = s.row_block
        c0, c1 = s.col_block
        po = ops.prepare(r1 - r0, n, s.r_rows, s.r_cols, s.r_vals)
        pc = ops.prepare(c1 - c0, m, s.c_rows, s.c_cols, s.c_vals)
        plan = sharding.ShardSweepPlan(s, po, pc, k)
        assert plan.ld == ref.ld
        plan.run(W, H)
        torch.cuda.synchronize()
        Rs.append(plan.R.clone())
        RHs[rank], RtWs[rank] = plan.RH.clone(), plan.RtW.clone()
        sums += plan.sums.cpu().numpy()
    # R: per-entry dots, same arithmetic -> bitwise; row blocks in CSR order
    assert torch.equal(torch.cat(Rs), ref.R)
    tol = lambda x: 2e-5 * (float(x.abs().max()) + 1.0)  # noqa: E731  fp32 accumulation order
    rh = torch.cat(RHs)
    rtw = torch.cat(RtWs)
    assert float((rh - ref.RH).abs().max()) <= tol(ref.RH)
    assert float((rtw - ref.RtW).abs().max()) <= tol(ref.RtW)
    full_sums = ref.sums.cpu().numpy()
    assert sums[0] == pytest.approx(full_sums[0], rel=1e-12)
    assert sums[1] == pytest.approx(full_sums[1], rel=1e-12)
    assert sums[2] == pytest.approx(full_sums[2], rel=1e-12)
