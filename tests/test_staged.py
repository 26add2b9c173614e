"""The shared-memory staged sweep (csrc/staged.cu, paper_2204_14067_b200/staged.py).

CPU: the plan is walked exactly as the kernel walks it (tiles -> chunks ->
pieces -> fold, gathers through the staged block slots or the cold ids) in
numpy, and must reproduce the oracle's sweep (mfg/data.py:253-293,
mfg/operators.py:108,117) -- this pins the planner's stream, chunk, piece
and block bookkeeping without a GPU.

GPU: mfg_sweep_staged against the oracle on fp32-rounded inputs (fp32
arithmetic: 2e-5 relative, the tolerance of the fp32 sweep tests), against
mfg_sweep, and bitwise run-to-run determinism.
"""

import numpy as np
import pytest
import torch

from oracle import mfg_oracle as orc
from conftest import rng_for

from paper_2204_14067_b200 import staged as ST


def _zipf_instance(seed, m, n, nnz, s=1.0):
    rng = rng_for(seed)
    pr = (np.arange(1, m + 1) ** -s)[rng.permutation(m)]
    pc = (np.arange(1, n + 1) ** -s)[rng.permutation(n)]
    keys = set()
    rows, cols = [], []
    while len(rows) < nnz:
        i = int(rng.choice(m, p=pr / pr.sum()))
        j = int(rng.choice(n, p=pc / pc.sum()))
        if (i, j) not in keys:
            keys.add((i, j))
            rows.append(i)
            cols.append(j)
    rows = np.array(rows)
    cols = np.array(cols)
    vals = rng.integers(1, 6, size=nnz).astype(np.float64)
    return m, n, rows, cols, vals


def _input_cpu(m, n, rows, cols, vals):
    om = orc.from_coo(m, n, rows, cols, vals)
    r = np.asarray(om.rows, np.int64)
    c = np.asarray(om.cols, np.int64)
    v = np.asarray(om.vals, np.float64)
    csc = np.lexsort((r, c))
    t = lambda a, dt=torch.int32: torch.from_numpy(np.ascontiguousarray(a)).to(dt)  # noqa: E731
    src = ST.StagedInput(m, n, t(c), t(r), t(v, torch.float32), t(r[csc]), t(c[csc]),
                         t(v[csc], torch.float32))
    return om, src


def _simulate(plan, w, h):
    """numpy walk of the plan in the kernel's order (fp64 arithmetic)."""
    nnz = plan.p[0].nnz
    R = np.full(nnz, np.nan)
    outs = []
    sq = 0.0
    chunks = plan.chunks.numpy()
    tiles = plan.tiles.numpy()
    for pi, (pp, self_f, other_f) in enumerate(zip(plan.p, (w, h), (h, w))):
        sidx, srow = pp.sidx.numpy(), pp.srow.numpy()
        sval = pp.svals.numpy().astype(np.float64)
        bm = pp.bmask.numpy().view(np.uint32)
        mem = pp.members.numpy()
        vpart = np.zeros((max(pp.npieces, 1), self_f.shape[1]))
        for (tp, block, c0, c1) in tiles:
            if tp != pi:
                continue
            for c in range(c0, c1):
                e0, e1, piece, cpass = chunks[c]
                assert cpass == pi and e0 % 32 == 0
                acc = np.zeros(self_f.shape[1])
                for e in range(e0, e1):
                    if e > e0 and (bm[e >> 5] >> (e & 31)) & 1:
                        vpart[piece] = acc
                        piece += 1
                        acc = np.zeros_like(acc)
                    g = mem[block * pp.S + sidx[e]] if block >= 0 else sidx[e]
                    r = self_f[srow[e]] @ other_f[g] - sval[e]
                    if pi == 0:
                        R[pp.spos.numpy()[e]] = r
                        sq += r * r
                    acc = acc + r * other_f[g]
                vpart[piece] = acc
        pptr, plist = pp.pptr.numpy(), pp.plist.numpy()
        out = np.zeros((pp.nrows, self_f.shape[1]))
        for i in range(pp.nrows):
            for p in plist[pptr[i]:pptr[i + 1]]:
                out[i] += vpart[p]
        outs.append(out)
    return R, outs[0], outs[1], sq


@pytest.mark.parametrize("seed,S,lmin,k", [(0, 7, 3.0, 5), (1, 3, 2.0, 8), (2, 50, 1e9, 4),
                                           (3, 1000, 1.0, 20), (4, 5, 0.0, 3), (5, 4, 2.0, 6)])
def test_plan_walk_matches_oracle(seed, S, lmin, k):
    m, n, rows, cols, vals = _zipf_instance(seed, 40, 60, 700)
    om, src = _input_cpu(m, n, rows, cols, vals)
    rng = rng_for(100 + seed)
    w = rng.standard_normal((m, k)).astype(np.float32).astype(np.float64)
    h = rng.standard_normal((n, k)).astype(np.float32).astype(np.float64)
    plan = ST.StagedPlan(src, k, S=min(S, ST.block_rows(k)), lmin=lmin, stage_min=0.5, grid=5,
                         tiles_per_cta=2)
    st = plan.stats()
    if lmin >= 1e9:
        assert st["blocks"] == [0, 0]          # everything cold
    R, RH, RtW, sq = _simulate(plan, w, h)
    rr, rh, rtw, sq0, _, _ = orc.sweep(om, w, h)
    assert not np.isnan(R).any()
    np.testing.assert_allclose(R, rr, rtol=0, atol=1e-12)
    np.testing.assert_allclose(RH, rh, rtol=0, atol=1e-11)
    np.testing.assert_allclose(RtW, rtw, rtol=0, atol=1e-11)
    assert abs(sq - sq0) <= 1e-12 * sq0
    # every chunk is 32-aligned inside one segment; tiles hold <= 64 chunks
    ch = plan.chunks.numpy()
    for (tp, block, c0, c1) in plan.tiles.numpy():
        assert 0 < c1 - c0 <= plan.groups
    assert (ch[:, 0] % 32 == 0).all()


def test_plan_rejects_bad_args():
    m, n, rows, cols, vals = _zipf_instance(5, 10, 12, 40)
    _, src = _input_cpu(m, n, rows, cols, vals)
    with pytest.raises(ValueError):
        ST.StagedPlan(src, 65)
    with pytest.raises(ValueError):
        ST.StagedPlan(src, 8, S=10 ** 6)
    empty = ST.StagedInput(3, 4, *(torch.zeros(0, dtype=torch.int32),) * 2,
                           torch.zeros(0, dtype=torch.float32),
                           *(torch.zeros(0, dtype=torch.int32),) * 2, torch.zeros(0, dtype=torch.float32))
    with pytest.raises(ValueError):
        ST.StagedPlan(empty, 8)


# --------------------------------------------------------------------- GPU


def _gpu_obs(m, n, rows, cols, vals):
    from paper_2204_14067_b200 import data as D
    return D.ObservationSet.from_coo(m, n, rows, cols, vals).with_dtype(torch.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 3, 8, 20, 30, 32, 40, 64])
@pytest.mark.parametrize("opts", [{}, {"S": 9, "lmin": 3.0, "stage_min": 0.5},
                                  {"S": 4, "lmin": 1e9}, {"S": 5, "lmin": 1.0, "stage_min": 0.0},
                                  {"l1_bytes": 2048, "lmin": 2.0, "stage_min": 0.5}])
def test_staged_sweep_matches_oracle(k, opts):
    from paper_2204_14067_b200 import mfsolver as MF
    m, n, rows, cols, vals = _zipf_instance(7 + k, 90, 130, 3000)
    obs = _gpu_obs(m, n, rows, cols, vals)
    om = orc.from_coo(m, n, rows, cols, vals)
    rng = rng_for(k)
    w = rng.standard_normal((m, k)).astype(np.float32)
    h = rng.standard_normal((n, k)).astype(np.float32)
    if "S" in opts:
        opts = dict(opts, S=min(opts["S"], ST.block_rows(k)))
    if "l1_bytes" in opts and k > 32:
        opts = dict(opts, l1_bytes=4096)
    plan = MF.SweepPlan(obs, k, staged=True, staged_opts=opts)
    wd = plan.pad(torch.from_numpy(w).cuda())
    hd = plan.pad(torch.from_numpy(h).cuda())
    plan.run(wd, hd)
    torch.cuda.synchronize()
    rr, rh, rtw, sq, w2, h2 = orc.sweep(om, w.astype(np.float64), h.astype(np.float64))
    R = plan.R.double().cpu().numpy()
    scale = np.abs(rr).max() + 1.0
    np.testing.assert_allclose(R, rr, rtol=0, atol=2e-5 * scale)
    np.testing.assert_allclose(plan.RH.double().cpu().numpy(), rh, rtol=0,
                               atol=2e-5 * (np.abs(rh).max() + 1.0))
    np.testing.assert_allclose(plan.RtW.double().cpu().numpy(), rtw, rtol=0,
                               atol=2e-5 * (np.abs(rtw).max() + 1.0))
    s = plan.sums.cpu().numpy()
    assert abs(s[0] - sq) <= 2e-5 * sq
    assert abs(s[1] - w2) <= 1e-12 * w2 and abs(s[2] - h2) <= 1e-12 * h2
    # bitwise deterministic
    R1, RH1, RtW1, s1 = plan.R.clone(), plan.RH.clone(), plan.RtW.clone(), plan.sums.clone()
    plan.run(wd, hd)
    torch.cuda.synchronize()
    assert torch.equal(R1, plan.R) and torch.equal(RH1, plan.RH) and torch.equal(RtW1, plan.RtW)
    assert torch.equal(s1, plan.sums)


@pytest.mark.gpu
def test_staged_sweep_matches_grouped_sweep_c2_scale():
    from paper_2204_14067_b200 import data as D
    from paper_2204_14067_b200 import mfsolver as MF
    from paper_2204_14067_b200 import synth
    m, n, r, c, v = synth.generate("c2", scale=0.25, seed=3)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    obs = D.ObservationSet.from_coo(m, n, r, c, v).with_dtype(torch.float32)
    k = 20
    w, h = synth.sweep_factors(m, n, k, seed=4, dtype=np.float32)
    a = MF.SweepPlan(obs, k)
    b = MF.SweepPlan(obs, k, staged=True)
    wa, ha = a.pad(torch.from_numpy(w).cuda()), a.pad(torch.from_numpy(h).cuda())
    a.run(wa, ha)
    b.run(b.pad(torch.from_numpy(w).cuda()), b.pad(torch.from_numpy(h).cuda()))
    torch.cuda.synchronize()
    for x, y in ((a.R, b.R), (a.RH, b.RH), (a.RtW, b.RtW)):
        x, y = x.double(), y.double()
        assert torch.max(torch.abs(x - y)).item() <= 2e-5 * (torch.max(torch.abs(x)).item() + 1.0)
    sa, sb = a.sums.cpu().numpy(), b.sums.cpu().numpy()
    assert abs(sa[0] - sb[0]) <= 1e-5 * sa[0]
    assert sa[1] == pytest.approx(sb[1], rel=1e-12) and sa[2] == pytest.approx(sb[2], rel=1e-12)
    # end to end through host buffers
    wh = torch.from_numpy(w).pin_memory()
    hh = torch.from_numpy(h).pin_memory()
    sums, RH, RtW = b.run_host(wh, hh)
    torch.cuda.synchronize()
    assert torch.equal(RH, b.RH.cpu()) and torch.equal(RtW, b.RtW.cpu())


def test_plan_walk_l1_blocked_matches_oracle():
    """L1-blocked plans: block-ordered stream, every tile gathers globally."""
    m, n, rows, cols, vals = _zipf_instance(6, 40, 60, 700)
    om, src = _input_cpu(m, n, rows, cols, vals)
    rng = rng_for(106)
    k = 6
    w = rng.standard_normal((m, k)).astype(np.float32).astype(np.float64)
    h = rng.standard_normal((n, k)).astype(np.float32).astype(np.float64)
    plan = ST.StagedPlan(src, k, S=5, lmin=2.0, stage_min=0.5, grid=5, l1_bytes=1)
    assert plan.stats()["mode"] == "l1-blocked" and max(plan.stats()["blocks"]) > 1
    assert (plan.tiles.numpy()[:, 1] == -1).all()
    R, RH, RtW, sq = _simulate(plan, w, h)
    rr, rh, rtw, sq0, _, _ = orc.sweep(om, w, h)
    np.testing.assert_allclose(R, rr, rtol=0, atol=1e-12)
    np.testing.assert_allclose(RH, rh, rtol=0, atol=1e-11)
    np.testing.assert_allclose(RtW, rtw, rtol=0, atol=1e-11)
    assert abs(sq - sq0) <= 1e-12 * sq0

