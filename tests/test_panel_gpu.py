"""The hybrid sweep (hot entries from shared-memory panels, csrc/panel.cu; cold
entries through the gather kernel) against the CPU oracle's sweep
(oracle/mfg_oracle.py: mfg/data.py:253-293, mfg/operators.py:108,117)."""
import numpy as np
import pytest
import torch

from oracle import mfg_oracle as orc
from paper_2204_14067_b200 import data as D
from paper_2204_14067_b200 import synth

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().double().cpu().numpy()


def _check(plan, om, wt, ht, k):
    plan.run(plan.pad(wt), plan.pad(ht))
    rr, rh, rtw, sq, w2, h2 = orc.sweep(om, _np(wt), _np(ht))
    tol = 2e-5  # fp32 storage and arithmetic against the fp64 oracle on the same fp32 inputs
    sc = lambda a: max(1.0, np.abs(a).max())  # noqa: E731
    assert np.max(np.abs(_np(plan.R) - rr)) <= tol * sc(rr)
    assert np.max(np.abs(_np(plan.RH) - rh)) <= tol * 10 * sc(rh)
    assert np.max(np.abs(_np(plan.RtW) - rtw)) <= tol * 10 * sc(rtw)
    sums = plan.sums.cpu().numpy()
    assert sums[0] == pytest.approx(sq, rel=tol * 10)
    assert sums[1] == pytest.approx(w2, rel=1e-12)
    assert sums[2] == pytest.approx(h2, rel=1e-12)
    keep = [plan.R.clone(), plan.RH.clone(), plan.RtW.clone(), plan.sums.clone()]
    plan.run(plan.pad(wt), plan.pad(ht))
    for a, b in zip(keep, [plan.R, plan.RH, plan.RtW, plan.sums]):
        assert torch.equal(a, b)  # bitwise run to run


@pytest.mark.parametrize("cold", ["pieces", "gather"])
@pytest.mark.parametrize("k", [40, 30, 32, 64])
@pytest.mark.parametrize("cfg", [
    dict(),                                              # defaults
    dict(lmin=1, lmax=5, max_panels=3),                   # short pieces, few panels
    dict(lmin=10 ** 9),                                   # nothing hot: all entries cold
    dict(lmin=1, max_panels=10 ** 6, min_panel_entries=1),  # every entry hot
])
def test_hybrid_sweep_vs_oracle(k, cfg, cold):
    from paper_2204_14067_b200.panel import HybridSweepPlan
    m, n, r, c, v = synth.generate("c3", scale=0.03, seed=200 + k)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    v32 = v.astype(np.float32).astype(np.float64)
    om = orc.from_coo(m, n, r, c, v32)
    w, h = synth.sweep_factors(m, n, k, seed=k)
    obs = D.ObservationSet.from_coo(m, n, r, c, v32, dtype=torch.float32)
    wt = torch.as_tensor(w).float().cuda()
    ht = torch.as_tensor(h).float().cuda()
    plan = HybridSweepPlan(obs, k, cold=cold, **cfg)
    assert plan.cold == (cold if k != 64 else "gather")
    if cfg.get("lmin", 0) >= 10 ** 9:
        assert plan.stats["csr_hot"] == 0 and plan.stats["csc_hot"] == 0
    if cfg.get("max_panels", 0) >= 10 ** 6:
        assert plan.stats["csr_hot"] == obs.size and plan.stats["csc_hot"] == obs.size
    _check(plan, om, wt, ht, k)


def test_hybrid_sweep_small_and_ragged():
    """Rows with no entries, a single entry, and a panel that is only partly filled."""
    from paper_2204_14067_b200.panel import HybridSweepPlan
    rng = np.random.default_rng(5)
    m, n, k = 37, 91, 40
    mask = rng.random((m, n)) < 0.2
    mask[3, :] = False
    mask[:, 7] = False
    mask[11, :] = False
    mask[11, 5] = True
    r, c = np.nonzero(mask)
    v = rng.integers(1, 6, size=len(r)).astype(np.float64)
    om = orc.from_coo(m, n, r, c, v)
    obs = D.ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    w, h = synth.sweep_factors(m, n, k, seed=3)
    wt = torch.as_tensor(w).float().cuda()
    ht = torch.as_tensor(h).float().cuda()
    for cfg in (dict(lmin=1, min_panel_entries=1), dict(lmin=2, lmax=3, min_panel_entries=1),
                dict(lmin=4, lmax=9, min_panel_entries=1, cold="gather")):
        plan = HybridSweepPlan(obs, k, **cfg)
        assert plan.stats["csr_hot"] > 0
        _check(plan, om, wt, ht, k)


def test_hybrid_rejects_unsupported():
    from paper_2204_14067_b200.panel import HybridSweepPlan
    m, n, r, c, v = synth.generate("c2", scale=0.05, seed=1)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    obs64 = D.ObservationSet.from_coo(m, n, r, c, v)
    with pytest.raises(ValueError):
        HybridSweepPlan(obs64, 40)
    obs32 = obs64.with_dtype(torch.float32)
    with pytest.raises(ValueError):
        HybridSweepPlan(obs32, 20)


def test_hybrid_run_host_and_plan_choice():
    """End to end from pinned host factors (eager and as a replayed CUDA graph)
    equals the resident run; best_sweep_plan returns a plan of either kind
    with the same results."""
    from paper_2204_14067_b200.panel import HybridSweepPlan, best_sweep_plan
    k = 40
    m, n, r, c, v = synth.generate("c3", scale=0.03, seed=77)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    obs = D.ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    w, h = synth.sweep_factors(m, n, k, seed=5)
    plan = HybridSweepPlan(obs, k)
    wt = torch.as_tensor(w).float().cuda()
    ht = torch.as_tensor(h).float().cuda()
    plan.run(plan.pad(wt), plan.pad(ht))
    ref = [plan.sums.clone().cpu(), plan.RH.clone().cpu(), plan.RtW.clone().cpu()]
    wa, ha = plan.pinned_factors()
    wa.copy_(torch.as_tensor(w).float())
    ha.copy_(torch.as_tensor(h).float())
    wh = torch.as_tensor(w).float().pin_memory()
    hh = torch.as_tensor(h).float().pin_memory()
    for (a, b) in ((wa, ha), (wh, hh)):
        for graph in (False, True, True):
            out = plan.run_host(a, b, graph=graph)
            torch.cuda.synchronize()
            for x, y in zip(out, ref):
                assert torch.equal(x, y)
    for mode in ("gather", "hybrid", "auto"):
        p = best_sweep_plan(obs, k, mode=mode)
        assert p.kind == (mode if mode != "auto" else p.kind)
        p.run(p.pad(wt), p.pad(ht))
        assert torch.allclose(p.RH.cpu(), ref[1], rtol=0, atol=2e-4 * float(ref[1].abs().max()))
        assert float(p.sums[0]) == pytest.approx(float(ref[0][0]), rel=1e-6)


@pytest.mark.parametrize("cold", ["pieces", "gather"])
def test_hybrid_out_scale_and_no_r(cold):
    """out_scale multiplies R.H and R^T.W on every path (folded rows, rows a
    single cold piece writes directly, the gather kernel's rows); want_r=False
    skips the residual output."""
    from paper_2204_14067_b200.panel import HybridSweepPlan
    k = 40
    m, n, r, c, v = synth.generate("c3", scale=0.02, seed=91)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    v32 = v.astype(np.float32).astype(np.float64)
    om = orc.from_coo(m, n, r, c, v32)
    obs = D.ObservationSet.from_coo(m, n, r, c, v32, dtype=torch.float32)
    w, h = synth.sweep_factors(m, n, k, seed=9)
    wt = torch.as_tensor(w).float().cuda()
    ht = torch.as_tensor(h).float().cuda()
    plan = HybridSweepPlan(obs, k, want_r=False, out_scale=2.0, cold=cold)
    assert plan.R is None
    if cold == "pieces":
        assert plan.p1.n_direct > 0          # light columns: one cold piece each
    plan.run(plan.pad(wt), plan.pad(ht))
    rr, rh, rtw, sq, w2, h2 = orc.sweep(om, _np(wt), _np(ht))
    sc = lambda a: max(1.0, np.abs(a).max())  # noqa: E731
    assert np.max(np.abs(_np(plan.RH) - 2.0 * rh)) <= 4e-4 * sc(rh)
    assert np.max(np.abs(_np(plan.RtW) - 2.0 * rtw)) <= 4e-4 * sc(rtw)
    sums = plan.sums.cpu().numpy()
    assert sums[0] == pytest.approx(sq, rel=2e-4)
    assert sums[1] == pytest.approx(w2, rel=1e-12) and sums[2] == pytest.approx(h2, rel=1e-12)
    # a second sweep with other factors reuses the plan (outputs fully rewritten)
    w3, h3 = synth.sweep_factors(m, n, k, seed=10)
    wt3 = torch.as_tensor(w3).float().cuda()
    ht3 = torch.as_tensor(h3).float().cuda()
    plan.run(plan.pad(wt3), plan.pad(ht3))
    _, rh3, rtw3, sq3, _, _ = orc.sweep(om, _np(wt3), _np(ht3))
    assert np.max(np.abs(_np(plan.RH) - 2.0 * rh3)) <= 4e-4 * sc(rh3)
    assert np.max(np.abs(_np(plan.RtW) - 2.0 * rtw3)) <= 4e-4 * sc(rtw3)
    assert plan.sums.cpu().numpy()[0] == pytest.approx(sq3, rel=2e-4)


@pytest.mark.parametrize("k", [40, 30])
@pytest.mark.parametrize("sizes", ["5,15,25,25,20,10", "100", "50,50", "1,1,1,1,1,1,1,1,1,1,1,1"])
def test_hybrid_run_host_chunk_profiles(k, sizes, monkeypatch):
    """The end-to-end pipeline over chunks of H (any chunk profile, padded and
    unpadded factor rows) is bitwise equal to the resident sweep, eagerly and as
    a replayed CUDA graph, and matches the oracle."""
    from paper_2204_14067_b200.panel import HybridSweepPlan
    monkeypatch.setenv("MFG_PANEL_CHUNK_SIZES", sizes)
    m, n, r, c, v = synth.generate("c3", scale=0.03, seed=300 + k)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    v32 = v.astype(np.float32).astype(np.float64)
    om = orc.from_coo(m, n, r, c, v32)
    obs = D.ObservationSet.from_coo(m, n, r, c, v32, dtype=torch.float32)
    w, h = synth.sweep_factors(m, n, k, seed=6)
    plan = HybridSweepPlan(obs, k)
    assert plan.nchunks == len(sizes.split(","))
    wt = torch.as_tensor(w).float().cuda()
    ht = torch.as_tensor(h).float().cuda()
    _check(plan, om, wt, ht, k)
    ref = [plan.sums.clone().cpu(), plan.RH.clone().cpu(), plan.RtW.clone().cpu()]
    R0 = plan.R.clone()
    wa, ha = plan.pinned_factors()
    wa.copy_(torch.as_tensor(w).float())
    ha.copy_(torch.as_tensor(h).float())
    for graph in (False, True, True):
        plan.R.zero_()
        out = plan.run_host(wa, ha, graph=graph)
        torch.cuda.synchronize()
        for x, y in zip(out, ref):
            assert torch.equal(x, y)
        assert torch.equal(plan.R, R0)
