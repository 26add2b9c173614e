"""GPU parity of the libmfg_b200 kernels against the oracle / reference goldens.

Tolerances: index handling bit-exact; fp64 values within 1e-12 (the
reference's own dense-comparison tolerance, tests/test_data.py:114-120);
fp32 storage within 1e-5 relative of the fp64 oracle (dot products of k
fp32 terms, fp32 accumulation).
"""

import numpy as np
import pytest
import torch

from oracle import mfg_oracle as orc

pytestmark = pytest.mark.gpu

from paper_2204_14067_b200 import data as D  # noqa: E402
from paper_2204_14067_b200 import mfsolver as MF  # noqa: E402
from paper_2204_14067_b200 import operators as OP  # noqa: E402
from paper_2204_14067_b200 import synth  # noqa: E402
from paper_2204_14067_b200.operators import FactorPair  # noqa: E402


def _np(t):
    return t.detach().double().cpu().numpy()


def test_omega_build_bit_exact(golden):
    g = golden("omega.npz")
    for ci in range(4):
        p = f"c{ci}_"
        obs = D.ObservationSet.from_coo(int(g[p + "m"]), int(g[p + "n"]), g[p + "in_rows"],
                                        g[p + "in_cols"], g[p + "in_vals"])
        assert np.array_equal(obs.rows, g[p + "rows"])
        assert np.array_equal(obs.cols, g[p + "cols"])
        assert np.array_equal(obs.vals, g[p + "vals"])
        assert np.array_equal(obs.indptr, g[p + "indptr"])
        d = obs.dev
        assert np.array_equal(d.csc.ptr.cpu().numpy(), g[p + "csc_ptr"])
        assert np.array_equal(d.csc.idx.cpu().numpy(), g[p + "csc_idx"])
        assert np.array_equal(d.vals_csc.cpu().numpy(), g[p + "csc_val"])


def test_omega_build_errors(golden):
    g = golden("omega.npz")
    with pytest.raises(D.DatasetError) as err:
        D.ObservationSet.from_coo(3, 3, [2, 0, 2, 1], [1, 0, 1, 2], [1.0, 2.0, 3.0, 4.0])
    assert str(err.value) == str(g["dup_msg"])
    for bad, args in [("row_range", (2, 2, [0, 2], [0, 0], [1.0, 1.0])),
                      ("col_range", (2, 2, [0, 1], [0, -1], [1.0, 1.0])),
                      ("length", (2, 2, [0, 1], [0], [1.0, 1.0]))]:
        with pytest.raises(D.DatasetError) as err:
            D.ObservationSet.from_coo(*args)
        assert str(err.value) == str(g["err_" + bad])
    obs = D.ObservationSet.from_coo(3, 4, [], [], [])
    assert np.array_equal(obs.indptr, g["empty_indptr"])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_sweep_matches_golden(golden, dtype):
    g = golden("sweep.npz")
    for name in g.names():
        p = name + "_"
        obs = D.ObservationSet.from_coo(*g.obs_args(p), dtype=dtype)
        wf = FactorPair(torch.as_tensor(g[p + "w"]).to(dtype), torch.as_tensor(g[p + "h"]).to(dtype))
        R, RH, RtW, sums = MF.sweep(obs, wf, want_r=True, want_rh=True, want_rtw=True,
                                    compute_f64=False)
        if dtype == torch.float64:
            tol = 1e-12
            assert np.max(np.abs(_np(R) - g[p + "r"]), initial=0) < tol, name
            assert np.max(np.abs(_np(RH) - g[p + "rh"]), initial=0) < tol, name
            assert np.max(np.abs(_np(RtW) - g[p + "rtw"]), initial=0) < tol, name
            assert sums[0] == pytest.approx(float(g[p + "loss"]), rel=1e-12, abs=1e-300)
            assert sums[1] + sums[2] == pytest.approx(float(g[p + "frob"]), rel=1e-12)
        else:
            # fp32 storage: compare with the oracle evaluated on the rounded inputs
            om = orc.from_coo(*g.obs_args(p))
            w32, h32 = _np(wf.w), _np(wf.h)
            om32 = orc.from_coo(om.m, om.n, om.rows, om.cols, om.vals.astype(np.float32))
            r, rh, rtw, sq, w2, h2 = orc.sweep(om32, w32, h32)
            scale = max(1.0, np.abs(r).max(initial=0))
            assert np.max(np.abs(_np(R) - r), initial=0) <= 1e-5 * scale, name
            assert np.max(np.abs(_np(RH) - rh), initial=0) <= 1e-5 * max(1.0, np.abs(rh).max(initial=0)), name
            assert np.max(np.abs(_np(RtW) - rtw), initial=0) <= 1e-5 * max(1.0, np.abs(rtw).max(initial=0)), name
            assert sums[0] == pytest.approx(sq, rel=1e-5, abs=1e-30)
            assert sums[1] == pytest.approx(w2, rel=1e-12)
            assert sums[2] == pytest.approx(h2, rel=1e-12)


def test_residual_and_loss_match_golden(golden):
    g = golden("sweep.npz")
    for name in g.names():
        p = name + "_"
        obs = D.ObservationSet.from_coo(*g.obs_args(p))
        wf = FactorPair(g[p + "w"], g[p + "h"])
        res = D.residual_on_omega(obs, wf)
        assert np.max(np.abs(_np(res.vals) - g[p + "r"]), initial=0) < 1e-12
        assert D.loss_quad(res) == pytest.approx(float(g[p + "loss"]), rel=1e-12, abs=1e-300)
        from paper_2204_14067_b200.kernels import SvdTriplet
        x = SvdTriplet(g[p + "tu"], g[p + "ts"], g[p + "tv"])
        rs = D.residual_on_omega_svd(obs, x)
        assert np.max(np.abs(_np(rs.vals) - g[p + "tres"]), initial=0) < 1e-12


def test_bcd_matches_golden(golden):
    g = golden("bcd.npz")
    for name in g.names():
        p = name + "_"
        obs = D.ObservationSet.from_coo(*g.obs_args(p))
        lam = float(g[p + "lam"])
        wf = FactorPair(g[p + "w"], g[p + "h"])
        e1 = MF.bcd_epoch(obs, wf, lam)
        # reference tolerance for BCD vs an independent dense BCD: 1e-10
        assert np.max(np.abs(_np(e1.w) - g[p + "w1"])) < 1e-10, name
        assert np.max(np.abs(_np(e1.h) - g[p + "h1"])) < 1e-10, name
        o0 = MF.mf_objective(obs, wf, lam)
        o1 = MF.mf_objective(obs, e1, lam)
        assert o0 == pytest.approx(float(g[p + "obj0"]), rel=1e-12)
        assert o1 == pytest.approx(float(g[p + "obj1"]), rel=1e-10)
        e3 = MF.mf_phase(obs, wf, lam, 3)
        assert MF.mf_objective(obs, e3, lam) == pytest.approx(float(g[p + "obj3"]), rel=1e-10)


def test_operator_matches_golden(golden):
    g = golden("operator.npz")
    for name in g.names():
        p = name + "_"
        obs = D.ObservationSet.from_coo(*g.obs_args(p))
        wf = FactorPair(g[p + "w"], g[p + "h"])
        grad = D.SparseResidual(obs.m, obs.n, obs, torch.as_tensor(g[p + "g"]).cuda())
        op = OP.ShiftedOperator(wf, grad, float(g[p + "alpha"]))
        for fn, blk, key in [(op.apply, "bn", "apply"), (op.apply_t, "bm", "apply_t"),
                             (op.apply_gram, "bm", "apply_gram"), (op.project_rows, "q", "project")]:
            ref = g[p + key]
            got = _np(fn(g[p + blk]))
            assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.abs(ref).max()), (name, key)
        assert op.frob_sq() == pytest.approx(float(g[p + "frob_sq"]), rel=1e-10)
        from paper_2204_14067_b200.kernels import SvdTriplet
        t1 = SvdTriplet(g[p + "t1u"], g[p + "t1s"], g[p + "t1v"])
        assert OP.inner_product(t1, wf) == pytest.approx(float(g[p + "ip_tf"]), rel=1e-10, abs=1e-12)
        assert OP.frob_dist_sq(t1, wf) == pytest.approx(float(g[p + "dist_tf"]), rel=1e-10)


@pytest.mark.parametrize("p", [1, 7, 32, 33, 128, 200, 300])
def test_spmm_widths_vs_oracle(p):
    m, n, r, c, v = synth.generate("c2", scale=0.05, seed=3)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    obs = D.ObservationSet.from_coo(m, n, r, c, v)
    om = orc.from_coo(m, n, r, c, v)
    rng = np.random.default_rng(p)
    gv = rng.standard_normal(om.size)
    grad = D.SparseResidual(m, n, obs, torch.as_tensor(gv).cuda())
    xb = rng.standard_normal((n, p))
    yb = rng.standard_normal((m, p))
    y0 = torch.as_tensor(rng.standard_normal((m, p))).cuda()
    got = OP.spmm(grad, torch.as_tensor(xb).cuda(), False, 0.5, -2.0, y0.clone())
    ref = 0.5 * orc.spmm_csr(om, gv, xb) - 2.0 * y0.cpu().numpy()
    assert np.max(np.abs(_np(got) - ref)) < 1e-11
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    got_t = OP.spmm(grad, torch.as_tensor(yb).cuda(), True, 1.0, 0.0, out)
    ref_t = orc.spmm_csc(om, gv, yb)
    assert np.max(np.abs(_np(got_t) - ref_t)) < 1e-11


@pytest.mark.parametrize("k", [1, 8, 20, 33, 40, 64, 100, 150])
def test_sweep_zipf_vs_oracle(k):
    """Zipf-skewed instance (saturated rows, hot columns), several k."""
    m, n, r, c, v = synth.generate("c3", scale=0.03, seed=k)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    om = orc.from_coo(m, n, r, c, v)
    w, h = synth.sweep_factors(m, n, k, seed=k)
    for dtype in (torch.float64, torch.float32):
        obs = D.ObservationSet.from_coo(m, n, r, c, v, dtype=dtype)
        wf = FactorPair(torch.as_tensor(w).to(dtype), torch.as_tensor(h).to(dtype))
        R, RH, RtW, sums = MF.sweep(obs, wf, want_r=True, want_rh=True, want_rtw=True,
                                    compute_f64=False)
        ww, hh = _np(wf.w), _np(wf.h)
        rr, rh, rtw, sq, w2, h2 = orc.sweep(om, ww, hh)
        tol = 1e-11 if dtype == torch.float64 else 2e-5
        sc = lambda a: max(1.0, np.abs(a).max())  # noqa: E731
        assert np.max(np.abs(_np(R) - rr)) <= tol * sc(rr)
        assert np.max(np.abs(_np(RH) - rh)) <= tol * sc(rh) * (10 if dtype == torch.float32 else 1)
        assert np.max(np.abs(_np(RtW) - rtw)) <= tol * sc(rtw) * (10 if dtype == torch.float32 else 1)
        assert sums[0] == pytest.approx(sq, rel=tol * 10)


def test_sweep_deterministic_and_identities():
    m, n, r, c, v = synth.generate("c2", scale=0.2, seed=5)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    obs = D.ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    w, h = synth.sweep_factors(m, n, 20, seed=2, dtype=np.float32)
    wf = FactorPair(torch.as_tensor(w), torch.as_tensor(h))
    a = MF.sweep(obs, wf, want_r=True, want_rh=True, want_rtw=True, compute_f64=False)
    b = MF.sweep(obs, wf, want_r=True, want_rh=True, want_rtw=True, compute_f64=False)
    for x, y in zip(a[:3], b[:3]):
        assert torch.equal(x, y)
    assert np.array_equal(a[3], b[3])
    # <R.H, W> = <R^T.W, H> = sum r (r + A)
    R, RH, RtW, _ = a
    lhs = float((RH.double() * wf.w.double()).sum())
    rhs = float((RtW.double() * wf.h.double()).sum())
    ra = float((R.double() * (R.double() + obs.dev.vals.double())).sum())
    assert lhs == pytest.approx(rhs, rel=1e-4)
    assert lhs == pytest.approx(ra, rel=1e-4)


@pytest.mark.parametrize("k", [3, 8, 16, 20, 24, 30, 32, 36, 40, 44, 48, 56, 64])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("layout", ["plan", "padded"])
def test_grouped_sweep_vs_oracle(k, dtype, layout):
    """The grouped (8-lane group) sweep kernel, with factors in the plan's
    layout (mfg_sweep_ld: unpadded ld = k where the kernel takes it) and
    zero-padded to kp; k > kp falls back to the warp-per-chunk kernel."""
    from paper_2204_14067_b200.mfsolver import SweepPlan
    m, n, r, c, v = synth.generate("c3", scale=0.03, seed=100 + k)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    om = orc.from_coo(m, n, r, c, v)
    w, h = synth.sweep_factors(m, n, k, seed=k)
    obs = D.ObservationSet.from_coo(m, n, r, c, v, dtype=dtype)
    plan = SweepPlan(obs, k)
    wt = torch.as_tensor(w).to(dtype).cuda()
    ht = torch.as_tensor(h).to(dtype).cuda()
    if layout == "padded" and plan.kp:
        def pad(f):
            out = torch.zeros((f.shape[0], plan.kp), dtype=dtype, device="cuda")
            out[:, :k] = f
            return out
        plan.pad = pad
    plan.run(plan.pad(wt), plan.pad(ht))
    rr, rh, rtw, sq, w2, h2 = orc.sweep(om, _np(wt), _np(ht))
    tol = 1e-11 if dtype == torch.float64 else 2e-5
    sc = lambda a: max(1.0, np.abs(a).max())  # noqa: E731
    amp = 1 if dtype == torch.float64 else 10
    assert np.max(np.abs(_np(plan.R) - rr)) <= tol * sc(rr)
    assert np.max(np.abs(_np(plan.RH) - rh)) <= tol * amp * sc(rh)
    assert np.max(np.abs(_np(plan.RtW) - rtw)) <= tol * amp * sc(rtw)
    sums = plan.sums.cpu().numpy()
    assert sums[0] == pytest.approx(sq, rel=tol * 10)
    assert sums[1] == pytest.approx(w2, rel=1e-12)
    assert sums[2] == pytest.approx(h2, rel=1e-12)
    # run-to-run bitwise determinism
    R0, RH0 = plan.R.clone(), plan.RH.clone()
    plan.run(plan.pad(wt), plan.pad(ht))
    assert torch.equal(R0, plan.R) and torch.equal(RH0, plan.RH)
    # end-to-end entry point from host factors: same results, eager and as a
    # replayed CUDA graph (which reads the host buffers at replay time)
    RtW0 = plan.RtW.clone()
    wh = torch.as_tensor(w).to(dtype).pin_memory()
    hh = torch.as_tensor(h).to(dtype).pin_memory()
    wa, ha = plan.pinned_factors()          # adjacent buffers: the one-copy path
    wa.copy_(wh)
    ha.copy_(hh)
    for wx, hx, graph in ((wh, hh, False), (wh, hh, True), (wh, hh, True), (wa, ha, False),
                          (wa, ha, True)):
        sums_h, rh_h, rtw_h = plan.run_host(wx, hx, graph=graph)
        torch.cuda.synchronize()
        assert torch.equal(rh_h, RH0.cpu()) and torch.equal(rtw_h, RtW0.cpu())
    for graph in (False, True, True):
        sums_h, rh_h, rtw_h = plan.run_host(wh, hh, graph=graph)
        torch.cuda.synchronize()
        assert torch.equal(rh_h, RH0.cpu()) and torch.equal(rtw_h, RtW0.cpu())
        sh = sums_h.numpy()
        assert sh[0] == sums[0]                              # same per-entry order
        assert np.allclose(sh[1:], sums[1:], rtol=1e-13)     # norms: layout-dependent slices
    wh.mul_(0.5)   # new contents in the same pinned buffers -> the graph sees them
    sums_h, rh_h, _ = plan.run_host(wh, hh)
    torch.cuda.synchronize()
    rr2, rh2, _, sq2, _, _ = orc.sweep(om, _np(wt) * 0.5, _np(ht))
    assert np.max(np.abs(rh_h.double().numpy() - rh2)) <= tol * amp * sc(rh2)
    assert sums_h.numpy()[0] == pytest.approx(sq2, rel=tol * 10)


@pytest.mark.parametrize("k", [130, 150, 200, 260, 300])
def test_bcd_large_k_packed_and_dual(k):
    """k > 128: packed shared-memory Cholesky; rows with fewer entries than k
    take the push-through (dual) d x d solve. Rows here have ~200 entries on
    the CSR side (primal for k <= 200) and ~15 on the CSC side (dual)."""
    rng = np.random.default_rng(k)
    m, n = 30, 400
    mask = rng.random((m, n)) < 0.5
    r, c = np.nonzero(mask)
    v = rng.standard_normal(r.size)
    om = orc.from_coo(m, n, r, c, v)
    w = rng.standard_normal((m, k)) * 0.3
    h = rng.standard_normal((n, k)) * 0.3
    obs = D.ObservationSet.from_coo(m, n, r, c, v)
    out = MF.bcd_epoch(obs, FactorPair(w, h), 1.7)
    w1, h1 = orc.bcd_epoch(om, w, h, 1.7)
    assert np.max(np.abs(_np(out.w) - w1)) < 1e-9 * max(1.0, np.abs(w1).max())
    assert np.max(np.abs(_np(out.h) - h1)) < 1e-9 * max(1.0, np.abs(h1).max())


@pytest.mark.parametrize("k", [1, 4, 5, 20, 37, 40, 41, 49, 57, 64, 65, 128])
def test_bcd_split_heavy_rows(k):
    """Rows with more than S = max(256, nnz/grid) entries are cut into
    segments whose partial Grams are summed in segment order by the CTA that
    finishes the row (bcd.cu SplitPlan). A few rows here hold 600-3000
    entries (2-12 segments) among many light ones, on both orientations;
    the epoch must match the oracle's per-row normal equations, and a second
    run must be bitwise identical (fixed reduction order). k <= 40 takes the
    small-k entry-group instantiation (bcd.cu small_k_path), 41 is the first
    k on the plain path, and 1, 5, 37 leave a ragged last 4x4 tile."""
    rng = np.random.default_rng(100 + k)
    m, n = 400, 3000
    deg = rng.integers(1, 30, size=m)
    deg[:6] = [3000, 2500, 1200, 800, 600, 257]
    rows, cols = [], []
    for i, d in enumerate(deg):
        cc = rng.choice(n, size=d, replace=False)
        if 7 not in cc:                  # column 7 in every row: a split CSC row too
            cc = np.append(cc, 7)
        rows.append(np.full(cc.size, i))
        cols.append(cc)
    r, c = np.concatenate(rows), np.concatenate(cols)
    perm = rng.permutation(m)           # heavy rows scattered, not first
    r = perm[r]
    v = rng.standard_normal(r.size)
    om = orc.from_coo(m, n, r, c, v)
    w = rng.standard_normal((m, k)) * 0.3
    h = rng.standard_normal((n, k)) * 0.3
    obs = D.ObservationSet.from_coo(m, n, r, c, v)
    out = MF.bcd_epoch(obs, FactorPair(w, h), 1.3)
    out2 = MF.bcd_epoch(obs, FactorPair(w, h), 1.3)
    w1, h1 = orc.bcd_epoch(om, w, h, 1.3)
    assert np.max(np.abs(_np(out.w) - w1)) < 1e-9 * max(1.0, np.abs(w1).max())
    assert np.max(np.abs(_np(out.h) - h1)) < 1e-9 * max(1.0, np.abs(h1).max())
    assert torch.equal(out.w, out2.w) and torch.equal(out.h, out2.h)
