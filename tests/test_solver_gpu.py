"""GPU parity of the lifting step and the end-to-end solvers against traces
produced by the reference itself (tests/golden/make_golden.py).

Bar (BASELINE.json north_star): identical identified rank at every outer
iteration and per-iteration objective within 1e-9 relative in fp64 mode.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2204_14067_b200 as P  # noqa: E402
from paper_2204_14067_b200 import data as D  # noqa: E402
from paper_2204_14067_b200 import eigensolver as E  # noqa: E402
from paper_2204_14067_b200 import kernels as K  # noqa: E402
from paper_2204_14067_b200 import operators as OP  # noqa: E402
from paper_2204_14067_b200 import proxlift as PL  # noqa: E402


def _np(t):
    return t.detach().double().cpu().numpy()


def test_dense_kernels_match_golden(golden):
    g = golden("kernels.npz")
    for name in [str(s) for s in g["orth_names"]]:
        q, rank = K.orthonormalize(g["orth_" + name + "_in"])
        assert rank == int(g["orth_" + name + "_rank"]), name
        qq = _np(q)
        # the near-dependent case keeps a direction fixed only to ~eps/1e-9
        atol = 1e-5 if name == "near" else 1e-10
        assert np.allclose(qq @ qq.T, g["orth_" + name + "_proj"], atol=atol), name
    for i in range(int(g["st_count"])):
        sig, kept, lt = K.soft_threshold(g[f"st{i}_in"], float(g[f"st{i}_beta"]))
        assert np.array_equal(sig, g[f"st{i}_sigma"])
        assert np.array_equal(kept, g[f"st{i}_kept"])
    for i in range(int(g["svd_count"])):
        mat = g[f"svd{i}_in"]
        u, s, v = K.exact_svd_short_fat(mat)
        assert np.allclose(s, g[f"svd{i}_s"], rtol=1e-10, atol=1e-10 * s.max())
        rec = (_np(u) * s) @ _np(v).T
        assert np.linalg.norm(rec - mat) <= 1e-10 * np.linalg.norm(mat)


def _op_from(g, p):
    obs = D.ObservationSet.from_coo(*g.obs_args(p))
    wf = OP.FactorPair(g[p + "w"], g[p + "h"])
    grad = D.SparseResidual(obs.m, obs.n, obs, torch.as_tensor(g[p + "g"]).cuda())
    return obs, wf, grad


def test_eigensolvers_match_golden(golden):
    g = golden("eigprox.npz")
    for seed in range(3):
        p = f"eig{seed}_"
        obs, wf, grad = _op_from(g, p)
        op = OP.ShiftedOperator(wf, grad, float(g[p + "alpha"]))
        for meth in ("lm-krylov", "power"):
            cfg = E.EigConfig(memory=3, max_iters=40, residual_tol=1e-9, method=meth)
            res = E.solve_topk(op, g[p + "r0"], cfg)
            ref_w = g[p + meth + "_w"]
            assert np.max(np.abs(res.eigvals - ref_w)) <= 1e-9 * ref_w[0], (seed, meth)
            # at residual_tol 3e-12 relative the sweep count depends on
            # LAPACK-vs-cuSOLVER rounding; it must stay close
            assert abs(res.iters_used - int(g[p + meth + "_iters"])) <= 5, (seed, meth)
            assert res.converged == bool(g[p + meth + "_conv"])


def test_prox_step_matches_golden(golden):
    g = golden("eigprox.npz")
    for seed in range(4):
        p = f"prox{seed}_"
        obs = D.ObservationSet.from_coo(*g.obs_args(p))
        wf = OP.FactorPair(g[p + "w"], g[p + "h"])
        grad = D.gradient(D.residual_on_omega(obs, wf))
        params = PL.StepParams(lam=1.0)
        cfg = E.EigConfig(memory=3, max_iters=200, residual_tol=1e-10)
        o = PL.inexact_prox_step(obs, wf, grad, 2.0, params, g[p + "r0"], cfg, eps_target=1e-4)
        assert o.x_next.rank == int(g[p + "rank"]), seed
        assert o.backtracks == int(g[p + "backtracks"])
        assert o.alpha_used == float(g[p + "alpha"])
        assert o.f_next == pytest.approx(float(g[p + "f_next"]), rel=1e-9)
        assert o.f_base == pytest.approx(float(g[p + "f_base"]), rel=1e-12)
        assert np.allclose(o.x_next.sigma, g[p + "sigma"], rtol=1e-9)
        assert np.max(np.abs(_np(o.x_next.dense()) - g[p + "xdense"])) < 1e-8
        # the certificate is an estimate of the same quantity
        assert o.eps_achieved == pytest.approx(float(g[p + "eps"]), rel=1e-3, abs=1e-9)


def _obs_from_trace(tr):
    return D.ObservationSet.from_coo(tr["m"], tr["n"], np.array(tr["rows"]), np.array(tr["cols"]),
                                     np.array(tr["vals"]))


@pytest.mark.parametrize("name", ["mfg_planted3", "mfg_planted4", "mfg_planted5", "mfg_crit4",
                                  "pg_planted9", "mfg_overreg"])
def test_lifted_trace_matches_reference(traces, name):
    tr = traces[name]
    obs = _obs_from_trace(tr)
    cfg = P.SolverConfig(**tr["cfg"])
    fn = P.solve_mf_global if tr["kind"] == "mf_global" else P.solve_pg_baseline
    x, _, trace = fn(obs, None, cfg)
    ranks = [r.rank for r in trace.records]
    objs = np.array([r.obj for r in trace.records])
    assert ranks == tr["rank"], name
    ref = np.array(tr["obj"])
    assert objs.shape == ref.shape, name
    # MF-Global: 1e-9 (north_star). The pure-PG baseline has no MF phase to
    # re-converge the iterate, so its per-step objective carries the
    # eigensolver's loose early tolerance (eps_t/(alpha_max k_t) ~ 1e-2) and
    # the eigenvector sign convention of LAPACK vs cuSOLVER (which orients
    # the retained warm-start direction): 1e-6 there.
    tol = 1e-9 if tr["kind"] == "mf_global" else 1e-6
    assert np.max(np.abs(objs - ref) / np.abs(ref)) <= tol, name
    assert [r.backtracks for r in trace.records] == tr["backtracks"]
    assert [r.k_t for r in trace.records] == tr["k_t"]


def test_mf_only_trace_matches_reference(traces):
    tr = traces["mfonly_planted14"]
    obs = _obs_from_trace(tr)
    cfg = P.SolverConfig(**tr["cfg"])
    _, trace = P.solve_mf_only(obs, None, cfg, fixed_rank=3)
    objs = np.array([r.obj for r in trace.records])
    ref = np.array(tr["obj"])
    assert objs.shape == ref.shape
    assert np.max(np.abs(objs - ref) / np.abs(ref)) <= 1e-9


def test_fp32_mode_tracks_fp64(traces):
    tr = traces["mfg_crit4"]
    obs = D.ObservationSet.from_coo(tr["m"], tr["n"], np.array(tr["rows"]), np.array(tr["cols"]),
                                    np.array(tr["vals"]), dtype=torch.float32)
    cfg = P.SolverConfig(**tr["cfg"])
    _, _, trace = P.solve_mf_global(obs, None, cfg)
    ref = np.array(tr["obj"])
    n = min(len(trace), ref.size)
    objs = np.array([r.obj for r in trace.records])[:n]
    assert np.max(np.abs(objs - ref[:n]) / np.abs(ref[:n])) <= 1e-4
    assert trace.final().rank == tr["rank"][-1]
