"""Generate golden fixtures by running the REFERENCE (mfglobal 0.1.0) itself.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--c1]

Writes small ``.npz`` / ``.json`` fixtures next to this file. Each fixture
stores its inputs as well as the reference outputs, so the tests never need
the reference (or its RNG conventions) at run time. ``--c1`` additionally
runs the full config-1 end-to-end solve (~10 min) and stores its trace.
"""

from __future__ import annotations

import json
import zlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import mfglobal  # noqa: E402  (the reference)
from mfglobal import data as rdata  # noqa: E402
from mfglobal import eigensolver as reig  # noqa: E402
from mfglobal import kernels as rker  # noqa: E402
from mfglobal import mfsolver as rmf  # noqa: E402
from mfglobal import operators as rops  # noqa: E402
from mfglobal import proxlift as rprox  # noqa: E402
from mfglobal import driver as rdrv  # noqa: E402

from paper_2204_14067_b200 import synth  # noqa: E402


def rng_for(seed):
    return np.random.Generator(np.random.Philox(seed))


def rand_obs(rng, m, n, frac=0.4, scale=1.0):
    mask = rng.random((m, n)) < frac
    mask[0, 0] = True
    rows, cols = np.nonzero(mask)
    vals = scale * rng.standard_normal(rows.size)
    return rdata.ObservationSet.from_coo(m, n, rows, cols, vals)


def planted(seed, m, n, r, frac, noise):
    rng = rng_for(seed)
    full = rng.standard_normal((m, r)) @ rng.standard_normal((n, r)).T
    mask = rng.random((m, n)) < frac
    rows, cols = np.nonzero(mask)
    vals = full[rows, cols] + noise * rng.standard_normal(rows.size)
    return rdata.ObservationSet.from_coo(m, n, rows, cols, vals)


def obs_arrays(prefix, obs, out):
    out[prefix + "m"] = obs.m
    out[prefix + "n"] = obs.n
    out[prefix + "rows"] = obs.rows
    out[prefix + "cols"] = obs.cols
    out[prefix + "vals"] = obs.vals
    out[prefix + "indptr"] = obs.indptr


def gen_omega():
    """Omega build: shuffled COO in, sorted CSR + scipy CSC out."""
    out = {}
    rng = rng_for(100)
    cases = [(7, 9, 0.5), (1, 1, 1.0), (30, 17, 0.3), (5, 40, 0.2)]
    for ci, (m, n, frac) in enumerate(cases):
        mask = rng.random((m, n)) < frac
        mask[0, 0] = True
        rows, cols = np.nonzero(mask)
        vals = rng.standard_normal(rows.size)
        perm = rng.permutation(rows.size)
        rows, cols, vals = rows[perm], cols[perm], vals[perm]
        obs = rdata.ObservationSet.from_coo(m, n, rows, cols, vals)
        p = f"c{ci}_"
        out[p + "in_rows"], out[p + "in_cols"], out[p + "in_vals"] = rows, cols, vals
        obs_arrays(p, obs, out)
        t = obs.a_csr_t
        out[p + "csc_ptr"], out[p + "csc_idx"], out[p + "csc_val"] = t.indptr, t.indices, t.data
    # empty Omega
    obs = rdata.ObservationSet.from_coo(3, 4, [], [], [])
    out["empty_indptr"] = obs.indptr
    # duplicate message
    try:
        rdata.ObservationSet.from_coo(3, 3, [2, 0, 2, 1], [1, 0, 1, 2], [1.0, 2.0, 3.0, 4.0])
    except rdata.DatasetError as exc:
        out["dup_msg"] = np.array(str(exc))
    for bad, args in [("row_range", (2, 2, [0, 2], [0, 0], [1.0, 1.0])),
                      ("col_range", (2, 2, [0, 1], [0, -1], [1.0, 1.0])),
                      ("length", (2, 2, [0, 1], [0], [1.0, 1.0]))]:
        try:
            rdata.ObservationSet.from_coo(*args)
        except rdata.DatasetError as exc:
            out["err_" + bad] = np.array(str(exc))
    np.savez_compressed(os.path.join(HERE, "omega.npz"), **out)


def gen_sweep():
    """R, loss, R.H, R^T.W on several instances (incl. empty rows / Omega)."""
    out = {}
    cases = []
    rng = rng_for(200)
    cases.append(("rand10x12k3", rand_obs(rng, 10, 12), 3))
    cases.append(("one", rdata.ObservationSet.from_coo(1, 1, [0], [0], [3.0]), 1))
    cases.append(("emptyrows", rdata.ObservationSet.from_coo(3, 4, [0, 0], [1, 3], [2.0, -1.0]), 2))
    cases.append(("emptyomega", rdata.ObservationSet.from_coo(3, 4, [], [], []), 2))
    cases.append(("rand40x60k5", rand_obs(rng, 40, 60, frac=0.5), 5))
    cases.append(("planted100x120k8", planted(2024, 100, 120, 5, 0.3, 0.1), 8))
    m, n, r, c, v = synth.generate("c2", scale=0.1)
    m, n, r, c, v, _ = synth.canonical(m, n, r, c, v)
    cases.append(("c2s01k20", rdata.ObservationSet.from_coo(m, n, r, c, v), 20))
    cases.append(("rand64x200k37", rand_obs(rng, 64, 200, frac=0.3), 37))
    names = []
    for name, obs, k in cases:
        names.append(name)
        wrng = rng_for(zlib.crc32(name.encode()) % 1000)
        w = wrng.standard_normal((obs.m, k)) * k ** -0.25
        h = wrng.standard_normal((obs.n, k)) * k ** -0.25
        wf = rops.FactorPair(w, h)
        res = rdata.residual_on_omega(obs, wf)
        p = name + "_"
        obs_arrays(p, obs, out)
        out[p + "k"] = k
        out[p + "w"], out[p + "h"] = w, h
        out[p + "r"] = res.vals
        out[p + "loss"] = rdata.loss_quad(res)
        out[p + "rh"] = res.csr @ h
        out[p + "rtw"] = res.csr_t @ w
        out[p + "frob"] = wf.frob_sq()
        # svd variant on a random triplet
        tr = rng_for(7 + len(names))
        kk = max(1, min(obs.m, obs.n, 3))
        qu, _ = np.linalg.qr(tr.standard_normal((obs.m, kk)))
        qv, _ = np.linalg.qr(tr.standard_normal((obs.n, kk)))
        sig = np.sort(0.1 + tr.random(kk))[::-1]
        x = rker.SvdTriplet(qu, sig, qv)
        out[p + "tu"], out[p + "ts"], out[p + "tv"] = qu, sig, qv
        out[p + "tres"] = rdata.residual_on_omega_svd(obs, x).vals
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "sweep.npz"), **out)


def gen_bcd():
    out = {}
    cases = []
    rng = rng_for(300)
    cases.append(("rand10x12k3", rand_obs(rng, 10, 12), 3, 0.8))
    cases.append(("scalar", rdata.ObservationSet.from_coo(1, 1, [0], [0], [3.0]), 1, 0.5))
    cases.append(("emptyrows", rdata.ObservationSet.from_coo(3, 4, [0, 0], [1, 3], [2.0, -1.0]), 2, 1.0))
    cases.append(("rand40x60k5", rand_obs(rng, 40, 60, frac=0.5), 5, 1.3))
    cases.append(("planted100x120k12", planted(2024, 100, 120, 5, 0.3, 0.1), 12, 8.0))
    cases.append(("rand50x70k70", rand_obs(rng, 50, 70, frac=0.6), 70, 2.0))
    names = []
    for name, obs, k, lam in cases:
        names.append(name)
        wrng = rng_for(len(names) + 31)
        w = wrng.standard_normal((obs.m, k))
        h = wrng.standard_normal((obs.n, k))
        if name == "scalar":
            w, h = np.array([[10.0]]), np.array([[1.0]])
        wf = rops.FactorPair(w, h)
        p = name + "_"
        obs_arrays(p, obs, out)
        out[p + "k"], out[p + "lam"] = k, lam
        out[p + "w"], out[p + "h"] = w, h
        e1 = rmf.bcd_epoch(obs, wf, lam)
        out[p + "w1"], out[p + "h1"] = e1.w, e1.h
        out[p + "obj0"] = rmf.mf_objective(obs, wf, lam)
        out[p + "obj1"] = rmf.mf_objective(obs, e1, lam)
        e3 = rmf.mf_phase(obs, wf, lam, 3)
        out[p + "w3"], out[p + "h3"] = e3.w, e3.h
        out[p + "obj3"] = rmf.mf_objective(obs, e3, lam)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "bcd.npz"), **out)


def gen_operator():
    out = {}
    names = []
    for seed, (m, n, k, alpha, p) in enumerate([(10, 12, 3, 0.7, 5), (40, 60, 5, 0.35, 9), (25, 30, 2, 0.0, 3)]):
        rng = rng_for(400 + seed)
        obs = rand_obs(rng, m, n)
        wf = rops.FactorPair(rng.standard_normal((m, k)), rng.standard_normal((n, k)))
        grad = rdata.gradient(rdata.residual_on_omega(obs, wf))
        op = rops.ShiftedOperator(wf, grad, alpha)
        bn = rng.standard_normal((n, p))
        bm = rng.standard_normal((m, p))
        q, _ = np.linalg.qr(rng.standard_normal((m, min(m, p))))
        name = f"op{seed}"
        names.append(name)
        pre = name + "_"
        obs_arrays(pre, obs, out)
        out[pre + "w"], out[pre + "h"], out[pre + "alpha"] = wf.w, wf.h, alpha
        out[pre + "g"] = grad.vals
        out[pre + "bn"], out[pre + "bm"], out[pre + "q"] = bn, bm, q
        out[pre + "apply"] = op.apply(bn)
        out[pre + "apply_t"] = op.apply_t(bm)
        out[pre + "apply_gram"] = op.apply_gram(bm)
        out[pre + "project"] = op.project_rows(q)
        out[pre + "frob_sq"] = op.frob_sq()
        t1 = rker.SvdTriplet(*_rand_triplet(rng, m, n, 3))
        out[pre + "t1u"], out[pre + "t1s"], out[pre + "t1v"] = t1.u, t1.sigma, t1.v
        out[pre + "ip_tf"] = rops.inner_product(t1, wf)
        out[pre + "dist_tf"] = rops.frob_dist_sq(t1, wf)
        out[pre + "ip_tt"] = rops.inner_product(t1, t1)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "operator.npz"), **out)


def _rand_triplet(rng, m, n, k, scale=1.0):
    qu, _ = np.linalg.qr(rng.standard_normal((m, k)))
    qv, _ = np.linalg.qr(rng.standard_normal((n, k)))
    sigma = np.sort(scale * (0.1 + rng.random(k)))[::-1]
    return qu, sigma, qv


def gen_kernels():
    out = {}
    rng = rng_for(500)
    mats = {}
    v = rng.standard_normal((60, 1))
    mats["dep2"] = np.hstack([v, 2 * v])
    mats["rand50x8"] = rng.standard_normal((50, 8))
    mats["wide3x5"] = rng.standard_normal((3, 5))
    b = rng.standard_normal((80, 6))
    # near-dependent columns straddling the 1e-10 screening threshold
    nb = np.linalg.norm(b)
    c1 = b[:, 0] + 1e-9 * nb * rng.standard_normal(80) / np.sqrt(80)
    c2 = b[:, 1] + 1e-12 * nb * rng.standard_normal(80) / np.sqrt(80)
    mats["near"] = np.hstack([b, c1[:, None], c2[:, None], b[:, 2:3] * 3.0])
    mats["zero"] = np.zeros((5, 3))
    names = []
    for name, mat in mats.items():
        names.append(name)
        q, rank = rker.orthonormalize(mat)
        out["orth_" + name + "_in"] = mat
        out["orth_" + name + "_rank"] = rank
        out["orth_" + name + "_proj"] = q @ q.T
    out["orth_names"] = np.array(names)
    # soft threshold cases
    st = [([3.0, 1.0, 0.5], 1.0), ([2.0, 1.0, 0.0], 0.0), ([3.0, 1.0], 5.0), ([2.0, 1.0], 1.0),
          ([5.0, 4.0], 1.0), ([1.0, 1e-13, 1e-14], 0.0), ([4.0, 3.0, 3.0, 2.0], 3.0)]
    for i, (s, beta) in enumerate(st):
        sig, kept, lt = rker.soft_threshold(np.array(s), beta)
        out[f"st{i}_in"], out[f"st{i}_beta"] = np.array(s), beta
        out[f"st{i}_sigma"], out[f"st{i}_kept"] = sig, kept
        out[f"st{i}_lt"] = np.nan if lt is None else lt
    out["st_count"] = len(st)
    # short-fat SVD
    for i, (k, n) in enumerate([(8, 40), (2, 5), (70, 90), (5, 30)]):
        mat = rng.standard_normal((k, n))
        if i == 3:
            base = rng.standard_normal((3, n))
            mat = np.vstack([base, base[0] + base[1], base[2]])
        u, s, vv = rker.exact_svd_short_fat(mat)
        out[f"svd{i}_in"], out[f"svd{i}_s"] = mat, s
    out["svd_count"] = 4
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def gen_eig_prox():
    out = {}
    # eigensolver on sparse-plus-low-rank operators
    for seed in range(3):
        rng = rng_for(600 + seed)
        m, n, k = 40, 60, 5
        obs = rand_obs(rng, m, n, frac=0.5)
        wf = rops.FactorPair(0.7 * rng.standard_normal((m, k)), 0.7 * rng.standard_normal((n, k)))
        grad = rdata.gradient(rdata.residual_on_omega(obs, wf))
        alpha = 0.6
        op = rops.ShiftedOperator(wf, grad, alpha)
        r0, _ = np.linalg.qr(rng.standard_normal((m, 6)))
        p = f"eig{seed}_"
        obs_arrays(p, obs, out)
        out[p + "w"], out[p + "h"], out[p + "g"], out[p + "alpha"], out[p + "r0"] = wf.w, wf.h, grad.vals, alpha, r0
        for meth in ("lm-krylov", "power"):
            cfg = reig.EigConfig(memory=3, max_iters=40, residual_tol=1e-9, method=meth)
            res = reig.solve_topk(op, r0, cfg)
            out[p + meth + "_w"] = res.eigvals
            out[p + meth + "_iters"] = res.iters_used
            out[p + meth + "_conv"] = res.converged
            out[p + meth + "_hist"] = np.array(res.history)
    # lifting step outcomes
    for seed in range(4):
        rng = rng_for(700 + seed)
        m, n, k = 40, 60, 5
        obs = rand_obs(rng, m, n, frac=0.5)
        wf = rops.FactorPair(0.7 * rng.standard_normal((m, k)), 0.7 * rng.standard_normal((n, k)))
        grad = rdata.gradient(rdata.residual_on_omega(obs, wf))
        r0, _ = np.linalg.qr(rng.standard_normal((m, 2 * k)))
        params = rprox.StepParams(lam=1.0)
        cfg = reig.EigConfig(memory=3, max_iters=200, residual_tol=1e-10)
        o = rprox.inexact_prox_step(obs, wf, grad, 2.0, params, r0, cfg, eps_target=1e-4)
        p = f"prox{seed}_"
        obs_arrays(p, obs, out)
        out[p + "w"], out[p + "h"], out[p + "r0"] = wf.w, wf.h, r0
        out[p + "rank"] = o.x_next.rank
        out[p + "sigma"] = o.x_next.sigma
        out[p + "alpha"] = o.alpha_used
        out[p + "backtracks"] = o.backtracks
        out[p + "f_next"] = o.f_next
        out[p + "f_base"] = o.f_base
        out[p + "eps"] = o.eps_achieved
        out[p + "dist_sq"] = o.dist_sq
        out[p + "sweeps"] = o.eig_sweeps
        out[p + "xdense"] = o.x_next.dense()
    np.savez_compressed(os.path.join(HERE, "eigprox.npz"), **out)


def trace_dict(trace):
    keys = ["iter", "obj", "rank", "alpha", "backtracks", "eps_target", "eps_achieved",
            "eig_sweeps", "k_t", "f_mf", "f_prev", "dist", "rmse"]
    return {k: [getattr(r, k) for r in trace.records] for k in keys}


def gen_traces():
    out = {}
    runs = []
    for seed in (3, 4, 5):
        obs = planted(seed, 30, 36, 3, 0.5, 0.05)
        runs.append((f"mfg_planted{seed}", "mf_global", obs,
                     dict(lam=2.0, k0=4, max_outer_iters=40, seed=seed)))
    obs = planted(2024, 100, 120, 5, 0.3, 0.1)
    runs.append(("mfg_crit4", "mf_global", obs, dict(lam=8.0, k0=8, max_outer_iters=60, stop_tol=1e-9, seed=7)))
    obs = planted(9, 30, 36, 3, 0.5, 0.05)
    runs.append(("pg_planted9", "pg", obs, dict(lam=2.5, k0=4, max_outer_iters=25, seed=9)))
    obs = planted(14, 30, 36, 3, 0.5, 0.05)
    runs.append(("mfonly_planted14", "mf_only", obs, dict(lam=2.0, max_outer_iters=30, seed=14)))
    rng = rng_for(800)
    obs = rand_obs(rng, 10, 12)
    runs.append(("mfg_overreg", "mf_global", obs, dict(lam=1e6, k0=3, max_outer_iters=30, seed=1)))
    for name, kind, obs, kw in runs:
        cfg = rdrv.SolverConfig(**kw)
        t0 = time.perf_counter()
        if kind == "mf_global":
            x, _, tr = rdrv.solve_mf_global(obs, None, cfg)
        elif kind == "pg":
            x, _, tr = rdrv.solve_pg_baseline(obs, None, cfg)
        else:
            _, tr = rdrv.solve_mf_only(obs, None, cfg, fixed_rank=3)
        el = time.perf_counter() - t0
        d = trace_dict(tr)
        d.update(kind=kind, cfg=kw, m=obs.m, n=obs.n, rows=obs.rows.tolist(),
                 cols=obs.cols.tolist(), vals=obs.vals.tolist(), elapsed_s=el)
        out[name] = d
        print(name, len(tr), "iters", f"{el:.1f}s", "final rank", d["rank"][-1], "obj", d["obj"][-1])
    with open(os.path.join(HERE, "traces.json"), "w") as fh:
        json.dump(out, fh)


def gen_traces_estimated():
    """Solver traces with the estimated certification mode (the only mode of
    the sharded driver), for the sharded-solver parity tests."""
    out = {}
    runs = [("mfg_est_planted3", planted(3, 30, 36, 3, 0.5, 0.05),
             dict(lam=2.0, k0=4, max_outer_iters=12, seed=3, cert_mode="estimated")),
            ("mfg_est_crit4", planted(2024, 100, 120, 5, 0.3, 0.1),
             dict(lam=8.0, k0=8, max_outer_iters=10, seed=7, cert_mode="estimated"))]
    for name, obs, kw in runs:
        cfg = rdrv.SolverConfig(**kw)
        t0 = time.perf_counter()
        x, _, tr = rdrv.solve_mf_global(obs, None, cfg)
        el = time.perf_counter() - t0
        d = trace_dict(tr)
        d.update(kind="mf_global", cfg=kw, m=obs.m, n=obs.n, rows=obs.rows.tolist(),
                 cols=obs.cols.tolist(), vals=obs.vals.tolist(), elapsed_s=el)
        out[name] = d
        print(name, len(tr), "iters", f"{el:.1f}s", "final rank", d["rank"][-1], "obj", d["obj"][-1])
    with open(os.path.join(HERE, "traces_estimated.json"), "w") as fh:
        json.dump(out, fh)


def gen_c1():
    m, n, r, c, v = synth.generate("c1")
    m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
    obs = rdata.ObservationSet.from_coo(m, n, r, c, v, transposed=tr)
    cfg = rdrv.SolverConfig(lam=5.0, k0=8, seed=0)
    t0 = time.perf_counter()
    x, _, trace = rdrv.solve_mf_global(obs, None, cfg)
    el = time.perf_counter() - t0
    d = trace_dict(trace)
    d.update(kind="mf_global", cfg=dict(lam=5.0, k0=8, seed=0), m=m, n=n, elapsed_s=el,
             time_s=[rec.time_s for rec in trace.records],
             numpy=np.__version__, instance="synth.generate('c1') canonical")
    with open(os.path.join(HERE, "trace_c1.json"), "w") as fh:
        json.dump(d, fh)
    print("c1", len(trace), "iters", el, "s; rank", x.rank, "F", d["obj"][-1])


def gen_extras():
    """rmse / rmse_factors (mfg/data.py:301-313), make_reference
    (mfg/driver.py:464-475, with a test split) and the rank-deficient
    _complete_basis / _prepare_block padding (mfg/eigensolver.py:53-78)."""
    out = {}
    rng = rng_for(4242)
    m, n, r = 40, 50, 3
    full = rng.standard_normal((m, r)) @ rng.standard_normal((n, r)).T
    mask = rng.random((m, n)) < 0.5
    test = (~mask) & (rng.random((m, n)) < 0.3)
    rows, cols = np.nonzero(mask)
    vals = full[rows, cols] + 0.05 * rng.standard_normal(rows.size)
    trow, tcol = np.nonzero(test)
    tval = full[trow, tcol] + 0.05 * rng.standard_normal(trow.size)
    obs = rdata.ObservationSet.from_coo(m, n, rows, cols, vals)
    split = rdata.EvalSplit(m, n, trow, tcol, tval)
    out.update(ex_m=m, ex_n=n, ex_rows=rows, ex_cols=cols, ex_vals=vals, ex_trows=trow,
               ex_tcols=tcol, ex_tvals=tval)
    u, sg, v = _rand_triplet(rng, m, n, 4)
    x = rker.SvdTriplet(u, sg, v)
    w = rng.standard_normal((m, 5))
    h = rng.standard_normal((n, 5))
    out.update(ex_u=u, ex_s=sg, ex_v=v, ex_w=w, ex_h=h,
               ex_rmse=rdata.rmse(split, x),
               ex_rmse0=rdata.rmse(split, rker.SvdTriplet.zero(m, n)),
               ex_rmsef=rdata.rmse_factors(split, rops.FactorPair(w, h)))
    cfg = rdrv.SolverConfig(lam=2.0, k0=4, max_outer_iters=15, seed=11)
    xs, metrics, tr = rdrv.make_reference(obs, split, cfg)
    out.update(ex_ref_fstar=metrics["f_star"], ex_ref_rmse_star=metrics["rmse_star"],
               ex_ref_rmse_zero=metrics["rmse_zero"], ex_ref_rank=xs.rank,
               ex_ref_obj=np.array([rec.obj for rec in tr.records]),
               ex_ref_ranks=np.array([rec.rank for rec in tr.records]),
               ex_ref_rmse=np.array([rec.rmse for rec in tr.records]))
    # _complete_basis: q spans e_0 and (e_1 + e_2)/sqrt(2): the next basis
    # vectors e_0, e_1 project to zero / survive, exercising both branches
    mq = 12
    q = np.zeros((mq, 2))
    q[0, 0] = 1.0
    q[1, 1] = q[2, 1] = 1.0 / np.sqrt(2.0)
    out.update(cb_q=q, cb_k=6, cb_out=reig._complete_basis(q, 6))
    # _prepare_block on a rank-deficient block (rank 2 of 5 columns)
    b = rng.standard_normal((30, 2)) @ rng.standard_normal((2, 5))
    out.update(pb_r0=b, pb_k=5, pb_out=reig._prepare_block(b, 5))
    try:
        reig._complete_basis(np.eye(3)[:, :1], 4)
    except ValueError as e:
        out["cb_err"] = str(e)
    np.savez_compressed(os.path.join(HERE, "extras.npz"), **out)
    print("extras", metrics)


def gen_c2(iters: int = 3):
    """BASELINE configs[1] (c2) in the reference's fp64, the first ``iters``
    outer iterations at the config's lambda; the GPU runs it in fp32 storage
    (tests/test_c2_fp32_gpu.py: identical ranks, objectives within 1e-4)."""
    m, n, r, c, v = synth.generate("c2")
    m, n, r, c, v, tr = synth.canonical(m, n, r, c, v)
    obs = rdata.ObservationSet.from_coo(m, n, r, c, v, transposed=tr)
    kw = dict(lam=float(synth.CONFIGS["c2"].lam), k0=synth.CONFIGS["c2"].k0, seed=0,
              max_outer_iters=iters)
    cfg = rdrv.SolverConfig(**kw)
    t0 = time.perf_counter()
    x, _, trace = rdrv.solve_mf_global(obs, None, cfg)
    el = time.perf_counter() - t0
    d = trace_dict(trace)
    d.update(kind="mf_global", cfg=kw, m=m, n=n, elapsed_s=el,
             time_s=[rec.time_s for rec in trace.records],
             numpy=np.__version__, instance="synth.generate('c2') canonical")
    with open(os.path.join(HERE, "trace_c2.json"), "w") as fh:
        json.dump(d, fh)
    print("c2", len(trace), "records", el, "s; rank", x.rank, "F", d["obj"][-1])


if __name__ == "__main__":
    print("reference", mfglobal.__version__, "numpy", np.__version__)
    if "--c1" in sys.argv:
        gen_c1()
        sys.exit(0)
    if "--c2" in sys.argv:
        gen_c2()
        sys.exit(0)
    if "--extras" in sys.argv:
        gen_extras()
        sys.exit(0)
    if "--estimated" in sys.argv:
        gen_traces_estimated()
        sys.exit(0)
    gen_omega()
    gen_sweep()
    gen_bcd()
    gen_operator()
    gen_kernels()
    gen_eig_prox()
    gen_traces()
