"""GPU parity for the rows round 1 left untested:
test-set RMSE on the device (mfg/data.py:301-313), make_reference
(mfg/driver.py:464-475), the rank-deficient basis padding of the
eigensolver (mfg/eigensolver.py:53-78), the fp32-storage BCD kernel against
the oracle's normal equations (mfg/mfsolver.py:53-75), and the BCD
non-SPD status word. Fixtures: tests/golden/extras.npz, written by running
the reference itself (tests/golden/make_golden.py --extras)."""

import numpy as np
import pytest
import torch

from oracle import mfg_oracle as orc

pytestmark = pytest.mark.gpu

import paper_2204_14067_b200 as P  # noqa: E402
from paper_2204_14067_b200 import data as D  # noqa: E402
from paper_2204_14067_b200 import eigensolver as E  # noqa: E402
from paper_2204_14067_b200 import mfsolver as MF  # noqa: E402
from paper_2204_14067_b200.operators import FactorPair  # noqa: E402


def _np(t):
    return t.detach().double().cpu().numpy()


def _split(g):
    return D.EvalSplit(int(g["ex_m"]), int(g["ex_n"]), g["ex_trows"], g["ex_tcols"], g["ex_tvals"])


def test_rmse_on_device_matches_reference(golden):
    g = golden("extras.npz")
    split = _split(g)
    x = P.SvdTriplet(g["ex_u"], g["ex_s"], g["ex_v"])
    assert D.rmse(split, x) == pytest.approx(float(g["ex_rmse"]), rel=1e-12)
    zero = P.SvdTriplet.zero(int(g["ex_m"]), int(g["ex_n"]))
    assert D.rmse(split, zero) == pytest.approx(float(g["ex_rmse0"]), rel=1e-12)
    wf = FactorPair(g["ex_w"], g["ex_h"])
    assert D.rmse_factors(split, wf) == pytest.approx(float(g["ex_rmsef"]), rel=1e-12)
    empty = D.EvalSplit(3, 4, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    with pytest.raises(ValueError, match="empty test set"):
        D.rmse(empty, x)
    with pytest.raises(ValueError, match="empty test set"):
        D.rmse_factors(empty, wf)


def test_make_reference_matches_reference(golden):
    g = golden("extras.npz")
    obs = P.ObservationSet.from_coo(int(g["ex_m"]), int(g["ex_n"]), g["ex_rows"], g["ex_cols"],
                                    g["ex_vals"])
    cfg = P.SolverConfig(lam=2.0, k0=4, max_outer_iters=15, seed=11)
    x, metrics, trace = P.make_reference(obs, _split(g), cfg)
    assert [rec.rank for rec in trace.records] == [int(r) for r in g["ex_ref_ranks"]]
    objs = np.array([rec.obj for rec in trace.records])
    assert np.max(np.abs(objs - g["ex_ref_obj"]) / np.abs(g["ex_ref_obj"])) <= 1e-9
    rm = np.array([rec.rmse for rec in trace.records], dtype=float)
    assert np.allclose(rm, g["ex_ref_rmse"], rtol=1e-8, atol=0)
    assert x.rank == int(g["ex_ref_rank"])
    assert metrics["f_star"] == pytest.approx(float(g["ex_ref_fstar"]), rel=1e-9)
    assert metrics["rmse_star"] == pytest.approx(float(g["ex_ref_rmse_star"]), rel=1e-8)
    assert metrics["rmse_zero"] == pytest.approx(float(g["ex_ref_rmse_zero"]), rel=1e-12)
    assert metrics["lam"] == 2.0 and metrics["seed"] == 11


def test_complete_basis_padding_branch(golden):
    g = golden("extras.npz")
    q = torch.as_tensor(g["cb_q"], device="cuda")
    out = E._complete_basis(q, int(g["cb_k"]))
    # e_0 lies in span(q) and is skipped (the nrm <= 1e-8 branch); e_1, e_2
    # survive projected; the padded columns are basis-independent
    assert np.allclose(_np(out), g["cb_out"], atol=1e-14, rtol=0)
    with pytest.raises(ValueError) as err:
        E._complete_basis(torch.eye(3, dtype=torch.float64, device="cuda")[:, :1], 4)
    assert str(err.value) == str(g["cb_err"])


def test_prepare_block_rank_deficient(golden):
    g = golden("extras.npz")
    k = int(g["pb_k"])
    out = _np(E._prepare_block(torch.as_tensor(g["pb_r0"], device="cuda"), k))
    ref = g["pb_out"]
    assert out.shape == ref.shape == (30, k)
    assert np.allclose(out.T @ out, np.eye(k), atol=1e-12)
    # the orthonormalised part (rank 2) spans the reference's: equal projectors
    pq, pr = out[:, :2], ref[:, :2]
    assert np.allclose(pq @ pq.T, pr @ pr.T, atol=1e-10)
    # the padding is the Gram-Schmidt completion against that span
    assert np.allclose(out[:, 2:], ref[:, 2:], atol=1e-10)


def _bcd_instance(seed, m=300, n=2000, heavy=(2000, 1500, 700, 300)):
    rng = np.random.default_rng(seed)
    deg = rng.integers(1, 25, size=m)
    deg[: len(heavy)] = heavy
    rows, cols = [], []
    for i, d in enumerate(deg):
        cc = rng.choice(n, size=d, replace=False)
        if 3 not in cc:
            cc = np.append(cc, 3)
        rows.append(np.full(cc.size, i))
        cols.append(cc)
    r, c = np.concatenate(rows), np.concatenate(cols)
    r = rng.permutation(m)[r]
    # integer ratings 1..5 like the fp32 configs (exact in fp32)
    v = rng.integers(1, 6, size=r.size).astype(np.float64)
    return rng, m, n, r, c, v


@pytest.mark.parametrize("k", [1, 5, 20, 24, 25, 30, 40, 41, 48, 56, 64, 65])
def test_bcd_fp32_storage_matches_oracle(k):
    """The fp32-storage instantiation (k_bcd<float,...>, what every c2-c5 MF
    phase runs): fp32 A and factors, fp64 Gram + Cholesky, fp32 rows out.
    Against the oracle's normal equations on the same fp32-rounded inputs,
    per half-sweep (the H half-sweep takes the GPU's W), with heavy rows
    split into segments on both orientations; the result must be the fp64
    solution rounded to fp32 (within a few fp32 ulps of the row's scale)
    and bitwise repeatable."""
    rng, m, n, r, c, v = _bcd_instance(700 + k)
    lam = 1.7
    obs = P.ObservationSet.from_coo(m, n, r, c, v, dtype=torch.float32)
    om = orc.from_coo(m, n, r, c, v)
    h = (rng.standard_normal((n, k)) * 0.3).astype(np.float32)
    ht = torch.as_tensor(h, device="cuda")
    w_gpu = MF._half_sweep(obs, False, ht, lam)
    w_gpu2 = MF._half_sweep(obs, False, ht, lam)
    MF.check_bcd_status()
    assert w_gpu.dtype == torch.float32 and torch.equal(w_gpu, w_gpu2)
    w_ref = orc.half_sweep(om.a_csr, om.pattern_csr, h.astype(np.float64), lam)
    scale = np.abs(w_ref).max(axis=1, keepdims=True) + 1e-30
    assert np.max(np.abs(_np(w_gpu) - w_ref) / scale) <= 4e-7
    h_gpu = MF._half_sweep(obs, True, w_gpu, lam)
    MF.check_bcd_status()
    h_ref = orc.half_sweep(om.a_csr_t, om.pattern_csr_t, _np(w_gpu), lam)
    scale = np.abs(h_ref).max(axis=1, keepdims=True) + 1e-30
    assert np.max(np.abs(_np(h_gpu) - h_ref) / scale) <= 4e-7


def test_bcd_non_spd_raises_numerical_error():
    """A NaN factor makes a pivot NaN: the kernel's status word is read back
    and the Python layer raises NumericalError instead of returning NaN rows
    (ADVICE round 1)."""
    rng, m, n, r, c, v = _bcd_instance(5, m=50, n=80, heavy=(60,))
    obs = P.ObservationSet.from_coo(m, n, r, c, v)
    w = rng.standard_normal((m, 4))
    h = rng.standard_normal((n, 4))
    MF.bcd_epoch(obs, FactorPair(w, h), 1.0)     # finite: no error
    h[3, 2] = np.nan                             # column 3 is in every row
    with pytest.raises(P.NumericalError, match="non-SPD"):
        MF.bcd_epoch(obs, FactorPair(w, h), 1.0)
    MF.bcd_epoch(obs, FactorPair(w, np.nan_to_num(h)), 1.0)   # state cleared
