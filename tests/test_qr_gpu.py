"""Our tall-skinny QR (csrc/qr.cu via dense.qr: Householder TSQR of 32-column
panels inside a block Gram-Schmidt with re-orthogonalisation) against
np.linalg.qr, the call the reference's orthonormalize makes
(mfg/kernels.py:94): orthonormality and B = Q R to 1e-13, |R_jj| equal to
LAPACK's to 1e-12 relative on full-rank blocks, the same kept/dropped columns
under the reference's threshold on rank-deficient blocks, Q equal up to
column signs, bitwise run-to-run reproducibility, and orthonormalize /
svd_from_factors on top of it."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2204_14067_b200 import dense, kernels as K  # noqa: E402


def _t(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


@pytest.fixture(autouse=True)
def _own_qr():
    prev = K.set_qr_backend("own")
    yield
    K.set_qr_backend(prev)


def _block(m, p, kind, seed):
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((m, p))
    if kind == "graded":
        b *= np.logspace(4, -6, p)
    elif kind == "krylov":
        a = rng.standard_normal((m, m))
        a = (a + a.T) / np.sqrt(m)
        x = b[:, : p // 3]
        b = np.concatenate([x, a @ x, a @ (a @ x)], axis=1)
    elif kind == "deficient":
        r = max(1, min(5, p // 4))
        b[:, p // 2: p // 2 + r] = b[:, :r] @ rng.standard_normal((r, r))
        b[:, -1] = 2.0 * b[:, 0]
    return b


SHAPES = [(1, 1, "rand"), (5, 3, "rand"), (40, 33, "rand"), (50, 50, "rand"), (256, 32, "rand"),
          (257, 31, "rand"), (2000, 300, "rand"), (2000, 300, "graded"), (900, 90, "krylov"),
          (3706, 80, "rand"), (20000, 70, "graded"), (70000, 64, "rand"), (300000, 40, "rand")]


@pytest.mark.parametrize("m,p,kind", SHAPES)
def test_qr_matches_lapack(m, p, kind):
    b = _block(m, p, kind, m + p)
    q_t, d_t = dense.qr(_t(b))
    q, d = q_t.cpu().numpy(), d_t.cpu().numpy()
    q0, r0 = np.linalg.qr(b)
    d0 = np.abs(np.diag(r0))
    scale = np.linalg.norm(b)
    assert q.shape == (m, p) and d.shape == (p,)
    assert np.max(np.abs(q.T @ q - np.eye(p))) <= 1e-13
    assert np.max(np.abs(d - d0) / d0) <= 1e-11
    # same columns up to sign; then B = Q R with R = Q^T B
    sign = np.sign(np.sum(q * q0, axis=0))
    assert np.max(np.abs(q * sign - q0)) <= 1e-9 * max(1.0, scale / d0.min() * 1e-4)
    assert np.linalg.norm(q @ (q.T @ b) - b) <= 1e-13 * scale * np.sqrt(p)
    q2, d2 = dense.qr(_t(b))
    assert torch.equal(q2, q_t) and torch.equal(d2, d_t)


@pytest.mark.parametrize("m,p", [(40, 33), (2000, 300), (5000, 97)])
def test_qr_screens_dependent_columns_like_householder(m, p):
    b = _block(m, p, "deficient", 7 * m + p)
    q_t, d_t = dense.qr(_t(b))
    q, d = q_t.cpu().numpy(), d_t.cpu().numpy()
    d0 = np.abs(np.diag(np.linalg.qr(b)[1]))
    thr = K.ORTH_TOL * np.linalg.norm(b)
    assert np.array_equal(d > thr, d0 > thr)
    assert (d <= thr).sum() >= 2
    assert np.max(np.abs(q.T @ q - np.eye(p))) <= 1e-12
    # orthonormalize: the reference's decision (drop, re-factor) and span
    qo, rank = K.orthonormalize(_t(b))
    keep = d0 > thr
    assert rank == int(keep.sum())
    qo = qo.cpu().numpy()
    qr0 = np.linalg.qr(b[:, keep])[0]
    assert np.max(np.abs(qo.T @ qo - np.eye(rank))) <= 1e-12
    assert np.linalg.norm(qo - qr0 @ (qr0.T @ qo)) <= 1e-9


def test_orthonormalize_wide_block_uses_first_m_columns():
    rng = np.random.default_rng(5)
    b = rng.standard_normal((6, 9))
    q, rank = K.orthonormalize(_t(b))
    assert rank == 6 and q.shape == (6, 6)
    qn = q.cpu().numpy()
    assert np.max(np.abs(qn.T @ qn - np.eye(6))) <= 1e-13


def test_svd_from_factors_on_own_qr():
    from paper_2204_14067_b200 import FactorPair, mfsolver

    rng = np.random.default_rng(11)
    w = rng.standard_normal((700, 12))
    h = rng.standard_normal((500, 12))
    x = mfsolver.svd_from_factors(FactorPair(_t(w), _t(h)))
    s0 = np.linalg.svd(w @ h.T, compute_uv=False)[:12]
    assert np.max(np.abs(x.sigma - s0)) <= 1e-10 * s0[0]
    assert np.max(np.abs(x.dense().cpu().numpy() - w @ h.T)) <= 1e-10 * s0[0]


@pytest.mark.parametrize("name", ["mfg_planted3", "mfg_planted4", "mfg_planted5", "mfg_crit4"])
def test_reference_traces_hold_with_own_qr(name):
    """The reference's traces (tests/golden/traces.json, made by make_golden.py
    from /root/reference) through solve_mf_global with every Householder QR on
    dense.qr: identical ranks, backtracks and k_t, objectives within 1e-9."""
    import json
    import os

    import paper_2204_14067_b200 as P

    with open(os.path.join(os.path.dirname(__file__), "golden", "traces.json")) as fh:
        tr = json.load(fh)[name]
    obs = P.ObservationSet.from_coo(tr["m"], tr["n"], np.array(tr["rows"]), np.array(tr["cols"]),
                                    np.array(tr["vals"]))
    _, _, trace = P.solve_mf_global(obs, None, P.SolverConfig(**tr["cfg"]))
    assert [r.rank for r in trace.records] == tr["rank"]
    assert [r.backtracks for r in trace.records] == tr["backtracks"]
    assert [r.k_t for r in trace.records] == tr["k_t"]
    objs = np.array([r.obj for r in trace.records])
    ref = np.array(tr["obj"])
    assert np.max(np.abs(objs - ref) / np.abs(ref)) <= 1e-9
