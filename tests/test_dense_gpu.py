"""The lifting step's dense fp64 contractions on our DMMA kernels
(csrc/dense.cu via paper_2204_14067_b200.dense) against numpy fp64: the
tall-skinny Gram a^T b with its split-K slices (bitwise reproducible), the
tall-times-small product with alpha/beta and the projection x - q q^T x. Tolerance: 1e-13 relative to the operands' scale
(fp64 sums of up to 1e6 terms in a fixed but different order)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2204_14067_b200 import dense  # noqa: E402


def _t(x):
    return torch.as_tensor(x, device="cuda")


@pytest.mark.parametrize("m,p,q", [(1, 1, 1), (7, 3, 5), (100, 64, 64), (1000, 65, 130),
                                   (20000, 40, 40), (300000, 8, 3), (5000, 600, 600), (0, 4, 4)])
def test_gram_matches_numpy(m, p, q):
    rng = np.random.default_rng(m + p + q)
    a = rng.standard_normal((m, p))
    b = rng.standard_normal((m, q))
    c = dense.gram(_t(a), _t(b)).cpu().numpy()
    ref = a.T @ b
    scale = np.sqrt(max(m, 1)) * 4.0
    assert c.shape == (p, q)
    assert np.max(np.abs(c - ref), initial=0.0) <= 1e-13 * scale * max(1.0, np.sqrt(m))
    c2 = dense.gram(_t(a), _t(b)).cpu().numpy()
    assert np.array_equal(c, c2)                      # fixed slice order
    g = dense.gram(_t(a), alpha=-2.0).cpu().numpy()
    assert np.allclose(g, -2.0 * (a.T @ a), rtol=0, atol=1e-12 * scale * max(1.0, np.sqrt(m)))


@pytest.mark.parametrize("m,p,q", [(1, 1, 1), (130, 17, 9), (4096, 64, 64), (70000, 40, 1),
                                   (3000, 600, 150), (50, 0, 3)])
def test_matmul_matches_numpy(m, p, q):
    rng = np.random.default_rng(10 * m + p)
    a = rng.standard_normal((m, p))
    b = rng.standard_normal((p, q))
    c0 = rng.standard_normal((m, q))
    out = _t(c0.copy())
    dense.matmul(_t(a), _t(b), alpha=0.5, beta=-1.5, out=out)
    ref = 0.5 * (a @ b) - 1.5 * c0
    tol = 1e-13 * max(1.0, np.sqrt(p)) * 4.0
    assert np.max(np.abs(out.cpu().numpy() - ref), initial=0.0) <= tol
    plain = dense.matmul(_t(a), _t(b)).cpu().numpy()
    assert np.max(np.abs(plain - a @ b), initial=0.0) <= tol


def test_matmul_vector_and_project_out():
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((5000, 12)))
    x = rng.standard_normal(5000)
    y = dense.project_out(_t(q), _t(x)).cpu().numpy()
    assert y.shape == (5000,)
    assert np.allclose(y, x - q @ (q.T @ x), atol=1e-12)
    xb = rng.standard_normal((5000, 3))
    yb = dense.project_out(_t(q), _t(xb)).cpu().numpy()
    assert np.allclose(yb, xb - q @ (q.T @ xb), atol=1e-12)
    v = dense.matmul(_t(q), _t(rng.standard_normal(12)))
    assert v.shape == (5000,)


def test_inner_product_on_own_grams():
    """inner_product / frob_dist_sq (mfg/operators.py:67-81) on the DMMA
    Grams against dense numpy."""
    import paper_2204_14067_b200 as P

    rng = np.random.default_rng(5)
    wa, ha = rng.standard_normal((300, 7)), rng.standard_normal((200, 7))
    wb, hb = rng.standard_normal((300, 4)), rng.standard_normal((200, 4))
    a, b = P.FactorPair(wa, ha), P.FactorPair(wb, hb)
    xa, xb = wa @ ha.T, wb @ hb.T
    assert P.inner_product(a, b) == pytest.approx(float(np.sum(xa * xb)), rel=1e-12)
    assert P.frob_dist_sq(a, b) == pytest.approx(float(np.sum((xa - xb) ** 2)), rel=1e-10)


def test_gram_workspace_shared_across_shapes():
    """Calls of different tile counts share one workspace: the arrival
    counters live in a fixed region, so one call's partial tiles never land
    on another call's counters (a first version placed them after
    ntiles * 4 bytes and corrupted later calls)."""
    torch.manual_seed(0)
    for _ in range(2):
        for m, p in [(1500, 762), (1500, 600), (5000, 600), (2000, 100), (1500, 762)]:
            a = torch.randn(m, p, dtype=torch.float64, device="cuda")
            b = torch.randn(m, p, dtype=torch.float64, device="cuda")
            assert float((dense.gram(a, b) - a.T @ b).abs().max()) < 1e-10
