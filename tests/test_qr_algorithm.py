"""Host check of the QR algorithm csrc/qr.cu implements, restated in numpy
(the same chunk split, Householder steps, dorg2r back-accumulation, TSQR tree
and BCGS2 panel loop): on full-rank, graded, Krylov-like and rank-deficient
blocks it must give LAPACK's |R_jj| and the reference's kept/dropped columns
(mfg/kernels.py:94-104). This is a test of the method, not of the CUDA code
(tests/test_qr_gpu.py does that)."""

import numpy as np
import pytest


def chunk_qr(a):
    a = a.copy()
    rows, nb = a.shape
    tau = np.zeros(nb)
    for j in range(nb):
        x = a[j + 1:, j]
        xn2 = float(x @ x)
        alpha = a[j, j]
        if xn2 > 0:
            beta = -np.copysign(np.sqrt(alpha * alpha + xn2), alpha)
            tau[j] = (beta - alpha) / beta
            a[j + 1:, j] = x / (alpha - beta)
            a[j, j] = beta
            v = np.r_[1.0, a[j + 1:, j]]
            a[j:, j + 1:] -= tau[j] * np.outer(v, v @ a[j:, j + 1:])
    r = np.triu(a[:nb, :nb]).copy()
    for j in range(nb - 1, -1, -1):
        v = np.r_[1.0, a[j + 1:, j]]
        if tau[j] != 0:
            a[j:, j + 1:] -= tau[j] * np.outer(v, v @ a[j:, j + 1:])
        a[j + 1:, j] = -tau[j] * a[j + 1:, j]
        a[j, j] = 1 - tau[j]
        a[:j, j] = 0
    return a, r


def split(rows, nb, ch=256):
    nch = max(1, min(-(-rows // ch), rows // nb))
    return nch, rows // nch, rows % nch


def tsqr(p):
    rows, nb = p.shape
    nch, base, rem = split(rows, nb)
    if nch == 1:
        return chunk_qr(p)
    q = np.empty_like(p)
    rs = np.empty((nch * nb, nb))
    spans = []
    for i in range(nch):
        r0 = i * base + min(i, rem)
        r = base + (i < rem)
        q[r0:r0 + r], rs[i * nb:(i + 1) * nb] = chunk_qr(p[r0:r0 + r])
        spans.append((r0, r))
    q2, rtop = tsqr(rs)
    for i, (r0, r) in enumerate(spans):
        q[r0:r0 + r] = q[r0:r0 + r] @ q2[i * nb:(i + 1) * nb]
    return q, rtop


def bcgs2_qr(b):
    m, p = b.shape
    q = np.empty((m, p))
    d = np.empty(p)
    for j0 in range(0, p, 32):
        nb = min(32, p - j0)
        pan = b[:, j0:j0 + nb].copy()
        if j0 == 0:
            q[:, :nb], r = tsqr(pan)
            d[:nb] = np.abs(np.diag(r))
            continue
        qp = q[:, :j0]
        pan -= qp @ (qp.T @ pan)
        q1, r1 = tsqr(pan)
        q1 = q1 - qp @ (qp.T @ q1)
        q[:, j0:j0 + nb], r2 = tsqr(q1)
        d[j0:j0 + nb] = np.abs(np.diag(r2) * np.diag(r1))
    return q, d


@pytest.mark.parametrize("m,p,kind", [(900, 130, "rand"), (900, 130, "graded"), (700, 90, "krylov"),
                                      (600, 100, "deficient"), (40, 33, "deficient"), (5, 3, "rand")])
def test_bcgs2_tsqr_matches_householder(m, p, kind):
    rng = np.random.default_rng(m + p)
    b = rng.standard_normal((m, p))
    if kind == "graded":
        b *= np.logspace(4, -8, p)
    elif kind == "krylov":
        a = rng.standard_normal((m, m))
        a = a + a.T
        x = b[:, :30]
        b = np.c_[x, a @ x, a @ (a @ x)]
    elif kind == "deficient":
        b[:, p // 2:p // 2 + 5] = b[:, :5] @ rng.standard_normal((5, 5))
        b[:, -1] = b[:, 0]
    q, d = bcgs2_qr(b)
    d0 = np.abs(np.diag(np.linalg.qr(b)[1]))
    thr = 1e-10 * np.linalg.norm(b)
    assert np.max(np.abs(q.T @ q - np.eye(p))) < 1e-13
    assert np.array_equal(d > thr, d0 > thr)
    if kind != "deficient":
        keep = d0 > thr
        assert np.max(np.abs(d - d0)[keep] / d0[keep]) < 1e-11
