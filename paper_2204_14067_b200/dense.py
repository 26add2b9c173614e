"""Dense fp64 contractions of the lifting step on our own tensor-core kernels
(csrc/dense.cu, mma.sync.m8n8k4.f64), replacing the cuBLAS GEMMs the
reference's numpy ``@`` calls map to (mfg/operators.py:67-81,102-118,
mfg/kernels.py:76-135, mfg/eigensolver.py:81-92,151-160,
mfg/proxlift.py:127-314).

* ``gram(a, b)``      a^T b   (tall a, b: rows are the contraction; split-K
                      over row slices, partials added in slice order)
* ``matmul(a, b)``    a b     (tall a times a small b), optional
                      ``alpha``, ``beta`` and ``out``
* ``project_out(q, x)``  x - q (q^T x)
* ``qr(b)``           (Q, |diag R|) of the tall-skinny QR b = Q R (csrc/qr.cu:
                      block Gram-Schmidt with re-orthogonalisation around a
                      Householder TSQR of 32-column panels), replacing
                      LAPACK/cuSOLVER geqrf + orgqr (mfg/kernels.py:94)

Inputs are fp64 device tensors (made contiguous, 1-d vectors as columns);
results are bitwise reproducible run to run."""

from __future__ import annotations

import torch

from . import _lib

_WS: dict = {}


def _ws(nbytes: int, device) -> torch.Tensor:
    key = (device.type, device.index)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        # zero-filled: the Gram kernel's arrival counters (at the front) must
        # start at zero; the kernel leaves them zero
        buf = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _mat(x: torch.Tensor) -> torch.Tensor:
    if x.dtype != torch.float64:
        x = x.double()
    if x.ndim == 1:
        x = x[:, None]
    if x.ndim != 2:
        raise ValueError("expected a matrix")
    return x if x.is_contiguous() else x.contiguous()


def gram(a: torch.Tensor, b: torch.Tensor | None = None, alpha: float = 1.0) -> torch.Tensor:
    """alpha * a^T b (p x q) for a (m x p), b (m x q); b defaults to a."""
    a = _mat(a)
    b = a if b is None else _mat(b)
    m, p = a.shape
    if b.shape[0] != m:
        raise ValueError(f"gram: row counts differ ({m} vs {b.shape[0]})")
    q = b.shape[1]
    out = torch.empty((p, q), dtype=torch.float64, device=a.device)
    if p == 0 or q == 0:
        return out
    lib = _lib.lib()
    wsb = int(lib.mfg_gemm_tn_workspace(m, p, q))
    ws = _ws(wsb, a.device) if wsb else None
    _lib.check(lib.mfg_gemm_tn(m, p, q, a.data_ptr(), p, b.data_ptr(), q, float(alpha),
                               out.data_ptr(), q, ws.data_ptr() if ws is not None else None,
                               wsb, _lib.stream_ptr()), "gemm_tn")
    return out


def matmul(a: torch.Tensor, b: torch.Tensor, alpha: float = 1.0, beta: float = 0.0,
           out: torch.Tensor | None = None) -> torch.Tensor:
    """alpha * a b + beta * out for a (m x p), b (p x q)."""
    vec = b.ndim == 1
    a = _mat(a)
    b = _mat(b)
    m, p = a.shape
    if b.shape[0] != p:
        raise ValueError(f"matmul: inner dimensions differ ({p} vs {b.shape[0]})")
    q = b.shape[1]
    if out is None:
        out = torch.empty((m, q), dtype=torch.float64, device=a.device)
        beta = 0.0
    elif not (out.dtype == torch.float64 and out.is_contiguous() and tuple(out.shape[:1]) == (m,)):
        raise ValueError("matmul: out must be a contiguous fp64 (m x q) tensor")
    if m and q:
        _lib.check(_lib.lib().mfg_gemm_nn(m, p, q, a.data_ptr(), p, b.data_ptr(), q, float(alpha),
                                          float(beta), out.data_ptr(), q, _lib.stream_ptr()),
                   "gemm_nn")
    return out[:, 0] if vec and out.ndim == 2 and q == 1 else out


def project_out(q: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """x - q (q^T x), a new tensor (x's shape)."""
    vec = x.ndim == 1
    xm = _mat(x)
    if q.shape[1] == 0:
        return x.clone() if not vec else xm[:, 0].clone()
    out = xm.clone()
    matmul(q, gram(q, xm), alpha=-1.0, beta=1.0, out=out)
    return out[:, 0] if vec else out


def qr(b: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(Q, d): Q (m x p) with orthonormal columns and d[j] = |R_jj| of the
    unpivoted QR factorisation b = Q R (m >= p). Q equals the Householder Q
    of np.linalg.qr (mfg/kernels.py:94) up to column signs; d is what the
    reference's |R_jj| <= tol ||b||_F screening reads."""
    b = _mat(b)
    m, p = b.shape
    if p > m:
        raise ValueError(f"qr: expected a tall block, got {m}x{p}")
    q = torch.empty((m, p), dtype=torch.float64, device=b.device)
    d = torch.empty((p,), dtype=torch.float64, device=b.device)
    if p == 0:
        return q, d
    lib = _lib.lib()
    wsb = int(lib.mfg_qr_workspace(m, p))
    ws = _ws(wsb, b.device)
    _lib.check(lib.mfg_qr(m, p, b.data_ptr(), p, q.data_ptr(), p, d.data_ptr(), ws.data_ptr(), wsb,
                          _lib.stream_ptr()), "qr")
    return q, d
