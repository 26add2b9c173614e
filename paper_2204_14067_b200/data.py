"""Omega storage on the device, SDDMM residuals, quadratic loss, RMSE.

Mirror of the reference module mfg/data.py (mfglobal 0.1.0). Same names,
argument meaning and errors; the observed set lives in HBM as int32 CSR + CSC
index arrays with the flat-chunk scheduling metadata the kernels use, and
every Omega-sized computation runs in libmfg_b200 (no CPU path).

f(X) = ||P_Omega(X - A)||_F^2 with no 1/2 (mfg/data.py:1-7), so the gradient
is 2 * P_Omega(X - A) and L = 2.
"""

from __future__ import annotations

import ctypes
import io
import os
from dataclasses import dataclass, field
from typing import TYPE_CHECKING

import numpy as np
import torch

from . import _lib
from .kernels import SvdTriplet, as_device

if TYPE_CHECKING:
    from .operators import FactorPair

LIPSCHITZ = 2.0                  # mfg/data.py:25
_EVAL_CHUNK = 1 << 18            # mfg/data.py:29 (kept for API parity; the GPU path is unchunked)


class DatasetError(ValueError):
    """Malformed or unusable rating data (mfg/data.py:32-33)."""


class EmptyDatasetError(DatasetError):
    pass


class ParseError(DatasetError):
    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


def _i32(n):
    return torch.empty(max(int(n), 0), dtype=torch.int32, device="cuda")


# Entry-stream arrays (column / row indices, values) are allocated with
# OMEGA_PAD zero entries past nnz: the grouped sweep kernel prefetches a
# block ahead without bounds guards (include/mfg_b200.h).
OMEGA_PAD = 64


def _padded(n, dtype, device="cuda"):
    return torch.zeros(max(int(n), 0) + OMEGA_PAD, dtype=dtype, device=device)[: max(int(n), 0)]


def _padded_copy(t):
    out = _padded(t.numel(), t.dtype, t.device)
    out.copy_(t)
    return out


class _LayoutBuffers:
    """One orientation's device arrays + its ctypes ``mfg_layout``."""

    def __init__(self, nrows, ncols, nnz, ptr, idx, row_of):
        self.nrows, self.ncols, self.nnz = int(nrows), int(ncols), int(nnz)
        self.ptr, self.idx, self.row_of = ptr, idx, row_of
        nb = (self.nnz + 31) // 32
        self.bmask = _i32(max(nb, 1))
        self.brank = _i32(max(nb, 1))
        self.nzrows = _i32(max(self.nrows, 1))
        self.empty_rows = _i32(max(self.nrows, 1))
        lib = _lib.lib()
        wsb = lib.mfg_layout_workspace(self.nnz, self.nrows)
        ws = _lib.WS.get(wsb, ptr.device)
        nne, ne = ctypes.c_int32(0), ctypes.c_int32(0)
        _lib.check(lib.mfg_layout_build(self.nrows, self.nnz, ptr.data_ptr(), row_of.data_ptr(),
                                        self.bmask.data_ptr(), self.brank.data_ptr(),
                                        self.nzrows.data_ptr(), self.empty_rows.data_ptr(),
                                        ctypes.byref(nne), ctypes.byref(ne), ws.data_ptr(), wsb,
                                        _lib.stream_ptr()), "layout build")
        self.n_nonempty, self.n_empty = nne.value, ne.value
        self.c = _lib.Layout(self.nrows, self.ncols, self.nnz, ptr.data_ptr(), idx.data_ptr(),
                             row_of.data_ptr(), self.bmask.data_ptr(), self.brank.data_ptr(),
                             self.nzrows.data_ptr(), self.n_nonempty, self.empty_rows.data_ptr(),
                             self.n_empty)

    @property
    def ref(self):
        return ctypes.byref(self.c)


class OmegaDevice:
    """Omega in HBM: CSR (row-major sorted) and CSC views plus metadata.

    Data layout (int32 indices, |Omega| < 2^31):
      csr: ptr[m+1], idx=cols[nnz], row_of=rows[nnz], vals[nnz] (storage dtype)
      csc: ptr[n+1], idx=rows_in_csc[nnz], row_of=cols_sorted[nnz],
           perm[nnz] (CSR position of each CSC entry), vals_csc[nnz]
    """

    def __init__(self, m, n, rows64, cols64, vals64, dtype):
        _lib.require_cuda()
        lib = _lib.lib()
        self.m, self.n = int(m), int(n)
        self.dtype = dtype
        nnz = int(vals64.numel())
        self.nnz = nnz
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        rows = _padded(nnz, torch.int32, dev)
        cols = _padded(nnz, torch.int32, dev)
        vals = _padded(nnz, torch.float64, dev)
        ptr = _i32(self.m + 1)
        csc_ptr = _i32(self.n + 1)
        csc_rows = _padded(nnz, torch.int32, dev)
        csc_cols = _padded(nnz, torch.int32, dev)
        csc_perm = _i32(nnz)
        wsb = lib.mfg_omega_build_workspace(nnz, self.m, self.n)
        ws = _lib.WS.get(wsb, dev)
        dup = ctypes.c_int64(-1)
        rerr = ctypes.c_int32(0)
        st = lib.mfg_omega_build(self.m, self.n, nnz, rows64.data_ptr(), cols64.data_ptr(),
                                 vals64.data_ptr(), rows.data_ptr(), cols.data_ptr(),
                                 vals.data_ptr(), ptr.data_ptr(), csc_ptr.data_ptr(),
                                 csc_rows.data_ptr(), csc_cols.data_ptr(), csc_perm.data_ptr(),
                                 ctypes.byref(dup), ctypes.byref(rerr), ws.data_ptr(), wsb,
                                 _lib.stream_ptr())
        if st == _lib.MFG_ERR_DATASET:
            if rerr.value == 1:
                raise DatasetError("row index out of range")
            if rerr.value == 2:
                raise DatasetError("column index out of range")
            i = int(dup.value)
            r = int(rows[i].item())
            c = int(cols[i].item())
            raise DatasetError(f"duplicate entry at ({r}, {c}); refusing to aggregate")
        _lib.check(st, "omega build")
        self.vals64 = vals
        self.vals = vals if dtype == torch.float64 else _padded_copy(vals.to(dtype))
        self.csr = _LayoutBuffers(self.m, self.n, nnz, ptr, cols, rows)
        self.csc = _LayoutBuffers(self.n, self.m, nnz, csc_ptr, csc_rows, csc_cols)
        self.csc_perm = csc_perm
        self.vals_csc = self.gather_csc(self.vals)

    def gather_csc(self, vals: torch.Tensor) -> torch.Tensor:
        """Values in CSR order -> CSC order (one gather kernel)."""
        out = _padded(vals.numel(), vals.dtype, vals.device)
        _lib.check(_lib.lib().mfg_gather(_lib.dtype_code(vals.dtype), self.nnz,
                                         self.csc_perm.data_ptr(), vals.data_ptr(),
                                         out.data_ptr(), _lib.stream_ptr()), "gather")
        return out

    def workspace(self, nbytes):
        return _lib.WS.get(nbytes, self.device)


@dataclass
class ObservationSet:
    """Sparse observed ratings A restricted to Omega (mfg/data.py:46-119).

    Immutable after construction. Entries are sorted by (row, col); the
    device copy (``dev``) is the one every kernel reads. ``rows``/``cols``/
    ``vals``/``indptr`` are host numpy views materialised on first access
    (int64/float64, exactly as the reference stores them). ``dtype`` is the
    storage precision of Omega values and MF factors on the device
    (float64 = the reference's precision; float32 = "fp32 mode").
    """

    m: int
    n: int
    dev: OmegaDevice = field(repr=False)
    transposed: bool = False
    row_ids: np.ndarray | None = None
    col_ids: np.ndarray | None = None
    _host: dict = field(default_factory=dict, repr=False)

    @property
    def size(self) -> int:
        return int(self.dev.nnz)

    @property
    def dtype(self) -> torch.dtype:
        return self.dev.dtype

    def _h(self, name):
        if name not in self._host:
            d = self.dev
            if name == "rows":
                self._host[name] = d.csr.row_of.cpu().numpy().astype(np.int64)
            elif name == "cols":
                self._host[name] = d.csr.idx.cpu().numpy().astype(np.int64)
            elif name == "vals":
                self._host[name] = d.vals64.cpu().numpy()
            elif name == "indptr":
                self._host[name] = d.csr.ptr.cpu().numpy().astype(np.int64)
        return self._host[name]

    rows = property(lambda self: self._h("rows"))
    cols = property(lambda self: self._h("cols"))
    vals = property(lambda self: self._h("vals"))
    indptr = property(lambda self: self._h("indptr"))

    @staticmethod
    def from_coo(
        m: int,
        n: int,
        rows,
        cols,
        vals,
        transposed: bool = False,
        row_ids: np.ndarray | None = None,
        col_ids: np.ndarray | None = None,
        dtype=torch.float64,
    ) -> "ObservationSet":
        """mfg/data.py:70-102 on the device (validation, sort, dedupe, CSR/CSC)."""
        _lib.require_cuda()
        rows = torch.as_tensor(np.asarray(rows, dtype=np.int64) if not torch.is_tensor(rows) else rows,
                               dtype=torch.int64).reshape(-1)
        cols = torch.as_tensor(np.asarray(cols, dtype=np.int64) if not torch.is_tensor(cols) else cols,
                               dtype=torch.int64).reshape(-1)
        vals = torch.as_tensor(np.asarray(vals, dtype=np.float64) if not torch.is_tensor(vals) else vals,
                               dtype=torch.float64).reshape(-1)
        if rows.numel() != cols.numel() or rows.numel() != vals.numel():
            raise DatasetError("index/value arrays disagree in length")
        dev = OmegaDevice(m, n, rows.cuda(), cols.cuda(), vals.cuda(), dtype)
        return ObservationSet(int(m), int(n), dev, transposed, row_ids, col_ids)

    def with_dtype(self, dtype) -> "ObservationSet":
        """Same Omega, other storage precision (shares the index arrays)."""
        if dtype == self.dtype:
            return self
        d = object.__new__(OmegaDevice)
        d.__dict__.update(self.dev.__dict__)
        d.dtype = dtype
        d.vals = self.dev.vals64 if dtype == torch.float64 else _padded_copy(self.dev.vals64.to(dtype))
        d.vals_csc = self.dev.gather_csc(d.vals)
        return ObservationSet(self.m, self.n, d, self.transposed, self.row_ids, self.col_ids)


@dataclass
class EvalSplit:
    """Held-out test entries over the same (m, n) grid (mfg/data.py:122-135).

    Test entries are evaluated with the same SDDMM kernel; the device copy is
    built lazily as an ObservationSet-like layout (duplicates allowed here in
    the reference, so no dedupe is applied: entries are kept as given)."""

    m: int
    n: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    transposed: bool = False
    _dev: object = field(default=None, repr=False)

    @property
    def size(self) -> int:
        return int(np.asarray(self.vals).size)


@dataclass
class SparseResidual:
    """Values on the training pattern Omega (mfg/data.py:138-161).

    ``vals`` is a device tensor in CSR order sharing the index arrays of the
    ObservationSet. ``sumsq`` caches the fused fp64 sum of squares produced
    by the SDDMM that created it (loss_quad reads it)."""

    m: int
    n: int
    obs: ObservationSet = field(repr=False)
    vals: torch.Tensor = field(repr=False)
    sumsq: float | None = None
    _csc: torch.Tensor | None = field(default=None, repr=False)
    _v64: torch.Tensor | None = field(default=None, repr=False)

    @property
    def rows(self):
        return self.obs.rows

    @property
    def cols(self):
        return self.obs.cols

    @property
    def indptr(self):
        return self.obs.indptr

    def scaled(self, c: float) -> "SparseResidual":
        ss = None if self.sumsq is None else self.sumsq * c * c
        return SparseResidual(self.m, self.n, self.obs, self.vals * c, ss)

    def vals64(self) -> torch.Tensor:
        """fp64 values (the lifting operator always runs in fp64)."""
        if self._v64 is None:
            self._v64 = self.vals if self.vals.dtype == torch.float64 else self.vals.double()
        return self._v64

    def vals_csc64(self) -> torch.Tensor:
        """fp64 values in CSC order (cached: one gather per gradient object,
        the analogue of the reference's cached csr_t, mfg/data.py:156-158)."""
        if self._csc is None:
            self._csc = self.obs.dev.gather_csc(self.vals64())
        return self._csc

    def norm(self) -> float:
        return float(np.sqrt(_dot(self.vals, self.vals)))

    def host_vals(self) -> np.ndarray:
        return self.vals.double().cpu().numpy()


def _dot(x: torch.Tensor, y: torch.Tensor) -> float:
    """fp64 dot product on the device, deterministic (one kernel + 8 B D2H)."""
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    ws = _lib.WS.get(1 << 16, x.device)
    x = x.contiguous()
    y = y.contiguous().to(x.dtype)
    _lib.check(_lib.lib().mfg_dot(_lib.dtype_code(x.dtype), x.numel(), x.data_ptr(), y.data_ptr(),
                                  out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
               "dot")
    return float(out.item())


def sddmm(obs: ObservationSet, left: torch.Tensor, right: torch.Tensor, *, scale=None,
          a=True, g: torch.Tensor | None = None, out_mult: float = 1.0, want_out=True,
          dtype=None, compute_f64=True):
    """Device SDDMM with fused fp64 reductions (see mfg_sddmm in the header).

    Returns (out or None, sums[3] as a host numpy array)."""
    dev = obs.dev
    dtype = dtype or left.dtype
    k = int(left.shape[1])
    left = left.to(dtype).contiguous()
    right = right.to(dtype).contiguous()
    if left.shape[0] != obs.m or right.shape[0] != obs.n or right.shape[1] != k:
        raise ValueError("sddmm operand shapes do not match Omega")
    A = None
    if a:
        A = dev.vals if dtype == dev.dtype else (dev.vals64 if dtype == torch.float64 else dev.vals.to(dtype))
    G = None if g is None else g.to(dtype).contiguous()
    out = torch.empty(obs.size, dtype=dtype, device=dev.device) if want_out else None
    sums = torch.empty(3, dtype=torch.float64, device=dev.device)
    sc = None
    if scale is not None:
        sc = torch.as_tensor(np.asarray(scale, dtype=np.float64)).to(dev.device)
    lib = _lib.lib()
    wsb = lib.mfg_sddmm_workspace(dev.csr.ref, max(k, 1))
    ws = dev.workspace(wsb)
    _lib.check(lib.mfg_sddmm(_lib.dtype_code(dtype), 1 if compute_f64 else 0, dev.csr.ref, k,
                             left.data_ptr(), max(k, 1), _lib.ptr(sc), right.data_ptr(), max(k, 1),
                             _lib.ptr(A), _lib.ptr(G), float(out_mult), _lib.ptr(out),
                             sums.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()), "sddmm")
    return out, sums.cpu().numpy()


def pair_values(left, right, rows=None, cols=None, obs: ObservationSet | None = None):
    """Entrywise values of left @ right.T on Omega (mfg/data.py:253-263).

    The device path evaluates on an ObservationSet's pattern (``obs``); the
    explicit-index form of the reference is supported for arbitrary index
    lists through a temporary pattern (duplicates allowed)."""
    left = as_device(left)
    right = as_device(right)
    if obs is None:
        obs = _adhoc_pattern(left.shape[0], right.shape[0], rows, cols)
        vals, _ = sddmm(obs.obs, left, right, a=False, dtype=torch.float64)
        return vals[obs.inverse]
    vals, _ = sddmm(obs, left, right, a=False, dtype=torch.float64)
    return vals


@dataclass
class _Adhoc:
    obs: ObservationSet
    inverse: torch.Tensor


def _adhoc_pattern(m, n, rows, cols) -> _Adhoc:
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    key = rows * n + cols
    uk, inv = np.unique(key, return_inverse=True)
    obs = ObservationSet.from_coo(m, n, uk // n, uk % n, np.zeros(uk.size))
    return _Adhoc(obs, torch.as_tensor(inv, device="cuda"))


def triplet_values(x: SvdTriplet, obs: ObservationSet) -> torch.Tensor:
    """mfg/data.py:266-269 on Omega: values of U diag(sigma) V^T."""
    if x.rank == 0:
        return torch.zeros(obs.size, dtype=torch.float64, device=obs.dev.device)
    out, _ = sddmm(obs, x.u, x.v, scale=x.sigma, a=False, dtype=torch.float64)
    return out


def residual_on_omega(obs: ObservationSet, wf: "FactorPair") -> SparseResidual:
    """r_ij = (W H^T)_ij - A_ij on Omega (mfg/data.py:272-280)."""
    if wf.w.shape[0] != obs.m or wf.h.shape[0] != obs.n:
        raise ValueError(
            f"factor dims ({wf.w.shape[0]}, {wf.h.shape[0]}) do not match data "
            f"({obs.m}, {obs.n})"
        )
    # Residuals (hence gradients) are stored in fp64 in both precision modes:
    # they feed the lifting step, whose Eq. 5 test compares O(f) quantities
    # with a 1e-12 relative slack. In fp32 mode the factors are fp32 and the
    # products are formed exactly in fp64.
    w = wf.w.to(obs.dtype).double()
    h = wf.h.to(obs.dtype).double()
    vals, sums = sddmm(obs, w, h, dtype=torch.float64)
    return SparseResidual(obs.m, obs.n, obs, vals, float(sums[0]))


def residual_on_omega_svd(obs: ObservationSet, x: SvdTriplet) -> SparseResidual:
    """Same with X as an SVD triplet (mfg/data.py:283-288); fp64 always."""
    if x.m != obs.m or x.n != obs.n:
        raise ValueError(f"triplet dims ({x.m}, {x.n}) do not match data ({obs.m}, {obs.n})")
    if x.rank == 0:
        vals = -obs.dev.vals64
        return SparseResidual(obs.m, obs.n, obs, vals.clone(), _dot(obs.dev.vals64, obs.dev.vals64))
    vals, sums = sddmm(obs, x.u, x.v, scale=x.sigma, dtype=torch.float64)
    return SparseResidual(obs.m, obs.n, obs, vals, float(sums[0]))


def loss_quad(res: SparseResidual) -> float:
    """f(X) = sum of squared residuals on Omega (mfg/data.py:291-293)."""
    if res.sumsq is not None:
        return float(res.sumsq)
    return _dot(res.vals, res.vals)


def gradient(res: SparseResidual) -> SparseResidual:
    """grad f(X) = 2 * P_Omega(X - A) (mfg/data.py:296-298)."""
    return res.scaled(LIPSCHITZ)


def _split_obs(split: EvalSplit) -> _Adhoc:
    if split._dev is None:
        split._dev = _adhoc_pattern(split.m, split.n, split.rows, split.cols)
        split._dev_vals = torch.as_tensor(np.asarray(split.vals, dtype=np.float64), device="cuda")
    return split._dev


def rmse(split: EvalSplit, x: SvdTriplet) -> float:
    """sqrt(||P_test(X - A)||^2 / |Omega_test|) (mfg/data.py:301-306)."""
    if split.size == 0:
        raise ValueError("empty test set")
    ad = _split_obs(split)
    if x.rank == 0:
        pred = torch.zeros(split.size, dtype=torch.float64, device="cuda")
    else:
        vals, _ = sddmm(ad.obs, x.u, x.v, scale=x.sigma, a=False, dtype=torch.float64)
        pred = vals[ad.inverse]
    diff = pred - split._dev_vals
    return float(np.sqrt(_dot(diff, diff) / split.size))


def rmse_factors(split: EvalSplit, wf: "FactorPair") -> float:
    """mfg/data.py:309-313."""
    if split.size == 0:
        raise ValueError("empty test set")
    ad = _split_obs(split)
    vals, _ = sddmm(ad.obs, wf.w, wf.h, a=False, dtype=torch.float64)
    diff = vals[ad.inverse] - split._dev_vals
    return float(np.sqrt(_dot(diff, diff) / split.size))


# --- text ingest (host side, mirrors mfg/data.py:164-250) -------------------

def _parse_stream(stream, what: str):
    users, items, ratings = [], [], []
    for line_no, raw in enumerate(stream, start=1):
        if isinstance(raw, bytes):
            raw = raw.decode("utf-8", errors="replace")
        line = raw.strip()
        if not line:
            continue
        parts = line.split()
        if len(parts) not in (3, 4):
            raise ParseError(line_no, f"expected 3 or 4 fields, got {len(parts)}")
        try:
            u, i, r = int(parts[0]), int(parts[1]), float(parts[2])
        except ValueError as exc:
            raise ParseError(line_no, f"cannot parse '{line}': {exc}") from None
        if u <= 0 or i <= 0:
            raise ParseError(line_no, "user/item ids must be positive integers")
        users.append(u)
        items.append(i)
        ratings.append(r)
    if not users:
        raise EmptyDatasetError(f"no ratings found in {what}")
    return (np.asarray(users, dtype=np.int64), np.asarray(items, dtype=np.int64),
            np.asarray(ratings, dtype=np.float64))


def _parse_native(buf: bytes):
    """libmfg_b200 mfg_parse_ratings on an in-memory file (multi-threaded);
    None when a line needs the reference's rules (the caller re-parses)."""
    import ctypes

    from . import _lib

    lib = _lib.lib()
    cap = int(lib.mfg_count_lines(buf, len(buf)))
    users = np.empty(cap, dtype=np.int64)
    items = np.empty(cap, dtype=np.int64)
    ratings = np.empty(cap, dtype=np.float64)
    count = ctypes.c_size_t(0)
    odd = ctypes.c_int64(0)
    st = lib.mfg_parse_ratings(buf, len(buf), 0, users.ctypes.data, items.ctypes.data,
                               ratings.ctypes.data, cap, ctypes.byref(count), ctypes.byref(odd))
    if st != _lib.MFG_OK:
        return None
    c = int(count.value)
    return users[:c], items[:c], ratings[:c]


def _parse_source(source, what: str):
    """Parse a path, bytes or an iterable of lines. Files and bytes go through
    the native parser; a line it does not take (or an iterable source) is
    parsed with the reference's rules (mfg/data.py:164-200), so accepted
    values and raised errors are the reference's."""
    if isinstance(source, (str, os.PathLike, bytes)):
        if isinstance(source, bytes):
            buf = source
        else:
            with open(source, "rb") as fh:
                buf = fh.read()
        out = _parse_native(buf)
        if out is not None:
            if out[0].size == 0:
                raise EmptyDatasetError(f"no ratings found in {what}")
            return out
        return _parse_stream(io.BytesIO(buf), what)
    return _parse_stream(source, what)


INSTANCE_MAGIC = b"MFGOMEG1"
_INSTANCE_FIELDS = 8   # int64 header words after the magic


def write_instance(path, m: int, n: int, rows, cols, vals, transposed: bool = False,
                   row_ids=None, col_ids=None, split: "EvalSplit | None" = None) -> None:
    """Binary Omega instance, the at-scale stand-in
    for re-parsing text with load_ratings (mfg/data.py:203-250): the magic,
    8 little-endian int64 words (m, n, nnz, transposed, value bytes, #row ids,
    #col ids, #test entries), then 8-byte aligned arrays: rows, cols (int32),
    values (f32 or f64), row ids, col ids (int64), test rows, cols (int32) and
    values (f64). Entries are stored as given (canonical order when written
    from an ObservationSet)."""
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    vals = np.ascontiguousarray(vals)
    if vals.dtype not in (np.float32, np.float64):
        vals = vals.astype(np.float64)
    if not (rows.size == cols.size == vals.size):
        raise ValueError("rows, cols and vals must have the same length")
    rid = np.zeros(0, np.int64) if row_ids is None else np.ascontiguousarray(row_ids, dtype=np.int64)
    cid = np.zeros(0, np.int64) if col_ids is None else np.ascontiguousarray(col_ids, dtype=np.int64)
    if split is not None:
        tr, tc = np.asarray(split.rows, np.int32), np.asarray(split.cols, np.int32)
        tv = np.asarray(split.vals, np.float64)
    else:
        tr = tc = np.zeros(0, np.int32)
        tv = np.zeros(0, np.float64)
    head = np.array([m, n, rows.size, int(bool(transposed)), vals.itemsize, rid.size, cid.size, tr.size],
                    dtype="<i8")
    with open(path, "wb") as fh:
        fh.write(INSTANCE_MAGIC)
        fh.write(head.tobytes())
        for a in (rows, cols, vals, rid, cid, tr, tc, tv):
            b = a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()
            fh.write(b)
            if len(b) % 8:
                fh.write(b"\0" * (8 - len(b) % 8))


def read_instance(path) -> dict:
    """Host arrays of a binary Omega instance (one read per array)."""
    with open(path, "rb") as fh:
        if fh.read(len(INSTANCE_MAGIC)) != INSTANCE_MAGIC:
            raise DatasetError(f"{path}: not an Omega instance file")
        head = np.frombuffer(fh.read(8 * _INSTANCE_FIELDS), dtype="<i8")
        if head.size != _INSTANCE_FIELDS:
            raise DatasetError(f"{path}: truncated header")
        m, n, nnz, tr, vb, nr, nc, nt = (int(x) for x in head)
        if vb not in (4, 8) or min(m, n, nnz, nr, nc, nt) < 0:
            raise DatasetError(f"{path}: corrupt header")
        out = {"m": m, "n": n, "transposed": bool(tr)}

        def arr(name, dt, count):
            a = np.fromfile(fh, dtype=dt, count=count)
            if a.size != count:
                raise DatasetError(f"{path}: truncated {name}")
            pad = (-count * np.dtype(dt).itemsize) % 8
            if pad:
                fh.read(pad)
            out[name] = a

        arr("rows", "<i4", nnz)
        arr("cols", "<i4", nnz)
        arr("vals", "<f4" if vb == 4 else "<f8", nnz)
        arr("row_ids", "<i8", nr)
        arr("col_ids", "<i8", nc)
        arr("test_rows", "<i4", nt)
        arr("test_cols", "<i4", nt)
        arr("test_vals", "<f8", nt)
    return out


def save_instance(path, obs: "ObservationSet", split: "EvalSplit | None" = None) -> None:
    """Write an ObservationSet (and optional test split) as a binary instance."""
    vals = obs.vals
    write_instance(path, obs.m, obs.n, obs.rows, obs.cols,
                   vals.astype(np.float32) if obs.dtype == torch.float32 else vals,
                   obs.transposed, obs.row_ids, obs.col_ids, split)


def load_instance(path, dtype=None):
    """(ObservationSet, EvalSplit | None) from a binary instance; the device
    build validates the entries exactly as from_coo does."""
    a = read_instance(path)
    if dtype is None:
        dtype = torch.float32 if a["vals"].dtype == np.float32 else torch.float64
    obs = ObservationSet.from_coo(a["m"], a["n"], a["rows"], a["cols"], a["vals"], a["transposed"],
                                  a["row_ids"] if a["row_ids"].size else None,
                                  a["col_ids"] if a["col_ids"].size else None, dtype=dtype)
    split = None
    if a["test_rows"].size:
        split = EvalSplit(a["m"], a["n"], a["test_rows"].astype(np.int64), a["test_cols"].astype(np.int64),
                          a["test_vals"], a["transposed"])
    return obs, split


def load_ratings(source, test_source=None, fmt: str = "movielens-tsv", dtype=torch.float64):
    """Whitespace "user item rating [timestamp]" loader (mfg/data.py:203-250):
    id compaction over train+test, transpose to m <= n."""
    if fmt != "movielens-tsv":
        raise DatasetError(f"unsupported format: {fmt}")
    users, items, ratings = _parse_source(source, "training data")
    test_raw = None
    if test_source is not None:
        test_raw = _parse_source(test_source, "test data")
    all_users = users if test_raw is None else np.concatenate([users, test_raw[0]])
    all_items = items if test_raw is None else np.concatenate([items, test_raw[1]])
    uniq_users, uniq_items = np.unique(all_users), np.unique(all_items)
    u_idx = np.searchsorted(uniq_users, users)
    i_idx = np.searchsorted(uniq_items, items)
    m, n = uniq_users.size, uniq_items.size
    transposed = m > n
    if transposed:
        m, n = n, m
        u_idx, i_idx = i_idx, u_idx
        row_ids, col_ids = uniq_items, uniq_users
    else:
        row_ids, col_ids = uniq_users, uniq_items
    obs = ObservationSet.from_coo(m, n, u_idx, i_idx, ratings, transposed, row_ids, col_ids,
                                  dtype=dtype)
    split = None
    if test_raw is not None:
        tu = np.searchsorted(uniq_users, test_raw[0])
        ti = np.searchsorted(uniq_items, test_raw[1])
        if transposed:
            tu, ti = ti, tu
        order = np.lexsort((ti, tu))
        split = EvalSplit(m, n, tu[order], ti[order], test_raw[2][order], transposed)
    return obs, split
