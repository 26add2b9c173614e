"""Nonconvex factorisation phase on the device (mirror of mfg/mfsolver.py).

Lemma-1 factors, the MF objective (one fused Omega sweep), and exact
block-coordinate descent whose per-row normal equations are assembled and
solved inside libmfg_b200 (mfg_bcd_half_sweep) without ever materialising
the (m, k, k) normal tensor of the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .data import ObservationSet
from .kernels import SIGMA_FLOOR, SvdTriplet, as_device
from .operators import FactorPair
from ._nvtx import annotate

_GUARD_SLACK = 1e-9          # mfg/mfsolver.py:15
_GUARD_SLACK_F32 = 1e-6      # fp32 storage: rounding of the stored factors
_PAIR_CHUNK = 1 << 25        # mfg/mfsolver.py:18 (API parity; unused on device)


def guard_slack(dtype) -> float:
    return _GUARD_SLACK if dtype == torch.float64 else _GUARD_SLACK_F32


class MfPhaseError(RuntimeError):
    """The BCD sweep increased the objective: indicates a kernel bug."""


def factors_from_svd(x: SvdTriplet) -> FactorPair:
    """W = U sqrt(s), H = V sqrt(s) (mfg/mfsolver.py:25-32)."""
    root = torch.as_tensor(np.sqrt(x.sigma), device=x.u.device)
    return FactorPair(x.u * root, x.v * root)


def svd_from_factors(wf: FactorPair) -> SvdTriplet:
    """Compact SVD of W H^T via QR of the factors and a k x k SVD (35-45)."""
    if wf.k == 0:
        return SvdTriplet.zero(wf.m, wf.n)
    from . import dense

    def qr(a):
        # our TSQR-panel QR (csrc/qr.cu); R = Q^T A on the DMMA Gram kernel
        a = a.double()
        if a.shape[1] > a.shape[0]:
            return torch.linalg.qr(a)       # wide factor (test scale only)
        q, _ = dense.qr(a)
        return q, dense.gram(q, a)

    qw, rw = qr(wf.w)
    qh, rh = qr(wf.h)
    u_mid, s, vt_mid = torch.linalg.svd(rw @ rh.T)
    sh = s.cpu().numpy()
    if sh.size == 0 or sh[0] == 0.0:
        return SvdTriplet.zero(wf.m, wf.n)
    kept = np.flatnonzero(sh > SIGMA_FLOOR * sh[0])
    idx = torch.as_tensor(kept, device=qw.device)
    return SvdTriplet(qw @ u_mid.index_select(1, idx), sh[kept], qh @ vt_mid.T.index_select(1, idx))


def grouped_width(k: int, dtype, compute_f64: bool = False) -> int:
    """Padded factor width of the grouped sweep kernel for k (0 = not used)."""
    if dtype == torch.float32:
        if compute_f64:
            return 32 if k <= 32 else 0
        return 32 if k <= 32 else (64 if k <= 64 else 0)
    return 16 if k <= 16 else (32 if k <= 32 else 0)


def grouped_ld(k: int, dtype, compute_f64: bool = False) -> int:
    """Factor row stride the single-launch grouped sweep kernel takes for
    width k (``mfg_sweep_ld``): k itself when a row is whole 16-byte chunks
    (k * elem % 16 == 0), else the padded width kp (0 = kernel not used)."""
    if k < 1 or not grouped_width(k, dtype, compute_f64):
        return 0
    return int(_lib.lib().mfg_sweep_ld(_lib.dtype_code(dtype), 1 if compute_f64 else 0, int(k)))


class SweepPlan:
    """Pre-planned Omega sweep (mfg_sweep) with resident outputs and workspace.

    ``run(w, h)`` enqueues one sweep on the current stream without any host
    synchronisation; outputs land in ``R``, ``RH``, ``RtW`` and the fp64 device
    vector ``sums`` = [sum r^2, ||W||^2, ||H||^2]. This is the unit of work of
    the BASELINE metric."""

    def __init__(self, obs: ObservationSet, k: int, *, want_r=True, want_rh=True, want_rtw=True,
                 out_scale: float = 1.0, compute_f64: bool = False):
        self.obs = obs
        dev = obs.dev
        dt = obs.dtype
        self.k = int(k)
        self.dt = dt
        self.compute_f64 = 1 if compute_f64 else 0
        self.out_scale = float(out_scale)
        self.R = torch.empty(obs.size, dtype=dt, device=dev.device) if want_r else None
        # host-facing results in one buffer [sums (32 B) | RH | RtW], so the
        # end-to-end path reads them back with a single D2H copy
        es = torch.empty(0, dtype=dt).element_size()
        nb_rh = obs.m * k * es if want_rh else 0
        nb_rtw = obs.n * k * es if want_rtw else 0
        self._out = torch.zeros(32 + nb_rh + nb_rtw, dtype=torch.uint8, device=dev.device)
        self.sums = self._out[:24].view(torch.float64)
        self.RH = self._out[32:32 + nb_rh].view(dt).view(obs.m, k) if want_rh else None
        self.RtW = self._out[32 + nb_rh:].view(dt).view(obs.n, k) if want_rtw else None
        lib = _lib.lib()
        self.wsb = lib.mfg_sweep_workspace(dev.csr.ref, dev.csc.ref, max(self.k, 1))
        # zero-filled once: the grouped kernel keeps zero-at-rest counters here
        self.ws = torch.zeros(self.wsb, dtype=torch.uint8, device=dev.device)
        self.kp = grouped_width(self.k, dt, compute_f64)
        self.ld = grouped_ld(self.k, dt, compute_f64) or self.k
        self._host = None

    def pad(self, f: torch.Tensor) -> torch.Tensor:
        """Factor in the grouped kernel's layout: contiguous (rows x k) when
        the kernel takes k unpadded (``ld == k``), else a zero-padded
        (rows x kp) copy (one 16-byte vector per lane gathers a whole row)."""
        if self.ld == self.k:
            return f.to(self.dt).contiguous()
        out = torch.zeros((f.shape[0], self.ld), dtype=self.dt, device=self.obs.dev.device)
        out[:, : f.shape[1]] = f
        return out

    def _args(self, w: torch.Tensor, h: torch.Tensor, stream: int) -> tuple:
        dev = self.obs.dev
        return (_lib.dtype_code(self.dt), self.compute_f64, dev.csr.ref, dev.csc.ref, max(self.k, 1),
                dev.vals.data_ptr(), dev.vals_csc.data_ptr(), w.data_ptr(), int(w.stride(0)),
                h.data_ptr(), int(h.stride(0)),
                _lib.ptr(self.R), _lib.ptr(self.RH), _lib.ptr(self.RtW), self.out_scale,
                self.sums.data_ptr(), self.ws.data_ptr(), self.wsb, stream)

    def run(self, w: torch.Tensor, h: torch.Tensor) -> None:
        """w, h: (rows x ld) with ld = k, or the zero-padded width ``kp``."""
        _lib.check(_lib.lib().mfg_sweep(*self._args(w, h, _lib.stream_ptr())), "sweep")

    def run_host(self, w_host: torch.Tensor, h_host: torch.Tensor, *, graph: bool = True):
        """End-to-end sweep from host factors through one ABI call
        (mfg_sweep_host): H2D of W and H into resident device factors, the
        sweep, and one D2H of the packed results [sums | RH | RtW]. Host
        factors are contiguous (rows x k) CPU tensors, pinned for the copies
        to be asynchronous. Returns pinned host views (sums, RH, RtW), valid
        once the current stream reaches this point and until the next call.

        With ``graph`` (default) the call is captured once per (host buffers,
        stream) into a CUDA graph -- H2D copies, sweep kernels and D2H copy as
        one graph -- and replayed, so a step costs one graph launch on the
        host instead of the copy and kernel enqueues. The buffers' contents
        are read at replay time, as with the eager call."""
        if self.RH is None or self.RtW is None:
            raise ValueError("run_host needs a plan with want_rh and want_rtw")
        for t, rows in ((w_host, self.obs.m), (h_host, self.obs.n)):
            if t.device.type != "cpu" or t.dtype != self.dt or tuple(t.shape) != (rows, self.k) \
                    or not t.is_contiguous():
                raise ValueError(f"host factor must be a contiguous CPU ({rows} x {self.k}) {self.dt} tensor")
        stream = torch.cuda.current_stream()
        if self._host is None:
            dev = self.obs.dev.device
            # W and H resident in one allocation (one H2D when the host
            # factors are adjacent too, see pinned_factors)
            whd = torch.zeros((self.obs.m + self.obs.n) * self.ld, dtype=self.dt, device=dev)
            self._wd = whd[: self.obs.m * self.ld].view(self.obs.m, self.ld)
            self._hd = whd[self.obs.m * self.ld:].view(self.obs.n, self.ld)
            self._host = torch.empty(self._out.numel(), dtype=torch.uint8).pin_memory()
            nb_rh = self.RH.numel() * self.RH.element_size()
            self._host_views = (self._host[:24].view(torch.float64),
                                self._host[32:32 + nb_rh].view(self.dt).view(self.obs.m, self.k),
                                self._host[32 + nb_rh:].view(self.dt).view(self.obs.n, self.k))
            dev = self.obs.dev
            self._host_args = (
                _lib.dtype_code(self.dt), self.compute_f64, dev.csr.ref, dev.csc.ref, self.k,
                dev.vals.data_ptr(), dev.vals_csc.data_ptr())
            self._host_tail = (
                self._wd.data_ptr(), self.ld, self._hd.data_ptr(), self.ld, _lib.ptr(self.R),
                self._out.data_ptr(), self._host.data_ptr(), self.out_scale, self.ws.data_ptr(),
                self.wsb)
            self._graph_key = None
        if not graph:
            self._host_call(w_host, h_host, stream.cuda_stream)
            return self._host_views
        key = (w_host.data_ptr(), h_host.data_ptr(), stream.cuda_stream)
        if self._graph_key != key:
            self._host_call(w_host, h_host, stream.cuda_stream)  # warm-up, eager
            g = self._capture(w_host, h_host, stream)
            if g is None:       # capture not possible here: stay eager for this plan
                return self._host_views
            self._graph, self._graph_key = g, key
        self._graph.replay()
        return self._host_views

    def pinned_factors(self):
        """Pinned host buffers (W: m x k, H: n x k) for ``run_host``, adjacent
        in one allocation so the end-to-end call moves both with one H2D copy.
        Fill them in place between calls."""
        whh = torch.zeros((self.obs.m + self.obs.n) * self.k, dtype=self.dt).pin_memory()
        return (whh[: self.obs.m * self.k].view(self.obs.m, self.k),
                whh[self.obs.m * self.k:].view(self.obs.n, self.k))

    def _capture(self, w_host, h_host, stream):
        """Capture one end-to-end call as a CUDA graph (None if the capture is
        invalidated, e.g. by an unrelated thread's synchronising call)."""
        if getattr(self, "_no_graph", False):
            return None
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                self._host_call(w_host, h_host, side.cuda_stream)
        except RuntimeError:
            torch.cuda.synchronize()
            self._no_graph = True
            return None
        stream.wait_stream(side)
        return g

    def _host_call(self, w_host: torch.Tensor, h_host: torch.Tensor, stream: int) -> None:
        _lib.check(_lib.lib().mfg_sweep_host(*self._host_args, w_host.data_ptr(), h_host.data_ptr(),
                                             *self._host_tail, stream), "sweep_host")


def sweep(obs: ObservationSet, wf: FactorPair, *, want_r=False, want_rh=False, want_rtw=False,
          out_scale: float = 1.0, compute_f64: bool = True):
    """One fused Omega sweep (mfg_sweep): R, R.H, R^T.W and fp64 sums.

    Returns (R, RH, RtW, sums) with sums = [sum r^2, ||W||^2, ||H||^2] on the
    host; unrequested outputs are None."""
    dt = obs.dtype
    w = wf.w.to(dt).contiguous()
    h = wf.h.to(dt).contiguous()
    plan = SweepPlan(obs, wf.k, want_r=want_r, want_rh=want_rh, want_rtw=want_rtw,
                     out_scale=out_scale, compute_f64=compute_f64)
    plan.run(w, h)
    return plan.R, plan.RH, plan.RtW, plan.sums.cpu().numpy()


@annotate("mfg.mf_objective")
def mf_objective(obs: ObservationSet, wf: FactorPair, lam: float) -> float:
    """f(W H^T) + (lam/2)(||W||^2 + ||H||^2) (mfg/mfsolver.py:48-50)."""
    if wf.w.shape[0] != obs.m or wf.h.shape[0] != obs.n:
        raise ValueError("factor dimensions do not match the data")
    if wf.k == 0:
        from .data import _dot
        return _dot(obs.dev.vals64, obs.dev.vals64)
    _, _, _, s = sweep(obs, wf)
    return float(s[0]) + 0.5 * lam * (float(s[1]) + float(s[2]))


@annotate("mfg._half_sweep")
def _half_sweep(obs: ObservationSet, transpose: bool, other: torch.Tensor, lam: float) -> torch.Tensor:
    dev = obs.dev
    lay = dev.csc if transpose else dev.csr
    vals = dev.vals_csc if transpose else dev.vals
    dt = obs.dtype
    other = other.to(dt).contiguous()
    k = int(other.shape[1])
    out = torch.empty((lay.nrows, k), dtype=dt, device=dev.device)
    lib = _lib.lib()
    wsb = lib.mfg_bcd_workspace(lay.ref, k)
    ws = dev.workspace(wsb)
    _lib.check(lib.mfg_bcd_half_sweep(_lib.dtype_code(dt), lay.ref, k, vals.data_ptr(),
                                      other.data_ptr(), k, float(lam), out.data_ptr(), k,
                                      ws.data_ptr(), wsb, _lib.stream_ptr()), "bcd half sweep")
    if k and lay.nrows:
        flag = torch.zeros(1, dtype=torch.int32).pin_memory()
        _lib.check(lib.mfg_bcd_status(ws.data_ptr(), flag.data_ptr(), _lib.stream_ptr()),
                   "bcd status")
        _PENDING_FLAGS.append(flag)
    return out


_PENDING_FLAGS: list = []


def check_bcd_status(sync: bool = True) -> None:
    """Raise NumericalError if a half-sweep enqueued since the last check met
    a non-SPD normal matrix (a pivot <= 0 or NaN: non-finite inputs). With
    ``sync`` the current stream is synchronised first; without it the caller
    must already have synchronised past the half-sweeps."""
    if not _PENDING_FLAGS:
        return
    if sync:
        torch.cuda.current_stream().synchronize()
    bad = any(int(f[0]) != 0 for f in _PENDING_FLAGS)
    _PENDING_FLAGS.clear()
    if bad:
        from .driver import NumericalError

        raise NumericalError("BCD half-sweep: non-SPD normal matrix (non-finite factors or data)")


@annotate("mfg.bcd_epoch")
def bcd_epoch(obs: ObservationSet, wf: FactorPair, lam: float) -> FactorPair:
    """All rows of W given H, then all rows of H given the new W (78-93)."""
    if lam <= 0:
        raise ValueError("lam must be positive")
    if wf.w.shape[0] != obs.m or wf.h.shape[0] != obs.n:
        raise ValueError("factor dimensions do not match the data")
    if wf.k == 0:
        return wf
    w_new = _half_sweep(obs, False, wf.h, lam)
    h_new = _half_sweep(obs, True, w_new, lam)
    check_bcd_status()
    return FactorPair(w_new, h_new)


@annotate("mfg.mf_phase")
def mf_phase(obs: ObservationSet, start: FactorPair, lam: float, epochs: int) -> FactorPair:
    """``epochs`` BCD sweeps with the monotone-descent guard (96-112)."""
    wf = start
    if epochs <= 0:
        return wf
    wf = wf.to(obs.dtype)
    slack = guard_slack(obs.dtype)
    prev = mf_objective(obs, wf, lam)
    for _ in range(epochs):
        wf = bcd_epoch(obs, wf, lam)
        cur = mf_objective(obs, wf, lam)
        if cur > prev + slack * (1.0 + abs(prev)):
            raise MfPhaseError(f"BCD sweep increased the objective: {prev!r} -> {cur!r}")
        prev = cur
    return wf
