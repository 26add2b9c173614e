"""ctypes binding of libmfg_b200.so (the C ABI in include/mfg_b200.h).

The product path has no CPU fallback: importing a kernel entry point when the
shared library is missing, or calling one without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MFG_LIB_PATH") or os.path.join(HERE, "libmfg_b200.so")

MFG_OK, MFG_ERR_ARG, MFG_ERR_DATASET, MFG_ERR_CAPACITY, MFG_ERR_CUDA, MFG_ERR_NUMERICAL = range(6)
MFG_F32, MFG_F64 = 0, 1


class MfgKernelError(RuntimeError):
    """A CUDA-side failure reported by libmfg_b200."""


class Layout(ctypes.Structure):
    """mirror of ``mfg_layout`` (include/mfg_b200.h)."""

    _fields_ = [
        ("nrows", ctypes.c_int32),
        ("ncols", ctypes.c_int32),
        ("nnz", ctypes.c_int64),
        ("ptr", ctypes.c_void_p),
        ("idx", ctypes.c_void_p),
        ("row_of", ctypes.c_void_p),
        ("bmask", ctypes.c_void_p),
        ("brank", ctypes.c_void_p),
        ("nzrows", ctypes.c_void_p),
        ("n_nonempty", ctypes.c_int32),
        ("empty_rows", ctypes.c_void_p),
        ("n_empty", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_LP = ctypes.POINTER(Layout)


class PanelPass(ctypes.Structure):
    """mirror of ``mfg_panel_pass`` (include/mfg_b200.h)."""

    _fields_ = [
        ("n_pieces", ctypes.c_int32),
        ("n_frows", ctypes.c_int32),
        ("n_light", ctypes.c_int32),
        ("panel_ids", ctypes.c_void_p),
        ("pieces", ctypes.c_void_p),
        ("recs", ctypes.c_void_p),
        ("frows", ctypes.c_void_p),
        ("fbeg", ctypes.c_void_p),
        ("fcnt", ctypes.c_void_p),
        ("r_hot", ctypes.c_void_p),
        ("piece_out", ctypes.c_void_p),
        ("piece_sq", ctypes.c_void_p),
    ]


_PP = ctypes.POINTER(PanelPass)

_SIGS = {
    "mfg_last_error": (ctypes.c_char_p, []),
    "mfg_version": (_INT, []),
    "mfg_launch_count": (_I64, []),
    "mfg_count_lines": (_I64, [_P, _SZ]),
    "mfg_parse_ratings": (_INT, [_P, _SZ, _INT, _P, _P, _P, _SZ, _P, _P]),
    "mfg_omega_build_workspace": (_SZ, [_I64, _I32, _I32]),
    "mfg_omega_build": (_INT, [_I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                               ctypes.POINTER(_I64), ctypes.POINTER(_I32), _P, _SZ, _P]),
    "mfg_layout_workspace": (_SZ, [_I64, _I32]),
    "mfg_layout_build": (_INT, [_I32, _I64, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_I32),
                                ctypes.POINTER(_I32), _P, _SZ, _P]),
    "mfg_gather": (_INT, [_INT, _I64, _P, _P, _P, _P]),
    "mfg_convert": (_INT, [_INT, _INT, _I64, _P, _P, _P]),
    "mfg_sweep_workspace": (_SZ, [_LP, _LP, _INT]),
    "mfg_sweep_ld": (_INT, [_INT, _INT, _INT]),
    "mfg_sweep": (_INT, [_INT, _INT, _LP, _LP, _INT, _P, _P, _P, _INT, _P, _INT, _P, _P, _P, _D,
                         _P, _P, _SZ, _P]),
    "mfg_sweep_sharded": (_INT, [_INT, _INT, _LP, _LP, _INT, _P, _P, _P, _P, _INT, _P, _P, _INT, _P,
                                 _P, _P, _D, _P, _P, _SZ, _P]),
    "mfg_sweep_host": (_INT, [_INT, _INT, _LP, _LP, _INT, _P, _P, _P, _P, _P, _INT, _P, _INT, _P,
                              _P, _P, _D, _P, _SZ, _P]),
    "mfg_panel_rows": (_INT, [_INT]),
    "mfg_panel_ctas": (_INT, []),
    "mfg_panel_sweep": (_INT, [_INT, _INT, _P, _P, _PP, _PP, _P, _P, _P, _P]),
    "mfg_cold_sweep": (_INT, [_INT, _PP, _PP, _P, _P, _P, _P, _D, _P, _P]),
    "mfg_panel_fold": (_INT, [_INT, _INT, _PP, _P, _INT, _D, _INT, _P, _P, _P]),
    "mfg_sddmm_workspace": (_SZ, [_LP, _INT]),
    "mfg_sddmm": (_INT, [_INT, _INT, _LP, _INT, _P, _INT, _P, _P, _INT, _P, _P, _D, _P, _P, _P,
                         _SZ, _P]),
    "mfg_spmm_workspace": (_SZ, [_LP, _INT]),
    "mfg_spmm": (_INT, [_INT, _LP, _INT, _P, _P, _INT, _D, _D, _P, _INT, _P, _SZ, _P]),
    "mfg_bcd_workspace": (_SZ, [_LP, _INT]),
    "mfg_bcd_half_sweep": (_INT, [_INT, _LP, _INT, _P, _P, _INT, _D, _P, _INT, _P, _SZ, _P]),
    "mfg_bcd_status": (_INT, [_P, _P, _P]),
    "mfg_gemm_tn_workspace": (_SZ, [_INT, _INT, _INT]),
    "mfg_gemm_tn": (_INT, [_INT, _INT, _INT, _P, _INT, _P, _INT, _D, _P, _INT, _P, _SZ, _P]),
    "mfg_qr_workspace": (_SZ, [_INT, _INT]),
    "mfg_qr": (_INT, [_INT, _INT, _P, _INT, _P, _INT, _P, _P, _SZ, _P]),
    "mfg_gemm_nn": (_INT, [_INT, _INT, _INT, _P, _INT, _P, _INT, _D, _D, _P, _INT, _P]),
    "mfg_dot": (_INT, [_INT, _I64, _P, _P, _P, _P, _SZ, _P]),
    "mfg_profile_enable": (_INT, [_INT]),
    "mfg_profile_collect": (_INT, [ctypes.POINTER(_D), ctypes.POINTER(_INT)]),
    "mfg_set_probe": (_INT, [_P]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the shared library; raise if it is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -m paper_2204_14067_b200.build_lib` (no CPU fallback exists)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int, what: str):
    if status == MFG_OK:
        return
    msg = lib().mfg_last_error().decode(errors="replace")
    from .data import DatasetError  # local import: avoid a cycle
    from .operators import CapacityError

    if status == MFG_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    if status == MFG_ERR_DATASET:
        raise DatasetError(msg)
    if status == MFG_ERR_CAPACITY:
        raise CapacityError(f"{what}: {msg}")
    raise MfgKernelError(f"{what}: {msg} (status {status})")


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2204_14067_b200 runs its hot path on a CUDA device (sm_100a); "
            "no GPU is visible and there is no CPU fallback")


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float64:
        return MFG_F64
    if dt == torch.float32:
        return MFG_F32
    raise TypeError(f"unsupported dtype {dt}")


class Workspace:
    """Grow-only device scratch buffer shared by consecutive calls on a stream."""

    def __init__(self):
        self._buf = {}

    def get(self, nbytes: int, device) -> torch.Tensor:
        key = (str(device), torch.cuda.current_stream(device).cuda_stream)
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            size = max(int(nbytes), 1 << 16)
            size = int(size * 1.25)
            buf = torch.empty(size, dtype=torch.uint8, device=device)
            self._buf[key] = buf
        return buf


WS = Workspace()
