"""NVTX ranges around the solver's phases (tracing). The ranges
show up in nsys / ncu timelines; they cost ~1 us each and wrap phase-level
calls only. ``MFG_NVTX=0`` turns them off."""

from __future__ import annotations

import functools
import os

import torch

_ON = os.environ.get("MFG_NVTX", "1") not in ("0", "")


def annotate(name: str):
    """Decorator: run the function inside an NVTX range ``name``."""

    def deco(fn):
        if not _ON:
            return fn

        @functools.wraps(fn)
        def wrapped(*args, **kwargs):
            if not torch.cuda.is_available():
                return fn(*args, **kwargs)
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()

        return wrapped

    return deco
