"""Tensor plumbing shared by the public API (reference: tensorops.py).

Inputs may be numpy arrays (the reference's convention: coerced to C-contiguous
f32) or torch tensors (f32 or bf16, any device).  Host inputs produce host
(numpy) outputs; CUDA tensor inputs stay on the device.  All arithmetic runs
in the sm_100a library.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _lib as L
from . import engine as E
from .errors import DimensionError

__all__ = ["as_f32", "l2_normalize_rows", "NormalizedRows", "to_device", "to_host"]

DEGENERATE_NORM = 1e-12


def as_f32(x) -> np.ndarray:
    """C-contiguous float32 host copy (tensorops.py:24-26)."""
    if isinstance(x, torch.Tensor):
        return x.detach().float().cpu().contiguous().numpy()
    return np.ascontiguousarray(x, dtype=np.float32)


def to_device(x, keep_bf16: bool = True) -> tuple[torch.Tensor, bool]:
    """(contiguous CUDA tensor f32/bf16, caller_was_host)."""
    dev = L.device()
    if isinstance(x, torch.Tensor):
        host = x.device.type != "cuda"
        t = x.detach()
        if not (keep_bf16 and t.dtype == torch.bfloat16):
            t = t.float()
        return t.to(dev).contiguous(), host
    a = np.ascontiguousarray(x, dtype=np.float32)
    return torch.from_numpy(a).to(dev), True


def to_host(t: torch.Tensor | None, host: bool):
    if t is None or not host:
        return t
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.cpu().numpy()


class NormalizedRows(NamedTuple):
    rows: object
    degenerate: object  # indices of rows with norm < DEGENERATE_NORM


def l2_normalize_rows(x) -> NormalizedRows:
    """tensorops.py:59-76 on the device (bit-identical f32 result)."""
    t, host = to_device(x)
    if t.ndim != 2:
        raise DimensionError(f"l2_normalize_rows expects [N, D], got {tuple(t.shape)}")
    rows, deg = E.l2norm(t)
    idx = torch.nonzero(deg, as_tuple=False).flatten()
    if host:
        return NormalizedRows(rows.cpu().numpy(), idx.cpu().numpy().astype(np.int64))
    return NormalizedRows(rows, idx)
