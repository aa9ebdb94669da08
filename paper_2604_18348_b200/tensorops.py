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

__all__ = ["as_f32", "matmul", "row_softmax", "l2_normalize_rows", "NormalizedRows",
           "to_device", "to_host"]

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


def matmul(a, b):
    """f32 matrix product a @ b (tensorops.py:29-37) on the device, in the
    accumulation order the reference's OpenBLAS call uses for the shape."""
    ta, host = to_device(a, keep_bf16=False)
    tb, _ = to_device(b, keep_bf16=False)
    if ta.ndim != 2 or tb.ndim != 2:
        raise DimensionError(f"matmul expects 2-D operands, got {tuple(ta.shape)} and "
                             f"{tuple(tb.shape)}")
    if ta.shape[1] != tb.shape[0]:
        raise DimensionError(f"matmul inner dimensions differ: {tuple(ta.shape)} x "
                             f"{tuple(tb.shape)}")
    m, kd, n = int(ta.shape[0]), int(ta.shape[1]), int(tb.shape[1])
    out = torch.zeros((m, n), dtype=torch.float32, device=ta.device)
    if kd > 0:
        order = L.gemm_order(m, n, kd)
        for r0 in range(0, m, 65535):  # grid.y limit per launch
            r1 = min(m, r0 + 65535)
            L.call("ac_matmul", ta[r0:r1].data_ptr(), r1 - r0, kd, tb.data_ptr(), n,
                   out[r0:r1].data_ptr(), order, L.stream_ptr())
    return to_host(out, host)


def row_softmax(s, scale: float = 1.0):
    """Stable softmax over the last axis of ``scale * s`` (tensorops.py:40-51)."""
    t, host = to_device(s, keep_bf16=False)
    t = t.contiguous()
    out = torch.empty_like(t)
    cols = int(t.shape[-1]) if t.ndim else 1
    rows = t.numel() // cols if cols else 0
    L.call("ac_row_softmax", t.data_ptr(), rows, cols, float(scale), out.data_ptr(),
           L.stream_ptr())
    return to_host(out, host)


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
