"""Real-model tensor ingestion: strict npy v1.0 f32 files
and ``step<t>/layer<l>/head<h>/{q,k,v}.npy`` dump trees, staged for the GPU.

Same accepted format and error behaviour as the reference's ``npyio.py:22-77``
(``write_npy`` / ``read_npy``: little-endian f32, C order, version (1, 0)
only, header padded to 64 bytes; anything else -> ``FormatError`` naming the
file and the field) and ``harness/dump.py:19-82`` (``write_dump`` /
``ingest_dump``: contiguous ``step``/``layer``/``head`` indices, rank-2
tensors, consistent q/k/v shapes, no shape drift across steps ->
``FormatError`` / ``ContractError``).

The B200 side: ``load_layer`` reads one layer's heads straight into a pinned
``[H, L, D]`` staging buffer (payload bytes land in place with
``readinto``, no intermediate arrays) and moves them to the device in the
compute dtype with one copy per tensor -- the same pinned-host -> HBM path the
steady step uses, so a captured dump can drive ``LayerSession.step``.
"""

from __future__ import annotations

import ast
import re
import struct
from pathlib import Path

import numpy as np

from .errors import ContractError, FormatError

__all__ = ["write_npy", "read_npy", "npy_header", "write_dump", "ingest_dump", "load_layer"]

_MAGIC = b"\x93NUMPY"
_PREFIX = len(_MAGIC) + 4  # magic + version (2 bytes) + header length (u16)


def write_npy(path, arr) -> None:
    """``arr`` as little-endian f32, C order, npy v1.0 (header padded so the
    payload starts on a 64-byte boundary)."""
    a = np.ascontiguousarray(arr, dtype="<f4")
    shape = "(%d,)" % a.shape[0] if a.ndim == 1 else repr(tuple(a.shape))
    text = "{'descr': '<f4', 'fortran_order': False, 'shape': %s, }" % shape
    text += " " * ((-(_PREFIX + len(text) + 1)) % 64) + "\n"
    with open(path, "wb") as f:
        f.write(_MAGIC + bytes((1, 0)) + struct.pack("<H", len(text)) + text.encode("latin1"))
        f.write(a.tobytes(order="C"))


def npy_header(path, size: int | None = None) -> tuple[tuple, int]:
    """Validate a strict f32 npy v1.0 header: returns (shape, payload offset).
    ``size`` (file bytes) enables the payload-length check."""
    path = Path(path)
    with open(path, "rb") as f:
        pre = f.read(_PREFIX)
        if len(pre) < _PREFIX or pre[:6] != _MAGIC:
            raise FormatError(f"{path}: bad magic, not an npy file")
        if (pre[6], pre[7]) != (1, 0):
            raise FormatError(f"{path}: unsupported npy version {(pre[6], pre[7])}, need (1, 0)")
        (hlen,) = struct.unpack("<H", pre[8:10])
        raw = f.read(hlen)
    if len(raw) < hlen:
        raise FormatError(f"{path}: truncated header")
    try:
        hdr = ast.literal_eval(raw.decode("latin1"))
    except (ValueError, SyntaxError) as exc:
        raise FormatError(f"{path}: unparseable header: {exc}") from exc
    if not isinstance(hdr, dict):
        raise FormatError(f"{path}: header is not a dict")
    for key in ("descr", "fortran_order", "shape"):
        if key not in hdr:
            raise FormatError(f"{path}: header missing field '{key}'")
    if hdr["descr"] != "<f4":
        raise FormatError(f"{path}: descr is {hdr['descr']!r}, only '<f4' accepted")
    if hdr["fortran_order"] is not False:
        raise FormatError(f"{path}: fortran_order is {hdr['fortran_order']!r}, must be False")
    shape = hdr["shape"]
    if not isinstance(shape, tuple) or not all(isinstance(d, int) and d >= 0 for d in shape):
        raise FormatError(f"{path}: malformed shape {shape!r}")
    off = _PREFIX + hlen
    if size is not None:
        need = 4 * (int(np.prod(shape, dtype=np.int64)) if shape else 1)
        if size - off != need:
            raise FormatError(f"{path}: payload is {size - off} bytes, shape {shape} needs {need}")
    return shape, off


def read_npy(path) -> np.ndarray:
    """A strict f32 npy v1.0 file as a C-contiguous float32 array."""
    path = Path(path)
    shape, off = npy_header(path, path.stat().st_size)
    out = np.empty(shape, dtype=np.float32)
    if out.size == 0:  # e.g. shape (0, 64): nothing to read
        return out
    with open(path, "rb") as f:
        f.seek(off)
        f.readinto(out.reshape(-1).view(np.uint8))
    return out


def write_dump(directory, step_inputs) -> None:
    """``step_inputs[step][layer][head] = (q, k, v)`` as a dump tree."""
    root = Path(directory)
    for t, layers in enumerate(step_inputs):
        for l, heads in enumerate(layers):
            for h, qkv in enumerate(heads):
                d = root / f"step{t}" / f"layer{l}" / f"head{h}"
                d.mkdir(parents=True, exist_ok=True)
                for name, a in zip("qkv", qkv):
                    write_npy(d / f"{name}.npy", a)


def _children(parent: Path, prefix: str) -> list[Path]:
    """``<prefix><n>`` subdirectories, which must be numbered 0..N-1."""
    pat = re.compile(rf"^{prefix}(\d+)$")
    found = {}
    for c in parent.iterdir():
        m = pat.match(c.name)
        if m and c.is_dir():
            found[int(m.group(1))] = c
    if not found:
        raise FormatError(f"{parent}: no {prefix}<n> subdirectories")
    idx = sorted(found)
    if idx != list(range(len(idx))):
        raise FormatError(f"{parent}: non-contiguous {prefix} indices {idx}")
    return [found[i] for i in idx]


def _head_shapes(hd: Path):
    shapes = []
    for name in "qkv":
        p = hd / f"{name}.npy"
        if not p.is_file():
            raise FormatError(f"{p}: missing tensor file")
        shape, _ = npy_header(p, p.stat().st_size)
        if len(shape) != 2:
            raise FormatError(f"{p}: expected rank 2, got shape {shape}")
        shapes.append(shape)
    q, k, v = shapes
    if q[1] != k[1] or k != v:
        raise ContractError(f"{hd}: inconsistent q/k/v shapes {q}, {k}, {v}")
    return q, k, v


def _tree(directory) -> list[list[list[Path]]]:
    """Head directories ``[step][layer][head]``, shapes validated (headers
    only) and checked for drift against step 0."""
    root = Path(directory)
    if not root.is_dir():
        raise FormatError(f"{root}: not a directory")
    tree, ref = [], None
    for sd in _children(root, "step"):
        layers = [[hd for hd in _children(ld, "head")] for ld in _children(sd, "layer")]
        shapes = [[_head_shapes(hd) for hd in heads] for heads in layers]
        if ref is None:
            ref = shapes
        elif shapes != ref:
            raise ContractError(f"{sd}: shapes drift relative to step0")
        tree.append(layers)
    return tree


def ingest_dump(directory):
    """The dump tree back as ``out[step][layer][head] = (q, k, v)`` f32 arrays."""
    return [[[tuple(read_npy(hd / f"{n}.npy") for n in "qkv") for hd in heads] for heads in layers]
            for layers in _tree(directory)]


def load_layer(directory, step: int, layer: int, dtype=None, device="cuda"):
    """One layer of a dump as device tensors ``(Q, K, V)``, each ``[H, L, D]``
    in ``dtype`` (default bfloat16), via one pinned staging buffer per tensor.
    Heads of a layer must share one shape (the steady step's contract)."""
    import torch
    dtype = torch.bfloat16 if dtype is None else dtype
    tree = _tree(directory)
    if not (0 <= step < len(tree)) or not (0 <= layer < len(tree[step])):
        raise FormatError(f"{directory}: no step{step}/layer{layer}")
    heads = tree[step][layer]
    shapes = {_head_shapes(hd) for hd in heads}
    if len(shapes) != 1:
        raise ContractError(f"{directory}: step{step}/layer{layer} heads differ in shape")
    out = []
    for i, name in enumerate("qkv"):
        L, D = next(iter(shapes))[i]
        stage = torch.empty((len(heads), L, D), dtype=torch.float32, pin_memory=True)
        buf = stage.numpy()
        for h, hd in enumerate(heads):
            p = hd / f"{name}.npy"
            _, off = npy_header(p)
            if buf[h].size == 0:
                continue
            with open(p, "rb") as f:
                f.seek(off)
                f.readinto(buf[h].reshape(-1).view(np.uint8))
        out.append(stage.to(device, non_blocking=True).to(dtype))
    return tuple(out)
