"""ctypes binding of ``libadacluster_sm100.so`` (include/adacluster_sm100.h).

The library is the only compute path: if it is missing, or no CUDA device is
present, every entry point raises — there is no CPU fallback.  Status codes
map onto the reference exception classes (errors.py:8-29).
"""

from __future__ import annotations

import contextlib
import ctypes
import functools
import os
from pathlib import Path

import numpy as np
import torch

from .errors import ContractError, DimensionError, ParameterError

LIB_PATH = Path(__file__).resolve().parent / "libadacluster_sm100.so"

AC_OK, AC_ERR_PARAM, AC_ERR_DIM, AC_ERR_CONTRACT, AC_ERR_CUDA = range(5)
DTYPE_F32, DTYPE_BF16 = 0, 1
ORDER_SEQ, ORDER_LANES16, ORDER_GEMV8 = 0, 1, 2
SCORERS = {"quest": 0, "mean": 1, "clamped": 2, "given": 3}
ASSIGN_MERGE, ASSIGN_ALL = 1, 2
ASSIGN_LABELS_ONLY = 4
ST_ACTIVE, ST_NITER, ST_DONE, ST_FLAGS, ST_KPP_STOP, ST_REPAIRS, ST_FIXUPS, ST_WIDE = range(8)
ASSIGN_MODE_AUTO, ASSIGN_MODE_EXACT, ASSIGN_MODE_TC = range(3)
LLOYD_NO_INERTIA = 1
LLOYD_PREPARED = 2
LLOYD_PREPARED = 2
STATUS_WORDS = 8

# struct layouts (must match the header; checked in tests/test_abi.py)
PROBLEM_DTYPE = np.dtype([
    ("x", "u8"), ("xx", "u8"), ("centers", "u8"), ("cc", "u8"), ("labels", "u8"),
    ("best", "u8"), ("counts", "u8"), ("perm", "u8"), ("starts", "u8"), ("tile_hist", "u8"),
    ("inertia", "u8"), ("movement", "u8"), ("status", "u8"), ("plan_n", "u8"),
    ("plan_k", "u8"), ("dscratch", "u8"), ("planes", "u8"),
    ("csum", "u8"), ("cabs", "u8"), ("clsb", "u8"), ("n", "i8"), ("k", "i4"),
    ("order", "i4"),
])
SELECT_DTYPE = np.dtype([
    ("reps", "u8"), ("emax", "u8"), ("emin", "u8"), ("counts", "u8"), ("kstarts", "u8"),
    ("scores", "u8"), ("selected", "u8"), ("runs", "u8"), ("nruns", "u8"), ("covered", "u8"),
    ("density", "u8"), ("gq", "i4"), ("c", "i4"), ("topk", "i4"), ("order", "i4"),
    ("run_stride", "i4"), ("pad_", "i4"),
])
ITEM_DTYPE = np.dtype([("q_row0", "i8"), ("q_rows", "i4"), ("head", "i4"), ("run0", "i4"),
                       ("nruns", "i4")])

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double
_F = ctypes.c_float

# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGS = {
    "ac_last_error": [],
    "ac_abi_version": [],
    "ac_struct_sizes": [_P],
    "ac_device_info": [_P, _P, _P],
    "ac_pw_plan_len": [_I64],
    "ac_pw_plan_build": [_I64, _P, _I64],
    "ac_gemm_order": [_I64, _I64, _I64],
    "ac_workspace_bytes": [_I, _P, _I, _P, _I],
    "ac_matmul": [_P, _I64, _I, _P, _I64, _P, _I, _P],
    "ac_row_softmax": [_P, _I64, _I64, _F, _P, _P],
    "ac_quest_pairs": [_P, _I, _I, _P, _P, _I, _P, _P],
    "ac_l2norm": [_P, _I, _I64, _I, _P, _P, _P, _P],
    "ac_l2norm_ex": [_P, _I, _I64, _I, _P, _P, _P, _P, _I64, _P],
    "ac_row_sqnorm": [_P, _I, _I64, _I, _P, _P],
    "ac_kmeanspp": [_P, _I, _I, _I, _I64, _I, _P, _P],
    "ac_lloyd": [_P, _I, _I, _I, _I64, _I, _I, _D, _I, _P, _P],
    "ac_lloyd_ex": [_P, _I, _I, _I, _I64, _I, _I, _D, _I, _P, _P],
    "ac_lloyd_prepare": [_P, _I, _I, _I, _I64, _I, _P],
    "ac_assign": [_P, _I, _I, _I, _I64, _I, _I, _I, _P],
    "ac_assign_ordered": [_P, _I, _I, _I, _I64, _I, _I, _I, _I, _P, _P],
    "ac_set_assign_mode": [_I],
    "ac_get_assign_mode": [],
    "ac_set_update_mode": [_I],
    "ac_get_update_mode": [],
    "ac_set_pdl": [_I],
    "ac_get_pdl": [],
    "ac_repair_sort": [_P, _I, _I, _I, _I64, _I, _I, _I, _P],
    "ac_segment_mean": [_P, _I, _I, _I, _I, _P, _P],
    "ac_sort_by_label": [_P, _I, _I64, _I, _P],
    "ac_reduce_best": [_P, _I, _I64, _P, _P, _P],
    "ac_tau": [_P, _I, _I, _I, _I64, _D, _P, _P],
    "ac_mse_f64": [_P, _I, _I, _I, _I64, _P, _P],
    "ac_retire": [_P, _I, _I, _I, _I64, _P, _P, _P, _P, _P],
    "ac_gather_rows": [_P, _I, _I, _P, _I64, _P, _P],
    "ac_drop_empty": [_P, _I, _I, _I64, _I, _P, _P],
    "ac_envelopes": [_P, _I, _I, _I, _I, _P, _P, _P],
    "ac_select": [_P, _I, _I, _I, _I, _I, _I, _P],
    "ac_select_topp": [_P, _I, _I, _I, _I, _I, _I, _F, _F, _P],
    "ac_permute_rows": [_P, _I, _I, _P, _I64, _P, _P],
    "ac_permute_rows_heads": [_P, _I, _I, _P, _I64, _I, _P, _P],
    "ac_build_q_layout": [_P, _I, _I, _I64, _I, _P, _P, _P, _P, _P, _I, _P, _I, _P, _P, _I64,
                          _P, _I, _I, _P],
    "ac_attention_item_rows": [_I, _I],
    "ac_order_items": [_P, _I, _P, _P, _P],
    "ac_sparse_attention": [_P, _I64, _P, _P, _P, _I, _I, _I64, _I, _P, _I, _P, _F, _P, _I, _P],
    "ac_sparse_attention_fa4": [_P, _I64, _P, _P, _P, _I, _I64, _I, _P, _I, _P, _F, _P, _I, _P],
    "ac_sparse_attention_fa4_d128": [_P, _I64, _P, _P, _P, _I, _I64, _I, _P, _I, _P, _F, _P, _I, _P],
    "ac_sparse_attention_simt": [_P, _P, _P, _P, _I, _I, _I64, _P, _I, _P, _F, _P, _I, _P],
}
_RESTYPES = {"ac_last_error": ctypes.c_char_p, "ac_pw_plan_len": _I64, "ac_workspace_bytes": _I64}

EXPORTED = tuple(_SIGS)


@functools.lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH.name} is not built; run `python -m paper_2604_18348_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, _I)
    return L


def check(rc: int, what: str = "") -> None:
    if rc == AC_OK:
        return
    msg = lib().ac_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == AC_ERR_PARAM:
        raise ParameterError(text)
    if rc == AC_ERR_DIM:
        raise DimensionError(text)
    if rc == AC_ERR_CONTRACT:
        raise ContractError(text)
    raise RuntimeError(text)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


@contextlib.contextmanager
def pdl(on: bool = True):
    """Programmatic dependent launch of the Lloyd-chain kernels enqueued (or
    captured) inside the block, on this thread (ac_set_pdl)."""
    prev = int(lib().ac_get_pdl())
    call("ac_set_pdl", int(bool(on)))
    try:
        yield
    finally:
        call("ac_set_pdl", prev)


# where the engine turns it on (A/B knobs): steady steps of at most this
# many rows per layer (default: all), the multi-stage planner's rounds
PDL_STEADY_ROWS = int(os.environ.get("AC_PDL_STEADY_ROWS", str(1 << 62)))
PDL_PLANNER = os.environ.get("AC_PDL_PLANNER", "1") != "0"


@functools.lru_cache(maxsize=None)
def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2604_18348_b200 needs a CUDA device (sm_100a); no CPU fallback")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int:
    return 0 if t is None else t.data_ptr()


@functools.lru_cache(maxsize=None)
def gemm_order(m: int, n: int, d: int) -> int:
    return int(lib().ac_gemm_order(m, n, d))


_PLANS: dict[tuple[int, int], torch.Tensor] = {}


def pw_plan(n: int) -> torch.Tensor:
    """Device copy of the numpy pairwise-sum tree for a length-n reduction."""
    dev = device()
    key = (n, dev.index)
    t = _PLANS.get(key)
    if t is None:
        L = lib()
        ln = int(L.ac_pw_plan_len(n))
        host = np.empty(ln, np.int32)
        check(L.ac_pw_plan_build(n, host.ctypes.data, ln), "ac_pw_plan_build")
        t = torch.from_numpy(host).to(dev)
        _PLANS[key] = t
    return t


WS_CLUSTER, WS_SELECT, WS_ATTENTION = 0, 1, 2
WS_FIELDS = {
    WS_CLUSTER: ("xx", "centers", "cc", "labels", "best", "counts", "perm", "starts",
                 "tile_hist", "inertia", "movement", "status", "plan_n", "plan_k", "dscratch",
                 "planes", "csum", "cabs", "clsb"),
    WS_SELECT: ("scores", "selected", "runs", "nruns", "covered", "density"),
    WS_ATTENTION: ("qp", "qidx", "items", "kp", "vp"),
}


def workspace_bytes(op: int, *dims: int) -> dict:
    """Per-buffer byte sizes of one problem / launch (ac_workspace_bytes)."""
    return dict(_workspace_bytes(op, tuple(int(x) for x in dims)))


@functools.lru_cache(maxsize=4096)
def _workspace_bytes(op: int, dims: tuple) -> tuple:
    names = WS_FIELDS.get(op, ())
    d = np.asarray(dims, np.int64)
    f = np.zeros(max(len(names), 1), np.int64)
    tot = int(lib().ac_workspace_bytes(op, d.ctypes.data, len(d), f.ctypes.data, len(names)))
    if tot < 0:
        check(AC_ERR_PARAM, "ac_workspace_bytes")
    return tuple(zip(names, (int(x) for x in f)))


def to_device_struct(arr: np.ndarray) -> torch.Tensor:
    """Upload a structured numpy array (descriptor table) to the device."""
    raw = np.ascontiguousarray(arr).view(np.uint8)
    host = torch.from_numpy(raw.copy()).pin_memory()
    return host.to(device(), non_blocking=True)


def upload(t: torch.Tensor) -> torch.Tensor:
    """Small host tensor -> device without a stream sync: a pageable copy
    waits for the stream's queued work; a pinned one is enqueued."""
    return t.pin_memory().to(device(), non_blocking=True)


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return DTYPE_F32
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    raise ParameterError(f"unsupported token dtype {t.dtype} (float32 or bfloat16)")
