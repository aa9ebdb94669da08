"""C-ABI checks that need no GPU: the library loads, exports every entry
point declared in include/adacluster_sm100.h, descriptor structs have the
layout the Python binding assumes, and the host-side helpers (numpy
pairwise-sum plan, OpenBLAS order rule) agree with numpy / the oracle."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2604_18348_b200 import _lib as L

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "adacluster_sm100.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ac_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(str(L.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 30


def test_binding_covers_header():
    assert set(declared_symbols()) <= set(L.EXPORTED)


def test_abi_version_and_struct_sizes():
    lib = L.lib()
    assert lib.ac_abi_version() == 1
    sizes = np.zeros(3, np.int64)
    lib.ac_struct_sizes(sizes.ctypes.data)
    assert list(sizes) == [L.PROBLEM_DTYPE.itemsize, L.SELECT_DTYPE.itemsize,
                           L.ITEM_DTYPE.itemsize]


def eval_plan(plan: np.ndarray, a: np.ndarray) -> np.float32:
    """Host interpretation of the device pairwise plan (pairwise.cuh)."""
    nl, ni, nh = int(plan[0]), int(plan[1]), int(plan[2])
    lo = plan[3:3 + nl + 1]
    lev = plan[4 + nl:4 + nl + nh + 1]
    nodes = plan[5 + nl + nh:].reshape(-1, 3)
    vals = np.zeros(nl + ni, np.float32)
    for i in range(nl):
        seg = a[lo[i]:lo[i + 1]]
        n = seg.size
        if n < 8:
            r = np.float32(0)
            for v in seg:
                r = np.float32(r + v)
        else:
            acc = seg[:8].copy()
            j = 8
            while j < n - n % 8:
                acc = (acc + seg[j:j + 8]).astype(np.float32)
                j += 8
            r = np.float32(np.float32(np.float32(acc[0] + acc[1]) + np.float32(acc[2] + acc[3]))
                           + np.float32(np.float32(acc[4] + acc[5]) + np.float32(acc[6] + acc[7])))
            for v in seg[j:]:
                r = np.float32(r + v)
        vals[i] = r
    for h in range(nh):
        for dst, x, y in nodes[lev[h]:lev[h + 1]]:
            vals[dst] = np.float32(vals[x] + vals[y])
    return vals[nl + ni - 1] if ni else vals[0]


@pytest.mark.parametrize("n", [1, 5, 8, 100, 128, 129, 1000, 4097, 70000])
def test_pairwise_plan_matches_numpy(n):
    lib = L.lib()
    ln = int(lib.ac_pw_plan_len(n))
    plan = np.empty(ln, np.int32)
    assert lib.ac_pw_plan_build(n, plan.ctypes.data, ln) == 0
    a = (np.random.default_rng(n).random(n) * 10).astype(np.float32)
    assert eval_plan(plan, a) == a.sum()


def test_gemm_order_rule_matches_oracle(oracle):
    lib = L.lib()
    for m in (1, 2, 8, 30, 34, 35, 40, 65, 145, 1000, 70000):
        for n in (1, 3, 8, 17, 30, 32, 100, 1000):
            for d in (4, 16, 31, 32, 64, 128):
                assert lib.ac_gemm_order(m, n, d) == oracle.gemm_order(m, n, d)


def test_gemm_order_rule_matches_numpy_blas(oracle):
    """The dispatch rule reproduces numpy/OpenBLAS `x @ c.T` bit-for-bit
    (only meaningful on the oracle host's BLAS)."""
    rng = np.random.default_rng(0)
    for (m, n, d) in [(1500, 100, 64), (30, 30, 64), (145, 8, 64), (40, 32, 64), (20, 4, 6)]:
        x = (rng.normal(size=(m, d)) * 40).astype(np.float32)
        c = (rng.normal(size=(n, d)) * 40).astype(np.float32)
        ours = oracle.matmul_nt(x, c)
        if not np.array_equal(ours, x @ c.T):
            pytest.skip("this host's BLAS uses a different kernel than the oracle host")


def test_error_codes_map_to_reference_exceptions():
    from paper_2604_18348_b200.errors import ContractError, DimensionError, ParameterError
    with pytest.raises(ParameterError):
        L.check(L.AC_ERR_PARAM)
    with pytest.raises(DimensionError):
        L.check(L.AC_ERR_DIM)
    with pytest.raises(ContractError):
        L.check(L.AC_ERR_CONTRACT)
    with pytest.raises(RuntimeError):
        L.check(L.AC_ERR_CUDA)


@pytest.mark.parametrize("n,k,d,dtype", [(70000, 100, 64, L.DTYPE_BF16), (4096, 65, 64, L.DTYPE_F32),
                                         (300, 7, 17, L.DTYPE_F32), (1, 1, 128, L.DTYPE_BF16)])
def test_workspace_bytes_cluster(n, k, d, dtype):
    """ac_workspace_bytes(AC_WS_CLUSTER) sizes every buffer of one
    ac_cluster_problem; the Python Batch allocates exactly the sum."""
    from paper_2604_18348_b200.engine import batch_buffer_bytes
    f = L.workspace_bytes(L.WS_CLUSTER, n, k, d, dtype, 25)
    fast = d in (64, 128)
    assert f["xx"] == f["labels"] == f["best"] == f["perm"] == 4 * n
    assert f["centers"] == 4 * k * d and f["starts"] == 4 * (k + 1)
    assert f["tile_hist"] == 4 * ((n + 127) // 128) * k
    assert f["dscratch"] == 8 * n and f["status"] == 32 and f["inertia"] == 100
    assert f["plan_n"] == 4 * int(L.lib().ac_pw_plan_len(n))
    assert f["planes"] == (6 * n * d if (fast and dtype == L.DTYPE_F32) else 0)
    assert f["csum"] == (8 * k * d if fast else 0)
    tot = batch_buffer_bytes([n, n], [k, k], d, dtype, 25)
    assert all(tot[x] == 2 * f[x] for x in f)


def test_workspace_bytes_select_attention_and_errors():
    s = L.workspace_bytes(L.WS_SELECT, 65, 100, 25, 25)
    assert s == {"scores": 4 * 65 * 100, "selected": 8 * 65 * 25, "runs": 4 * 65 * 25 * 2,
                 "nruns": 4 * 65, "covered": 8 * 65, "density": 8}
    a = L.workspace_bytes(L.WS_ATTENTION, 70000, 30, 65, 25, 64, L.DTYPE_BF16)
    qp_cap = 70000 + 128 * 65
    assert a["qp"] == 30 * qp_cap * 64 * 2
    assert a["items"] == 30 * ((70000 + 127) // 128 + 65) * L.ITEM_DTYPE.itemsize
    assert a["kp"] == a["vp"] == 30 * 70000 * 64 * 2
    from paper_2604_18348_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        L.workspace_bytes(7, 1, 2, 3)
    with pytest.raises(ParameterError):
        L.workspace_bytes(L.WS_CLUSTER, 10, 2)
