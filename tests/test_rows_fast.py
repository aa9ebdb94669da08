"""Row kernels of the D=64/128 fast path (k_l2norm_v, k_problem_xx_v) vs the
validated references: the oracle's l2 normalisation, numpy's pairwise
``(x * x).sum(axis=1)`` and the staged thread-per-row kernel (ac_row_sqnorm);
the fused bf16 planes must re-join to the normalised rows exactly.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rows(n, d, seed, dtype):
    rng = np.random.default_rng(seed)
    m = max(n, 8)
    x = (rng.normal(size=(m, d)) * rng.lognormal(size=(m, 1))).astype(np.float32)
    x[3] = 0
    x[5] = x[5] / np.linalg.norm(x[5])
    x[7] = 1e-30
    t = torch.from_numpy(np.ascontiguousarray(x[:n]))
    if dtype == "bf16":
        t = t.bfloat16()
    return t


def _sqnorm_ref(x: torch.Tensor) -> torch.Tensor:
    from paper_2604_18348_b200 import _lib as L
    out = torch.empty(x.shape[0], dtype=torch.float32, device="cuda")
    L.call("ac_row_sqnorm", x.data_ptr(), L.dtype_code(x), x.shape[0], x.shape[1], out.data_ptr(),
           L.stream_ptr())
    return out


def _join(planes: torch.Tensor) -> torch.Tensor:
    hi, mid, lo = (planes[i].float() for i in range(3))
    return (hi + mid) + lo


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [1, 63, 1000, 4099])
def test_l2norm_fast_matches_oracle(gpu, oracle, d, dtype, n):
    from paper_2604_18348_b200 import _lib as L
    x = _rows(n, d, n + d, dtype)
    xd = x.cuda()
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    sq = torch.empty(n, dtype=torch.float32, device="cuda")
    deg = torch.empty(n, dtype=torch.uint8, device="cuda")
    L.call("ac_l2norm", xd.data_ptr(), L.dtype_code(xd), n, d, out.data_ptr(), sq.data_ptr(),
           deg.data_ptr(), L.stream_ptr())
    torch.cuda.synchronize()
    ro, rdeg = oracle.l2_normalize(x.float().numpy())
    assert np.array_equal(out.cpu().numpy().view(np.int32), ro.view(np.int32))
    assert list(np.flatnonzero(deg.cpu().numpy())) == list(rdeg)
    assert torch.equal(sq.view(torch.int32), _sqnorm_ref(out).view(torch.int32))


@pytest.mark.parametrize("d", [64, 128])
def test_l2norm_ex_planes_and_xx(gpu, d):
    """The fused query prepare: per-problem [3][n][d] planes + xx."""
    from paper_2604_18348_b200 import _lib as L
    H, n = 3, 1111
    x = _rows(H * n, d, 9, "bf16").cuda()
    out = torch.empty((H * n, d), dtype=torch.float32, device="cuda")
    sq = torch.empty(H * n, dtype=torch.float32, device="cuda")
    deg = torch.empty(H * n, dtype=torch.uint8, device="cuda")
    planes = torch.empty((H, 3, n, d), dtype=torch.bfloat16, device="cuda")
    L.call("ac_l2norm_ex", x.data_ptr(), L.DTYPE_BF16, H * n, d, out.data_ptr(), sq.data_ptr(),
           deg.data_ptr(), planes.data_ptr(), n, L.stream_ptr())
    torch.cuda.synchronize()
    for h in range(H):
        assert torch.equal(_join(planes[h]), out[h * n:(h + 1) * n])
    assert torch.equal(sq.view(torch.int32), _sqnorm_ref(out).view(torch.int32))
    ref = (out.cpu().numpy() ** 2).sum(axis=1, dtype=np.float32)
    assert np.array_equal(sq.cpu().numpy(), ref)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_problem_xx_fast(gpu, d, dtype):
    """ac_lloyd_prepare on a ragged multi-problem batch: xx (+ f32 planes)."""
    from paper_2604_18348_b200 import engine as E
    xs = [_rows(n, d, n, dtype).cuda() for n in (100, 700, 64 * 37 + 5)]
    b = E.Batch(xs, [16, 16, 16], 2)
    b.prepare()
    torch.cuda.synchronize()
    off = 0
    for x in xs:
        n = x.shape[0]
        assert torch.equal(b.xx[off:off + n].view(torch.int32), _sqnorm_ref(x).view(torch.int32))
        if b.planes is not None:
            pl = b.planes[3 * off * d:3 * (off + n) * d].view(3, n, d)
            assert torch.equal(_join(pl), x.float())
        off += n
