"""Tensor-core assignment (k_assign_tc) vs the all-FFMA exact kernel.

The tcgen05 kernel computes x·c with a 3-way bf16 split and re-derives every
near-tie candidate with the reference's exact sequential FMA chain, so its
labels, winning distances and per-tile histograms must equal the exact
kernel's bit for bit (which in turn equals the oracle — test_gpu_parity.py).
Includes adversarial near-ties: duplicated centres and points equidistant
from two centres.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(xs, centers, mode, c_lo=0, merge_from=None):
    from paper_2604_18348_b200 import _lib as L
    from paper_2604_18348_b200 import engine as E
    ks = [int(c.shape[0]) for c in centers]
    b = E.Batch(xs, ks, 1)
    for p, c in enumerate(centers):
        b.centers_of(p).copy_(c)
    b.prepare()
    flags = L.ASSIGN_ALL
    if merge_from is not None:
        b.labels.copy_(merge_from[0])
        b.best.copy_(merge_from[1])
        flags |= L.ASSIGN_MERGE
    L.call("ac_set_assign_mode", mode)
    try:
        b.assign(c_lo, flags)
    finally:
        L.call("ac_set_assign_mode", L.ASSIGN_MODE_AUTO)
    torch.cuda.synchronize()
    return (b.labels.clone(), b.best.clone(), b.tile_hist.clone(),
            b.status.view(b.P, L.STATUS_WORDS)[:, L.ST_FIXUPS].clone())


def _compare(xs, centers, c_lo=0, merge_from=None):
    from paper_2604_18348_b200 import _lib as L
    a = _run(xs, centers, L.ASSIGN_MODE_TC, c_lo, merge_from)
    e = _run(xs, centers, L.ASSIGN_MODE_EXACT, c_lo, merge_from)
    assert torch.equal(a[0], e[0]), f"labels differ in {(a[0] != e[0]).sum().item()} rows"
    assert torch.equal(a[1].view(torch.int32), e[1].view(torch.int32)), "best distances differ"
    if merge_from is None:
        assert torch.equal(a[2], e[2]), "tile histograms differ"
    return a[3].cpu().numpy()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,k", [(200, 16), (127, 16), (128, 65), (129, 100), (5000, 128),
                                 (70000, 65), (70000, 100)])
def test_tc_assign_random(gpu, dtype, n, k, d):
    g = torch.Generator().manual_seed(n * 131 + k + d)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    x = (torch.randn(n, d, generator=g) * 20).to(tdt).cuda()
    idx = torch.randint(0, n, (k,), generator=g)
    c = (x.float().cpu()[idx] + torch.randn(k, d, generator=g) * 0.5).cuda()
    _compare([x], [c])


@pytest.mark.parametrize("d", [64, 128])
def test_tc_assign_normalised_queries_batch(gpu, d):
    """Unit-norm f32 rows (the query side), several heads per launch."""
    g = torch.Generator().manual_seed(7)
    xs, cs = [], []
    for h in range(5):
        n = 3000 + 977 * h
        x = torch.randn(n, d, generator=g)
        x = (x / x.norm(dim=1, keepdim=True)).cuda()
        c = x[torch.randint(0, n, (65,), generator=g).cuda()] * 0.9
        xs.append(x.contiguous())
        cs.append(c.contiguous())
    fix = _compare(xs, cs)
    assert (fix >= 0).all()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_tc_assign_exact_ties(gpu, dtype, d):
    """Duplicated centres and rows exactly between two centres: the first
    index must win, exactly as numpy's argmin."""
    g = torch.Generator().manual_seed(3)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    base = torch.randn(40, d, generator=g) * 10
    c = torch.cat([base, base[:10], base[5:15]])           # 60 centres, 20 duplicated
    mid = 0.5 * (base[:20] + base[20:40])                   # equidistant from pairs
    pts = torch.cat([mid.repeat(30, 1), base.repeat(20, 1),
                     torch.randn(2000, d, generator=g) * 10])
    x = pts.to(tdt).cuda().contiguous()
    fix = _compare([x], [c.cuda()])
    assert fix[0] > 0  # the duplicates must have gone through the exact fix-up


def test_tc_assign_degenerate_rows(gpu):
    """All-zero rows are equidistant from every centre (many candidates)."""
    g = torch.Generator().manual_seed(5)
    x = torch.randn(1000, 64, generator=g)
    x[::7] = 0
    c = torch.randn(100, 64, generator=g)
    _compare([x.cuda()], [c.cuda()])


@pytest.mark.parametrize("dtype,d", [("bf16", 64), ("bf16", 128), ("f32", 64), ("f32", 128)])
def test_tc_assign_merge(gpu, dtype, d):
    """Running multi-stage assignment: merge new centres [c_lo, k) into the
    existing (label, best) with strict '<' (earlier centres win ties)."""
    from paper_2604_18348_b200 import _lib as L
    g = torch.Generator().manual_seed(11 + d)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    x = (torch.randn(9000, d, generator=g) * 30).to(tdt).cuda()
    c_old = torch.randn(100, d, generator=g) * 30
    c_new = torch.cat([c_old[:7], torch.randn(93, d, generator=g) * 30])  # 7 exact duplicates
    both = torch.cat([c_old, c_new]).cuda()
    lab, best, _, _ = _run([x], [both[:100].contiguous()], L.ASSIGN_MODE_EXACT)
    _compare([x], [both.contiguous()], c_lo=100, merge_from=(lab, best))


@pytest.mark.parametrize("d", [64, 128])
def test_tc_assign_lloyd_parity(gpu, oracle, d):
    """A full Lloyd run through the tensor-core path equals the oracle."""
    rng = np.random.default_rng(1)
    x = (rng.normal(size=(20000, d)) * 5).astype(np.float32)
    a = gpu.kmeans(x, 100, seed=4)
    b = oracle.kmeans(x, 100, 4)
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centers, b.centers)
    assert a.n_iter == b.n_iter
    assert list(a.inertia_history) == list(b.inertia_history)


@pytest.mark.parametrize("dtype,d,k", [("f32", 64, 65), ("bf16", 64, 100), ("f32", 128, 40),
                                       ("bf16", 128, 128)])
def test_split_chain_update_matches_member_order(gpu, dtype, d, k):
    """k_usum/k_ufin (split f64 chains + exact f32 enclosure test, member-order
    fallback) and k_ustream/k_ufin (the same sums streamed in token order)
    give the same Lloyd run as the member-order chains, bit for bit."""
    from paper_2604_18348_b200 import _lib as L
    from paper_2604_18348_b200 import engine as E
    g = torch.Generator().manual_seed(d + k)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    xs = [(torch.randn(12000 + 777 * h, d, generator=g) * (1 + h)).to(tdt).cuda() for h in range(3)]
    runs = []
    prev = int(L.lib().ac_get_update_mode())
    for mode in (1, 0, 2, 3):
        L.call("ac_set_update_mode", mode)
        try:
            ms = E.kmeans_batch(xs, [k] * 3, [1, 2, 3], 25, 1e-4)
        finally:
            L.call("ac_set_update_mode", prev)
        torch.cuda.synchronize()
        runs.append([(m.centers.clone(), m.labels.clone(), m.n_iter()) for m in ms])
    for other in runs[1:]:
        for (c0, l0, n0), (c1, l1, n1) in zip(runs[0], other):
            assert n0 == n1
            assert torch.equal(l0, l1)
            assert torch.equal(c0, c1)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_labels_only_lloyd_with_empty_cluster_repair(gpu, oracle, dtype):
    """Lloyd without inertia (labels-only tensor-core assign, approximate
    `best`) must still repair empty clusters exactly like the reference:
    same labels, centres and iteration count as the exact-distance run and
    as the oracle."""
    import numpy as np
    from paper_2604_18348_b200 import _lib as L
    from paper_2604_18348_b200 import engine as E
    g = torch.Generator().manual_seed(21)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    x = (torch.randn(6000, 64, generator=g) * 3).to(tdt)
    init = x.float()[torch.randperm(6000, generator=g)[:40]].clone()
    init[7] = 500.0   # far away: empty after the first assignment -> repair
    init[23] = -500.0
    res = []
    for inertia in (True, False):
        b = E.Batch([x.cuda()], [40], 25)
        b.centers_of(0).copy_(init.cuda())
        b.lloyd_range(0, 1, 25, 1e-4, inertia=inertia)
        torch.cuda.synchronize()
        st = b.status.view(b.P, L.STATUS_WORDS)[0].cpu().numpy()
        res.append((b.labels.cpu().numpy(), b.centers_of(0).cpu().numpy(), int(st[L.ST_NITER]),
                    int(st[L.ST_REPAIRS])))
    (l0, c0, n0, r0), (l1, c1, n1, r1) = res
    assert r0 > 0 and r0 == r1
    assert n0 == n1
    assert np.array_equal(l0, l1)
    assert np.array_equal(c0, c1)
    ref = oracle.lloyd(x.float().numpy(), init.numpy(), 25, 1e-4)
    assert np.array_equal(l1, ref.assignments)
    assert np.array_equal(c1, ref.centers)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("ks", [(129,), (200,), (300, 100), (100, 257, 140)])
def test_tc_assign_chunked_over_128_centres(gpu, dtype, ks, d):
    """k > 128: 128-centre tensor-core passes merged with strict '<' (first
    index wins across chunks) + rebuilt tile histograms == the exact kernel."""
    g = torch.Generator().manual_seed(sum(ks) * 7 + d)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    xs, cs = [], []
    for j, k in enumerate(ks):
        n = 4000 + 1500 * j
        x = (torch.randn(n, d, generator=g) * 20).to(tdt).cuda()
        c = (x.float().cpu()[torch.randint(0, n, (k,), generator=g)] +
             torch.randn(k, d, generator=g) * 0.5)
        c[k // 2] = c[3]  # duplicated centres across chunks: ties -> the lower index
        xs.append(x)
        cs.append(c.cuda())
    _compare(xs, cs)


def test_lloyd_with_chunked_assign_matches_oracle(gpu, oracle):
    """A 200-centre Lloyd run (chunked tensor-core assign) equals the oracle."""
    rng = np.random.default_rng(11)
    x = (rng.normal(size=(9000, 64)) * 5).astype(np.float32)
    init = x[rng.choice(9000, 200, replace=False)] + 0.1
    a = gpu.warm_start_update(x, init)
    b = oracle.warm_start(x, init)
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centers, b.centers)
    assert a.n_iter == b.n_iter


@pytest.mark.parametrize("dtype,d", [("f32", 64), ("bf16", 128)])
def test_pdl_launches_match_plain_launches(gpu, dtype, d):
    """Programmatic dependent launches of the Lloyd-chain kernels (ac_set_pdl)
    give the same k-means as plain stream-ordered launches, bit for bit."""
    from paper_2604_18348_b200 import _lib as L
    from paper_2604_18348_b200 import engine as E
    g = torch.Generator().manual_seed(5 + d)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    xs = [(torch.randn(9000 + 501 * h, d, generator=g) * (1 + h)).to(tdt).cuda() for h in range(2)]
    runs = []
    for on in (0, 1):
        with L.pdl(on):
            ms = E.kmeans_batch(xs, [65, 40], [3, 4], 25, 1e-4)
        torch.cuda.synchronize()
        runs.append([(m.centers.clone(), m.labels.clone(), m.n_iter()) for m in ms])
    for (c0, l0, n0), (c1, l1, n1) in zip(*runs):
        assert n0 == n1
        assert torch.equal(l0, l1)
        assert torch.equal(c0, c1)
