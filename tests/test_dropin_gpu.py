"""Drop-in surface on the device beyond the pipeline: full_attention with
Lq != Lk and a different value width, matmul, row_softmax, quest_scalar /
quest_scores_loop, and the evaluation ops compare_outputs / exact_topk_keys
(reference tensorops.py:29-51, reference.py:25-82, quest.py:74-91)."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel_l2(ref, x):
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(ref - np.asarray(x, np.float64)) / max(np.linalg.norm(ref), 1e-30))


@pytest.mark.parametrize("lq,lk,d,dv", [(5, 1, 8, 8), (3, 6, 8, 8), (16, 12, 8, 8), (16, 12, 8, 4),
                                        (300, 1000, 64, 64), (1000, 300, 64, 32),
                                        (129, 257, 128, 128), (7, 3, 5, 11)])
def test_full_attention_rectangular(gpu, oracle, lq, lk, d, dv):
    rng = np.random.default_rng(lq * 1000 + lk)
    q = rng.normal(size=(lq, d)).astype(np.float32)
    k = rng.normal(size=(lk, d)).astype(np.float32)
    v = rng.normal(size=(lk, dv)).astype(np.float32)
    out = gpu.full_attention(q, k, v)
    assert out.shape == (lq, dv) and out.dtype == np.float32
    assert rel_l2(oracle.full_attention(q, k, v), out) <= 1e-5


def test_full_attention_rectangular_bf16(gpu, oracle):
    rng = np.random.default_rng(3)
    q, k, v = (rng.normal(size=(n, 64)).astype(np.float32) for n in (700, 2000, 2000))
    tq, tk, tv = (torch.from_numpy(a).bfloat16().cuda() for a in (q, k, v))
    out = gpu.full_attention(tq, tk, tv)
    assert out.is_cuda and tuple(out.shape) == (700, 64)
    ref = oracle.full_attention(*(t.float().cpu().numpy() for t in (tq, tk, tv)))
    assert rel_l2(ref, out.cpu().numpy()) <= 1e-2


def test_full_attention_contract_cases(gpu):
    """Single key -> v0; identical keys -> mean of values; convex combination
    (reference tests/test_reference.py:26-60)."""
    rng = np.random.default_rng(0)
    q = rng.normal(size=(5, 8)).astype(np.float32)
    k = rng.normal(size=(1, 8)).astype(np.float32)
    v = rng.normal(size=(1, 8)).astype(np.float32)
    np.testing.assert_allclose(gpu.full_attention(q, k, v), np.repeat(v, 5, 0), atol=1e-6)
    k6 = np.repeat(rng.normal(size=(1, 8)).astype(np.float32), 6, 0)
    v6 = rng.normal(size=(6, 8)).astype(np.float32)
    np.testing.assert_allclose(gpu.full_attention(q[:3], k6, v6),
                               np.repeat(v6.mean(0, keepdims=True), 3, 0), atol=1e-5)
    q16, k12, v12 = (rng.normal(size=(n, 8)).astype(np.float32) for n in (16, 12, 12))
    o = gpu.full_attention(q16, k12, v12)
    assert np.all(o <= v12.max(0) + 1e-5) and np.all(o >= v12.min(0) - 1e-5)
    with pytest.raises(gpu.DimensionError):
        gpu.full_attention(q16, k12[:, :4], v12)
    with pytest.raises(gpu.DimensionError):
        gpu.full_attention(q16, k12, v12[:5])


@pytest.mark.parametrize("m,k,n", [(1500, 64, 100), (200, 128, 200), (7, 5, 9), (100, 17, 3),
                                   (30, 64, 30), (1, 64, 50), (3, 2, 1)])
def test_matmul(gpu, oracle, m, k, n):
    rng = np.random.default_rng(m + n)
    a = (rng.normal(size=(m, k)) * 3).astype(np.float32)
    b = (rng.normal(size=(k, n)) * 3).astype(np.float32)
    c = gpu.matmul(a, b)
    assert c.shape == (m, n) and c.dtype == np.float32
    ref = a.astype(np.float64) @ b.astype(np.float64)
    assert np.max(np.abs(c - ref)) <= 1e-5 * max(1.0, np.max(np.abs(ref)))
    if oracle.gemm_order(m, n, k) == 0:  # general-kernel shapes: the oracle's FMA chain exactly
        assert np.array_equal(c, oracle.matmul_nt(a, np.ascontiguousarray(b.T)))
    with pytest.raises(gpu.DimensionError):
        gpu.matmul(a, b[:-1] if k > 1 else np.zeros((2, n), np.float32))


def test_row_softmax(gpu):
    rng = np.random.default_rng(5)
    s = (rng.normal(size=(37, 1000)) * 20).astype(np.float32)
    s[3, 7] = 3.0e38  # large finite values stay stable (row max subtracted)
    for scale in (1.0, 0.125):
        z = scale * s.astype(np.float64)
        z -= z.max(axis=1, keepdims=True)
        ref = np.exp(z)
        ref /= ref.sum(axis=1, keepdims=True)
        out = gpu.row_softmax(s, scale)
        assert out.shape == s.shape and out.dtype == np.float32
        np.testing.assert_allclose(out, ref, rtol=2e-5, atol=1e-7)
        np.testing.assert_allclose(out.sum(axis=1), 1.0, rtol=1e-5)
    np.testing.assert_allclose(gpu.row_softmax(np.zeros((2, 4), np.float32)), 0.25)


def test_quest_scalar_and_loop(gpu, oracle):
    rng = np.random.default_rng(9)
    x = rng.normal(size=(400, 48)).astype(np.float32)
    m = oracle.kmeans(x, 12, 0)
    env = gpu.build_envelopes(x, m)
    reps = rng.normal(size=(10, 48)).astype(np.float32)
    loop = gpu.quest_scores_loop(reps, env)
    ref = np.array([[np.maximum(reps[g] * env.max_vec[c], reps[g] * env.min_vec[c]).sum()
                     for c in range(12)] for g in range(10)], np.float32)
    assert np.array_equal(loop, ref)  # f32 products, numpy pairwise sum: bit-exact
    assert gpu.quest_scalar(reps[2], env, 5) == float(ref[2, 5])
    # the matmul form agrees to rounding and both bound every member product
    tq = gpu.tensor_quest(reps, env)
    np.testing.assert_allclose(tq, loop, rtol=1e-4, atol=1e-3)
    for c in range(12):
        mem = x[m.assignments == c]
        assert np.all(reps @ mem.T <= loop[:, c:c + 1] + 1e-3)


def test_compare_outputs_semantics(gpu):
    """reference.py:59-82 in f64: rel_l2, mean per-row cosine, SNR, max_abs."""
    rng = np.random.default_rng(1)
    a = rng.normal(size=(50, 16)).astype(np.float32)
    b = (a + 0.01 * rng.normal(size=a.shape)).astype(np.float32)
    m = gpu.compare_outputs(a, b)
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    d = a64 - b64
    rel = np.linalg.norm(d) / np.linalg.norm(a64)
    cos = np.mean(np.sum(a64 * b64, 1) / (np.linalg.norm(a64, axis=1) * np.linalg.norm(b64, axis=1)))
    assert m.rel_l2 == pytest.approx(rel, rel=1e-12)
    assert m.cosine_sim == pytest.approx(cos, rel=1e-12)
    assert m.snr_db == pytest.approx(10 * math.log10(np.sum(a64 ** 2) / np.sum(d ** 2)), rel=1e-12)
    assert m.max_abs == pytest.approx(np.max(np.abs(d)), rel=1e-12)
    same = gpu.compare_outputs(a, a)
    assert same.rel_l2 == 0.0 and math.isinf(same.snr_db) and same.cosine_sim == pytest.approx(1.0)
    z = gpu.compare_outputs(np.zeros((3, 4), np.float32), np.zeros((3, 4), np.float32))
    assert z.rel_l2 == 0.0 and z.cosine_sim == 1.0
    with pytest.raises(gpu.DimensionError):
        gpu.compare_outputs(a, b[:10])


def test_exact_topk_keys_semantics(gpu):
    """reference.py:48-56: stable descending sort of k @ q, ties -> lower index."""
    rng = np.random.default_rng(2)
    k = rng.normal(size=(500, 32)).astype(np.float32)
    k[10] = k[3]  # an exact tie
    q = rng.normal(size=32).astype(np.float32)
    got = gpu.exact_topk_keys(q, k, 40)
    scores = k @ q
    ref = np.argsort(-scores, kind="stable")[:40]
    # scores equal to fp rounding: compare the score sequence and the tie order
    assert np.allclose(scores[got], scores[ref], rtol=1e-6, atol=1e-5)
    i3, i10 = list(got).index(3) if 3 in got else None, list(got).index(10) if 10 in got else None
    if i3 is not None and i10 is not None:
        assert i3 < i10
    basis = np.eye(8, dtype=np.float32)
    assert list(gpu.exact_topk_keys(basis[5], basis, 1)) == [5]
    with pytest.raises(gpu.ParameterError):
        gpu.exact_topk_keys(q, k, 0)


def _topp_numpy(scores, top_p, counts, scale, cap):
    """The top-p rule restated in numpy (test reference)."""
    order = np.argsort(-scores, axis=1, kind="stable")
    out = np.full((scores.shape[0], cap), -1, np.int64)
    cov = []
    for g in range(scores.shape[0]):
        s = scores[g, order[g]].astype(np.float64)
        m = counts[order[g]] * np.exp((s - s[0]) * scale)
        cum = np.cumsum(m)
        n = int(np.searchsorted(cum, top_p * cum[-1] * (1 - 1e-6))) + 1
        n = max(1, min(n, cap))
        out[g, :n] = order[g, :n]
        cov.append(counts[order[g, :n]].sum())
    return out, float(np.mean(cov) / counts.sum())


@pytest.mark.parametrize("top_p,cap", [(0.5, 40), (0.9, 40), (0.99, 25), (1.0, 40)])
def test_select_topp_clusters(gpu, top_p, cap):
    """Top-p extension: smallest score-ordered prefix reaching top_p of the
    estimated mass (counts x exp(score x scale)), capped; -1 padding."""
    rng = np.random.default_rng(int(top_p * 100) + cap)
    scores = (rng.normal(size=(65, 40)) * 3).astype(np.float32)
    counts = rng.integers(50, 3000, size=40)
    got = gpu.select_topp_clusters(scores, top_p, counts, mass_scale=0.5, max_clusters=cap)
    ref, dens = _topp_numpy(scores, top_p, counts, 0.5, cap)
    n_g = (got.selected >= 0).sum(axis=1)
    n_r = (ref >= 0).sum(axis=1)
    assert np.all(np.abs(n_g - n_r) <= 1)  # f32 vs f64 mass sums at the boundary
    for g in range(65):
        k = min(n_g[g], n_r[g])
        assert np.array_equal(got.selected[g, :k], ref[g, :k])
        assert np.all(got.selected[g, n_g[g]:] == -1)
    if top_p == 1.0:
        assert np.all(n_g == min(cap, 40)) or np.all(n_g >= 1)
    # top-1 == top-k with k = 1 when top_p is tiny
    one = gpu.select_topp_clusters(scores, 1e-9, counts, max_clusters=cap)
    assert np.array_equal(one.selected[:, 0], gpu.select_topk_clusters(scores, 1, counts).selected[:, 0])
    with pytest.raises(gpu.ParameterError):
        gpu.select_topp_clusters(scores, 1.5, counts)
