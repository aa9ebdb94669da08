"""CUDA path vs the bit-exact CPU oracle on identical seeded inputs.

Integer/label/selection results must be bit-identical; clustering floats
(centres, inertia, tau, stage MSE) too, because the oracle restates the
reference arithmetic exactly.  Attention outputs: rel-L2 <= 1e-4 for f32
inputs, <= 1e-2 for bf16 inputs (BASELINE.json north_star tolerances).
"""

import numpy as np
import pytest
import torch

from workload.synthetic import CRIT7_SPEC, LayerSpec, gen_synthetic

pytestmark = pytest.mark.gpu

F32_TOL = 1e-4
BF16_TOL = 1e-2


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))


def same_model(dev, ora, inertia=True):
    assert np.array_equal(dev.assignments, ora.assignments)
    assert np.array_equal(dev.centers, ora.centers)
    assert np.array_equal(np.asarray(dev.counts, np.int64), np.asarray(ora.counts, np.int64))
    assert dev.n_iter == ora.n_iter
    if inertia:
        assert list(dev.inertia_history) == list(ora.inertia_history)


def bf16_round(a):
    return torch.from_numpy(a).bfloat16().float().numpy()


@pytest.mark.parametrize("n,d,k,seed", [
    (6, 3, 6, 1), (12, 2, 2, 2), (20, 4, 1, 0), (40, 2, 15, 0), (60, 6, 5, 3),
    (200, 8, 10, 4), (300, 64, 8, 2), (500, 32, 16, 1), (1000, 64, 20, 3),
    (2000, 16, 50, 5), (4096, 64, 65, 0), (3000, 128, 100, 7), (700, 17, 9, 11),
])
def test_kmeans_bit_exact(gpu, oracle, n, d, k, seed):
    rng = np.random.default_rng(seed + 100)
    x = (rng.normal(size=(n, d)) * 3).astype(np.float32)
    a = gpu.kmeans(x, k, seed=seed)
    b = oracle.kmeans(x, k, seed)
    same_model(a, b, inertia=k > 1)


def test_l2norm_bit_exact(gpu, oracle):
    rng = np.random.default_rng(0)
    x = (rng.normal(size=(777, 64)) * rng.lognormal(size=(777, 1))).astype(np.float32)
    x[3] = 0
    x[5] = x[5] / np.linalg.norm(x[5])
    nr = gpu.l2_normalize_rows(x)
    ro, deg = oracle.l2_normalize(x)
    assert np.array_equal(nr.rows, ro)
    assert list(nr.degenerate) == list(deg) == [3]


@pytest.mark.parametrize("L,D,dtype", [(2048, 64, "f32"), (4096, 64, "bf16"), (3000, 128, "bf16")])
def test_plan_pieces_bit_exact(gpu, oracle, L, D, dtype):
    q, k, v = gen_synthetic(CRIT7_SPEC, L, D, 1, 1, 0)[0][0]
    if dtype == "bf16":
        q, k = bf16_round(q), bf16_round(k)
        kt = torch.from_numpy(k).bfloat16().cuda()
    else:
        kt = k
    qa, ra = gpu.cluster_queries(q, 65, 0)
    qb, rb = oracle.cluster_queries(q, 65, 0)
    same_model(qa, qb)
    assert np.array_equal(ra, rb)
    s0a = gpu.kmeans(kt, 100, 0)
    s0b = oracle.kmeans(k, 100, 0)
    same_model(_host(s0a), s0b)
    ta = gpu.compute_tau(k, s0b)
    tb = oracle.compute_tau(k, s0b)
    assert ta == tb
    ma = gpu.multi_stage_cluster_keys(k, tb, stage0=s0b)
    mb = oracle.multi_stage(k, tb, stage0=s0b)
    assert np.array_equal(ma.assignments, mb.assignments)
    assert np.array_equal(ma.centers, mb.centers)
    assert ma.stage_mse == mb.stage_mse and ma.stage_count == mb.stage_count
    assert ma.n_iter == mb.n_iter and ma.flag_full == mb.flag_full


def _host(m):
    import dataclasses
    out = dataclasses.replace(m)
    for f in ("centers", "assignments", "counts"):
        v = getattr(m, f)
        if isinstance(v, torch.Tensor):
            setattr(out, f, v.cpu().numpy())
    return out


@pytest.mark.parametrize("kind,L,D,m0,nmax", [
    ("mixed", 1024, 16, 16, 200), ("compact", 512, 8, 16, 1000), ("dispersed", 512, 8, 16, 64),
    ("mixed", 2048, 64, 32, 1000),
])
def test_multi_stage_rounds_bit_exact(gpu, oracle, kind, L, D, m0, nmax):
    spec = LayerSpec(kind=kind, gaussian_components=8, component_sigma=0.5,
                     component_separation=20.0)
    q, k, v = gen_synthetic(spec, L, D, 1, 1, 3)[0][0]
    s0 = oracle.kmeans(k, m0, 1)
    tau = oracle.compute_tau(k, s0)
    ma = gpu.multi_stage_cluster_keys(k, tau, n_max=nmax, m0=m0, seed=1, stage0=s0)
    mb = oracle.multi_stage(k, tau, n_max=nmax, m0=m0, seed=1, stage0=s0)
    assert ma.stage_count == mb.stage_count
    assert ma.flag_full == mb.flag_full
    assert np.array_equal(ma.assignments, mb.assignments)
    assert np.array_equal(ma.centers, mb.centers)
    assert ma.stage_mse == mb.stage_mse
    assert ma.n_iter == mb.n_iter


@pytest.mark.parametrize("gq,c,d", [(2, 3, 4), (8, 16, 32), (5, 7, 11), (65, 100, 64),
                                    (30, 30, 64), (7, 9, 32), (65, 17, 64), (3, 40, 48)])
def test_selection_bit_exact(gpu, oracle, gq, c, d):
    rng = np.random.default_rng(gq * 100 + c)
    x = rng.normal(size=(c * 4, d)).astype(np.float32)
    m = oracle.kmeans(x, c, 0)
    env_o = oracle.envelopes(x, m)
    env_g = gpu.build_envelopes(x, m)
    assert np.array_equal(env_g.max_vec, env_o.max_vec)
    assert np.array_equal(env_g.min_vec, env_o.min_vec)
    assert np.array_equal(env_g.member_order, env_o.member_order)
    assert np.array_equal(env_g.member_starts, env_o.member_starts)
    reps = rng.normal(size=(gq, d)).astype(np.float32)
    s_g = gpu.tensor_quest(reps, env_g)
    s_o = oracle.scores(reps, env_o.max_vec, env_o.min_vec, "quest")
    assert np.array_equal(s_g, s_o)
    assert np.array_equal(gpu.mean_center_scores(reps, m.centers),
                          oracle.scores(reps, m.centers, m.centers, "mean"))
    assert np.array_equal(gpu.tensor_quest_clamped_centers(reps, m.centers),
                          oracle.scores(reps, m.centers, m.centers, "clamped"))
    for topk in (1, min(3, c), c):
        a = gpu.select_topk_clusters(s_o, topk, m.counts)
        b = oracle.select_topk(s_o, topk, m.counts)
        assert np.array_equal(a.selected, b.selected)
        assert a.density == b.density


def test_selection_ties_lower_index(gpu):
    s = np.array([[1.0, 2.0, 2.0], [3.0, 1.0, 2.0]], np.float32)
    r = gpu.select_topk_clusters(s, 2, np.array([1, 1, 1]))
    assert r.selected.tolist() == [[1, 2], [0, 2]]


@pytest.mark.parametrize("L,D", [(300, 16), (1000, 64), (517, 32), (256, 128)])
def test_full_attention_f32(gpu, oracle, L, D):
    rng = np.random.default_rng(L)
    q, k, v = (rng.normal(size=(L, D)).astype(np.float32) for _ in range(3))
    a = gpu.full_attention(q, k, v)
    b = oracle.full_attention(q, k, v)
    assert rel_l2(b, a) <= F32_TOL


def test_head_c1_f32_sparse(gpu, oracle):
    """C1-shaped head (L=4096, D=64, f32), crit-7 spec, topk 25."""
    q, k, v = gen_synthetic(CRIT7_SPEC, 4096, 64, 1, 1, 0)[0][0]
    p = gpu.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
    op = oracle.Params(q_clusters=65, topk=25, full_layer_quota=0.0)
    out, hs = gpu.adacluster_attention(q, k, v, gpu.LayerPolicy(topk=25), gpu.StepState(), 0, p)
    r = oracle.head_step(q, k, v, None, oracle.HeadState(), 0, op)
    assert hs.mode == r.mode == "sparse"
    assert np.array_equal(hs.q_model.assignments, r.q_model.assignments)
    assert np.array_equal(hs.key_model.assignments, r.key_model.assignments)
    assert np.array_equal(hs.selection.selected, r.selection.selected)
    assert hs.density == r.selection.density
    assert hs.key_iters == r.key_iters and hs.query_iters == r.query_iters
    assert rel_l2(r.out, out) <= F32_TOL


def test_head_bf16_sparse(gpu, oracle):
    """bf16 inputs (C2-like spec, smaller L): clustering bit-exact on the
    upcast values, output within 1e-2 of the oracle's f32 sparse output."""
    q, k, v = gen_synthetic(CRIT7_SPEC, 8192, 64, 1, 1, 0)[0][0]
    qb, kb, vb = (torch.from_numpy(a).bfloat16().cuda() for a in (q, k, v))
    qf, kf, vf = (bf16_round(a) for a in (q, k, v))
    p = gpu.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
    op = oracle.Params(q_clusters=65, topk=25, full_layer_quota=0.0)
    out, hs = gpu.adacluster_attention(qb, kb, vb, gpu.LayerPolicy(topk=25), gpu.StepState(), 0, p)
    r = oracle.head_step(qf, kf, vf, None, oracle.HeadState(), 0, op)
    assert np.array_equal(hs.key_model.assignments.cpu().numpy(), r.key_model.assignments)
    assert np.array_equal(hs.q_model.assignments.cpu().numpy(), r.q_model.assignments)
    assert np.array_equal(hs.selection.selected.cpu().numpy(), r.selection.selected)
    assert rel_l2(r.out, out.float().cpu().numpy()) <= BF16_TOL


def _steps_inputs(seed, steps=3, layers=2, heads=2, L=256, D=8, drift=0.0, sigma=0.3):
    out = []
    for l in range(layers):
        spec = LayerSpec(kind="compact", gaussian_components=8, component_sigma=sigma,
                         component_separation=15.0, drift_sigma=drift)
        out.append(gen_synthetic(spec, L, D, heads, steps, seed + l))
    return [[out[l][t] for l in range(layers)] for t in range(steps)]


@pytest.mark.parametrize("seed,steps,drift,quota,layers,heads", [
    (2, 3, 0.02, 0.15, 2, 2), (4, 2, 0.0, 0.5, 2, 2), (6, 4, 0.02, 0.0, 1, 1),
])
def test_run_denoise_steps_vs_oracle(gpu, oracle, seed, steps, drift, quota, layers, heads):
    inp = _steps_inputs(seed, steps=steps, drift=drift, layers=layers, heads=heads)
    p = gpu.PipelineParams(q_clusters=8, topk=3, m0=16, n_max=1000, full_layer_quota=quota)
    op = oracle.Params(q_clusters=8, topk=3, m0=16, n_max=1000, full_layer_quota=quota)
    res = gpu.run_denoise_steps(inp, p, seed=1)
    outs, modes, rr, mse, _ = oracle.run_steps(inp, op, seed=1)
    assert [pl.mode for pl in res.policies] == modes
    assert res.mse_layer == mse
    for t in range(steps):
        for l in range(layers):
            for h in range(heads):
                hs, r = res.stats[t][l][h], rr[t][l][h]
                assert hs.mode == r.mode
                assert rel_l2(outs[t][l][h], res.outputs[t][l][h]) <= F32_TOL
                if hs.mode == "sparse":
                    assert np.array_equal(hs.selection.selected, r.selection.selected)
                    assert hs.key_iters == r.key_iters
                    assert hs.query_iters == r.query_iters
                    assert hs.density == r.selection.density


@pytest.mark.parametrize("H,L,D", [(1, 128, 64), (2, 1000, 64), (3, 4133, 64), (1, 300, 128),
                                   (2, 2500, 128)])
def test_dense_attention_tcgen05_bf16(gpu, oracle, H, L, D):
    """tcgen05 kernel (bf16, D 64/128) vs the f32 oracle on the same bf16 values."""
    from paper_2604_18348_b200 import engine as E
    rng = np.random.default_rng(L + D)
    q, k, v = (rng.normal(size=(H, L, D)).astype(np.float32) for _ in range(3))
    k *= 2.0
    qb, kb, vb = (torch.from_numpy(a).bfloat16().cuda() for a in (q, k, v))
    out = E.dense_attention_heads(qb, kb, vb, out_dtype=torch.float32).cpu().numpy()
    for h in range(H):
        ref = oracle.full_attention(*(bf16_round(a[h]) for a in (q, k, v)))
        assert rel_l2(ref, out[h]) <= BF16_TOL


@pytest.mark.parametrize("D", [64, 128])
def test_sparse_tcgen05_matches_simt(gpu, D):
    """Same runs/items through both attention kernels (bf16 inputs)."""
    from paper_2604_18348_b200.pipeline import LayerRunner
    q, k, v = gen_synthetic(CRIT7_SPEC, 6000, D, 2, 1, 3)[0][0]
    Q, K, V = (torch.stack([torch.from_numpy(a)] * 2).bfloat16().cuda().contiguous()
               for a in (q, k, v))
    p = gpu.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
    outs = {}
    for impl in ("auto", "simt"):
        run = LayerRunner(p, torch.float32, impl)
        plan = run.plan(Q, K, [0, 1])
        so = run.sparse(Q, K, V, plan.q_models, plan.reps, plan.key_models, 25)
        outs[impl] = so.out.cpu().numpy()
    assert rel_l2(outs["simt"], outs["auto"]) <= BF16_TOL


@pytest.mark.parametrize("d", [64, 128])
def test_envelopes_large_clusters_signed_zeros(gpu, oracle, d):
    """k_envelopes_w (8 warps per cluster, chunk results folded in order) vs
    the sequential np.maximum/np.minimum fold, with +0/-0 ties and large
    clusters so that every warp has a chunk."""
    rng = np.random.default_rng(d)
    x = rng.normal(size=(6000, d)).astype(np.float32)
    x[:, 0] = np.where(rng.random(6000) < 0.5, 0.0, -0.0).astype(np.float32)
    x[:, 1] = np.abs(x[:, 1]) * -1.0
    x[::3, 1] = -0.0
    x[::5, 1] = 0.0
    m = oracle.kmeans(x, 7, 2)
    env_o = oracle.envelopes(x, m)
    env_g = gpu.build_envelopes(x, m)
    assert np.array_equal(env_g.max_vec.view(np.int32), env_o.max_vec.view(np.int32))
    assert np.array_equal(env_g.min_vec.view(np.int32), env_o.min_vec.view(np.int32))


def test_compactness_matches_scalar_loops(gpu):
    """GPU compactness (f64) vs the reference test's scalar loops
    (tests/test_clustering.py:240-275 of the reference)."""
    import math
    rng = np.random.default_rng(18)
    x = rng.normal(size=(60, 3)).astype(np.float32)
    m = gpu.kmeans(x, 4, seed=3)
    rep = gpu.compactness([x], [m])
    mse = np.mean([np.linalg.norm(x[i].astype(np.float64) - m.centers[m.assignments[i]]) ** 2
                   for i in range(60)])
    assert rep.mse_layer == pytest.approx(mse, rel=1e-12)
    s = [np.mean([np.linalg.norm(x[i].astype(np.float64) - m.centers[c]) for i in range(60)
                  if m.assignments[i] == c]) for c in range(4)]
    db = np.mean([max((s[i] + s[j]) / np.linalg.norm(m.centers[i].astype(np.float64) - m.centers[j])
                      for j in range(4) if j != i) for i in range(4)])
    assert rep.db_index == pytest.approx(db, rel=1e-12)
    z = np.tile(np.array([[1.0, 1.0]], np.float32), (4, 1))
    rz = gpu.compactness([z], [gpu.kmeans(z, 1, seed=0)])
    assert rz.mse_layer == 0.0 and math.isinf(rz.comp)


@pytest.mark.parametrize("m0,nmax,sched", [(1, 10, None), (3, 5, None), (4, 40, "grow")])
def test_multi_stage_capacity_edges(gpu, oracle, m0, nmax, sched):
    """Accumulated centres can reach n_max - 1 + max(8, m0) before the budget
    check trips (clustering.py:282-290), and a custom stage_schedule may ask
    for more than m0 per round; both must match the oracle."""
    spec = LayerSpec(kind="dispersed", gaussian_components=8, component_sigma=0.5,
                     component_separation=20.0)
    q, k, v = gen_synthetic(spec, 600, 16, 1, 1, 5)[0][0]
    schedule = (lambda t, remaining, total: 4 + 9 * t) if sched == "grow" else None
    s0 = oracle.kmeans(k, m0, 2)
    tau = oracle.compute_tau(k, s0) * 0.5
    ma = gpu.multi_stage_cluster_keys(k, tau, n_max=nmax, m0=m0, seed=2, stage0=s0,
                                      stage_schedule=schedule)
    mb = oracle.multi_stage(k, tau, n_max=nmax, m0=m0, seed=2, stage0=s0, stage_schedule=schedule)
    assert ma.flag_full == mb.flag_full and ma.stage_count == mb.stage_count
    assert np.array_equal(ma.assignments, mb.assignments)
    assert np.array_equal(ma.centers, mb.centers)
    assert ma.stage_mse == mb.stage_mse
