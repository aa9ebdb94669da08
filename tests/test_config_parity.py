"""Parity at the BASELINE.json configs' per-head sizes.

One or two heads of each config (C1 f32 2x4096x64 in both the criterion-7 /
topk-25 setting and the reference "as-is" setting; C2 70000x64, C3 32760x128
and C4 118800x128 in bf16) run step 0 and two warm steps through the public
streaming driver ``LayerSession`` with the CUDA-graph steady step, and are
compared step by step with the CPU oracle carrying the same state
(oracle.head_step, which restates pipeline.py:237-275 and is pinned to the
reference by tests/golden).

Bars (BASELINE.json north_star): query/key labels, key counts and selected
cluster sets bit-identical (the oracle reproduces the reference's arithmetic
exactly); carried key/query centres bit-identical; sparse
output rel-L2 <= 1e-2 (bf16 inputs) / <= 1e-4 (f32) of the oracle's sparse
output on the same (bf16-rounded) values.  The rel-L2 of both outputs
against dense attention is printed for the record.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

from workload.synthetic import CRIT7_SPEC, LayerSpec, gen_outlier_steps, gen_synthetic

pytestmark = pytest.mark.gpu

DRIFT = 5e-4
T_STEPS = 3


def rel_l2(ref, x):
    ref = np.asarray(ref, np.float64)
    x = np.asarray(x, np.float64)
    return float(np.linalg.norm(ref - x) / max(np.linalg.norm(ref), 1e-30))


def _inputs(spec, L, D, heads, seeds, dtype):
    """[t] -> (Q, K, V) [H, L, D] torch (CPU) in ``dtype``; plus the f32
    values the oracle sees (bf16-rounded when dtype is bf16)."""
    if isinstance(spec, tuple):  # ("outlier", frac_tail): the adaptive-count workload
        per = [gen_outlier_steps(L, D, T_STEPS, s, spec[1], drift_sigma=DRIFT) for s in seeds[:heads]]
    else:
        per = [gen_synthetic(spec, L, D, 1, T_STEPS, s) for s in seeds[:heads]]
    dev, ora = [], []
    for t in range(T_STEPS):
        trip = [torch.from_numpy(np.stack([per[h][t][0][j] for h in range(heads)])).to(dtype)
                for j in range(3)]
        dev.append(trip)
        ora.append([x.float().numpy() for x in trip])
    return dev, ora


def _dense_f32(q, k, v):
    """Dense softmax attention in f32 on the device (torch SDPA; an
    evaluation reference only, not the product path)."""
    import torch.nn.functional as F
    tq, tk, tv = (torch.from_numpy(a).cuda()[None, None] for a in (q, k, v))
    with torch.nn.attention.sdpa_kernel([torch.nn.attention.SDPBackend.EFFICIENT_ATTENTION,
                                         torch.nn.attention.SDPBackend.MATH]):
        return F.scaled_dot_product_attention(tq, tk, tv)[0, 0].cpu().numpy()


def _gpu_view(sess, h):
    """Per-head results of the session's last step as numpy."""
    if sess.steady is None:
        qm, km, so = sess.last
        sel = so.selections[h]
        return dict(qlab=qm[h].labels.cpu().numpy(), klab=km[h].labels.cpu().numpy(),
                    kcounts=km[h].counts.cpu().numpy(), selected=sel.selected.cpu().numpy(),
                    density=float(sel.density.item()))
    st = sess.steady
    qm, km = st.qmodels[h], st.kmodels[h]
    return dict(qlab=qm.labels.cpu().numpy(), klab=km.labels.cpu().numpy(),
                kcounts=km.counts.cpu().numpy(), selected=st.selected[h].cpu().numpy(),
                density=float(st.density[h].item()))


def _run(P, O, spec, L, D, heads, seeds, dtype, q_clusters, topk, tol, label):
    dev_in, ora_in = _inputs(spec, L, D, heads, seeds, dtype)
    params = P.PipelineParams(q_clusters=q_clusters, topk=topk, full_layer_quota=0.0)
    op = O.Params(q_clusters=q_clusters, topk=topk, full_layer_quota=0.0)
    # LayerSession seeds head h with seed + 7919*layer + h (pipeline.py:315)
    sess = P.LayerSession(params, seed=0, graph=True)
    states = [O.HeadState() for _ in range(heads)]
    report = []
    for t in range(T_STEPS):
        Q, K, V = (x.cuda() for x in dev_in[t])
        out = sess.step(Q, K, V).float().cpu().numpy()
        if t >= 1:
            assert sess.steady is not None, "warm step did not take the graph path"
        for h in range(heads):
            q, k, v = (a[h] for a in ora_in[t])
            r = O.head_step(q, k, v, None, states[h], h, op)
            g = _gpu_view(sess, h)
            where = f"{label} step {t} head {h}"
            assert r.mode == "sparse" and sess.mode == "sparse", where
            qa = float(np.mean(g["qlab"] == r.q_model.assignments))
            ka = float(np.mean(g["klab"] == r.key_model.assignments))
            same_sel = float(np.mean(np.all(g["selected"] == r.selection.selected, axis=1)))
            e_sparse = rel_l2(r.out, out[h])
            dense = _dense_f32(q, k, v)
            report.append(dict(step=t, head=h, q_labels=qa, k_labels=ka, selected=same_sel,
                               rel_l2=e_sparse, gpu_vs_dense=rel_l2(dense, out[h]),
                               ref_vs_dense=rel_l2(dense, r.out), density=g["density"]))
            print(where, report[-1])
            assert qa == 1.0, f"{where}: query label agreement {qa}"
            assert ka == 1.0, f"{where}: key label agreement {ka}"
            assert np.array_equal(g["kcounts"], r.key_model.counts), where
            assert same_sel == 1.0, f"{where}: selected-set agreement {same_sel}"
            assert g["density"] == r.selection.density, where
            assert e_sparse <= tol, f"{where}: rel-L2 {e_sparse}"
            # carried state (next step's warm start)
            assert np.array_equal(sess.key_centers[h].cpu().numpy(), states[h].key_centers), where
            assert np.array_equal(sess.query_centers[h].cpu().numpy(),
                                  states[h].query_centers), where
    return report, sess


def test_c1_crit7_f32(gpu, oracle):
    """C1: 2 heads x 64, L=4096, f32; criterion-7 spec, topk 25."""
    spec = dataclasses.replace(CRIT7_SPEC, drift_sigma=DRIFT)
    _run(gpu, oracle, spec, 4096, 64, 2, [1000, 1001], torch.float32, 65, 25, 1e-4, "C1-crit7")


def test_c1_as_is_f32(gpu, oracle):
    """C1 as the reference runs it out of the box: default LayerSpec and
    default PipelineParams (topk 64), quota 0 for a single layer."""
    _run(gpu, oracle, LayerSpec(), 4096, 64, 2, [1000, 1001], torch.float32, 65, 64, 1e-4,
         "C1-as-is")


def test_c2_head_bf16(gpu, oracle):
    """C2: one CogVideoX-2B head, L=70000, D=64, bf16 (the bench's head 0)."""
    spec = dataclasses.replace(CRIT7_SPEC, drift_sigma=DRIFT)
    _run(gpu, oracle, spec, 70000, 64, 1, [1000], torch.bfloat16, 65, 25, 1e-2, "C2")


def test_c3_head_bf16(gpu, oracle):
    """C3: one Wan-2.1-1.3B head, L=32760, D=128, bf16."""
    spec = dataclasses.replace(CRIT7_SPEC, drift_sigma=DRIFT)
    _run(gpu, oracle, spec, 32760, 128, 1, [1000], torch.bfloat16, 65, 25, 1e-2, "C3")


def test_c4_head_bf16(gpu, oracle):
    """C4: one HunyuanVideo head, L=118800, D=128, bf16."""
    spec = dataclasses.replace(CRIT7_SPEC, drift_sigma=DRIFT)
    _run(gpu, oracle, spec, 118800, 128, 1, [1000], torch.bfloat16, 65, 25, 1e-2, "C4")


def test_c3_outlier_heads_adaptive_counts(gpu, oracle):
    """C3-sized heads of the outlier-cloud workload (bench C3 spec mix): the
    multi-stage planner runs tens of rounds and the key-cluster count adapts
    (> m0 = 100); everything still bit-exact against the oracle."""
    _, sess = _run(gpu, oracle, ("outlier", 0.002), 32760, 128, 2, [1001, 1002], torch.bfloat16,
                   65, 25, 1e-2, "C3-outlier")
    counts = [int(c.shape[0]) for c in sess.key_centers]
    print("key clusters", counts)
    assert all(c > 100 for c in counts)
