"""StackSession (the streamed, graph-captured run_denoise_steps of a layer
stack) vs the oracle's run_steps (pipeline.py:296-386): step-0 planning of
every layer, per-layer MSE, the quota forcing the worst layers to full
attention, frozen policies, warm steps -- outputs, selections and carried
centres identical to the oracle (bit-exact clustering; attention rel-L2)."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

from workload.synthetic import CRIT7_SPEC, LayerSpec, gen_synthetic

pytestmark = pytest.mark.gpu


def rel_l2(ref, x):
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(ref - np.asarray(x, np.float64)) / max(np.linalg.norm(ref), 1e-30))


SPECS = [dataclasses.replace(CRIT7_SPEC, drift_sigma=5e-4),
         LayerSpec(kind="compact", gaussian_components=16, component_sigma=2.0,
                   component_separation=40.0, drift_sigma=5e-4, scale_spread=0.3),
         LayerSpec(kind="compact", gaussian_components=24, component_sigma=1.5,
                   component_separation=60.0, drift_sigma=5e-4, scale_spread=0.3),
         LayerSpec(kind="compact", gaussian_components=8, component_sigma=3.0,
                   component_separation=30.0, drift_sigma=5e-4, scale_spread=0.3)]


@pytest.mark.parametrize("dtype,quota", [(torch.bfloat16, 0.25), (torch.float32, 0.5)])
def test_stack_session_matches_oracle_run_steps(gpu, oracle, dtype, quota):
    n_layers, H, Ln, D, T = 4, 2, 2048, 64, 3
    per_layer = [gen_synthetic(SPECS[l], Ln, D, H, T, 40 + l) for l in range(n_layers)]
    # step_inputs[t][l][h] = (q, k, v) in the device dtype's values
    dev = [[[tuple(torch.from_numpy(a).to(dtype) for a in per_layer[l][t][h]) for h in range(H)]
            for l in range(n_layers)] for t in range(T)]
    ora = [[[tuple(x.float().numpy() for x in dev[t][l][h]) for h in range(H)]
            for l in range(n_layers)] for t in range(T)]
    params = gpu.PipelineParams(q_clusters=65, topk=25, full_layer_quota=quota)
    op = oracle.Params(q_clusters=65, topk=25, full_layer_quota=quota)
    outs_o, modes_o, res_o, mse_o, _ = oracle.run_steps(ora, op, seed=3)

    def stacked(t, l, j):
        return torch.stack([dev[t][l][h][j] for h in range(H)]).cuda()

    st = gpu.StackSession(n_layers, H, params, seed=3)
    modes = st.plan([(stacked(0, l, 0), stacked(0, l, 1)) for l in range(n_layers)])
    assert modes == modes_o and st.mse_layer == mse_o
    assert "full" in modes and "sparse" in modes
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-4
    for t in range(T):
        outs = st.step([(stacked(t, l, 0), stacked(t, l, 1), stacked(t, l, 2))
                        for l in range(n_layers)])
        for l in range(n_layers):
            sess = st.layers[l]
            for h in range(H):
                e = rel_l2(outs_o[t][l][h], outs[l][h].float().cpu().numpy())
                assert e <= tol, f"step {t} layer {l} head {h}: rel-L2 {e}"
                r = res_o[t][l][h]
                if modes[l] == "sparse":
                    sel = (sess.last[2].selections[h].selected if sess.steady is None
                           else sess.steady.selected[h])
                    assert np.array_equal(sel.cpu().numpy(), r.selection.selected)
        if t >= 1:
            assert all(st.layers[l].steady is not None for l in range(n_layers)
                       if modes[l] == "sparse")
    # one shared workspace for all sparse layers' graphs
    assert len(st.pool) == 1
