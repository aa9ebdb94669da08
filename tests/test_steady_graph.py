"""The graph-captured steady-state step (steady.py) equals the eager warm
step bit for bit, step after step (same kernels, state carried in place)."""

import dataclasses

import pytest
import torch

from workload.synthetic import CRIT7_SPEC, gen_synthetic

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_graph_step_matches_eager(gpu, dtype):
    import paper_2604_18348_b200 as P
    H, Ln, D, T = 3, 4096, 64, 4
    spec = dataclasses.replace(CRIT7_SPEC, drift_sigma=5e-4)
    steps = [[], [], [], []]
    for h in range(H):
        s = gen_synthetic(spec, Ln, D, 1, T, 100 + h)
        for t in range(T):
            steps[t].append(s[t][0])
    ins = [[torch.stack([torch.from_numpy(x[j]) for x in steps[t]]).to(dtype).cuda()
            for j in range(3)] for t in range(T)]
    params = P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
    eager = P.LayerSession(params, graph=False)
    graph = P.LayerSession(params, graph=True)
    for t in range(T):
        a = eager.step(*ins[t])
        b = graph.step(*ins[t])
        torch.cuda.synchronize()
        assert torch.equal(a, b), f"step {t}: outputs differ"
        for x, y in zip(eager.key_centers, graph.key_centers):
            assert torch.equal(x, y), f"step {t}: key centres differ"
        for x, y in zip(eager.query_centers, graph.query_centers):
            assert torch.equal(x, y), f"step {t}: query centres differ"
    assert graph.steady is not None and graph.steady.graph is not None
    assert graph.density() == pytest.approx(eager.density())
    assert graph.useful_attention_flops() == pytest.approx(eager.useful_attention_flops())


def test_graph_step_from_pinned_host(gpu):
    """Pinned host inputs: the H2D/D2H copies run inside the graph; results
    equal the eager device path."""
    import paper_2604_18348_b200 as P
    H, Ln, D, T = 2, 4096, 64, 4
    spec = dataclasses.replace(CRIT7_SPEC, drift_sigma=5e-4)
    steps = [[] for _ in range(T)]
    for h in range(H):
        s = gen_synthetic(spec, Ln, D, 1, T, 200 + h)
        for t in range(T):
            steps[t].append(s[t][0])
    ins = [[torch.stack([torch.from_numpy(x[j]) for x in steps[t]]).bfloat16() for j in range(3)]
           for t in range(T)]
    params = P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
    eager = P.LayerSession(params, graph=False)
    graph = P.LayerSession(params, graph=True)
    pinned = [[x.pin_memory() for x in trip] for trip in ins]
    outs = [torch.empty((H, Ln, D), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    for t in range(T):
        a = eager.step(*[x.cuda() for x in ins[t]]).cpu()
        if t < 2:  # step 0 plans, step 1 builds the steady graph (device path)
            b = graph.step(*[x.cuda() for x in ins[t]]).cpu()
        else:
            b = graph.step(*pinned[t], host_out=outs[t % 2])
            torch.cuda.synchronize()
        assert torch.equal(a, b), f"step {t}"
    assert len(graph.steady.host_graphs) == 2
