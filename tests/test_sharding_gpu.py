"""The sharded drivers with real kernels: two ranks (gloo, both on cuda:0)
each run their balanced block of heads; the gathered outputs, the agreed
per-layer policies (quota included) and the carried centres equal a
single-process run over all heads bit for bit (heads are independent and
every kernel is deterministic)."""

from __future__ import annotations

import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

H, L, D, T, NL = 3, 2048, 64, 3, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    from workload.synthetic import CRIT7_SPEC, LayerSpec, gen_synthetic
    specs = [dataclasses.replace(CRIT7_SPEC, drift_sigma=5e-4),
             LayerSpec(kind="compact", gaussian_components=16, component_sigma=2.0,
                       component_separation=40.0, drift_sigma=5e-4, scale_spread=0.3),
             LayerSpec(kind="compact", gaussian_components=24, component_sigma=1.5,
                       component_separation=60.0, drift_sigma=5e-4, scale_spread=0.3)]
    per = [gen_synthetic(specs[l], L, D, H, T, 70 + l) for l in range(NL)]
    return [[[torch.from_numpy(np.stack([per[l][t][h][j] for h in range(H)])).bfloat16()
              for j in range(3)] for l in range(NL)] for t in range(T)]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import paper_2604_18348_b200 as P
    from paper_2604_18348_b200.sharding import ShardedLayerSession, head_block
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ins = _inputs()
    h0, h1 = head_block(H, world, rank)
    params = P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.3)
    st = P.StackSession(NL, H, params, seed=5)
    modes = st.plan([(ins[0][l][0][h0:h1].cuda(), ins[0][l][1][h0:h1].cuda()) for l in range(NL)])
    outs = []
    for t in range(T):
        o = st.step([tuple(x[h0:h1].cuda() for x in ins[t][l]) for l in range(NL)])
        outs.append([x.float().cpu().numpy() for x in o])
    one = ShardedLayerSession(H, P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0),
                              seed=5, layer=0)
    lo = [one.step(*(x[h0:h1].cuda() for x in ins[t][0])).float().cpu().numpy() for t in range(T)]
    q.put((rank, modes, st.mse_layer, outs, lo))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_equal_one_process(gpu):
    import paper_2604_18348_b200 as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ins = _inputs()
    params = P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.3)
    st = P.StackSession(NL, H, params, seed=5)
    modes = st.plan([(ins[0][l][0].cuda(), ins[0][l][1].cuda()) for l in range(NL)])
    ref = [[x.float().cpu().numpy() for x in st.step([tuple(x.cuda() for x in ins[t][l])
                                                      for l in range(NL)])] for t in range(T)]
    one = P.LayerSession(P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0), seed=5)
    lref = [one.step(*(x.cuda() for x in ins[t][0])).float().cpu().numpy() for t in range(T)]
    assert "full" in modes and "sparse" in modes  # ceil(0.3 * 3) = 1 layer forced dense
    for rank, rmodes, rmse, outs, lo in res:
        assert rmodes == modes and rmse == st.mse_layer
        for t in range(T):
            for l in range(NL):
                assert np.array_equal(outs[t][l], ref[t][l]), f"rank {rank} step {t} layer {l}"
            assert np.array_equal(lo[t], lref[t]), f"rank {rank} layer session step {t}"
