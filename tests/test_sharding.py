"""Multi-process host logic of head sharding on CPU (gloo, world size 2):
head blocks, the step-0 statistics exchange and the output all-gather are
the only cross-rank data flow (sharding.py)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_18348_b200.sharding import (decide_policies, exchange_step0, gather_heads,
                                            head_block)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h0, h1 = head_block(H, world, rank)
    L, D = 7, 4
    local = torch.stack([torch.full((L, D), float(h)) for h in range(h0, h1)]) if h1 > h0 else \
        torch.zeros((0, L, D))
    full = gather_heads(local, H)
    flags = torch.tensor([1 if h == 3 else 0 for h in range(h0, h1)], dtype=torch.uint8)
    mse = torch.tensor([10.0 * h for h in range(h0, h1)], dtype=torch.float64)
    fl, ms = exchange_step0(flags, mse, H)
    out_q.put((rank, full.numpy().copy(), fl.numpy().copy(), ms.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H", [5, 30, 1])
def test_gloo_gather_and_step0_exchange(H):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, full, fl, ms in res:
        assert full.shape == (H, 7, 4)
        for h in range(H):
            assert (full[h] == h).all()
        assert list(fl) == [h == 3 for h in range(H)]
        assert list(ms) == [10.0 * h for h in range(H)]


def test_head_blocks_cover_every_head_once():
    for H in (1, 5, 12, 24, 30, 40):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                h0, h1 = head_block(H, world, r)
                seen += list(range(h0, h1))
            assert seen == list(range(H))


def test_decide_policies_matches_reference_rule():
    # pipeline.py:326-339: quota forces the worst ceil(q*n) layers (ties -> lower index)
    assert decide_policies([1.0, 3.0, 2.0, 3.0], [False] * 4, 0.25) == ["sparse", "full", "sparse", "sparse"]
    assert decide_policies([1.0, 3.0], [True, False], 0.0) == ["full", "sparse"]
    assert decide_policies([5.0], [False], 0.15) == ["full"]  # ceil(0.15) = 1 forces a single layer


def _policy_worker(rank, world, port, H, n_layers, quota, out_q):
    import numpy as np
    from paper_2604_18348_b200.sharding import agree_policies
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h0, h1 = head_block(H, world, rank)
    rng = np.random.default_rng(7)
    mse_all = rng.random((n_layers, H)) * 10.0          # same on every rank
    flags_all = rng.random((n_layers, H)) < 0.05
    local_mse = [mse_all[l, h0:h1] for l in range(n_layers)]
    local_flags = [list(flags_all[l, h0:h1]) for l in range(n_layers)]
    modes, mse_layer, flagged = agree_policies(local_mse, local_flags, H, quota)
    out_q.put((rank, h1 - h0, modes, mse_layer, flagged))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H,world", [(5, 2), (1, 2), (3, 4), (12, 4)])
def test_gloo_policy_agreement_with_quota(H, world):
    """Every rank derives the same per-layer policies (quota 0.15 over 10
    layers, flagged heads) from its own heads' stats -- including ranks that
    own no head -- and they equal the single-process rule over all heads."""
    import numpy as np
    n_layers, quota = 10, 0.15
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_policy_worker, args=(r, world, port, H, n_layers, quota, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    mse_all = rng.random((n_layers, H)) * 10.0
    flags_all = rng.random((n_layers, H)) < 0.05
    mse_ref = [float(np.mean([float(m) for m in mse_all[l]])) for l in range(n_layers)]
    modes_ref = decide_policies(mse_ref, [bool(flags_all[l].any()) for l in range(n_layers)], quota)
    assert modes_ref.count("full") >= 2  # ceil(0.15 * 10) = 2 forced layers at least
    for rank, nh, modes, mse_layer, flagged in res:
        assert modes == modes_ref and mse_layer == mse_ref
    assert sum(r[1] for r in res) == H


def test_head_blocks_balanced():
    """Balanced split: sizes differ by at most one, larger blocks first."""
    assert [head_block(30, 8, r)[1] - head_block(30, 8, r)[0] for r in range(8)] == [4] * 6 + [3] * 2
    assert [head_block(12, 8, r)[1] - head_block(12, 8, r)[0] for r in range(8)] == [2] * 4 + [1] * 4
    assert [head_block(5, 4, r)[1] - head_block(5, 4, r)[0] for r in range(4)] == [2, 1, 1, 1]
    assert [head_block(3, 4, r)[1] - head_block(3, 4, r)[0] for r in range(4)] == [1, 1, 1, 0]
    for H in range(1, 50):
        for world in (1, 2, 3, 4, 8):
            sizes = [head_block(H, world, r)[1] - head_block(H, world, r)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1 and sum(sizes) == H
