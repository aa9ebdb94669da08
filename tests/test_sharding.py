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


@pytest.mark.parametrize("H", [5, 30])
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
