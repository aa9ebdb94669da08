"""Head sharding over GPUs of one box (one process per GPU).

Heads are independent (the reference proves it in
tests/test_pipeline.py:131-139: per-head seeds ``seed + 7919*l + h``), so a
layer's heads are split into contiguous blocks, one per rank, and the only
collectives are
  1. step 0: every rank learns every head's ``flag_full`` and clustering MSE,
     so all ranks apply the identical per-layer policy (pipeline.py:319-339);
  2. every step: an all-gather of the per-head outputs into the
     sequence-level [H, L, D] result (NCCL over NVLink/NVSwitch; gloo on CPU
     in the tests).
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

__all__ = ["head_block", "heads_per_rank", "gather_heads", "exchange_step0",
           "decide_policies", "ShardedLayerSession"]


def heads_per_rank(H: int, world: int) -> int:
    return math.ceil(H / world)


def head_block(H: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [h0, h1) block of heads owned by ``rank`` (may be empty)."""
    per = heads_per_rank(H, world)
    return min(H, rank * per), min(H, (rank + 1) * per)


def gather_heads(local: torch.Tensor, H: int, group=None) -> torch.Tensor:
    """All-gather per-rank head blocks [h_local, L, D] into [H, L, D]."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    per = heads_per_rank(H, world)
    shape = (per,) + tuple(local.shape[1:])
    pad = torch.zeros(shape, dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    if dist.get_backend(group) == "nccl":
        full = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype,
                           device=local.device)
        dist.all_gather_into_tensor(full, pad, group=group)
    else:
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        full = torch.cat(parts)
    return full[:H]


def exchange_step0(flags: torch.Tensor, mse: torch.Tensor, H: int, group=None):
    """All-gather the per-head step-0 statistics (flag_full u8, MSE f64)."""
    flags = flags.to(torch.float64).reshape(-1, 1)
    mse = mse.to(torch.float64).reshape(-1, 1)
    both = torch.cat([flags, mse], dim=1)
    full = gather_heads(both, H, group)
    return full[:, 0] > 0.5, full[:, 1]


def decide_policies(mse_layer: list, flagged: list, quota: float) -> list:
    """pipeline.py:326-339: a layer runs full attention if any head overflowed
    the centre budget or it is among the worst ceil(quota * n_layers) layers
    by step-0 MSE (ties to the lower layer index)."""
    n = len(mse_layer)
    forced = math.ceil(quota * n) if quota > 0 else 0
    worst = set(sorted(range(n), key=lambda l: (-mse_layer[l], l))[:forced])
    return ["full" if (flagged[l] or l in worst) else "sparse" for l in range(n)]


class ShardedLayerSession:
    """LayerSession over this rank's head block + output all-gather.  Step 0
    agrees on the layer policy across ranks before any attention runs."""

    def __init__(self, H: int, params=None, seed: int = 0, layer: int = 0, out_dtype=None,
                 group=None):
        from .pipeline import LayerSession
        self.H = H
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.h0, self.h1 = head_block(H, world, rank)
        self.session = LayerSession(params, seed=seed, layer=layer, out_dtype=out_dtype,
                                    head_offset=self.h0, reduce_flag=self._any_flag)

    def _any_flag(self, local: bool) -> bool:
        if not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return local
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([1 if local else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def step(self, Q, K, V) -> torch.Tensor:
        """Q/K/V: this rank's heads [h1-h0, L, D]; returns all heads [H, L, D]."""
        out = self.session.step(Q, K, V)
        return gather_heads(out, self.H, self.group)
