"""Head sharding over GPUs of one box (one process per GPU).

Heads are independent (the reference proves it in
tests/test_pipeline.py:131-139: per-head seeds ``seed + 7919*l + h``), so a
layer's heads are split into balanced contiguous blocks, one per rank
(30 heads on 8 ranks -> 4/4/4/4/4/4/3/3, 12 -> 2/2/2/2/1/1/1/1; a rank may
own no head when H < world), and the only collectives are
  1. step 0: every rank learns every head's ``flag_full`` and clustering MSE,
     so all ranks apply the identical per-layer policy, quota included
     (pipeline.py:319-339) -- ``agree_policies``;
  2. every step: an all-gather of the per-head outputs into the
     sequence-level [H, L, D] result (NCCL over NVLink/NVSwitch; gloo on CPU
     in the tests), asynchronous so it overlaps the next layer's compute.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["head_block", "heads_per_rank", "gather_heads", "gather_heads_async",
           "exchange_step0", "agree_policies", "decide_policies", "ShardedLayerSession"]


def _world_rank(group=None) -> tuple[int, int]:
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def heads_per_rank(H: int, world: int) -> int:
    """Largest block size (the padded all-gather slot)."""
    return math.ceil(H / world) if world > 0 else H


def head_block(H: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous [h0, h1) block of heads owned by ``rank``: the
    first H % world ranks own one head more (may be empty when H < world)."""
    base, extra = divmod(H, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


class _Pending:
    """An all-gather in flight; ``wait()`` returns the compacted [H, ...] result."""

    def __init__(self, work, parts, sizes, H, per, done=None):
        self.work, self.parts, self.sizes, self.H, self.per = work, parts, sizes, H, per
        self.done = done

    def wait(self) -> torch.Tensor:
        if self.done is not None:
            return self.done
        if self.work is not None:
            self.work.wait()
        if isinstance(self.parts, list):
            blocks = [p[:s] for p, s in zip(self.parts, self.sizes)]
        else:
            blocks = [self.parts[r * self.per:r * self.per + s] for r, s in enumerate(self.sizes)]
        self.done = torch.cat(blocks)
        return self.done


def gather_heads_async(local: torch.Tensor, H: int, group=None) -> _Pending:
    """Start the all-gather of per-rank head blocks [h_local, ...] into
    [H, ...] (blocks padded to the largest block, compacted on wait)."""
    world, rank = _world_rank(group)
    if world == 1:
        return _Pending(None, None, None, H, H, done=local)
    per = heads_per_rank(H, world)
    sizes = [head_block(H, world, r)[1] - head_block(H, world, r)[0] for r in range(world)]
    if local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank} holds {local.shape[0]} heads, expected {sizes[rank]}")
    shape = (per,) + tuple(local.shape[1:])
    if local.shape[0] == per:
        pad = local.contiguous()
    else:
        pad = torch.zeros(shape, dtype=local.dtype, device=local.device)
        pad[:local.shape[0]] = local
    if dist.get_backend(group) == "nccl":
        full = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype,
                           device=local.device)
        work = dist.all_gather_into_tensor(full, pad, group=group, async_op=True)
        return _Pending(work, full, sizes, H, per)
    dev = pad.device
    if pad.is_cuda:  # gloo moves host memory: stage through the host
        pad = pad.cpu()
    parts = [torch.empty_like(pad) for _ in range(world)]
    work = dist.all_gather(parts, pad, group=group, async_op=True)
    pend = _Pending(work, parts, sizes, H, per)
    if dev.type == "cuda":
        pend.wait()
        pend.done = pend.done.to(dev)
    return pend


def gather_heads(local: torch.Tensor, H: int, group=None) -> torch.Tensor:
    """All-gather per-rank head blocks [h_local, L, D] into [H, L, D]."""
    return gather_heads_async(local, H, group).wait()


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


def agree_policies(local_mse: list, local_flags: list, H: int, quota: float, group=None):
    """Identical per-layer policies on every rank (pipeline.py:319-339).

    ``local_mse[l]`` / ``local_flags[l]``: this rank's heads' step-0 key
    clustering MSE (f64) and flag_full for layer l.  One all-gather carries
    every layer; the per-layer MSE is the mean over ALL heads in head order,
    exactly the reference's ``float(np.mean([float(m) for m in mses]))``.
    Returns (modes, mse_layer, flagged)."""
    n_layers = len(local_mse)
    hl = len(local_mse[0]) if n_layers else 0
    st = torch.zeros((hl, 2 * n_layers), dtype=torch.float64)
    for l in range(n_layers):
        st[:, 2 * l] = torch.as_tensor(np.asarray(local_flags[l], np.float64).reshape(-1))
        st[:, 2 * l + 1] = torch.as_tensor(np.asarray(local_mse[l], np.float64).reshape(-1))
    world, _ = _world_rank(group)
    if world > 1 and dist.get_backend(group) == "nccl":
        full = gather_heads(st.cuda(), H, group).cpu()
    else:
        full = gather_heads(st, H, group)
    full = full.numpy()
    mse_layer = [float(np.mean([float(m) for m in full[:, 2 * l + 1]])) for l in range(n_layers)]
    flagged = [bool((full[:, 2 * l] > 0.5).any()) for l in range(n_layers)]
    return decide_policies(mse_layer, flagged, quota), mse_layer, flagged


class ShardedLayerSession:
    """LayerSession over this rank's head block + output all-gather.  Step 0
    agrees on the layer policy across ranks before any attention runs; a rank
    without heads joins the collectives and contributes an empty block."""

    def __init__(self, H: int, params=None, seed: int = 0, layer: int = 0, out_dtype=None,
                 group=None):
        from .pipeline import LayerSession
        self.H = H
        self.group = group
        world, rank = _world_rank(group)
        self.h0, self.h1 = head_block(H, world, rank)
        self.session = LayerSession(params, seed=seed, layer=layer, out_dtype=out_dtype,
                                    head_offset=self.h0, reduce_flag=self._any_flag)

    @property
    def local_heads(self) -> int:
        return self.h1 - self.h0

    def _any_flag(self, local: bool) -> bool:
        world, _ = _world_rank(self.group)
        if world == 1:
            return local
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([1 if local else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def step_local(self, Q, K, V, **kw) -> torch.Tensor:
        """This rank's heads only (no gather); a rank without heads returns
        an empty block after joining the step-0 flag all-reduce."""
        return self.session.step(Q, K, V, **kw)

    def step_async(self, Q, K, V):
        """Local step, then the output all-gather in flight (``.wait()``)."""
        return gather_heads_async(self.step_local(Q, K, V), self.H, self.group)

    def step(self, Q, K, V) -> torch.Tensor:
        """Q/K/V: this rank's heads [h1-h0, L, D]; returns all heads [H, L, D]."""
        return self.step_async(Q, K, V).wait()
