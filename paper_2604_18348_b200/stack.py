"""A layer stack of AdaCluster attention on the device, heads optionally
sharded over the GPUs of a box: the streamed form of ``run_denoise_steps``
(reference pipeline.py:296-386).

Step 0 plans EVERY layer before any layer's attention (pipeline.py:310-324),
because the per-layer policy needs every layer's step-0 key-clustering MSE:
a layer runs full attention when any of its heads overflowed the centre
budget or it is among the worst ``ceil(full_layer_quota * n_layers)`` layers
by MSE (pipeline.py:326-339).  With head sharding each rank plans its own
heads and one all-gather of (flag, MSE) per head gives every rank the same
policies (sharding.agree_policies).  Policies stay frozen for later steps.

Every later (warm) step runs each sparse layer as its own CUDA graph; the
layers share one set of [H, L, D]-sized buffers (steady.Workspace), so the
stack's HBM footprint is one layer's working set plus each layer's carried
state (centres, labels).  Under sharding the per-layer output all-gather is
issued asynchronously and overlaps the next layer's compute.
"""

from __future__ import annotations

import torch

from .pipeline import LayerPolicy, LayerSession, PipelineParams
from .sharding import _world_rank, agree_policies, gather_heads_async, head_block

__all__ = ["StackSession"]


class StackSession:
    """``n_layers`` layers of ``H`` heads (this rank owns heads [h0, h1)).

    plan(step0)   step0[l] = (Q, K) of this rank's heads of layer l, [h, L, D]
                  -> the per-layer modes (identical on every rank)
    step(inputs)  inputs[l] = (Q, K, V) of this rank's heads; the first call
                  is step 0 (reusing the plans), later calls are warm steps.
                  Returns per-layer outputs, all heads [H, L, D] when
                  ``gather`` (sharded), else this rank's heads.
    """

    def __init__(self, n_layers: int, H: int, params: PipelineParams | None = None,
                 seed: int = 0, out_dtype=None, group=None, graph: bool = True):
        self.params = params or PipelineParams()
        self.params.validate()
        self.n_layers, self.H, self.group = n_layers, H, group
        world, rank = _world_rank(group)
        self.world = world
        self.h0, self.h1 = head_block(H, world, rank)
        self.pool: dict = {}
        self.layers = []
        for l in range(n_layers):
            s = LayerSession(self.params, seed=seed, layer=l, out_dtype=out_dtype,
                             head_offset=self.h0, graph=graph)
            s.workspace_pool = self.pool
            self.layers.append(s)
        self.modes = None
        self.mse_layer = None
        self.flagged = None
        self.t = 0

    @property
    def local_heads(self) -> int:
        return self.h1 - self.h0

    def plan(self, step0) -> list:
        """Plan every layer (step 0), then agree on the per-layer policies."""
        if len(step0) != self.n_layers:
            raise ValueError(f"expected {self.n_layers} layers, got {len(step0)}")
        local_mse, local_flags = [], []
        for sess, (Q, K) in zip(self.layers, step0):
            mse, flags = sess.plan(Q, K)
            local_mse.append(mse.cpu().numpy())
            local_flags.append(flags)
        self.modes, self.mse_layer, self.flagged = agree_policies(
            local_mse, local_flags, self.H, self.params.full_layer_quota, self.group)
        for sess, m in zip(self.layers, self.modes):
            sess.set_mode(m)
        return self.modes

    def policies(self) -> list:
        """LayerPolicy per layer (key-cluster counts of this rank's heads)."""
        out = []
        for sess, m in zip(self.layers, self.modes or []):
            kc = [int(c.shape[0]) for c in sess.key_centers] if sess.key_centers else []
            out.append(LayerPolicy(mode=m, key_cluster_count=kc, topk=self.params.topk,
                                   q_clusters=self.params.q_clusters))
        return out

    def step_layer(self, l: int, Q, K, V, gather: bool = True):
        """One layer of the current step; returns a pending all-gather
        (``.wait()`` -> [H, L, D]) when sharded and ``gather``, else the
        local output."""
        out = self.layers[l].step(Q, K, V)
        if gather and self.world > 1:
            return gather_heads_async(out, self.H, self.group)
        return out

    def step(self, inputs, gather: bool = True) -> list:
        if self.modes is None:
            raise RuntimeError("plan() must run before the first step")
        if len(inputs) != self.n_layers:
            raise ValueError(f"expected {self.n_layers} layers, got {len(inputs)}")
        pend = [self.step_layer(l, Q, K, V, gather) for l, (Q, K, V) in enumerate(inputs)]
        self.t += 1
        return [p.wait() if hasattr(p, "wait") else p for p in pend]

    def key_centers(self, l: int) -> list:
        return self.layers[l].key_centers

    def query_centers(self, l: int) -> list:
        return self.layers[l].query_centers
