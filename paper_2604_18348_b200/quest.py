"""Critical-cluster selection on the device (reference: quest.py).

``build_envelopes`` (:61), ``tensor_quest`` (:94),
``tensor_quest_clamped_centers`` (:106), ``mean_center_scores`` (:119) and
``select_topk_clusters`` (:128) with the reference's signatures; scores and
selections are bit-identical (OpenBLAS accumulation order reproduced).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import engine as E
from .clustering import ClusterModel, import_model
from .errors import DimensionError, ParameterError
from .tensorops import to_device, to_host

__all__ = ["ClusterEnvelope", "SelectionResult", "build_envelopes", "quest_scalar",
           "quest_scores_loop", "tensor_quest", "tensor_quest_clamped_centers",
           "mean_center_scores", "select_topk_clusters", "select_topp_clusters"]

DEFAULT_TOPK = 64


@dataclass
class ClusterEnvelope:
    max_vec: object                   # [C, D] elementwise max of member keys
    min_vec: object                   # [C, D] elementwise min
    member_order: object | None = None   # token indices grouped by cluster (stable)
    member_starts: object | None = None  # group start offsets into member_order

    @property
    def num_clusters(self) -> int:
        return int(self.max_vec.shape[0])

    def members(self, c: int):
        starts = self.member_starts
        lo = starts[c]
        hi = starts[c + 1] if c + 1 < len(starts) else len(self.member_order)
        return self.member_order[lo:hi]


@dataclass
class SelectionResult:
    scores: object     # [Gq, C]
    selected: object   # [Gq, topk] cluster indices, descending score
    density: float     # mean selected key tokens / total key tokens


def _sorted_model(k: torch.Tensor, model: ClusterModel) -> E.DevModel:
    """Device model with member order / starts for the given labels."""
    dm = import_model(model, int(k.shape[0]))
    b = E.Batch([k], [dm.k], 1)
    b.centers_of(0).copy_(dm.centers)
    n = dm.n
    b.labels[:n].copy_(dm.labels)
    L.call("ac_sort_by_label", b.dev.data_ptr(), 1, b.max_n, b.max_k, L.stream_ptr())
    return b.model(0)


def build_envelopes(k, model: ClusterModel) -> ClusterEnvelope:
    """Per-cluster elementwise max/min over member keys (quest.py:61-71)."""
    t, host = to_device(k)
    m = _sorted_model(t, model)
    emax, emin = E.envelopes_batch([t], [m])
    order = m.perm.to(torch.int64)
    starts = m.starts[:-1].to(torch.int64)
    return ClusterEnvelope(to_host(emax[0], host), to_host(emin[0], host), to_host(order, host),
                           to_host(starts, host))


def _scores(q_reps, a, b, scorer: str):
    q, host = to_device(q_reps, keep_bf16=False)
    ta, _ = to_device(a, keep_bf16=False)
    tb, _ = to_device(b, keep_bf16=False)
    if q.shape[1] != ta.shape[1]:
        raise DimensionError(f"query dim {q.shape[1]} != envelope dim {ta.shape[1]}")
    C = int(ta.shape[0])
    dev = L.device()
    dummy = E.DevModel(centers=ta, labels=None, counts=torch.ones(C, dtype=torch.int32, device=dev),
                       perm=None, starts=torch.arange(C + 1, dtype=torch.int32, device=dev),
                       status=None, inertia=None, k=C, n=C)
    sels, _, _ = E.select_batch([q.contiguous()], [ta.contiguous()], [tb.contiguous()], [dummy], [1],
                                scorer)
    return to_host(sels[0].scores, host)


def _quest_pairs(q_reps, env: ClusterEnvelope, clusters=None):
    q, host = to_device(q_reps, keep_bf16=False)
    mx, _ = to_device(env.max_vec, keep_bf16=False)
    mn, _ = to_device(env.min_vec, keep_bf16=False)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    if q.shape[1] != mx.shape[1]:
        raise DimensionError(f"query dim {q.shape[1]} != envelope dim {mx.shape[1]}")
    if clusters is not None:
        mx, mn = mx[clusters:clusters + 1], mn[clusters:clusters + 1]
    q, mx, mn = q.contiguous(), mx.contiguous(), mn.contiguous()
    out = torch.empty((q.shape[0], mx.shape[0]), dtype=torch.float32, device=q.device)
    L.call("ac_quest_pairs", q.data_ptr(), int(q.shape[0]), int(q.shape[1]), mx.data_ptr(),
           mn.data_ptr(), int(mx.shape[0]), out.data_ptr(), L.stream_ptr())
    return out, host


def quest_scalar(q_row, env: ClusterEnvelope, c: int) -> float:
    """Upper bound on q·k over the members of cluster ``c`` in the scalar
    form sum_t max(q_t·max_ct, q_t·min_ct) (quest.py:74-77), on the device."""
    q, _ = to_device(q_row, keep_bf16=False)
    out, _ = _quest_pairs(q.reshape(1, -1), env, clusters=int(c))
    return float(out[0, 0].item())


def quest_scores_loop(q_reps, env: ClusterEnvelope):
    """Scalar-form scores of every (query rep, cluster) pair (quest.py:80-91):
    the same per-pair bound as ``quest_scalar``, one device thread per pair."""
    out, host = _quest_pairs(q_reps, env)
    return to_host(out, host)


def tensor_quest(q_reps, env: ClusterEnvelope):
    """max(Q,0) max_vecᵀ + min(Q,0) min_vecᵀ (quest.py:94-103)."""
    return _scores(q_reps, env.max_vec, env.min_vec, "quest")


def tensor_quest_clamped_centers(q_reps, centers):
    """Ablation scorer on clamped centres (quest.py:106-116)."""
    return _scores(q_reps, centers, centers, "clamped")


def mean_center_scores(q_reps, centers):
    """Plain Q_reps centersᵀ (quest.py:119-125)."""
    return _scores(q_reps, centers, centers, "mean")


def select_topk_clusters(scores, topk: int, counts) -> SelectionResult:
    """Top ``topk`` clusters per query cluster, ties to the lower index
    (quest.py:128-143)."""
    s, host = to_device(scores, keep_bf16=False)
    gq, C = int(s.shape[0]), int(s.shape[1])
    if not 1 <= topk <= C:
        raise ParameterError(f"topk={topk} out of range [1, {C}]")
    dev = L.device()
    cnt = torch.as_tensor(np.asarray(counts) if not isinstance(counts, torch.Tensor) else counts)
    cnt = cnt.to(dev, torch.int32).contiguous()
    starts = torch.zeros(C + 1, dtype=torch.int32, device=dev)
    starts[1:] = torch.cumsum(cnt, 0)
    dummy = E.DevModel(centers=None, labels=None, counts=cnt, perm=None, starts=starts,
                       status=None, inertia=None, k=C, n=int(starts[-1].item()))
    z = torch.zeros((1, 1), dtype=torch.float32, device=dev)
    sels, _, _ = E.select_batch([torch.zeros((gq, 1), dtype=torch.float32, device=dev)], [z], [z],
                                [dummy], [int(topk)], "given", scores_in=[s.contiguous()])
    sel = sels[0]
    return SelectionResult(scores=to_host(s, host), selected=to_host(sel.selected, host),
                           density=float(sel.density.item()))


def select_topp_clusters(scores, top_p: float, counts, mass_scale: float = 1.0,
                         max_clusters: int | None = None) -> SelectionResult:
    """Top-p critical-cluster selection (an extension; the reference selects
    top-k only, quest.py:128-143): per query cluster, the smallest prefix of
    the stable descending score order whose estimated attention mass
    ``counts[c] * exp((scores[c] - max scores) * mass_scale)`` reaches
    ``top_p`` of the row's total -- at least one cluster, at most
    ``max_clusters`` (default: all).  ``selected`` rows are padded with -1
    past the chosen count; density counts the chosen clusters' tokens.
    Scores are typically TensorQuest bounds and ``mass_scale`` 1/sqrt(D)."""
    s, host = to_device(scores, keep_bf16=False)
    gq, C = int(s.shape[0]), int(s.shape[1])
    if not 0.0 < top_p <= 1.0:
        raise ParameterError(f"top_p={top_p} not in (0, 1]")
    cap = C if max_clusters is None else int(max_clusters)
    if not 1 <= cap <= C:
        raise ParameterError(f"max_clusters={cap} out of range [1, {C}]")
    dev = L.device()
    cnt = torch.as_tensor(np.asarray(counts) if not isinstance(counts, torch.Tensor) else counts)
    cnt = cnt.to(dev, torch.int32).contiguous()
    starts = torch.zeros(C + 1, dtype=torch.int32, device=dev)
    starts[1:] = torch.cumsum(cnt, 0)
    dummy = E.DevModel(centers=None, labels=None, counts=cnt, perm=None, starts=starts,
                       status=None, inertia=None, k=C, n=int(starts[-1].item()))
    z = torch.zeros((1, 1), dtype=torch.float32, device=dev)
    sels, _, _ = E.select_batch([torch.zeros((gq, 1), dtype=torch.float32, device=dev)], [z], [z],
                                [dummy], [cap], "given", scores_in=[s.contiguous()],
                                top_p=float(top_p), mass_scale=float(mass_scale))
    sel = sels[0]
    return SelectionResult(scores=to_host(s, host), selected=to_host(sel.selected, host),
                           density=float(sel.density.item()))
