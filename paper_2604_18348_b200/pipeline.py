"""Cluster-sparse attention pipeline on the device (reference: pipeline.py).

Same public names and semantics as the reference: ``PipelineParams`` (:53),
``LayerPolicy`` (:76), ``StepState`` (:85), ``HeadStats`` (:93),
``count_flops`` (:125), ``adacluster_attention`` (:237), ``DenoiseResult``
(:278) and ``run_denoise_steps`` (:296).

Internally every layer's heads run as one batch: the clustering, selection
and attention kernels take all heads of a layer per launch, so a 30-head
layer costs the same number of launches as one head.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import engine as E
from .clustering import ClusterModel, export_model
from .errors import ContractError, ParameterError
from .profiling import phase
from .quest import SelectionResult
from .tensorops import to_device, to_host

__all__ = ["PipelineParams", "LayerPolicy", "StepState", "HeadStats", "FlopCounts",
           "count_flops", "clustering_flops", "adacluster_attention", "run_denoise_steps",
           "DenoiseResult", "LayerRunner", "LayerSession"]

SCORERS = ("quest", "mean", "clamped")


@dataclass
class PipelineParams:
    q_clusters: int = 65
    topk: int = 64
    tau_factor: float = 1.5
    m0: int = 100
    n_max: int = 1000
    max_iter: int = 25
    tol: float = 1e-4
    scorer: str = "quest"
    full_layer_quota: float = 0.15
    uniform_key_clusters: int | None = None

    def validate(self):
        if self.scorer not in SCORERS:
            raise ParameterError(f"unknown scorer {self.scorer!r}, expected one of {SCORERS}")
        if self.q_clusters < 1 or self.topk < 1 or self.m0 < 1 or self.n_max < self.m0:
            raise ParameterError("q_clusters, topk, m0 must be >= 1 and n_max >= m0")
        if not 0.0 <= self.full_layer_quota <= 1.0:
            raise ParameterError(f"full_layer_quota={self.full_layer_quota} not in [0, 1]")


@dataclass
class LayerPolicy:
    mode: str | None = None
    key_cluster_count: list = field(default_factory=list)
    tau: list = field(default_factory=list)
    topk: int = 64
    q_clusters: int = 65


@dataclass
class StepState:
    """Per-head carry-over between denoising steps (centres stay on device)."""
    step: int = 0
    key_centers: object = None
    query_centers: object = None


@dataclass
class HeadStats:
    mode: str
    num_key_clusters: int
    density: float
    flops_full: float
    flops_sparse: float
    flops_overhead: float
    est_speedup: float
    key_iters: int = 0
    query_iters: int = 0
    selection: object = None
    key_model: ClusterModel | None = None
    q_model: ClusterModel | None = None


@dataclass
class FlopCounts:
    flops_full: float
    flops_sparse: float
    flops_overhead: float

    @property
    def est_speedup(self) -> float:
        return self.flops_full / (self.flops_sparse + self.flops_overhead)


def clustering_flops(n: int, c: int, d: int, iters: int) -> float:
    """Assignment cost 2·N·C·D per Lloyd iteration (pipeline.py:120-122)."""
    return 2.0 * n * c * d * iters


def count_flops(L_: int, D: int, C: int, Gq: int, density: float, kmeans_iters: int,
                mode: str) -> FlopCounts:
    """(full, sparse, overhead) FLOPs of one head (pipeline.py:125-141)."""
    if L_ < 1 or D < 1 or C < 1 or Gq < 1:
        raise ParameterError("count_flops requires positive sizes")
    full = 4.0 * L_ * L_ * D
    if mode == "full":
        return FlopCounts(full, full, clustering_flops(L_, C, D, kmeans_iters))
    sparse = 4.0 * L_ * (density * L_) * D
    over = clustering_flops(L_, C, D, kmeans_iters) + L_ * D + 4.0 * Gq * C * D
    return FlopCounts(full, sparse, over)


# ---------------------------------------------------------------------------
# batched per-layer engine
# ---------------------------------------------------------------------------
@dataclass
class LayerPlan:
    q_models: list
    reps: list
    key_models: list
    taus: list


@dataclass
class SparseOut:
    out: torch.Tensor           # [H, L, D]
    selections: list            # DevSelection per head
    topks: list


class LayerRunner:
    """All heads of one layer on the device: step-0 planning, warm steps,
    selection and block-sparse attention.  Heads are independent
    (SPEC.md:242); batching only amortises launches."""

    def __init__(self, params: PipelineParams, out_dtype=torch.float32, attn_impl: str = "auto",
                 inertia: bool = True):
        self.p = params
        self.out_dtype = out_dtype
        self.attn_impl = attn_impl
        # inertia_history is only exported by the model-returning API
        # (adacluster_attention, run_denoise_steps); the streaming sessions
        # skip it in the WARM Lloyd passes (labels-only assignment).  Cold
        # k-means keeps it: starting from k-means++ seeds, empty clusters are
        # common and their repair needs the exact distances of every row,
        # which the labels-only path recomputes in one CTA per problem
        # (measured: C2 step 0 99 -> 145 ms when cold passes skipped it)
        self.inertia = inertia
        # the cold query k-means (65 centres, k-means++ seeds) with the
        # labels-only assignment when inertia is not exported; AC_COLD_Q_INERTIA=1 A/B
        import os
        self.cold_q_inertia = inertia or os.environ.get("AC_COLD_Q_INERTIA") == "1"

    def plan(self, Q: torch.Tensor, K: torch.Tensor, seeds: list[int]) -> LayerPlan:
        """_plan_head (pipeline.py:168-185) for every head."""
        p = self.p
        H, Ln, _ = Q.shape
        qs = [Q[h] for h in range(H)]
        ks = [K[h] for h in range(H)]
        # the query clustering (no host decisions) is enqueued sync-free on a
        # side stream and overlaps the key side, whose multi-stage rounds
        # read results on the host (C2 step 0: 22 + 26 ms -> concurrent)
        # The key side (the critical path: its multi-stage rounds read
        # results on the host) runs on a high-priority stream so that the
        # concurrent query chain only fills the SMs it leaves idle.
        main = torch.cuda.current_stream()
        side, hi = _side_stream(), _side_stream(high=True)
        side.wait_stream(main)
        hi.wait_stream(main)
        stops: list = []
        kstops: list = []
        kc = min(p.uniform_key_clusters if p.uniform_key_clusters is not None else p.m0, Ln)
        # keys first (sync-free k-means: stop flags read later), then the
        # query chain is enqueued while the key kernels already run
        with phase("plan_stage0"), torch.cuda.stream(hi):
            s0 = E.kmeans_batch(ks, [kc] * H, seeds, p.max_iter, p.tol, stops_out=kstops)
        with phase("plan_queries"), torch.cuda.stream(side):
            qm, reps, _ = E.cluster_queries_batch(qs, [min(p.q_clusters, Ln)] * H, seeds,
                                                  p.max_iter, p.tol, inertia=self.cold_q_inertia,
                                                  stops_out=stops)
        with torch.cuda.stream(hi):
            if any(bool((t >= 0).any()) for t in kstops):  # rare k-means++ stop: host replay
                s0 = E.kmeans_batch(ks, [kc] * H, seeds, p.max_iter, p.tol)
            if p.uniform_key_clusters is not None:
                km = s0
                taus = [None] * H
            else:
                with phase("plan_tau"):
                    taus = [float(t) for t in E.tau_batch(ks, s0, p.tau_factor).cpu().numpy()]
                with phase("plan_multistage"):
                    km = E.multi_stage_batch(ks, taus, p.n_max, kc, seeds, p.max_iter, p.tol, s0)
        main.wait_stream(side)
        main.wait_stream(hi)
        _adopt(main, qm, reps)
        _adopt(main, km, [])
        if any(bool((t >= 0).any()) for t in stops):  # rare k-means++ stop: redo with host replay
            qm, reps, _ = E.cluster_queries_batch(qs, [min(p.q_clusters, Ln)] * H, seeds,
                                                  p.max_iter, p.tol)
        return LayerPlan(qm, reps, km, taus)

    def warm(self, Q: torch.Tensor, K: torch.Tensor, key_centers: list, query_centers: list):
        """Warm-started clusterings of a later step (pipeline.py:263-267)."""
        p = self.p
        H = Q.shape[0]
        with phase("warm_keys"):
            km = E.lloyd_batch([K[h] for h in range(H)], key_centers, p.max_iter, p.tol,
                               self.inertia)
        with phase("warm_queries"):
            qm, reps, _ = E.cluster_queries_batch([Q[h] for h in range(H)], [0] * H, [0] * H,
                                                  p.max_iter, p.tol, inits=query_centers,
                                                  inertia=self.inertia)
        return qm, reps, km

    def sparse(self, Q, K, V, q_models, reps, key_models, topk: int) -> SparseOut:
        """_sparse_head (pipeline.py:188-195) for every head."""
        p = self.p
        H = Q.shape[0]
        ks = [K[h] for h in range(H)]
        with phase("select"):
            if p.scorer == "quest":
                emax, emin = E.envelopes_batch(ks, key_models)
            else:
                emax = emin = [m.centers for m in key_models]
            topks = [min(topk, m.k) for m in key_models]
            sels, runs, nruns = E.select_batch(reps, emax, emin, key_models, topks, p.scorer)
        out = E.sparse_attention_heads(Q, K, V, q_models, key_models, runs, nruns,
                                       self.out_dtype, self.attn_impl)
        return SparseOut(out, sels, topks)

    def dense(self, Q, K, V) -> torch.Tensor:
        return E.dense_attention_heads(Q, K, V, self.out_dtype, self.attn_impl)

    def consolidate(self, K, key_models) -> list:
        """_carry_centers at step 0 (pipeline.py:223-234): one warm Lloyd."""
        p = self.p
        H = K.shape[0]
        with phase("consolidate"):
            return E.lloyd_batch([K[h] for h in range(H)], [m.centers for m in key_models],
                                 p.max_iter, p.tol, self.inertia)


_SIDE: dict = {}


def _side_stream(high: bool = False) -> torch.cuda.Stream:
    key = (torch.cuda.current_device(), high)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=key[0], priority=-1 if high else 0)
    return _SIDE[key]


def _adopt(stream, models, reps) -> None:
    """Tensors made on the side stream and used on ``stream`` from now on:
    keep the caching allocator from reusing them before ``stream`` is done."""
    for m in models:
        for t in (m.centers, m.labels, m.counts, m.perm, m.starts, m.status, m.inertia):
            t.record_stream(stream)
    for r in reps:
        r.record_stream(stream)


def _stack(heads, keep_bf16=True):
    ts = [to_device(x, keep_bf16)[0] for x in heads]
    dt = torch.bfloat16 if all(t.dtype == torch.bfloat16 for t in ts) else torch.float32
    return torch.stack([t.to(dt) for t in ts]).contiguous()


def _is_host(x) -> bool:
    return not (isinstance(x, torch.Tensor) and x.device.type == "cuda")


def _selection(sel: E.DevSelection, host: bool) -> SelectionResult:
    return SelectionResult(scores=to_host(sel.scores, host), selected=to_host(sel.selected, host),
                           density=float(sel.density.item()))


def _head_stats(mode: str, Ln: int, D: int, key_model: ClusterModel | None,
                q_model: ClusterModel | None, sel: SelectionResult | None) -> HeadStats:
    c = key_model.num_clusters if key_model is not None else 1
    iters = (key_model.n_iter if key_model is not None else 0) + (
        q_model.n_iter if q_model is not None else 0)
    density = sel.density if sel is not None else 1.0
    gq = q_model.num_clusters if q_model is not None else 1
    fc = count_flops(Ln, D, c, gq, density, iters, mode)
    return HeadStats(mode=mode, num_key_clusters=c, density=density, flops_full=fc.flops_full,
                     flops_sparse=fc.flops_sparse, flops_overhead=fc.flops_overhead,
                     est_speedup=fc.est_speedup,
                     key_iters=key_model.n_iter if key_model is not None else 0,
                     query_iters=q_model.n_iter if q_model is not None else 0, selection=sel,
                     key_model=key_model, q_model=q_model)


def adacluster_attention(q, k, v, policy: LayerPolicy, state: StepState, seed: int,
                         params: PipelineParams | None = None):
    """One head of the pipeline for one denoising step (pipeline.py:237-275).
    Mutates ``policy`` and ``state`` like the reference."""
    params = params or PipelineParams()
    host = _is_host(q)
    Q, K, V = _stack([q]), _stack([k]), _stack([v])
    Ln, D = int(Q.shape[1]), int(Q.shape[2])
    run = LayerRunner(params)
    if policy.mode == "full":
        state.step += 1
        out = run.dense(Q, K, V)[0]
        return to_host(out, host), _head_stats("full", Ln, D, None, None, None)
    if state.step == 0 or state.key_centers is None:
        plan = run.plan(Q, K, [int(seed)])
        km_dev, qm_dev, reps = plan.key_models[0], plan.q_models[0], plan.reps
        if km_dev.flag_full:
            policy.mode = "full"
            state.step += 1
            km = export_model(km_dev, host, with_inertia=False)
            qm = export_model(qm_dev, host)
            out = run.dense(Q, K, V)[0]
            return to_host(out, host), _head_stats("full", Ln, D, km, qm, None)
        policy.mode = "sparse"
        policy.key_cluster_count = [km_dev.k]
        policy.tau = [plan.taus[0]]
        policy.topk = params.topk
        policy.q_clusters = params.q_clusters
        key_models, q_models = [km_dev], [qm_dev]
    else:
        kc = to_device(state.key_centers, keep_bf16=False)[0]
        qc = to_device(state.query_centers, keep_bf16=False)[0]
        q_models, reps, key_models = run.warm(Q, K, [kc], [qc])
    so = run.sparse(Q, K, V, q_models, reps, key_models, policy.topk)
    km = export_model(key_models[0], host, with_inertia=key_models[0].host_iters is None)
    qm = export_model(q_models[0], host)
    sel = _selection(so.selections[0], host)
    stats = _head_stats("sparse", Ln, D, km, qm, sel)
    if state.step == 0:
        cons = run.consolidate(K, key_models)[0]
        state.key_centers = to_host(cons.centers.clone(), host)
        stats.key_iters += cons.n_iter()
    else:
        state.key_centers = to_host(key_models[0].centers.clone(), host)
    state.query_centers = to_host(q_models[0].centers.clone(), host)
    state.step += 1
    return to_host(so.out[0], host), stats


@dataclass
class DenoiseResult:
    outputs: list          # [step][layer][head] -> [L, D]
    policies: list         # [layer] -> LayerPolicy
    stats: list            # [step][layer][head] -> HeadStats
    mse_layer: list        # [layer] step-0 mean-over-heads key clustering MSE


def _check_shapes(step_inputs):
    if not step_inputs or not step_inputs[0]:
        raise ParameterError("run_denoise_steps needs at least one step and one layer")
    ref = [[(tuple(q.shape), tuple(k.shape), tuple(v.shape)) for q, k, v in layer]
           for layer in step_inputs[0]]
    for t, layers in enumerate(step_inputs):
        got = [[(tuple(q.shape), tuple(k.shape), tuple(v.shape)) for q, k, v in layer]
               for layer in layers]
        if got != ref:
            raise ContractError(f"per-layer shapes at step {t} differ from step 0")


def run_denoise_steps(step_inputs, params: PipelineParams | None = None, seed: int = 0,
                      collect_stats: bool = True):
    """Multi-layer, multi-step driver (pipeline.py:296-386).  Step 0 plans
    every layer and applies the per-layer policy (flagged heads, worst
    ``full_layer_quota`` fraction by MSE); later steps warm-start."""
    params = params or PipelineParams()
    params.validate()
    _check_shapes(step_inputs)
    n_layers = len(step_inputs[0])
    host = _is_host(step_inputs[0][0][0][0])
    run = LayerRunner(params)

    plans, mse_layer, flagged = [], [], []
    for l, layer in enumerate(step_inputs[0]):
        Q = _stack([h[0] for h in layer])
        K = _stack([h[1] for h in layer])
        H = Q.shape[0]
        plan = run.plan(Q, K, [seed + 7919 * l + h for h in range(H)])
        plans.append(plan)
        mses = E.mse_batch([K[h] for h in range(H)], plan.key_models).cpu().numpy()
        mse_layer.append(float(np.mean([float(m) for m in mses])))
        flagged.append(any(m.flag_full for m in plan.key_models))

    from .sharding import decide_policies
    modes = decide_policies(mse_layer, flagged, params.full_layer_quota)
    policies = []
    for l in range(n_layers):
        policies.append(LayerPolicy(mode=modes[l],
                                    key_cluster_count=[m.k for m in plans[l].key_models],
                                    tau=list(plans[l].taus), topk=params.topk,
                                    q_clusters=params.q_clusters))

    key_c: list[list | None] = [None] * n_layers
    qry_c: list[list | None] = [None] * n_layers
    outputs, stats = [], []
    for t, layers in enumerate(step_inputs):
        s_out, s_stats = [], []
        for l, layer in enumerate(layers):
            Q = _stack([h[0] for h in layer])
            K = _stack([h[1] for h in layer])
            V = _stack([h[2] for h in layer])
            H, Ln, D = (int(x) for x in Q.shape)
            pol = policies[l]
            if pol.mode == "full":
                out = run.dense(Q, K, V)
                hs = []
                for h in range(H):
                    if not collect_stats:
                        hs.append(None)
                    elif t == 0:
                        km = export_model(plans[l].key_models[h], host, with_inertia=False)
                        qm = export_model(plans[l].q_models[h], host)
                        hs.append(_head_stats("full", Ln, D, km, qm, None))
                    else:
                        hs.append(_head_stats("full", Ln, D, None, None, None))
            else:
                if t == 0:
                    qms, reps, kms = plans[l].q_models, plans[l].reps, plans[l].key_models
                else:
                    qms, reps, kms = run.warm(Q, K, key_c[l], qry_c[l])
                so = run.sparse(Q, K, V, qms, reps, kms, pol.topk)
                out = so.out
                extra = [0] * H
                if t == 0:
                    cons = run.consolidate(K, kms)
                    key_c[l] = [m.centers for m in cons]
                    if collect_stats:
                        extra = [m.n_iter() for m in cons]
                else:
                    key_c[l] = [m.centers for m in kms]
                qry_c[l] = [m.centers for m in qms]
                hs = []
                for h in range(H):
                    if not collect_stats:
                        hs.append(None)
                        continue
                    km = export_model(kms[h], host, with_inertia=kms[h].host_iters is None)
                    qm = export_model(qms[h], host)
                    st = _head_stats("sparse", Ln, D, km, qm, _selection(so.selections[h], host))
                    st.key_iters += extra[h]
                    hs.append(st)
            s_out.append([to_host(out[h], host) for h in range(H)])
            s_stats.append(hs)
        outputs.append(s_out)
        stats.append(s_stats)
    return DenoiseResult(outputs=outputs, policies=policies, stats=stats, mse_layer=mse_layer)


class LayerSession:
    """Stateful driver of one layer across denoising steps (the streamed form
    of ``run_denoise_steps`` for a single layer).  ``step(Q, K, V)`` takes
    [H, L, D] tensors (CUDA, or host/pinned — then the copies are part of the
    call) and returns [H, L, D] outputs (on the inputs' side).  Step 0 plans
    every head and fixes the layer policy (any flagged head -> full, as the
    reference's per-layer rule with quota 0); later steps warm-start."""

    def __init__(self, params: PipelineParams | None = None, seed: int = 0, layer: int = 0,
                 out_dtype=None, attn_impl: str = "auto", head_offset: int = 0,
                 reduce_flag=None, graph: bool = True):
        self.reduce_flag = reduce_flag or (lambda local: local)
        self.params = params or PipelineParams()
        self.params.validate()
        self.seed, self.layer, self.head_offset = seed, layer, head_offset
        self.out_dtype = out_dtype
        self.attn_impl = attn_impl
        self.t = 0
        self.mode = None
        self._key_centers = None
        self._query_centers = None
        self.last = None
        self.graph = graph
        self.steady = None  # SteadyStep (CUDA graph) once the warm step is fixed
        self._plan = None   # step-0 plan made by plan() ahead of step 0
        self.workspace_pool = None  # dict shared by the layers of a StackSession

    # carried state (pipeline.py:85-90); lives in the steady step's batches
    @property
    def key_centers(self):
        return self.steady.key_centers() if self.steady is not None else self._key_centers

    @key_centers.setter
    def key_centers(self, v):
        self._key_centers = v

    @property
    def query_centers(self):
        return self.steady.query_centers() if self.steady is not None else self._query_centers

    @query_centers.setter
    def query_centers(self, v):
        self._query_centers = v

    def useful_attention_flops(self) -> float:
        """4·D·Σ_heads Σ_g |Q_g|·|S_g| of the last sparse step (no tile padding)."""
        if self.steady is not None:
            return float(self.steady.useful_attention_flops().item())
        if self.last is None:
            return 0.0
        qm, _, so = self.last
        D = so.out.shape[-1]
        tot = sum(float((m.counts.double() * sel._covered.double()).sum().item())
                  for m, sel in zip(qm, so.selections))
        return tot * 4.0 * D

    def density(self) -> float:
        if self.steady is not None:
            return float(self.steady.density[0].item())
        if self.last is None:
            return float("nan")
        return float(self.last[2].selections[0].density.item())

    def _seeds(self, H: int) -> list:
        return [self.seed + 7919 * self.layer + self.head_offset + h for h in range(H)]

    def plan(self, Q, K):
        """Step-0 planning of this layer's heads without attention
        (run_denoise_steps' planning pass, pipeline.py:310-324): returns the
        per-head key-clustering MSE (f64, device) and flag_full list.  The
        caller then fixes the layer policy (``set_mode``) -- across layers for
        the quota, across ranks for sharded heads -- and step 0 reuses the plan."""
        if self.t != 0:
            raise ContractError("plan() is the step-0 planning pass")
        dev = L.device()
        Q, K = (x if (isinstance(x, torch.Tensor) and x.device.type == "cuda")
                else torch.as_tensor(x).to(dev) for x in (Q, K))
        H = int(Q.shape[0])
        if H == 0:
            self._plan = "empty"
            return torch.zeros(0, dtype=torch.float64, device=dev), []
        run = LayerRunner(self.params, None, self.attn_impl, inertia=False)
        plan = run.plan(Q, K, self._seeds(H))
        self._plan = plan
        mse = E.mse_batch([K[h] for h in range(H)], plan.key_models)
        return mse, [bool(m.flag_full) for m in plan.key_models]

    def set_mode(self, mode: str):
        """Fix the layer policy decided from plan() (``full`` or ``sparse``)."""
        if mode not in ("full", "sparse"):
            raise ParameterError(f"mode must be 'full' or 'sparse', got {mode!r}")
        self.mode = mode

    def step(self, Q, K, V, host_out=None, async_out: bool = False):
        """One denoising step of the layer.  With host (pinned) inputs the
        result is written to ``host_out`` (a pinned host tensor of the output
        shape, e.g. preallocated by a serving loop) or to a fresh pinned
        tensor, and is ready when the call returns (like the reference's
        numpy result); ``async_out=True`` returns as soon as the device->host
        copy is enqueued on the current stream (synchronise before reading)."""
        host = not (isinstance(Q, torch.Tensor) and Q.device.type == "cuda")
        dev = L.device()
        if host:
            st = self.steady
            Q, K, V = (torch.as_tensor(x) for x in (Q, K, V))
            if (st is not None and st.Q.shape == Q.shape and st.dtype == Q.dtype
                    and host_out is not None and all(x.is_pinned() for x in (Q, K, V, host_out))):
                # steady state from pinned buffers: copies inside the graph
                self.t += 1
                res = st.step_host(Q, K, V, host_out)
                if not async_out:
                    torch.cuda.current_stream().synchronize()
                return res
            Q, K, V = (x.to(dev, non_blocking=True) for x in (Q, K, V))
        odt = self.out_dtype or (torch.bfloat16 if Q.dtype == torch.bfloat16 else torch.float32)
        run = LayerRunner(self.params, odt, self.attn_impl, inertia=False)
        H = Q.shape[0]
        if H == 0:  # a rank without heads of this layer (head sharding)
            if self.t == 0 and self._plan is None:
                self.mode = "full" if self.reduce_flag(False) else "sparse"
            self.t += 1
            return torch.empty(tuple(Q.shape), dtype=odt, device=Q.device)
        if self.t == 0:
            if self._plan is not None:  # planned ahead; policy fixed by set_mode
                plan = self._plan
                self._plan = None
                if self.mode is None:
                    raise ContractError("plan() was called but set_mode() was not")
            else:
                plan = run.plan(Q, K, self._seeds(H))
                flagged = self.reduce_flag(any(m.flag_full for m in plan.key_models))
                self.mode = "full" if flagged else "sparse"
            if self.mode == "sparse":
                so = run.sparse(Q, K, V, plan.q_models, plan.reps, plan.key_models,
                                self.params.topk)
                cons = run.consolidate(K, plan.key_models)
                self.key_centers = [m.centers for m in cons]
                self.query_centers = [m.centers for m in plan.q_models]
                self.last = (plan.q_models, plan.key_models, so)
                out = so.out
            else:
                with phase("attention_dense"):
                    out = run.dense(Q, K, V)
        elif self.mode == "full":
            with phase("attention_dense"):
                out = run.dense(Q, K, V)
        elif (self.graph and self.attn_impl == "auto" and self.params.scorer == "quest"
              and int(Q.shape[2]) in E.ATTN_DIMS):
            from .steady import SteadyStep
            if self.steady is None or self.steady.Q.shape != Q.shape or self.steady.dtype != Q.dtype:
                from .steady import Workspace
                kc, qc = self.key_centers, self.query_centers
                self.steady = None
                ws = None
                if self.workspace_pool is not None:
                    key = (H, int(Q.shape[1]), int(Q.shape[2]), Q.dtype, int(qc[0].shape[0]), odt)
                    ws = self.workspace_pool.get(key)
                    if ws is None:
                        ws = self.workspace_pool[key] = Workspace(*key)
                self.steady = SteadyStep(H, Q.shape[1], Q.shape[2], Q.dtype, self.params, kc, qc,
                                         odt, workspace=ws)
                self.last = None
            with phase("steady_step"):
                out = self.steady.step(Q, K, V)
            if not host:
                out = out.clone()  # the graph's output buffer is reused next step
        else:
            qm, reps, km = run.warm(Q, K, self.key_centers, self.query_centers)
            so = run.sparse(Q, K, V, qm, reps, km, self.params.topk)
            self.key_centers = [m.centers for m in km]
            self.query_centers = [m.centers for m in qm]
            self.last = (qm, km, so)
            out = so.out
        self.t += 1
        if host:
            res = host_out if host_out is not None else torch.empty(out.shape, dtype=out.dtype,
                                                                     pin_memory=True)
            res.copy_(out, non_blocking=True)
            if not async_out:
                torch.cuda.current_stream().synchronize()
            return res
        return out
