"""Device-side orchestration of the AdaCluster hot path.

Everything here drives ``libadacluster_sm100.so`` through the C-ABI on the
current torch CUDA stream.  A *batch* is a set of independent clustering
problems (the heads of a layer, or one multi-stage round of several heads)
laid out in a few flat device buffers with one descriptor per problem
(``ac_cluster_problem``).  Control flow that the reference decides on data
(Lloyd convergence, empty-cluster repair) stays on the device; the host only
synchronises where the reference's control flow needs a size it cannot
bound (multi-stage round sizes, k-means++ ``total <= 0`` replays) or when a
caller asks for host results.

Reference call sites: clustering.py:78-320, quest.py:61-143,
pipeline.py:154-275.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .errors import DimensionError, ParameterError
from .profiling import phase

F32 = torch.float32
I32 = torch.int32
TILE = 128


def _draws(seed: int, n: int, k: int, forced_from: int | None = None) -> np.ndarray:
    """k-means++ random stream of clustering.py:78-91 (numpy PCG64 default_rng):
    ``rng.integers(n)`` then one ``rng.random()`` per step; steps from
    ``forced_from`` on take ``rng.integers(n)`` (the ``total <= 0`` branch),
    encoded as -(idx + 1)."""
    rng = np.random.default_rng(seed)
    out = np.empty(max(k, 1), np.float64)
    out[0] = float(rng.integers(n))
    if forced_from is None:
        if k > 1:
            out[1:k] = rng.random(k - 1)  # the same stream as k - 1 scalar draws
        return out
    for s in range(1, k):
        if s >= forced_from:
            out[s] = -(float(rng.integers(n)) + 1.0)
        else:
            out[s] = rng.random()
    return out


@dataclass
class DevModel:
    """Device-resident clustering result of one problem (views into a batch)."""
    centers: torch.Tensor     # [k, D] f32
    labels: torch.Tensor      # [n] int32
    counts: torch.Tensor      # [k] int32
    perm: torch.Tensor        # [n] int32 member order (stable argsort of labels)
    starts: torch.Tensor      # [k+1] int32
    status: torch.Tensor      # [8] int32
    inertia: torch.Tensor     # [max_iter] f32
    k: int
    n: int
    # multi-stage bookkeeping (host-known)
    flag_full: bool = False
    stage_count: int = 1
    stage_mse: list = field(default_factory=list)
    tau: float | None = None
    host_iters: int | None = None   # when set, n_iter is host-known (multi-stage)

    def n_iter(self) -> int:
        if self.host_iters is not None:
            return self.host_iters
        return int(self.status[L.ST_NITER].item())


class Batch:
    """Flat device buffers + descriptor table for a batch of problems that
    share D, dtype and the reference's GEMM accumulation order."""

    def __init__(self, xs: list[torch.Tensor], ks: list[int], max_iter: int,
                 kcaps: list[int] | None = None, planes: torch.Tensor | None = None):
        if not xs:
            raise ParameterError("empty batch")
        dev = L.device()
        self.xs = xs
        self.D = int(xs[0].shape[1])
        self.dtype = L.dtype_code(xs[0])
        self.P = len(xs)
        self.ns = [int(x.shape[0]) for x in xs]
        self.ks = [int(k) for k in ks]
        self.kcaps = [int(c) for c in (kcaps or ks)]
        self.max_iter = max(int(max_iter), 1)
        self.orders = [L.gemm_order(n, k, self.D) for n, k in zip(self.ns, self.ks)]
        # the general (OpenBLAS sgemm) order has its own kernels; the small-
        # shape orders share k_assign_generic, which reads each problem's order
        if len({o == L.ORDER_SEQ for o in self.orders}) != 1:
            raise ParameterError("batch mixes the general GEMM order with small-shape orders")
        N, K, D, P = sum(self.ns), sum(self.kcaps), self.D, self.P
        tiles = [(n + TILE - 1) // TILE for n in self.ns]
        # buffer sizes from the C-ABI's workspace query (ac_workspace_bytes),
        # summed over the problems: the header is the single source of truth
        ws = batch_buffer_bytes(self.ns, self.kcaps, D, self.dtype, self.max_iter)

        def buf(name, dtype, fill=None):
            n = ws[name] // torch.empty((), dtype=dtype).element_size()
            if n == 0:
                return None
            if fill is None:
                return torch.empty(n, dtype=dtype, device=dev)
            return torch.full((n,), fill, dtype=dtype, device=dev)

        self.xx = buf("xx", F32)
        self.labels = buf("labels", I32)
        self.best = buf("best", F32)
        self.perm = buf("perm", I32)
        self.dscratch = buf("dscratch", torch.float64)
        self.centers = buf("centers", F32)
        self.cc = buf("cc", F32)
        self.counts = buf("counts", I32)
        self.starts = buf("starts", I32)
        self.movement = buf("movement", F32)
        self.tile_hist = buf("tile_hist", I32) if ws["tile_hist"] else torch.empty(
            1, dtype=I32, device=dev)
        self.inertia = buf("inertia", F32, 0.0)
        # f32 points: exact bf16 hi/mid/lo planes for the tensor-core assign
        # (written by ac_lloyd_prepare), [3][n][D] per problem
        if planes is not None and ws["planes"]:  # caller-provided (shared workspace)
            if planes.numel() * planes.element_size() < ws["planes"]:
                raise ParameterError("planes workspace too small")
            self.planes = planes
        else:
            self.planes = buf("planes", torch.bfloat16)
        # split-chain centroid update workspaces (zeroed; the kernels re-zero)
        self.csum = buf("csum", torch.float64, 0.0)
        self.cabs = buf("cabs", F32, 0.0)
        self.clsb = buf("clsb", I32, 0x7F800000)
        self.status = buf("status", I32, 0)
        desc = np.zeros(P, dtype=L.PROBLEM_DTYPE)
        self.n_off, self.k_off, self.t_off = [], [], []
        no = ko = to = 0
        for p in range(P):
            x = xs[p]
            if not x.is_contiguous() or x.shape[1] != D or x.dtype != xs[0].dtype:
                raise DimensionError("batch inputs must be contiguous [n, D] of one dtype")
            self.n_off.append(no)
            self.k_off.append(ko)
            self.t_off.append(to)
            e = desc[p]
            e["x"] = x.data_ptr()
            e["xx"] = self.xx.data_ptr() + 4 * no
            e["centers"] = self.centers.data_ptr() + 4 * ko * D
            e["cc"] = self.cc.data_ptr() + 4 * ko
            e["labels"] = self.labels.data_ptr() + 4 * no
            e["best"] = self.best.data_ptr() + 4 * no
            e["counts"] = self.counts.data_ptr() + 4 * ko
            e["perm"] = self.perm.data_ptr() + 4 * no
            e["starts"] = self.starts.data_ptr() + 4 * (ko + p)
            e["tile_hist"] = self.tile_hist.data_ptr() + 4 * to
            e["inertia"] = self.inertia.data_ptr() + 4 * p * self.max_iter
            e["movement"] = self.movement.data_ptr() + 4 * ko
            e["status"] = self.status.data_ptr() + 4 * p * L.STATUS_WORDS
            e["plan_n"] = L.pw_plan(self.ns[p]).data_ptr()
            e["plan_k"] = 0
            e["dscratch"] = self.dscratch.data_ptr() + 8 * no
            e["planes"] = (self.planes.data_ptr() + 2 * 3 * no * D) if self.planes is not None else 0
            e["csum"] = (self.csum.data_ptr() + 8 * ko * D) if self.csum is not None else 0
            e["cabs"] = (self.cabs.data_ptr() + 4 * ko * D) if self.cabs is not None else 0
            e["clsb"] = (self.clsb.data_ptr() + 4 * ko * D) if self.clsb is not None else 0
            e["n"] = self.ns[p]
            e["k"] = self.ks[p]
            e["order"] = self.orders[p]
            no += self.ns[p]
            ko += self.kcaps[p]
            to += tiles[p] * self.kcaps[p]
        self.desc = desc
        self.dev = L.to_device_struct(desc)
        self.max_n = max(self.ns)
        self.max_k = max(self.kcaps)

    # views -------------------------------------------------------------
    def centers_of(self, p: int, k: int | None = None) -> torch.Tensor:
        k = self.ks[p] if k is None else k
        o = self.k_off[p] * self.D
        return self.centers[o:o + k * self.D].view(k, self.D)

    def model(self, p: int) -> DevModel:
        n, k, no, ko = self.ns[p], self.ks[p], self.n_off[p], self.k_off[p]
        return DevModel(
            centers=self.centers_of(p), labels=self.labels[no:no + n],
            counts=self.counts[ko:ko + k], perm=self.perm[no:no + n],
            starts=self.starts[ko + p:ko + p + k + 1],
            status=self.status[p * L.STATUS_WORDS:(p + 1) * L.STATUS_WORDS],
            inertia=self.inertia[p * self.max_iter:(p + 1) * self.max_iter], k=k, n=n)

    def best_of(self, p: int) -> torch.Tensor:
        return self.best[self.n_off[p]:self.n_off[p] + self.ns[p]]

    # kernels -------------------------------------------------------------
    def args(self):
        return (self.dev.data_ptr(), self.P, self.dtype, self.D, self.max_n, self.max_k)

    def kmeanspp(self, draws: torch.Tensor, max_k: int):
        L.call("ac_kmeanspp", self.dev.data_ptr(), self.P, self.dtype, self.D, self.max_n, max_k,
               draws.data_ptr(), L.stream_ptr())

    def lloyd(self, max_iter: int, tol: float, poll_every: int = 0, group: int = 0):
        """Lloyd on every problem; ``group`` > 0 runs the problems in blocks of
        that many, so a block's points stay resident in the 126 MB L2 across
        its iterations (each assign/update pass then reads L2, not HBM)."""
        if group <= 0 or group >= self.P:
            L.call("ac_lloyd", *self.args(), int(max_iter), float(tol), int(poll_every),
                   self.desc.ctypes.data, L.stream_ptr())
            return
        isz = self.desc.dtype.itemsize
        for g0 in range(0, self.P, group):
            g1 = min(self.P, g0 + group)
            L.call("ac_lloyd", self.dev.data_ptr() + g0 * isz, g1 - g0, self.dtype, self.D,
                   max(self.ns[g0:g1]), max(self.kcaps[g0:g1]), int(max_iter), float(tol),
                   int(poll_every), self.desc.ctypes.data + g0 * isz, L.stream_ptr())

    def lloyd_range(self, g0: int, g1: int, max_iter: int, tol: float, inertia: bool = True,
                    prepared: bool = False):
        """Lloyd on problems [g0, g1) of the batch (current stream);
        ``inertia=False`` skips the inertia_history reductions; ``prepared``:
        xx/planes were written by ac_l2norm_ex (see SteadyStep)."""
        isz = self.desc.dtype.itemsize
        flags = (0 if inertia else L.LLOYD_NO_INERTIA) | (L.LLOYD_PREPARED if prepared else 0)
        L.call("ac_lloyd_ex", self.dev.data_ptr() + g0 * isz, g1 - g0, self.dtype, self.D,
               max(self.ns[g0:g1]), max(self.kcaps[g0:g1]), int(max_iter), float(tol),
               flags, self.desc.ctypes.data + g0 * isz, L.stream_ptr())

    def l2_group(self, budget: float = 48e6) -> int:
        """Problems per block so that a block's points fit in ~`budget` bytes of L2."""
        esz = 2 if self.dtype == L.DTYPE_BF16 else 4
        per = max(1, max(self.ns) * self.D * esz)
        return max(1, int(budget // per))

    def prepare(self):
        L.call("ac_lloyd_prepare", *self.args(), L.stream_ptr())

    def assign(self, c_lo: int = 0, flags: int = L.ASSIGN_ALL):
        L.call("ac_assign_ordered", *self.args(), int(c_lo), int(flags), self.orders[0],
               self.desc.ctypes.data, L.stream_ptr())

    def sort(self):
        """tile histograms must be current (written by assign)."""
        L.call("ac_repair_sort", *self.args(), -1, L.ASSIGN_ALL, L.stream_ptr())


def batch_buffer_bytes(ns, kcaps, d: int, dtype: int, max_iter: int) -> dict:
    """Byte size of every flat buffer of a batch: the per-problem sizes of
    ac_workspace_bytes(AC_WS_CLUSTER) summed over the problems."""
    tot: dict[str, int] = {}
    for n, k in zip(ns, kcaps):
        for name, b in L.workspace_bytes(L.WS_CLUSTER, n, k, d, dtype, max(max_iter, 1)).items():
            tot[name] = tot.get(name, 0) + b
    return tot


def _group_by_order(ns, ks, D):
    """Problems that can share one batch: the general GEMM order apart from
    the small-shape orders (LANES16 / GEMV8 problems batch together)."""
    groups: dict[bool, list[int]] = {}
    for i, (n, k) in enumerate(zip(ns, ks)):
        groups.setdefault(L.gemm_order(n, k, D) == L.ORDER_SEQ, []).append(i)
    return list(groups.values())


# ---------------------------------------------------------------------------
# k-means / Lloyd
# ---------------------------------------------------------------------------
def kmeans_batch(xs: list[torch.Tensor], ks: list[int], seeds: list[int], max_iter: int,
                 tol: float, inertia: bool = True, stops_out: list | None = None,
                 poll_every: int = 0) -> list[DevModel]:
    """clustering.py:155-167 for every problem (k-means++ then Lloyd).
    ``inertia=False``: no inertia_history (callers that never read it -- the
    streaming sessions and the multi-stage rounds -- get the labels-only
    assignment, same labels / centres / n_iter).  ``stops_out``: instead of
    reading the k-means++ `total <= 0` stop flags on the host (a sync), append
    them (device int32 tensors) to this list; a caller that finds any flag
    >= 0 must redo the call without ``stops_out`` (sync-free enqueue, used to
    run the query clustering concurrently with the keys')."""
    out: list[DevModel | None] = [None] * len(xs)
    D = int(xs[0].shape[1])
    for idx in _group_by_order([x.shape[0] for x in xs], ks, D):
        sub_x = [xs[i] for i in idx]
        sub_k = [ks[i] for i in idx]
        sub_s = [seeds[i] for i in idx]
        b = Batch(sub_x, sub_k, max_iter)
        mk = max(sub_k)
        draws = np.zeros((len(idx), mk), np.float64)
        for j, (x, k, s) in enumerate(zip(sub_x, sub_k, sub_s)):
            draws[j, :k] = _draws(s, int(x.shape[0]), k)
        dd = L.upload(torch.from_numpy(draws))
        b.kmeanspp(dd, mk)
        if stops_out is not None:
            stops_out.append(b.status.view(b.P, L.STATUS_WORDS)[:, L.ST_KPP_STOP].clone())
            stops = np.full(1, -1)
        else:
            # k-means++ `total <= 0` replay (all remaining points coincide with
            # a chosen centre): rare; requires a host look at the stop flags
            stops = b.status.view(b.P, L.STATUS_WORDS)[:, L.ST_KPP_STOP].cpu().numpy()
        if (stops >= 0).any():
            for j in np.flatnonzero(stops >= 0):
                draws[j, :sub_k[j]] = _draws(sub_s[j], int(sub_x[j].shape[0]), sub_k[j],
                                             forced_from=int(stops[j]))
            dd = torch.from_numpy(draws).to(L.device())
            b.kmeanspp(dd, mk)
        if inertia:
            b.lloyd(max_iter, tol, poll_every)
        else:
            b.lloyd_range(0, b.P, max_iter, tol, inertia=False)
        for j, i in enumerate(idx):
            out[i] = b.model(j)
    return out  # type: ignore[return-value]


def lloyd_batch(xs: list[torch.Tensor], inits: list[torch.Tensor], max_iter: int,
                tol: float, inertia: bool = True) -> list[DevModel]:
    """clustering.py:119-152 from given initial centres (warm starts)."""
    out: list[DevModel | None] = [None] * len(xs)
    D = int(xs[0].shape[1])
    ks = [int(c.shape[0]) for c in inits]
    for idx in _group_by_order([x.shape[0] for x in xs], ks, D):
        b = Batch([xs[i] for i in idx], [ks[i] for i in idx], max_iter)
        for j, i in enumerate(idx):
            b.centers_of(j).copy_(inits[i].to(F32))
        if inertia:
            b.lloyd(max_iter, tol)
        else:
            b.lloyd_range(0, b.P, max_iter, tol, inertia=False)
        for j, i in enumerate(idx):
            out[i] = b.model(j)
    return out  # type: ignore[return-value]


def l2norm(x: torch.Tensor):
    """tensorops.py:59-76 on device: (rows f32, degenerate mask u8)."""
    rows, d = x.shape
    out = torch.empty((rows, d), dtype=F32, device=x.device)
    deg = torch.empty(rows, dtype=torch.uint8, device=x.device)
    L.call("ac_l2norm", x.data_ptr(), L.dtype_code(x), rows, d, out.data_ptr(), 0,
           deg.data_ptr(), L.stream_ptr())
    return out, deg


def segment_means(xs: list[torch.Tensor], models: list[DevModel]) -> list[torch.Tensor]:
    """f64 member means in member order (cluster_queries reps, clustering.py:197-200)."""
    outs = [torch.empty((m.k, x.shape[1]), dtype=F32, device=x.device) for x, m in zip(xs, models)]
    # a minimal descriptor table pointing at the models' buffers
    desc = np.zeros(len(xs), dtype=L.PROBLEM_DTYPE)
    for p, (x, m) in enumerate(zip(xs, models)):
        e = desc[p]
        e["x"] = x.data_ptr()
        e["counts"] = m.counts.data_ptr()
        e["perm"] = m.perm.data_ptr()
        e["starts"] = m.starts.data_ptr()
        e["n"] = m.n
        e["k"] = m.k
    dv = L.to_device_struct(desc)
    ptrs = L.upload(torch.tensor([o.data_ptr() for o in outs], dtype=torch.int64))
    L.call("ac_segment_mean", dv.data_ptr(), len(xs), L.dtype_code(xs[0]), int(xs[0].shape[1]),
           max(m.k for m in models), ptrs.data_ptr(), L.stream_ptr())
    return outs


def cluster_queries_batch(qs: list[torch.Tensor], num_clusters: list[int], seeds: list[int],
                          max_iter: int, tol: float, inits: list[torch.Tensor] | None = None,
                          inertia: bool = True, stops_out: list | None = None):
    """clustering.py:182-200: normalise, cluster (cold or warm), representatives."""
    qns = [l2norm(q)[0] for q in qs]
    if inits is None:
        models = kmeans_batch(qns, num_clusters, seeds, max_iter, tol, inertia, stops_out)
    else:
        models = lloyd_batch(qns, inits, max_iter, tol, inertia)
    reps = segment_means(qns, models)
    return models, reps, qns


# ---------------------------------------------------------------------------
# tau / mse / multi-stage
# ---------------------------------------------------------------------------
def _model_desc(xs: list[torch.Tensor], models: list[DevModel], scratch: list[torch.Tensor]):
    desc = np.zeros(len(xs), dtype=L.PROBLEM_DTYPE)
    for p, (x, m, s) in enumerate(zip(xs, models, scratch)):
        e = desc[p]
        e["x"] = x.data_ptr()
        e["centers"] = m.centers.data_ptr()
        e["labels"] = m.labels.data_ptr()
        e["plan_n"] = L.pw_plan(m.n).data_ptr()
        e["dscratch"] = s.data_ptr()
        e["n"] = m.n
        e["k"] = m.k
    return L.to_device_struct(desc)


def tau_batch(ks: list[torch.Tensor], stage0: list[DevModel], factor: float) -> torch.Tensor:
    """compute_tau (clustering.py:209-215) for every problem -> f64 [P] device."""
    scratch = [torch.empty(m.n, dtype=torch.float64, device=L.device()) for m in stage0]
    dv = _model_desc(ks, stage0, scratch)
    out = torch.empty(len(ks), dtype=torch.float64, device=L.device())
    L.call("ac_tau", dv.data_ptr(), len(ks), L.dtype_code(ks[0]), int(ks[0].shape[1]),
           max(m.n for m in stage0), float(factor), out.data_ptr(), L.stream_ptr())
    return out


def mse_batch(ks: list[torch.Tensor], models: list[DevModel]) -> torch.Tensor:
    """pipeline.py:319-323 per-head clustering MSE (f64) -> [P] device."""
    scratch = [torch.empty(m.n, dtype=torch.float64, device=L.device()) for m in models]
    dv = _model_desc(ks, models, scratch)
    out = torch.empty(len(ks), dtype=torch.float64, device=L.device())
    L.call("ac_mse_f64", dv.data_ptr(), len(ks), L.dtype_code(ks[0]), int(ks[0].shape[1]),
           max(m.n for m in models), out.data_ptr(), L.stream_ptr())
    return out


class _RunningAssign:
    """nearest-centre state of all N keys against the accumulated multi-stage
    centres: running (best, label) merged round by round with strict '<'
    (earlier centres win ties, exactly like argmin over the concatenation)."""

    def __init__(self, k: torch.Tensor, kcap: int, max_iter: int):
        self.k = k
        self.batch = Batch([k], [1], max_iter, kcaps=[kcap])
        self.batch.prepare()  # ||x||^2 of every key (the centres are set per round)
        self.nc = 0
        self.orders: list[int] = []

    def _grow(self, need: int):
        """Re-home the running state into a batch with room for ``need``
        centres (a custom stage_schedule can exceed the default bound)."""
        old = self.batch
        cap = max(need, 2 * old.kcaps[0])
        nb = Batch([self.k], [1], old.max_iter, kcaps=[cap])
        nb.xx.copy_(old.xx)
        if self.nc:
            nb.centers_of(0, self.nc).copy_(old.centers_of(0, self.nc))
            nb.labels.copy_(old.labels)
            nb.best.copy_(old.best)
        nb.desc[0]["k"] = old.desc[0]["k"]
        nb.desc[0]["order"] = old.desc[0]["order"]
        self.batch = nb

    def add(self, centers: torch.Tensor):
        m = centers.shape[0]
        if self.nc + m > self.batch.kcaps[0]:
            self._grow(self.nc + m)
        b = self.batch
        b.centers_of(0, self.nc + m)[self.nc:].copy_(centers)
        new_nc = self.nc + m
        order = L.gemm_order(b.ns[0], new_nc, b.D)
        full = not self.orders or any(o != order for o in self.orders) or self.nc == 0
        b.desc[0]["k"] = new_nc
        b.desc[0]["order"] = order
        b.orders = [order]
        b.ks = [new_nc]
        b.dev = L.to_device_struct(b.desc)
        if full:
            b.assign(0, L.ASSIGN_ALL)
        else:
            b.assign(self.nc, L.ASSIGN_ALL | L.ASSIGN_MERGE)
        self.orders.append(order)
        self.nc = new_nc

    def mean_best(self) -> torch.Tensor:
        b = self.batch
        out = torch.empty(1, dtype=F32, device=L.device())
        L.call("ac_reduce_best", b.dev.data_ptr(), 1, b.max_n, 0, out.data_ptr(), L.stream_ptr())
        return out


class _RunningAssignBatch:
    """The running nearest-centre state of several heads' keys at once (one
    Batch, one problem per head): each round's centres are appended per
    head and merged into (best, label) with strict '<' -- earlier centres win
    ties, exactly argmin over the concatenation (clustering.py:301-302) --
    in one assignment launch per group of heads that share the merge offset
    and the GEMM order (all of them in lock-step rounds)."""

    def __init__(self, ks: list[torch.Tensor], kcap: int, max_iter: int):
        self.ks = ks
        self.max_iter = max_iter
        self.batch = Batch(ks, [1] * len(ks), max_iter, kcaps=[kcap] * len(ks))
        self.batch.prepare()  # ||x||^2 of every key (the centres are set per round)
        self.nc = [0] * len(ks)
        self.orders: list[list[int]] = [[] for _ in ks]

    def _grow(self, need: list[int]):
        old = self.batch
        caps = [max(n, c) for n, c in zip(need, old.kcaps)]
        caps = [c if c <= k else max(c, 2 * k) for c, k in zip(caps, old.kcaps)]
        nb = Batch(self.ks, [1] * len(self.ks), self.max_iter, kcaps=caps)
        nb.xx.copy_(old.xx)
        nb.labels.copy_(old.labels)
        nb.best.copy_(old.best)
        for p, nc in enumerate(self.nc):
            if nc:
                nb.centers_of(p, nc).copy_(old.centers_of(p, nc))
            nb.desc[p]["k"] = old.desc[p]["k"]
            nb.desc[p]["order"] = old.desc[p]["order"]
            nb.ks[p] = old.ks[p]
        self.batch = nb

    def add(self, heads: list[int], centers: list[torch.Tensor]):
        b = self.batch
        need = list(b.kcaps)
        for p, c in zip(heads, centers):
            need[p] = self.nc[p] + int(c.shape[0])
        if any(n > c for n, c in zip(need, b.kcaps)):
            self._grow(need)
            b = self.batch
        groups: dict[tuple, list[int]] = {}
        for p, c in zip(heads, centers):
            m = int(c.shape[0])
            nc = self.nc[p]
            b.centers_of(p, nc + m)[nc:].copy_(c)
            order = L.gemm_order(b.ns[p], nc + m, b.D)
            full = nc == 0 or any(o != order for o in self.orders[p])
            b.desc[p]["k"] = nc + m
            b.desc[p]["order"] = order
            b.ks[p] = nc + m
            groups.setdefault((0 if full else nc, order), []).append(p)
            self.orders[p].append(order)
            self.nc[p] = nc + m
        b.dev = L.to_device_struct(b.desc)
        for (c_lo, order), ps in groups.items():
            host = np.ascontiguousarray(b.desc[ps])
            dev = b.dev if len(ps) == b.P else L.to_device_struct(host)
            flags = L.ASSIGN_ALL | (L.ASSIGN_MERGE if c_lo else 0)
            L.call("ac_assign_ordered", dev.data_ptr(), len(ps), b.dtype, b.D,
                   max(b.ns[p] for p in ps), max(b.ks[p] for p in ps), int(c_lo), flags, order,
                   host.ctypes.data, L.stream_ptr())

    def mean_best(self, heads: list[int]) -> torch.Tensor:
        """f32 mean of the running best distances (nearest_center_mse over the
        accumulated centres) of ``heads`` -> device [len(heads)]."""
        b = self.batch
        out = torch.empty(len(heads), dtype=F32, device=L.device())
        if len(heads) == b.P and heads == list(range(b.P)):
            dev = b.dev
        else:
            dev = L.to_device_struct(np.ascontiguousarray(b.desc[heads]))
        L.call("ac_reduce_best", dev.data_ptr(), len(heads), max(b.ns[p] for p in heads), 0,
               out.data_ptr(), L.stream_ptr())
        self._keep_mb = dev
        return out


_MS_POLL = int(os.environ.get("AC_MS_POLL", "4"))  # C3 cold 108 -> 98 ms (8: 102)


def multi_stage_batch(ks: list[torch.Tensor], taus: list[float], n_max: int, m0: int,
                      seeds: list[int], max_iter: int, tol: float,
                      stage0: list[DevModel | None], schedule=None) -> list[DevModel]:
    """multi_stage_cluster_keys (clustering.py:218-320) for several keys
    tensors in lock-step rounds, batched across heads: per round one
    k-means batch over the heads still splitting, one retire launch, one
    merged assignment per group of heads and ONE host read (|U| and the
    stage MSE of every head); the final drop-empty / member sort run once
    for all heads.  Rounds need |U| on the host (it sizes the next round)."""
    dev = L.device()
    H = len(ks)
    D = int(ks[0].shape[1])
    dt = L.dtype_code(ks[0])
    results: list[DevModel | None] = [None] * H
    st = []
    for h in range(H):
        n = int(ks[h].shape[0])
        st.append(dict(n=n, pool=None, size=n, nc=0, rnd=0, flag=False, iters=0, mse=[]))
    live = [h for h in range(H) if taus[h] > 0.0]
    # centres accumulate while nc < n_max, each round adding m_t <= max(STAGE_FLOOR=8, m0)
    # (clustering.py:272-286); a custom schedule may exceed it (then the batch grows)
    run = _RunningAssignBatch(ks, n_max - 1 + max(8, m0), max_iter) if live else None
    for h in range(H):
        if taus[h] <= 0.0:
            base = stage0[h] if stage0[h] is not None else kmeans_batch(
                [ks[h]], [min(m0, st[h]["n"])], [seeds[h]], max_iter, tol)[0]
            ra = _RunningAssign(ks[h], max(base.k, 1), max_iter)
            ra.add(base.centers)
            base.flag_full = True
            base.stage_count = 1
            base.stage_mse = [float(ra.mean_best().item())]
            base.tau = float(taus[h])
            base.host_iters = base.n_iter()
            results[h] = base
    with L.pdl(L.PDL_PLANNER):
        _multi_stage_rounds(ks, taus, n_max, m0, seeds, max_iter, tol, stage0, schedule, st, live,
                            run, D, dt, dev)
    # final labels = running argmin over every accumulated centre; drop empty
    # centres and sort members -- one launch each for every head
    fin = [h for h in range(H) if results[h] is None]
    if fin:
        b = run.batch
        sub = L.to_device_struct(np.ascontiguousarray(b.desc[fin]))
        newk = torch.empty(len(fin), dtype=I32, device=dev)
        L.call("ac_drop_empty", sub.data_ptr(), len(fin), D, b.max_n, b.max_k, newk.data_ptr(),
               L.stream_ptr())
        kk = newk.cpu().numpy()
        for j, p in enumerate(fin):
            b.desc[p]["k"] = int(kk[j])
            b.ks[p] = int(kk[j])
        b.dev = L.to_device_struct(b.desc)
        sub = L.to_device_struct(np.ascontiguousarray(b.desc[fin]))
        L.call("ac_sort_by_label", sub.data_ptr(), len(fin), b.max_n, b.max_k, L.stream_ptr())
        for h in fin:
            s = st[h]
            m = b.model(h)
            m.flag_full = s["flag"]
            m.stage_count = s["rnd"]
            m.stage_mse = s["mse"]
            m.tau = float(taus[h])
            m.host_iters = s["iters"]
            results[h] = m
    return results  # type: ignore[return-value]


def _multi_stage_rounds(ks, taus, n_max, m0, seeds, max_iter, tol, stage0, schedule, st, live,
                        run, D, dt, dev):
    """The round loop of multi_stage_batch (mutates st / live)."""
    while live:
        todo = []
        for h in live:
            s = st[h]
            if s["nc"] >= n_max:
                s["flag"] = True
                continue
            if schedule is not None:
                want = int(schedule(s["rnd"], s["size"], s["n"]))
            else:
                want = m0 if s["rnd"] == 0 else max(8, math.ceil(m0 * s["size"] / s["n"]))
            s["m_t"] = min(want, s["size"])
            todo.append(h)
        if not todo:
            break
        # this round's clustering (stage 0 reused for round 0)
        need, subx = [], {}
        for h in todo:
            s = st[h]
            if s["rnd"] == 0 and stage0[h] is not None and stage0[h].k == s["m_t"]:
                s["model"], s["sub"] = stage0[h], ks[h]
            else:
                if s["size"] == s["n"]:
                    sub = ks[h]
                else:
                    sub = torch.empty((s["size"], D), dtype=ks[h].dtype, device=dev)
                    L.call("ac_gather_rows", ks[h].data_ptr(), dt, D, s["pool"].data_ptr(),
                           s["size"], sub.data_ptr(), L.stream_ptr())
                subx[h] = sub
                need.append(h)
        if need:
            # small late-round problems converge in a few iterations: poll
            # the active flags every _MS_POLL iterations instead of launching
            # all max_iter iterations
            ms = kmeans_batch([subx[h] for h in need], [st[h]["m_t"] for h in need],
                              [seeds[h] + st[h]["rnd"] for h in need], max_iter, tol,
                              poll_every=_MS_POLL)
            for h, m in zip(need, ms):
                st[h]["model"], st[h]["sub"] = m, subx[h]
        # retire: U = U[dist >= tau] (f32 compare, NEP 50)
        desc = np.zeros(len(todo), dtype=L.PROBLEM_DTYPE)
        outs = []
        scratch = []
        for j, h in enumerate(todo):
            s = st[h]
            m = s["model"]
            if s["pool"] is None:
                s["pool"] = torch.arange(s["n"], dtype=torch.int64, device=dev)
            sc = torch.empty(s["size"], dtype=torch.float64, device=dev)
            scratch.append(sc)
            e = desc[j]
            e["x"] = s["sub"].data_ptr()
            e["centers"] = m.centers.data_ptr()
            e["labels"] = m.labels.data_ptr()
            e["dscratch"] = sc.data_ptr()
            e["n"] = s["size"]
            e["k"] = m.k
            outs.append(torch.empty(s["size"], dtype=torch.int64, device=dev))
        dv = L.to_device_struct(desc)
        tau32 = L.upload(torch.tensor([np.float32(taus[h]) for h in todo], dtype=F32))
        pin = L.upload(torch.tensor([st[h]["pool"].data_ptr() for h in todo], dtype=torch.int64))
        pout = L.upload(torch.tensor([o.data_ptr() for o in outs], dtype=torch.int64))
        cnt = torch.empty(len(todo), dtype=torch.int64, device=dev)
        L.call("ac_retire", dv.data_ptr(), len(todo), dt, D, max(st[h]["size"] for h in todo),
               tau32.data_ptr(), pin.data_ptr(), pout.data_ptr(), cnt.data_ptr(), L.stream_ptr())
        run.add(todo, [st[h]["model"].centers for h in todo])
        mses = run.mean_best(todo)
        zero = torch.zeros((), dtype=I32, device=dev)
        nits = torch.stack([zero if st[h]["model"].host_iters is not None
                            else st[h]["model"].status[L.ST_NITER] for h in todo])
        for h in todo:
            st[h]["nc"] += st[h]["model"].k
        # the round's one sync: |U|, the stage MSE and the Lloyd iterations
        host = torch.cat([cnt.double(), mses.double(), nits.double()]).cpu().numpy()
        nt = len(todo)
        for j, h in enumerate(todo):
            s = st[h]
            s["pool"] = outs[j][:int(host[j])]
            s["size"] = int(host[j])
            s["mse"].append(float(np.float32(host[nt + j])))
            m = s["model"]
            s["iters"] += m.host_iters if m.host_iters is not None else int(host[2 * nt + j])
            s["rnd"] += 1
        live = [h for h in live if st[h]["size"] > 0 and not st[h]["flag"]]
        for h in list(live):
            if st[h]["nc"] >= n_max:
                st[h]["flag"] = True
                live.remove(h)


# ---------------------------------------------------------------------------
# selection + attention
# ---------------------------------------------------------------------------
def envelopes_batch(ks: list[torch.Tensor], models: list[DevModel]):
    D = int(ks[0].shape[1])
    emax = [torch.empty((m.k, D), dtype=F32, device=L.device()) for m in models]
    emin = [torch.empty((m.k, D), dtype=F32, device=L.device()) for m in models]
    desc = np.zeros(len(ks), dtype=L.PROBLEM_DTYPE)
    for p, (x, m) in enumerate(zip(ks, models)):
        e = desc[p]
        e["x"] = x.data_ptr()
        e["counts"] = m.counts.data_ptr()
        e["perm"] = m.perm.data_ptr()
        e["starts"] = m.starts.data_ptr()
        e["n"] = m.n
        e["k"] = m.k
    dv = L.to_device_struct(desc)
    pmax = L.upload(torch.tensor([t.data_ptr() for t in emax], dtype=torch.int64))
    pmin = L.upload(torch.tensor([t.data_ptr() for t in emin], dtype=torch.int64))
    L.call("ac_envelopes", dv.data_ptr(), len(ks), L.dtype_code(ks[0]), D,
           max(m.k for m in models), pmax.data_ptr(), pmin.data_ptr(), L.stream_ptr())
    return emax, emin


@dataclass
class DevSelection:
    scores: torch.Tensor     # [gq, C] f32
    selected: torch.Tensor   # [gq, topk] int64
    runs: torch.Tensor       # [gq, run_stride, 2] int32
    nruns: torch.Tensor      # [gq] int32
    density: torch.Tensor    # [1] f64


def select_batch(reps: list[torch.Tensor], emax: list[torch.Tensor], emin: list[torch.Tensor],
                 kmodels: list[DevModel], topks: list[int], scorer: str,
                 run_stride: int | None = None, scores_in: list[torch.Tensor] | None = None,
                 top_p: float | None = None, mass_scale: float = 1.0):
    """quest.py:94-143: scores, stable top-k (or the top-p extension, at most
    topk clusters), merged runs, density."""
    dev = L.device()
    P = len(reps)
    D = int(reps[0].shape[1])
    stride = run_stride or max(topks)
    out = []
    desc = np.zeros(P, dtype=L.SELECT_DTYPE)
    gq_max = max(int(r.shape[0]) for r in reps)
    runs = torch.zeros((P, gq_max, stride, 2), dtype=I32, device=dev)
    nruns = torch.zeros((P, gq_max), dtype=I32, device=dev)
    for p in range(P):
        gq, C = int(reps[p].shape[0]), kmodels[p].k
        sel = DevSelection(
            scores=(scores_in[p] if scores_in is not None
                    else torch.empty((gq, C), dtype=F32, device=dev)),
            selected=torch.empty((gq, topks[p]), dtype=torch.int64, device=dev),
            runs=runs[p], nruns=nruns[p],
            density=torch.empty(1, dtype=torch.float64, device=dev))
        cov = torch.empty(gq, dtype=torch.int64, device=dev)
        sel._covered = cov  # keep alive
        e = desc[p]
        e["reps"] = reps[p].data_ptr()
        e["emax"] = emax[p].data_ptr()
        e["emin"] = emin[p].data_ptr()
        e["counts"] = kmodels[p].counts.data_ptr()
        e["kstarts"] = kmodels[p].starts.data_ptr()
        e["scores"] = sel.scores.data_ptr()
        e["selected"] = sel.selected.data_ptr()
        e["runs"] = sel.runs.data_ptr()
        e["nruns"] = sel.nruns.data_ptr()
        e["covered"] = cov.data_ptr()
        e["density"] = sel.density.data_ptr()
        e["gq"], e["c"], e["topk"] = gq, C, topks[p]
        e["order"] = L.gemm_order(gq, C, D)
        e["run_stride"] = stride
        out.append(sel)
    dv = L.to_device_struct(desc)
    if top_p is None:
        L.call("ac_select", dv.data_ptr(), P, D, L.SCORERS[scorer], gq_max,
               max(m.k for m in kmodels), stride, L.stream_ptr())
    else:
        L.call("ac_select_topp", dv.data_ptr(), P, D, L.SCORERS[scorer], gq_max,
               max(m.k for m in kmodels), stride, float(top_p), float(mass_scale), L.stream_ptr())
    return out, runs, nruns


ATTN_DIMS = (16, 32, 64, 128)


def _attn_dim(d: int) -> int:
    for a in ATTN_DIMS:
        if d <= a:
            return a
    raise DimensionError(f"head_dim {d} > 128 is not supported by the attention kernel")


def _pad_dim(x: torch.Tensor, da: int) -> torch.Tensor:
    if x.shape[-1] == da:
        return x.contiguous()
    return torch.nn.functional.pad(x, (0, da - x.shape[-1])).contiguous()


def sparse_attention_heads(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                           qmodels: list[DevModel], kmodels: list[DevModel],
                           runs: torch.Tensor, nruns: torch.Tensor, out_dtype=F32,
                           impl: str = "auto") -> torch.Tensor:
    """_gathered_attention (pipeline.py:154-165) for H heads of one layer.
    q/k/v: [H, L, D] (f32 or bf16).  Returns [H, L, D] out_dtype."""
    H, Ln, D = q.shape
    dev = L.device()
    da = _attn_dim(D)
    dt = L.dtype_code(q)
    qa, ka, va = (_pad_dim(t, da) for t in (q, k, v))
    kp = torch.empty_like(ka)
    vp = torch.empty_like(va)
    kperm = torch.stack([m.perm for m in kmodels])
    L.call("ac_permute_rows_heads", ka.data_ptr(), dt, da, kperm.data_ptr(), Ln, H, kp.data_ptr(),
           L.stream_ptr())
    L.call("ac_permute_rows_heads", va.data_ptr(), dt, da, kperm.data_ptr(), Ln, H, vp.data_ptr(),
           L.stream_ptr())
    gq = L.upload(torch.tensor([m.k for m in qmodels], dtype=I32))
    gq_max = int(runs.shape[1])
    topk_max = int(runs.shape[2])
    qperm = torch.stack([m.perm for m in qmodels])
    qlab = torch.stack([m.labels for m in qmodels])
    qcounts = torch.zeros((H, gq_max), dtype=I32, device=dev)
    qstarts = torch.zeros((H, gq_max + 1), dtype=I32, device=dev)
    for h, m in enumerate(qmodels):
        qcounts[h, :m.k] = m.counts
        qstarts[h, :m.k + 1] = m.starts
    qp_cap = Ln + TILE * gq_max
    item_cap = (Ln + TILE - 1) // TILE + gq_max
    item_rows = 128 if impl == "simt" else int(L.lib().ac_attention_item_rows(dt, da))
    qp = torch.empty((H * qp_cap, da), dtype=q.dtype, device=dev)
    qidx = torch.empty(H * qp_cap + H * gq_max, dtype=I32, device=dev)
    items = torch.empty(H * item_cap * L.ITEM_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    L.call("ac_build_q_layout", qa.data_ptr(), dt, da, Ln, H, qperm.data_ptr(), qstarts.data_ptr(),
           qcounts.data_ptr(), qlab.data_ptr(), gq.data_ptr(), gq_max, nruns.data_ptr(), topk_max,
           qp.data_ptr(), qidx.data_ptr(), qp_cap, items.data_ptr(), item_cap, item_rows,
           L.stream_ptr())
    out = torch.empty((H, Ln, da), dtype=out_dtype, device=dev)
    odt = L.dtype_code(out) if out_dtype != F32 else L.DTYPE_F32
    scale = float(1.0 / math.sqrt(D))
    with phase("attention"):
        if impl == "simt":
            L.call("ac_sparse_attention_simt", qp.data_ptr(), qidx.data_ptr(), kp.data_ptr(),
                   vp.data_ptr(), dt, da, Ln, items.data_ptr(), H * item_cap, runs.data_ptr(),
                   scale, out.data_ptr(), odt, L.stream_ptr())
        else:
            L.call("ac_sparse_attention", qp.data_ptr(), H * qp_cap, qidx.data_ptr(),
                   kp.data_ptr(), vp.data_ptr(), dt, da, Ln, H, items.data_ptr(), H * item_cap,
                   runs.data_ptr(), scale, out.data_ptr(), odt, L.stream_ptr())
    return out[..., :D] if da != D else out


def dense_attention_1h(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out_dtype=F32,
                       impl: str = "auto") -> torch.Tensor:
    """full_attention (reference.py:25-45) for one head with any Lq, Lk >= 1
    and value width Dv: q [Lq, D], k [Lk, D], v [Lk, Dv] -> [Lq, Dv].

    One query cluster of Lq rows in identity order attends over the single
    key run [0, Lk).  q and k are zero-padded to a common kernel width
    (zero columns add nothing to q·k; the softmax scale stays 1/sqrt(D)),
    v likewise (padded output columns are dropped)."""
    Lq, D = int(q.shape[0]), int(q.shape[1])
    Lk, Dv = int(k.shape[0]), int(v.shape[1])
    dev = L.device()
    da = _attn_dim(max(D, Dv))
    dt = L.dtype_code(q)
    qa, ka, va = (_pad_dim(t, da) for t in (q, k, v))
    item_rows = 128 if impl == "simt" else int(L.lib().ac_attention_item_rows(dt, da))
    ident = torch.arange(Lq, dtype=I32, device=dev)
    counts = torch.tensor([Lq], dtype=I32, device=dev)
    starts = torch.tensor([0, Lq], dtype=I32, device=dev)
    labels = torch.zeros(Lq, dtype=I32, device=dev)
    gq = torch.ones(1, dtype=I32, device=dev)
    nruns = torch.ones((1, 1), dtype=I32, device=dev)
    runs = torch.tensor([[[[0, Lk]]]], dtype=I32, device=dev)
    qp_cap = Lq + TILE
    item_cap = (Lq + TILE - 1) // TILE + 1
    qp = torch.empty((qp_cap, da), dtype=q.dtype, device=dev)
    qidx = torch.empty(qp_cap + 1, dtype=I32, device=dev)
    items = torch.empty(item_cap * L.ITEM_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    L.call("ac_build_q_layout", qa.data_ptr(), dt, da, Lq, 1, ident.data_ptr(), starts.data_ptr(),
           counts.data_ptr(), labels.data_ptr(), gq.data_ptr(), 1, nruns.data_ptr(), 1,
           qp.data_ptr(), qidx.data_ptr(), qp_cap, items.data_ptr(), item_cap, item_rows,
           L.stream_ptr())
    out = torch.empty((Lq, da), dtype=out_dtype, device=dev)
    odt = L.dtype_code(out) if out_dtype != F32 else L.DTYPE_F32
    scale = float(1.0 / math.sqrt(D))
    # one head: the head stride L of the K/V tensors is Lk; the output rows
    # are addressed through qidx (tokens < Lq)
    if impl == "simt":
        L.call("ac_sparse_attention_simt", qp.data_ptr(), qidx.data_ptr(), ka.data_ptr(),
               va.data_ptr(), dt, da, Lk, items.data_ptr(), item_cap, runs.data_ptr(), scale,
               out.data_ptr(), odt, L.stream_ptr())
    else:
        L.call("ac_sparse_attention", qp.data_ptr(), qp_cap, qidx.data_ptr(), ka.data_ptr(),
               va.data_ptr(), dt, da, Lk, 1, items.data_ptr(), item_cap, runs.data_ptr(), scale,
               out.data_ptr(), odt, L.stream_ptr())
    return out[:, :Dv] if da != Dv else out


def dense_attention_heads(q, k, v, out_dtype=F32, impl: str = "auto") -> torch.Tensor:
    """full_attention (reference.py:25-45) for H heads: one run covering all keys."""
    H, Ln, D = q.shape
    dev = L.device()
    qm = []
    km = []
    ar = torch.arange(Ln, dtype=I32, device=dev)
    for _ in range(H):
        qm.append(DevModel(centers=None, labels=torch.zeros(Ln, dtype=I32, device=dev),
                           counts=torch.tensor([Ln], dtype=I32, device=dev), perm=ar,
                           starts=torch.tensor([0, Ln], dtype=I32, device=dev), status=None,
                           inertia=None, k=1, n=Ln))
        km.append(DevModel(centers=None, labels=None, counts=None, perm=ar, starts=None,
                           status=None, inertia=None, k=1, n=Ln))
    runs = torch.zeros((H, 1, 1, 2), dtype=I32, device=dev)
    runs[..., 1] = Ln
    nruns = torch.ones((H, 1), dtype=I32, device=dev)
    return sparse_attention_heads(q, k, v, qm, km, runs, nruns, out_dtype, impl)
