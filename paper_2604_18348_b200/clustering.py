"""Query and key clustering on the device (reference: clustering.py).

Same names, signatures, defaults, errors and return types as the reference's
``kmeans`` (:155), ``warm_start_update`` (:170), ``cluster_queries`` (:182),
``nearest_center_mse`` (:203), ``compute_tau`` (:209) and
``multi_stage_cluster_keys`` (:218).  Results are bit-identical to the
reference (labels, centres, counts, iteration counts, inertia history,
stage MSEs) — see DESIGN.md "Parity model".
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import engine as E
from .errors import ParameterError
from .tensorops import to_device, to_host

__all__ = [
    "ClusterModel", "kmeans", "cluster_queries", "multi_stage_cluster_keys", "compute_tau",
    "warm_start_update", "nearest_center_mse",
]

DEFAULT_MAX_ITER = 25
DEFAULT_TOL = 1e-4
DEFAULT_QUERY_CLUSTERS = 65
DEFAULT_STAGE0_CLUSTERS = 100
DEFAULT_TAU_FACTOR = 1.5
STAGE_FLOOR = 8


@dataclass
class ClusterModel:
    centers: object          # [C, D] f32
    assignments: object      # [N] int32
    counts: object           # [C] int64, all >= 1
    flag_full: bool = False
    stage_count: int = 1
    n_iter: int = 0
    inertia_history: list = field(default_factory=list)
    stage_mse: list = field(default_factory=list)
    tau: float | None = None

    @property
    def num_clusters(self) -> int:
        return int(self.centers.shape[0])


def export_model(m: E.DevModel, host: bool, with_inertia: bool = True) -> ClusterModel:
    """Device model -> reference ClusterModel (numpy when the caller was host)."""
    n_iter = m.n_iter()
    inertia = []
    if with_inertia and m.host_iters is None and n_iter > 0:
        inertia = [float(v) for v in m.inertia[:n_iter].cpu().numpy()]
    counts = m.counts.to(torch.int64)
    return ClusterModel(
        centers=to_host(m.centers.clone(), host), assignments=to_host(m.labels.clone(), host),
        counts=to_host(counts, host), flag_full=bool(m.flag_full), stage_count=int(m.stage_count),
        n_iter=int(n_iter), inertia_history=inertia, stage_mse=list(m.stage_mse), tau=m.tau)


def import_model(model: ClusterModel, n: int) -> E.DevModel:
    """Reference ClusterModel (host or device) -> minimal DevModel."""
    dev = L.device()
    centers = torch.as_tensor(np.asarray(model.centers, np.float32) if not isinstance(
        model.centers, torch.Tensor) else model.centers).to(dev, torch.float32).contiguous()
    labels = torch.as_tensor(np.asarray(model.assignments, np.int32) if not isinstance(
        model.assignments, torch.Tensor) else model.assignments).to(dev, torch.int32).contiguous()
    counts = torch.as_tensor(np.asarray(model.counts) if not isinstance(
        model.counts, torch.Tensor) else model.counts).to(dev, torch.int32).contiguous()
    return E.DevModel(centers=centers, labels=labels, counts=counts, perm=None, starts=None,
                      status=None, inertia=None, k=int(centers.shape[0]), n=n,
                      host_iters=int(model.n_iter))


def _check_points(x: torch.Tensor, what: str):
    if x.ndim != 2 or x.shape[0] == 0:
        raise ParameterError(f"{what} needs a non-empty [N, D] input, got shape {tuple(x.shape)}")


def kmeans(x, k: int, seed: int, max_iter: int = DEFAULT_MAX_ITER,
           tol: float = DEFAULT_TOL) -> ClusterModel:
    """k-means++ seeded Lloyd clustering (clustering.py:155-167)."""
    t, host = to_device(x)
    _check_points(t, "kmeans")
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    if k > t.shape[0]:
        raise ParameterError(f"k={k} exceeds the number of points N={t.shape[0]}")
    m = E.kmeans_batch([t], [int(k)], [int(seed)], max_iter, tol)[0]
    return export_model(m, host)


def warm_start_update(k_next, prev_centers, max_iter: int = DEFAULT_MAX_ITER,
                      tol: float = DEFAULT_TOL) -> ClusterModel:
    """Lloyd from the previous step's centres (clustering.py:170-179)."""
    t, host = to_device(k_next)
    c, _ = to_device(prev_centers, keep_bf16=False)
    if c.shape[0] > t.shape[0]:
        raise ParameterError(f"C={c.shape[0]} centers exceed N={t.shape[0]} points")
    m = E.lloyd_batch([t], [c], max_iter, tol)[0]
    return export_model(m, host)


def cluster_queries(q, num_clusters: int = DEFAULT_QUERY_CLUSTERS, seed: int = 0,
                    max_iter: int = DEFAULT_MAX_ITER, tol: float = DEFAULT_TOL,
                    init_centers=None):
    """Cluster L2-normalised queries; returns (model, representatives)
    (clustering.py:182-200)."""
    t, host = to_device(q)
    inits = None
    if init_centers is not None:
        inits = [to_device(init_centers, keep_bf16=False)[0]]
    else:
        _check_points(t, "kmeans")
        if num_clusters < 1 or num_clusters > t.shape[0]:
            raise ParameterError(f"k={num_clusters} out of range for N={t.shape[0]}")
    models, reps, _ = E.cluster_queries_batch([t], [int(num_clusters)], [int(seed)], max_iter,
                                              tol, inits)
    return export_model(models[0], host), to_host(reps[0], host)


def nearest_center_mse(x, centers) -> float:
    """Mean squared distance to the nearest centre (clustering.py:203-206)."""
    t, _ = to_device(x)
    c, _ = to_device(centers, keep_bf16=False)
    ra = E._RunningAssign(t, int(c.shape[0]), 1)
    ra.add(c)
    return float(ra.mean_best().item())


def compute_tau(k, stage0: ClusterModel, factor: float = DEFAULT_TAU_FACTOR) -> float:
    """factor x mean token-to-assigned-centre distance (clustering.py:209-215)."""
    t, _ = to_device(k)
    dm = import_model(stage0, int(t.shape[0]))
    return float(E.tau_batch([t], [dm], factor).item())


def multi_stage_cluster_keys(k, tau: float, n_max: int = 1000, m0: int = DEFAULT_STAGE0_CLUSTERS,
                             seed: int = 0, max_iter: int = DEFAULT_MAX_ITER,
                             tol: float = DEFAULT_TOL, stage0: ClusterModel | None = None,
                             stage_schedule=None) -> ClusterModel:
    """Threshold-bounded multi-stage key clustering (clustering.py:218-320)."""
    t, host = to_device(k)
    if t.ndim != 2 or t.shape[0] == 0:
        raise ParameterError(f"multi-stage clustering needs a non-empty [N, D] input, got {tuple(t.shape)}")
    if m0 < 1:
        raise ParameterError(f"m0 must be >= 1, got {m0}")
    if n_max < m0:
        raise ParameterError(f"n_max={n_max} must be >= m0={m0}")
    if tau <= 0.0:
        warnings.warn("tau <= 0: no token can be retired, flagging layer as hard to compress")
    s0 = import_model(stage0, int(t.shape[0])) if stage0 is not None else None
    m = E.multi_stage_batch([t], [float(tau)], int(n_max), int(m0), [int(seed)], max_iter, tol,
                            [s0], schedule=stage_schedule)[0]
    return export_model(m, host, with_inertia=False)


def default_schedule(m0: int):
    def schedule(t, remaining, total):
        return m0 if t == 0 else max(STAGE_FLOOR, math.ceil(m0 * remaining / total))
    return schedule


# ---------------------------------------------------------------------------
# evaluation: per-layer compactness (clustering.py:323-362), on the device
# ---------------------------------------------------------------------------
@dataclass
class CompactnessReport:
    mse_per_head: list    # mean squared token-to-assigned-centre distance per head
    mse_layer: float      # mean over heads
    comp: float           # 1 / mse_layer (inf when exactly zero)
    db_index: float       # Davies-Bouldin index, averaged over heads


def _davies_bouldin(x: torch.Tensor, cen: torch.Tensor, lab: torch.Tensor, cnt: torch.Tensor) -> float:
    """DB = mean_i max_{j != i} (S_i + S_j) / M_ij in f64 (clustering.py:323-337)."""
    c = cen.shape[0]
    if c < 2:
        return 0.0
    dist = torch.linalg.norm(x - cen[lab], dim=1)
    # per-cluster sums without atomics (run-to-run deterministic, like the
    # reference's np.add.at): stable member order, f64 scan, segment ends
    order = torch.sort(lab, stable=True).indices
    csum = torch.cumsum(dist[order], 0)
    ends = torch.cumsum(torch.bincount(lab, minlength=c), 0)
    tot = csum[(ends - 1).clamp(min=0)]
    tot = torch.where(ends > 0, tot, torch.zeros_like(tot))
    s = torch.diff(tot, prepend=torch.zeros(1, dtype=tot.dtype, device=tot.device)) / cnt
    m = torch.cdist(cen, cen)
    ratio = (s[:, None] + s[None, :]) / torch.where(m > 0, m, torch.full_like(m, math.inf))
    ratio.fill_diagonal_(-math.inf)
    return float(ratio.max(dim=1).values.mean().item())


def compactness(k_heads, models) -> CompactnessReport:
    """Per-layer compactness of per-head key clusterings: per-head MSE, the
    layer's 1/MSE and the mean Davies-Bouldin index (clustering.py:340-362),
    evaluated on the GPU in f64 (agrees with the reference to f64 rounding:
    the reductions run in a different order)."""
    if len(k_heads) != len(models):
        raise ParameterError(f"{len(k_heads)} key tensors but {len(models)} models")
    mse, db = [], []
    for x, m in zip(k_heads, models):
        xd, _ = to_device(x, keep_bf16=False)
        xd = xd.double()
        cen = torch.as_tensor(np.asarray(m.centers) if not isinstance(m.centers, torch.Tensor)
                              else m.centers).to(xd.device).double()
        lab = torch.as_tensor(np.asarray(m.assignments) if not isinstance(m.assignments, torch.Tensor)
                              else m.assignments).to(xd.device).long()
        cnt = torch.as_tensor(np.asarray(m.counts) if not isinstance(m.counts, torch.Tensor)
                              else m.counts).to(xd.device).double()
        mse.append(float(((xd - cen[lab]) ** 2).sum(dim=1).mean().item()))
        db.append(_davies_bouldin(xd, cen, lab, cnt))
    mse_layer = float(np.mean(mse))
    return CompactnessReport(mse_per_head=mse, mse_layer=mse_layer,
                             comp=math.inf if mse_layer == 0.0 else 1.0 / mse_layer,
                             db_index=float(np.mean(db)))
