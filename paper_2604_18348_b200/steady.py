"""Steady-state denoising step of one layer as a single CUDA graph.

After step 0 the reference's per-head work is fixed in shape
(pipeline.py:344-385, t >= 1): warm-started key Lloyd from the carried
centres (``warm_start_update``, clustering.py:170-179), warm-started query
clustering (``cluster_queries(init_centers=...)``, clustering.py:182-200),
envelopes + TensorQuest + top-k (quest.py:61-143) and the gathered sparse
attention (pipeline.py:154-165).  Every data-dependent decision inside that
step (Lloyd convergence, empty-cluster repair, run lengths, work items) is
taken on the device, so the whole step is enqueued once, captured into a
CUDA graph and replayed: no host synchronisation and no per-launch host work
(descriptor uploads, TMA tensor-map encoding) in steady state.

The clustering batches persist across steps: a Lloyd run leaves its final
centres in the batch, which is exactly the next step's warm start
(``_carry_centers`` is a passthrough for t >= 1, pipeline.py:223-234).
"""

from __future__ import annotations

import math
import os

import numpy as np
import torch

from . import _lib as L
from . import engine as E

F32 = torch.float32
I32 = torch.int32


class Workspace:
    """The large per-step buffers of a warm step ([H, L, D]-sized: static
    inputs, normalised queries and their bf16 planes, permuted K/V, the
    padded query layout, output).  A layer stack shares one workspace across
    its layers' graphs (layers run one after another), so a 40-layer stack
    holds one layer's worth of these instead of forty."""

    def __init__(self, H: int, Ln: int, D: int, dtype: torch.dtype, gq: int, out_dtype=None):
        dev = L.device()
        odt = out_dtype or (torch.bfloat16 if dtype == torch.bfloat16 else F32)
        self.key = (H, Ln, D, dtype, gq, odt)
        self.Q = torch.empty((H, Ln, D), dtype=dtype, device=dev)
        self.K = torch.empty((H, Ln, D), dtype=dtype, device=dev)
        self.V = torch.empty((H, Ln, D), dtype=dtype, device=dev)
        self.qn = torch.empty((H, Ln, D), dtype=F32, device=dev)
        self.qdeg = torch.empty(H * Ln, dtype=torch.uint8, device=dev)
        self.planes = (torch.empty(3 * H * Ln * D, dtype=torch.bfloat16, device=dev)
                       if D in (64, 128) else None)
        self.kp = torch.empty_like(self.K)
        self.vp = torch.empty_like(self.V)
        self.qp_cap = Ln + E.TILE * gq
        self.item_cap = (Ln + E.TILE - 1) // E.TILE + gq
        self.qp = torch.empty((H * self.qp_cap, D), dtype=dtype, device=dev)
        self.qidx = torch.empty(H * self.qp_cap + H * gq, dtype=I32, device=dev)
        self.items = torch.empty(H * self.item_cap * L.ITEM_DTYPE.itemsize, dtype=torch.uint8,
                                 device=dev)
        self.items_scratch = torch.empty_like(self.items)  # ac_order_items
        self.out = torch.empty((H, Ln, D), dtype=odt, device=dev)


# AC_ITEM_ORDER=1 issues the attention work items longest first; off by
# default: the layout's head-major order keeps a head's K/V hot in L2 and
# measured the same or faster (C3 5.43-5.47 vs 5.44-5.49 ms, C4 71.7-71.9
# vs 72.2-72.5 ms same box)
_ORDER_ITEMS = os.environ.get("AC_ITEM_ORDER", "0") != "0"
# host path H2D order: every block's Q, then every block's K (default), or
# interleaved Q0 K0 Q1 K1 (AC_H2D_QFIRST=0); e2e C2 29.52 -> 28.04 ms, C4
# 79.4 -> 77.5, C3 8.39 -> 8.34 same box
_H2D_QFIRST = os.environ.get("AC_H2D_QFIRST", "1") != "0"


class SteadyStep:
    """Graph-captured warm step for H heads of [L, D] (bf16 or f32).

    ``step(Q, K, V)`` copies the inputs into the graph's static buffers,
    replays the graph and returns the static output buffer [H, L, D]
    (valid until the next call)."""

    def __init__(self, H: int, Ln: int, D: int, dtype: torch.dtype, params, key_centers: list,
                 query_centers: list, out_dtype=None, use_graph: bool = True, split: int = 0,
                 workspace: Workspace | None = None):
        dev = L.device()
        self.H, self.L, self.D, self.dtype = H, Ln, D, dtype
        self.p = params
        self.out_dtype = out_dtype or (torch.bfloat16 if dtype == torch.bfloat16 else F32)
        gq_set = {int(c.shape[0]) for c in query_centers}
        if len(gq_set) != 1:
            raise ValueError("steady step expects one query-cluster count for all heads")
        gq0 = next(iter(gq_set))
        ws = workspace or Workspace(H, Ln, D, dtype, gq0, self.out_dtype)
        if ws.key != (H, Ln, D, dtype, gq0, self.out_dtype):
            raise ValueError("workspace shape does not match the step")
        self.ws = ws
        self.Q, self.K, self.V = ws.Q, ws.K, ws.V
        p = params
        # ---- key clustering (warm Lloyd, in place across steps) ----
        self.kb = E.Batch([self.K[h] for h in range(H)], [int(c.shape[0]) for c in key_centers],
                          p.max_iter)
        for h, c in enumerate(key_centers):
            self.kb.centers_of(h).copy_(c.to(F32))
        # ---- query clustering on the normalised queries ----
        self.qn, self.qdeg = ws.qn, ws.qdeg
        self.gq = gq0
        self.qb = E.Batch([self.qn[h] for h in range(H)], [self.gq] * H, p.max_iter,
                          planes=ws.planes)
        for h, c in enumerate(query_centers):
            self.qb.centers_of(h).copy_(c.to(F32))
        self.qmodels = [self.qb.model(h) for h in range(H)]
        self.kmodels = [self.kb.model(h) for h in range(H)]
        # ---- representatives (f64 member means) ----
        self.reps = [torch.empty((self.gq, D), dtype=F32, device=dev) for _ in range(H)]
        desc = np.zeros(H, dtype=L.PROBLEM_DTYPE)
        for h, m in enumerate(self.qmodels):
            e = desc[h]
            e["x"] = self.qn[h].data_ptr()
            e["counts"], e["perm"], e["starts"] = m.counts.data_ptr(), m.perm.data_ptr(), m.starts.data_ptr()
            e["n"], e["k"] = m.n, m.k
        self.reps_desc = L.to_device_struct(desc)
        self.reps_ptrs = torch.tensor([r.data_ptr() for r in self.reps], dtype=torch.int64).to(dev)
        # ---- envelopes ----
        self.emax = [torch.empty((m.k, D), dtype=F32, device=dev) for m in self.kmodels]
        self.emin = [torch.empty((m.k, D), dtype=F32, device=dev) for m in self.kmodels]
        desc = np.zeros(H, dtype=L.PROBLEM_DTYPE)
        for h, m in enumerate(self.kmodels):
            e = desc[h]
            e["x"] = self.K[h].data_ptr()
            e["counts"], e["perm"], e["starts"] = m.counts.data_ptr(), m.perm.data_ptr(), m.starts.data_ptr()
            e["n"], e["k"] = m.n, m.k
        self.env_desc = L.to_device_struct(desc)
        self.pmax = torch.tensor([t.data_ptr() for t in self.emax], dtype=torch.int64).to(dev)
        self.pmin = torch.tensor([t.data_ptr() for t in self.emin], dtype=torch.int64).to(dev)
        # ---- selection ----
        self.topks = [min(p.topk, m.k) for m in self.kmodels]
        self.stride = max(self.topks)
        self.runs = torch.zeros((H, self.gq, self.stride, 2), dtype=I32, device=dev)
        self.nruns = torch.zeros((H, self.gq), dtype=I32, device=dev)
        self.scores = [torch.empty((self.gq, m.k), dtype=F32, device=dev) for m in self.kmodels]
        self.selected = [torch.empty((self.gq, t), dtype=torch.int64, device=dev) for t in self.topks]
        self.covered = torch.empty((H, self.gq), dtype=torch.int64, device=dev)
        self.density = torch.empty((H,), dtype=torch.float64, device=dev)
        desc = np.zeros(H, dtype=L.SELECT_DTYPE)
        for h in range(H):
            e = desc[h]
            e["reps"] = self.reps[h].data_ptr()
            e["emax"], e["emin"] = self.emax[h].data_ptr(), self.emin[h].data_ptr()
            e["counts"], e["kstarts"] = self.kmodels[h].counts.data_ptr(), self.kmodels[h].starts.data_ptr()
            e["scores"], e["selected"] = self.scores[h].data_ptr(), self.selected[h].data_ptr()
            e["runs"], e["nruns"] = self.runs[h].data_ptr(), self.nruns[h].data_ptr()
            e["covered"] = self.covered[h].data_ptr()
            e["density"] = self.density[h:h + 1].data_ptr()
            e["gq"], e["c"], e["topk"] = self.gq, self.kmodels[h].k, self.topks[h]
            e["order"] = L.gemm_order(self.gq, self.kmodels[h].k, D)
            e["run_stride"] = self.stride
        self.sel_desc = L.to_device_struct(desc)
        self.scorer = L.SCORERS[p.scorer]
        if p.scorer != "quest":
            raise ValueError("the graph-captured step implements the default 'quest' scorer")
        # ---- attention buffers ----
        da = E._attn_dim(D)
        if da != D:
            raise ValueError("graph-captured step needs head_dim in (16, 32, 64, 128)")
        self.dt = L.dtype_code(self.Q)
        self.kp, self.vp = ws.kp, ws.vp
        self.kperm = self.kb.perm.view(H, Ln)
        self.qperm = self.qb.perm.view(H, Ln)
        self.qlab = self.qb.labels.view(H, Ln)
        self.qcounts = self.qb.counts.view(H, self.gq)
        self.qstarts = self.qb.starts.view(H, self.gq + 1)
        self.gq_t = torch.full((H,), self.gq, dtype=I32, device=dev)
        self.qp_cap, self.item_cap = ws.qp_cap, ws.item_cap
        self.item_rows = int(L.lib().ac_attention_item_rows(self.dt, D))
        self.qp, self.qidx, self.items, self.out = ws.qp, ws.qidx, ws.items, ws.out
        self.items_scratch = ws.items_scratch
        self.odt = L.dtype_code(self.out) if self.out_dtype != F32 else L.DTYPE_F32
        self.scale = float(1.0 / math.sqrt(D))
        self.graph = None
        self.use_graph = use_graph
        # CUDA events recorded inside the graph around the attention kernel
        # and around the clustering (kernel time of the last replay)
        self.ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
        # concurrent clustering chains: head blocks x (keys, queries)
        # one chain pair for small layers (C3: 12 x 32760 -> 5.59 vs 5.70 ms), two
        # head blocks for large ones (C2: 25.97 vs 26.36 ms); AC_STEADY_SPLIT overrides
        if split <= 0:
            split = 1 if H * Ln <= 1_000_000 else 2
        split = int(os.environ.get("AC_STEADY_SPLIT", split))
        self.split = max(1, min(split, H))
        self.hb = (H + self.split - 1) // self.split
        # from pinned host inputs the last head block's data arrives last
        # (PCIe), so smaller blocks shorten the tail after it: twice the
        # device-resident split above 200k rows (e2e C3 8.59 vs 8.75 ms, C4
        # 79.3 vs 80.2; C1 is faster unsplit); AC_STEADY_SPLIT_HOST overrides
        split_h = self.split * 2 if H * Ln > 200_000 else self.split
        split_h = max(1, min(int(os.environ.get("AC_STEADY_SPLIT_HOST", split_h)), H))
        self.hb_host = (H + split_h - 1) // split_h
        nblk = max((H + self.hb - 1) // self.hb, (H + self.hb_host - 1) // self.hb_host)
        self.streams = [torch.cuda.Stream() for _ in range(2 * nblk)]
        self.fork = torch.cuda.Event()
        self.fork_v = torch.cuda.Event()
        self.h2d = torch.cuda.Stream()
        self.q_in = [torch.cuda.Event() for _ in range(nblk)]
        self.k_in = [torch.cuda.Event() for _ in range(nblk)]
        self.host_graphs = {}
        self.joins = [torch.cuda.Event() for _ in range(2 * nblk)]
        # host path: the attention runs in head chunks, each chunk's output
        # copied back (D2H stream) while the next chunk computes: about 34 MB
        # of output per chunk, at most 5 (e2e ms for 1/2/3/5 chunks: C1
        # 1.18/1.44/1.46/1.44, C3 9.93/8.61/8.42/8.62, C2 -/30.8/29.9/29.5,
        # C4 -/81.3/80.2/80.5); AC_STEADY_OUT_CHUNKS overrides
        out_bytes = H * Ln * D * self.out.element_size()
        chunks = min(5, max(1, -(-out_bytes // (34 << 20))))
        self.out_chunks = max(1, min(H, int(os.environ.get("AC_STEADY_OUT_CHUNKS", chunks))))
        self.d2h = torch.cuda.Stream()
        self.vstream = torch.cuda.Stream()
        self.v_in = [torch.cuda.Event() for _ in range(self.out_chunks)]
        self.v_done = [torch.cuda.Event() for _ in range(self.out_chunks)]
        self.chunk_done = [torch.cuda.Event() for _ in range(self.out_chunks)]
        self.d2h_done = torch.cuda.Event()
        # AC_STEADY_TRACE=1: timing events at phase boundaries (trace())
        self.tracing = int(os.environ.get("AC_STEADY_TRACE", "0")) != 0
        self.marks = []
        self._keep = []

    # ------------------------------------------------------------------
    def _mark(self, name: str):
        if self.tracing:
            e = torch.cuda.Event(enable_timing=True, external=True)
            e.record()
            self.marks.append((name, e))
            self._keep.append(e)  # captured graphs reference it: never freed

    def trace(self) -> list:
        """(phase, ms since the step start) of the last replay (AC_STEADY_TRACE=1)."""
        self.ev[2].synchronize()
        torch.cuda.synchronize()
        t0 = self.ev[0]
        return [(n, round(t0.elapsed_time(e), 3)) for n, e in self.marks]

    def _enqueue(self, host=None):
        # programmatic dependent launches of the Lloyd chains (ac_set_pdl)
        with L.pdl(self.H * self.L <= L.PDL_STEADY_ROWS):
            self._enqueue_impl(host)

    def _enqueue_impl(self, host=None):
        self.marks = []
        """Every kernel of one warm step.  Heads are independent and the key
        side (Lloyd, envelopes, K/V permutation) and query side (normalise,
        Lloyd, reps) only meet at selection, so the clustering runs as
        ``2 * self.split`` concurrent chains (key / query x head blocks) on
        separate streams: each Lloyd chain alone is a sequence of
        latency-bound launches that leaves most SMs idle.

        ``host = (hQ, hK, hV, hout)`` (pinned) puts the PCIe copies into the
        graph: every block's Q first (the query chains are the longest), then
        K, then V,
        each overlapping the clustering already running; the result is copied
        back at the end."""
        H, Ln, D = self.H, self.L, self.D
        p = self.p
        kb, qb = self.kb, self.qb
        main = torch.cuda.current_stream()
        hb = self.hb_host if host is not None else self.hb
        blocks = [(h0, min(H, h0 + hb)) for h0 in range(0, H, hb)]
        self.ev[0].record()
        self.fork.record(main)
        # host path: per-block H2D copies on their own stream in the order the
        # chains need them (Q0 Q1 .. K0 K1 .. V: the query chains are the
        # long ones), so block 0's query clustering starts after 1/(3*nblk)
        # of the input has arrived
        if host is not None:
            self.h2d.wait_event(self.fork)
            # AC_H2D_QFIRST=1: every block's Q before any K (the query chains
            # are the long ones), else interleaved Q0 K0 Q1 K1
            order = ([(0, i) for i in range(len(blocks))] + [(1, i) for i in range(len(blocks))]
                     if _H2D_QFIRST else [(t, i) for i in range(len(blocks)) for t in (0, 1)])
            with torch.cuda.stream(self.h2d):
                for t, i in order:
                    h0, h1 = blocks[i]
                    dst = self.Q if t == 0 else self.K
                    dst[h0:h1].copy_(host[t][h0:h1], non_blocking=True)
                    (self.q_in if t == 0 else self.k_in)[i].record(self.h2d)
        for i, (h0, h1) in enumerate(blocks):
            qs, ks = self.streams[2 * i + 1], self.streams[2 * i]
            if host is not None:
                qs.wait_event(self.q_in[i])
                ks.wait_event(self.k_in[i])
            else:
                qs.wait_event(self.fork)
                ks.wait_event(self.fork)
            with torch.cuda.stream(qs):
                # normalisation + the query Batch's prepare (xx, f32 planes) in one pass
                r0 = h0 * Ln
                L.call("ac_l2norm_ex", self.Q[h0].data_ptr(), self.dt, (h1 - h0) * Ln, D,
                       self.qn[h0].data_ptr(), qb.xx.data_ptr() + 4 * r0, self.qdeg.data_ptr() + r0,
                       qb.planes.data_ptr() + 2 * 3 * r0 * D if qb.planes is not None else 0, Ln,
                       L.stream_ptr())
                qb.lloyd_range(h0, h1, p.max_iter, p.tol, inertia=False, prepared=True)
                self._mark(f"qchain{i}")
            with torch.cuda.stream(ks):
                kb.lloyd_range(h0, h1, p.max_iter, p.tol, inertia=False)
                self._mark(f"kchain{i}")
        nc = self.out_chunks
        bounds = [(H * c) // nc for c in range(nc + 1)]
        if host is not None:
            # V per attention chunk, after every Q/K block: a chunk's attention
            # needs only its own heads' V (permuted by the final key clusters)
            with torch.cuda.stream(self.h2d):
                for c in range(nc):
                    h0, h1 = bounds[c], bounds[c + 1]
                    if h1 > h0:
                        self.V[h0:h1].copy_(host[2][h0:h1], non_blocking=True)
                    self.v_in[c].record(self.h2d)
        else:
            self.fork_v.record(main)
        esz = self.K.element_size()
        for i, (h0, h1) in enumerate(blocks):
            # per-block tails of each chain: query reps / key envelopes and
            # the K/V permutation (V after its copy) on the chain's stream
            qs, ks = self.streams[2 * i + 1], self.streams[2 * i]
            with torch.cuda.stream(qs):
                L.call("ac_segment_mean", self.reps_desc.data_ptr() + h0 * L.PROBLEM_DTYPE.itemsize,
                       h1 - h0, L.DTYPE_F32, D, self.gq, self.reps_ptrs.data_ptr() + h0 * 8,
                       L.stream_ptr())
                self.joins[2 * i + 1].record(qs)
            with torch.cuda.stream(ks):
                s = L.stream_ptr()
                hoff = h0 * Ln * D * esz
                L.call("ac_envelopes", self.env_desc.data_ptr() + h0 * L.PROBLEM_DTYPE.itemsize, h1 - h0,
                       self.dt, D, kb.max_k, self.pmax.data_ptr() + h0 * 8, self.pmin.data_ptr() + h0 * 8, s)
                L.call("ac_permute_rows_heads", self.K.data_ptr() + hoff, self.dt, D,
                       self.kperm[h0].data_ptr(), Ln, h1 - h0, self.kp.data_ptr() + hoff, s)
                if host is None:
                    ks.wait_event(self.fork_v)
                    L.call("ac_permute_rows_heads", self.V.data_ptr() + hoff, self.dt, D,
                           self.kperm[h0].data_ptr(), Ln, h1 - h0, self.vp.data_ptr() + hoff, s)
                self.joins[2 * i].record(ks)
        if host is not None:
            # V permutes per attention chunk on their own stream, as each
            # chunk's V arrives (the key clusters are final once the key
            # chains joined)
            for i in range(len(blocks)):
                self.vstream.wait_event(self.joins[2 * i])
            with torch.cuda.stream(self.vstream):
                for c in range(nc):
                    h0, h1 = bounds[c], bounds[c + 1]
                    self.vstream.wait_event(self.v_in[c])
                    if h1 > h0:
                        hoff = h0 * Ln * D * esz
                        L.call("ac_permute_rows_heads", self.V.data_ptr() + hoff, self.dt, D,
                               self.kperm[h0].data_ptr(), Ln, h1 - h0, self.vp.data_ptr() + hoff,
                               L.stream_ptr())
                    self.v_done[c].record(self.vstream)
        for i in range(2 * len(blocks)):
            main.wait_event(self.joins[i])
        s = L.stream_ptr()
        L.call("ac_select", self.sel_desc.data_ptr(), H, D, self.scorer, self.gq, kb.max_k,
               self.stride, s)
        L.call("ac_build_q_layout", self.Q.data_ptr(), self.dt, D, Ln, H, self.qperm.data_ptr(),
               self.qstarts.data_ptr(), self.qcounts.data_ptr(), self.qlab.data_ptr(),
               self.gq_t.data_ptr(), self.gq, self.nruns.data_ptr(), self.stride,
               self.qp.data_ptr(), self.qidx.data_ptr(), self.qp_cap, self.items.data_ptr(),
               self.item_cap, self.item_rows, s)
        self._mark("select+layout")
        self.ev[1].record()
        if host is None:
            self._attend(0, H)
        else:
            for c in range(nc):
                h0, h1 = bounds[c], bounds[c + 1]
                main.wait_event(self.v_done[c])
                if h1 <= h0:
                    continue
                self._attend(h0, h1)
                self.chunk_done[c].record(main)
                self.d2h.wait_event(self.chunk_done[c])
                with torch.cuda.stream(self.d2h):
                    host[3][h0:h1].copy_(self.out[h0:h1], non_blocking=True)
        self.ev[2].record()
        self._mark("attention")
        if host is not None:
            self.d2h_done.record(self.d2h)
            main.wait_event(self.d2h_done)
            self._mark("out")

    def _attend(self, h0: int, h1: int):
        """Attention of the work items of heads [h0, h1) (layout built for all
        heads: items carry absolute head indices), current stream."""
        isz = L.ITEM_DTYPE.itemsize
        if _ORDER_ITEMS:  # longest items first (LPT issue order)
            L.call("ac_order_items", self.items.data_ptr() + h0 * self.item_cap * isz,
                   (h1 - h0) * self.item_cap, self.runs.data_ptr(), self.items_scratch.data_ptr(),
                   L.stream_ptr())
        L.call("ac_sparse_attention", self.qp.data_ptr(), self.H * self.qp_cap, self.qidx.data_ptr(),
               self.kp.data_ptr(), self.vp.data_ptr(), self.dt, self.D, self.L, self.H,
               self.items.data_ptr() + h0 * self.item_cap * isz, (h1 - h0) * self.item_cap,
               self.runs.data_ptr(), self.scale, self.out.data_ptr(), self.odt, L.stream_ptr())

    def _capture(self, host=None):
        # one eager run on a side stream (lazy kernel attributes, workspaces),
        # then capture; the eager run advanced the warm start, so restore it
        kc = self.kb.centers.clone()
        qc = self.qb.centers.clone()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._enqueue(host)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.kb.centers.copy_(kc)
        self.qb.centers.copy_(qc)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._enqueue(host)
        torch.cuda.synchronize()
        return g

    def step_host(self, hQ, hK, hV, hout) -> torch.Tensor:
        """One warm step from pinned host inputs into a pinned host result
        (copies inside the graph, overlapped with the clustering).  One graph
        per distinct set of host buffers (a serving loop reuses a few)."""
        key = tuple(t.data_ptr() for t in (hQ, hK, hV, hout))
        g = self.host_graphs.get(key)
        if g is None:
            if len(self.host_graphs) >= 4:
                self.host_graphs.pop(next(iter(self.host_graphs)))
            g = self.host_graphs[key] = self._capture((hQ, hK, hV, hout))
        g.replay()
        return hout

    def step(self, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor) -> torch.Tensor:
        """One warm step; returns the static output buffer [H, L, D]."""
        for dst, src in ((self.Q, Q), (self.K, K), (self.V, V)):
            if src.data_ptr() != dst.data_ptr():
                dst.copy_(src, non_blocking=True)
        if not self.use_graph:
            self._enqueue()
        else:
            if self.graph is None:
                self.graph = self._capture()
            self.graph.replay()
        return self.out

    def last_times_ms(self) -> dict:
        """Device time of the last step's phases (synchronises)."""
        self.ev[2].synchronize()
        return {"cluster_select_layout": self.ev[0].elapsed_time(self.ev[1]),
                "attention": self.ev[1].elapsed_time(self.ev[2])}

    # ---- state views (device tensors, valid after step) ----
    def key_centers(self) -> list:
        return [self.kb.centers_of(h).clone() for h in range(self.H)]

    def query_centers(self) -> list:
        return [self.qb.centers_of(h).clone() for h in range(self.H)]

    def useful_attention_flops(self) -> torch.Tensor:
        """4·D·Σ_h Σ_g |Q_g|·|S_g| of the last step (device scalar, f64)."""
        return (self.qcounts.double() * self.covered.double()).sum() * 4.0 * self.D
