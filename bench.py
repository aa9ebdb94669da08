"""AdaCluster attention-layer benchmark (BASELINE.json metric).

Workload (default): config C2 — a CogVideoX-2B-shaped attention layer,
30 heads x head_dim 64, L = 70,000 tokens, bf16, synthetic Q/K/V from the
reference generator's criterion-7 spec (compact, 32 components, sigma 1,
separation 80) with per-step drift 5e-4; PipelineParams(q_clusters=65,
topk=25, m0=100, n_max=1000, quota 0).  A *step* is one steady-state
denoising step of the layer (t >= 1): warm-started key and query clustering,
envelopes, TensorQuest top-k, permutation, block-sparse attention and the
centre carry — exactly what the reference runs per step (pipeline.py:344-385).
The step-0 planning pass (k-means++, multi-stage clustering, consolidation)
is timed separately as ``cold_step_ms``.

Multi-GPU: heads are sharded in contiguous blocks over ranks (no cross-head
communication); the per-head outputs are all-gathered over NCCL inside the
timed region.  Time is the max over ranks.

``--impl reference`` times the reference's own CPU implementation of the
path — the unmodified ``adacluster`` package installed in baseline/_ref, run
through its public ``adacluster_attention`` with all host threads (the
bit-exact oracle port in oracle/ only if that install is missing): head 0's
warm steps (a bounded sample) extrapolated to the layer.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "AdaCluster attn-layer ms & tokens/s @70K seq, 1/2/4/8 B200, % TC/HBM roofline vs CPU"
CONFIGS = {
    "c2": dict(name="C2 CogVideoX-2B layer", heads=30, seq=70000, dim=64, dtype="bf16"),
    "c1": dict(name="C1 2x64 L=4096 f32", heads=2, seq=4096, dim=64, dtype="f32"),
    "c3": dict(name="C3 Wan-2.1-1.3B layer", heads=12, seq=32760, dim=128, dtype="bf16"),
    "c4": dict(name="C4 HunyuanVideo layer", heads=24, seq=118800, dim=128, dtype="bf16"),
    # one layer of the C5 40-layer stack (per-layer work; the stack is 40x)
    "c5": dict(name="C5 Wan-2.1-14B layer (1 of 40)", heads=40, seq=75600, dim=128, dtype="bf16"),
}
DRIFT = 5e-4


def _params(P):
    return P.PipelineParams(q_clusters=65, topk=25, m0=100, n_max=1000, full_layer_quota=0.0)


def gen_head(cfg, h: int):
    """Two consecutive steps of head h (per-head seed 1000 + h)."""
    from workload.synthetic import CRIT7_SPEC, gen_synthetic
    spec = dataclasses.replace(CRIT7_SPEC, drift_sigma=DRIFT)
    return gen_synthetic(spec, cfg["seq"], cfg["dim"], 1, 2, 1000 + h)


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------------------
# CPU arms (oracle port; test infrastructure used only as the baseline)
# ---------------------------------------------------------------------------
def cpu_warm_step(q, k, v, key_centers, query_centers):
    from oracle import oracle as O
    st = O.HeadState()
    st.step = 1
    st.key_centers = key_centers
    st.query_centers = query_centers
    p = O.Params(q_clusters=65, topk=25, m0=100, n_max=1000, full_layer_quota=0.0)
    t0 = time.perf_counter()
    r = O.head_step(q, k, v, "sparse", st, 0, p)
    return time.perf_counter() - t0, r, st


def cpu_threads():
    from oracle import oracle as O
    import ctypes
    L = O.lib()
    L.oc_num_threads.restype = ctypes.c_int
    return int(L.oc_num_threads())


def bf16_host(a):
    import torch
    return torch.from_numpy(a).bfloat16().float().numpy()


def _reference_pkg():
    """The UNMODIFIED reference package installed into baseline/_ref
    (pip install --no-index --no-build-isolation --no-deps --target baseline/_ref,
    see DESIGN.md), or None when it is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "adacluster" / "__init__.py").exists():
        return None
    sys.path.insert(0, str(ref))
    import adacluster
    return adacluster


def run_reference(args, cfg, rank):
    """Reference arm: the reference's own CPU implementation of the path on
    the host cores (all threads), through its public API
    (adacluster_attention, pipeline.py:237).  Bounded sample: head 0's warm
    denoising steps, extrapolated over the layer's heads."""
    if rank != 0:
        return
    R = _reference_pkg()
    steps = gen_head(cfg, 0)
    if cfg["dtype"] == "bf16":
        steps = [[tuple(bf16_host(a) for a in steps[t][0])] for t in range(2)]
    (q0, k0, v0), (q1, k1, v1) = steps[0][0], steps[1][0]
    inputs = [(q1, k1, v1), (q0, k0, v0)]
    times = []
    if R is not None:
        from threadpoolctl import threadpool_limits
        cores = os.cpu_count() or 1
        kind = "reference"
        with threadpool_limits(cores):
            p = R.PipelineParams(q_clusters=65, topk=25, m0=100, n_max=1000, full_layer_quota=0.0)
            pol, st = R.LayerPolicy(topk=25), R.StepState()
            t0 = time.perf_counter()
            R.adacluster_attention(q0, k0, v0, pol, st, 0, p)
            cold = time.perf_counter() - t0
            for i in range(args.warmup + args.steps):
                q, k, v = inputs[i % 2]
                t0 = time.perf_counter()
                R.adacluster_attention(q, k, v, pol, st, 0, p)
                dt = time.perf_counter() - t0
                if i >= args.warmup:
                    times.append(dt)
    else:  # reference not installed: the bit-exact oracle port
        from oracle import oracle as O
        kind = "port"
        cores = cpu_threads()
        p = O.Params(q_clusters=65, topk=25, m0=100, n_max=1000, full_layer_quota=0.0)
        st = O.HeadState()
        t0 = time.perf_counter()
        O.head_step(q0, k0, v0, None, st, 0, p)
        cold = time.perf_counter() - t0
        for i in range(args.warmup + args.steps):
            q, k, v = inputs[i % 2]
            t0 = time.perf_counter()
            O.head_step(q, k, v, "sparse", st, 0, p)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    head_s = statistics.mean(times)
    layer_s = head_s * cfg["heads"]
    value = cfg["seq"] / layer_s
    out = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": layer_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (bf16-valued inputs)" if cfg["dtype"] == "bf16" else "f32",
        "data": "synthetic (reference generator, criterion-7 spec, per-head seed 1000+h)",
        "impl": "reference",
        "config": config_block(cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "sample": f"head 0 of {cfg['heads']}, warm step at L={cfg['seq']}, "
                                   f"mean of {args.steps} steps ({head_s:.2f}s/head), "
                                   f"x{cfg['heads']} extrapolated; cold step-0 plan "
                                   f"{cold:.1f}s/head"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cold_step_ms": cold * cfg["heads"] * 1e3,
    }
    print(json.dumps(out), flush=True)


def config_block(cfg, n):
    return {"workload": f"{cfg['name']}: {cfg['heads']} heads x {cfg['dim']}, L={cfg['seq']}, "
                        f"{cfg['dtype']}, criterion-7 synthetic, topk 25, warm denoising step",
            "heads": cfg["heads"], "seq_len": cfg["seq"], "head_dim": cfg["dim"],
            "q_clusters": 65, "topk": 25, "drift_sigma": DRIFT,
            "parallelism": f"head-sharded x{n} + NCCL all-gather of outputs",
            "l2_policy": f"inputs larger than L2 ({3 * cfg['heads'] * cfg['seq'] * cfg['dim'] * (2 if cfg['dtype'] == 'bf16' else 4) / 1e6:.0f} MB of Q/K/V per step, alternating step inputs)"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--attn-impl", default="auto", choices=["auto", "simt"])
    ap.add_argument("--breakdown", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2604_18348_b200 as P
    from paper_2604_18348_b200.profiling import PhaseTimer

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    H, Ln, D = cfg["heads"], cfg["seq"], cfg["dim"]
    per = math.ceil(H / world)
    h0, h1 = min(H, rank * per), min(H, (rank + 1) * per)
    my = list(range(h0, h1))
    tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32

    # ---- inputs: two consecutive denoising steps per head ----
    steps = [[], []]
    for h in my:
        s = gen_head(cfg, h)
        for t in range(2):
            steps[t].append(s[t][0])
    host = []  # pinned host copies, [2][3] tensors [Hr, L, D]
    dev_in = []
    for t in range(2):
        trip = []
        for j in range(3):
            arr = np.stack([steps[t][i][j] for i in range(len(my))]) if my else np.zeros((0, Ln, D), np.float32)
            ht = torch.from_numpy(arr).to(tdt).pin_memory()
            trip.append(ht)
        host.append(trip)
        dev_in.append([x.cuda() for x in trip])
    del steps
    params = _params(P)
    from paper_2604_18348_b200.sharding import ShardedLayerSession, gather_heads

    # process warm-up: the first step-0 of a process also pays one-off costs
    # (library/module load, allocator growth, tensor maps); the reported
    # cold_step_ms is a fresh session's step 0 after it
    first = ShardedLayerSession(H, params, seed=0, layer=0, out_dtype=tdt)
    torch.cuda.synchronize()
    tf = time.perf_counter()
    first.session.step(*dev_in[0])
    torch.cuda.synchronize()
    cold_first_ms = (time.perf_counter() - tf) * 1e3
    del first
    torch.cuda.empty_cache()
    shard = ShardedLayerSession(H, params, seed=0, layer=0, out_dtype=tdt)
    sess = shard.session
    sess.attn_impl = args.attn_impl

    def gather(out):
        return gather_heads(out, H) if world > 1 else out

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- cold step (step 0 planning + sparse step + consolidation) ----
    barrier()
    cold_timer = PhaseTimer()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with cold_timer:
        t0.record()
        gather(sess.step(*dev_in[0]))
        t1.record()
    barrier()
    cold_ms = t0.elapsed_time(t1)
    cold_breakdown = cold_timer.summary()

    # ---- warm-up ----
    for i in range(args.warmup):
        gather(sess.step(*dev_in[(i + 1) % 2]))
    barrier()

    # ---- timed warm steps (device-resident inputs; one CUDA graph per step) ----
    with ClockSampler(local) as clocks:
        barrier()
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record()
        for i in range(args.steps):
            out = gather(sess.step(*dev_in[(args.warmup + i + 1) % 2]))
        stop.record()
        barrier()
    total_ms = start.elapsed_time(stop)
    ms_local = total_ms / max(args.steps, 1)
    ms = ms_local
    if world > 1:
        tt = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # attention kernel time: CUDA events recorded inside the graph around the
    # kernel, on its stream (last timed step); useful FLOPs of that step
    if sess.steady is not None:
        attn_ms = sess.steady.last_times_ms()["attention"]
    else:
        attn_ms = 0.0
    useful = sess.useful_attention_flops()
    # ---- launches per step (profiler replica of one step, untimed) ----
    launches = count_launches(sess, dev_in, gather, args) * args.steps

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        # a serving loop's preallocated pinned result buffers
        host_out = [torch.empty(host[0][0].shape, dtype=tdt).pin_memory() for _ in range(2)]
        for i in range(args.warmup):
            sess.step(*host[(i + 1) % 2], host_out=host_out[(i + 1) % 2])
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.steps):
            j = (args.warmup + i + 1) % 2
            res = sess.step(*host[j], host_out=host_out[j])
            if world > 1:
                gather(res.cuda(non_blocking=True))
        b.record()
        barrier()
        e_ms = a.elapsed_time(b) / max(args.steps, 1)
        if world > 1:
            tt = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        esz = 2 if tdt == torch.bfloat16 else 4
        e2e = {"value": Ln / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": 3 * len(my) * Ln * D * esz,
               "d2h_bytes_per_step": len(my) * Ln * D * esz,
               "api": "paper_2604_18348_b200.LayerSession.step(host pinned Q/K/V)"}

    phases = {}
    if args.breakdown:  # eager replica of one warm step with per-phase events
        timer = PhaseTimer()
        sess.graph = False
        steady, sess.steady = sess.steady, None
        if steady is not None:
            sess.key_centers, sess.query_centers = steady.key_centers(), steady.query_centers()
        with timer:
            sess.step(*dev_in[0])
        phases = timer.summary()
        sess.graph = True
        sess.steady = None
    # ---- dense baseline (torch SDPA: cuDNN / flash on sm_100) ----
    dense = None
    if not args.no_dense and rank == 0 and my:
        dense = dense_sdpa_ms(dev_in[0], tdt)

    # ---- CPU baseline: one head's warm step on the host cores ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(sess, host, args, cfg)
        except Exception as exc:  # baseline failures must not hide the GPU number
            cpu = {"value": None, "unit": "tokens/s", "cores": None, "kind": "port",
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        pk, pk_kind = peaks()
        peak = float(pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1590.0)))
        achieved = useful / (attn_ms / 1e3) / 1e12 if attn_ms > 0 else 0.0
        line = {
            "metric": METRIC, "value": Ln / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic (reference generator, criterion-7 spec, "
                                           "per-head seed 1000+h)",
            "config": config_block(cfg, world),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": attn_traffic(),
                         "kernel": "ac_sparse_attention", "peak_kind": f"{pk_kind} sustained bf16",
                         "useful_flops_per_step": useful, "kernel_ms_per_step": attn_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cold_step_ms": cold_ms,
            "cold_step_first_in_process_ms": cold_first_ms,
            "phases_ms_eager_step": phases,
            "dense_sdpa_ms": dense,
            "density": sess.density(),
        }
        if args.breakdown:
            line["cold_phases_ms"] = cold_breakdown
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def attn_traffic():
    """DRAM bytes (read + write) per launch of the attention kernel from the
    committed ncu --set full capture (profiles/r01_traffic.json), or None."""
    try:
        t = json.loads((ROOT / "profiles" / "r01_traffic.json").read_text())
        return t["k_attn_fa4"]["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


def count_launches(sess, dev_in, gather, args) -> int:
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        gather(sess.step(*dev_in[0]))
        torch.cuda.synchronize()
    n = 0
    for e in prof.events():
        if e.device_type.name == "CUDA" and ("ac::" in e.name or e.name.startswith("k_")):
            n += 1
    return n


def dense_sdpa_ms(trip, tdt):
    import torch
    import torch.nn.functional as F
    q, k, v = (x.unsqueeze(0) for x in trip)  # [1, H, L, D]
    try:
        for _ in range(2):
            F.scaled_dot_product_attention(q, k, v)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            F.scaled_dot_product_attention(q, k, v)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 3
    except RuntimeError as exc:
        return f"failed: {exc}"


def cpu_baseline(sess, host, args, cfg):
    """Head 0's next warm step on the host cores, started from the GPU
    session's carried state (bit-identical to the reference's own): the
    unmodified reference package (baseline/_ref) when installed, else the
    bit-exact oracle port."""
    import torch
    idx = (args.warmup + args.steps + 1) % 2
    q, k, v = (host[idx][j][0].float().numpy() for j in range(3))
    kc = sess.key_centers[0].cpu().numpy()
    qc = sess.query_centers[0].cpu().numpy()
    R = _reference_pkg()
    if R is not None:
        from threadpoolctl import threadpool_limits
        cores = os.cpu_count() or 1
        with threadpool_limits(cores):
            p = R.PipelineParams(q_clusters=65, topk=25, m0=100, n_max=1000, full_layer_quota=0.0)
            pol = R.LayerPolicy(mode="sparse", topk=25)
            st = R.StepState(step=1, key_centers=kc, query_centers=qc)
            t0 = time.perf_counter()
            R.adacluster_attention(q, k, v, pol, st, 0, p)
            dt = time.perf_counter() - t0
        kind, what = "reference", "adacluster (baseline/_ref) with all host threads"
    else:
        dt, _, _ = cpu_warm_step(q, k, v, kc, qc)
        cores, kind = cpu_threads(), "port"
        what = "oracle port: clustering in C threads, attention in numpy/OpenBLAS"
    layer = dt * cfg["heads"]
    return {"value": cfg["seq"] / layer, "unit": "tokens/s", "cores": cores, "kind": kind,
            "sample": f"head 0 of {cfg['heads']}, one warm step at L={cfg['seq']} "
                      f"({dt:.1f}s), x{cfg['heads']} extrapolated; {what}"}


if __name__ == "__main__":
    main()
