"""AdaCluster attention-layer benchmark (BASELINE.json metric).

Workload (default): config C2 -- a CogVideoX-2B-shaped attention layer,
30 heads x head_dim 64, L = 70,000 tokens, bf16, synthetic Q/K/V from the
reference generator's criterion-7 spec (compact, 32 components, sigma 1,
separation 80) with per-step drift 5e-4; PipelineParams(q_clusters=65,
topk=25, m0=100, n_max=1000, quota 0).  A *step* is one steady-state
denoising step of the layer (t >= 1): warm-started key and query clustering,
envelopes, TensorQuest top-k, permutation, block-sparse attention and the
centre carry -- exactly what the reference runs per step (pipeline.py:344-385).
The step-0 planning pass (k-means++, multi-stage clustering, consolidation)
is timed separately as ``cold_step_ms``.

Other configs (``--config``): c1 (2x64, L=4096, f32, criterion-7 / topk 25),
c1asis (c1 with the reference's defaults: LayerSpec(), topk 64), c3 (Wan-2.1
1.3B layer, 12x128, L=32760, a per-head spec mix so the key-cluster counts
adapt), c4 (HunyuanVideo layer, 24x128, L=118800) and c5 (the Wan-2.1-14B
40-layer stack, 40x128, L=75600, a per-layer spec cycle, quota 0.15: step 0
plans every layer, the worst layers run dense; a step is the whole stack).

Multi-GPU: heads are sharded in balanced contiguous blocks over ranks (no
cross-head communication); the per-head outputs are all-gathered over NCCL
inside the timed region.  Time is the max over ranks.

``--impl reference`` times the reference's own CPU implementation of the
path -- the unmodified ``adacluster`` package installed in baseline/_ref, run
through its public ``adacluster_attention`` with all host threads (the
bit-exact oracle port in oracle/ only if that install is missing): head 0's
warm steps (a bounded sample) extrapolated to the layer (x heads x layers).
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import platform
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
DRIFT = 5e-4


def _specs():
    from workload.synthetic import CRIT7_SPEC, LayerSpec
    crit7 = dataclasses.replace(CRIT7_SPEC, drift_sigma=DRIFT)
    # harder-to-compress compact heads: wider components relative to their
    # separation -> more multi-stage rounds and more key clusters (SURVEY
    # §8(d): adaptive key-cluster counts need a spec mix)
    wide = LayerSpec(kind="compact", gaussian_components=32, component_sigma=2.0,
                     component_separation=40.0, drift_sigma=DRIFT, scale_spread=0.3)
    mid = LayerSpec(kind="compact", gaussian_components=48, component_sigma=1.5,
                    component_separation=60.0, drift_sigma=DRIFT, scale_spread=0.3)
    return {"crit7": crit7, "wide": wide, "mid": mid,
            "default": dataclasses.replace(LayerSpec(), drift_sigma=DRIFT),
            # hard-to-compress heads: tight components plus a sparse outlier
            # cloud (the reference's own adaptive-count workload, scaled):
            # many multi-stage rounds, 120-210 key clusters at 32K-76K tokens
            "outlier1": ("outlier", 0.001), "outlier2": ("outlier", 0.002)}


CONFIGS = {
    "c2": dict(name="C2 CogVideoX-2B layer", heads=30, seq=70000, dim=64, dtype="bf16",
               specs=["crit7"], topk=25, layers=1, quota=0.0),
    "c1": dict(name="C1 2x64 L=4096 f32 (criterion-7, topk 25)", heads=2, seq=4096, dim=64,
               dtype="f32", specs=["crit7"], topk=25, layers=1, quota=0.0),
    "c1asis": dict(name="C1 as the reference runs it (LayerSpec(), PipelineParams() topk 64)",
                   heads=2, seq=4096, dim=64, dtype="f32", specs=["default"], topk=64, layers=1,
                   quota=0.0),
    "c3": dict(name="C3 Wan-2.1-1.3B layer (per-head spec mix, adaptive key counts)", heads=12,
               seq=32760, dim=128, dtype="bf16", specs=["crit7", "outlier1", "outlier2"], topk=25,
               layers=1, quota=0.0),
    "c4": dict(name="C4 HunyuanVideo layer", heads=24, seq=118800, dim=128, dtype="bf16",
               specs=["crit7"], topk=25, layers=1, quota=0.0),
    "c5": dict(name="C5 Wan-2.1-14B 40-layer stack (per-layer spec cycle, quota 0.15)", heads=40,
               seq=75600, dim=128, dtype="bf16", specs=["crit7", "mid", "wide"], topk=25,
               layers=40, quota=0.15, pool=4),
}


def _params(P, cfg):
    return P.PipelineParams(q_clusters=65, topk=cfg["topk"], m0=100, n_max=1000,
                            full_layer_quota=cfg["quota"])


def head_spec(cfg, layer: int, h: int):
    """Spec of (layer, head): per-head cycle for single layers, per-layer cycle
    for the stack."""
    names = cfg["specs"]
    key = names[layer % len(names)] if cfg["layers"] > 1 else names[h % len(names)]
    return _specs()[key]


def gen_spec(spec, L: int, D: int, seed: int):
    """Two consecutive steps of one head of ``spec``."""
    from workload.synthetic import gen_outlier_steps, gen_synthetic
    if isinstance(spec, tuple):
        return gen_outlier_steps(L, D, 2, seed, spec[1], drift_sigma=DRIFT)
    return gen_synthetic(spec, L, D, 1, 2, seed)


def gen_head(cfg, h: int, layer: int = 0):
    """Two consecutive steps of head h (per-head seed 1000 + h)."""
    return gen_spec(head_spec(cfg, layer, h), cfg["seq"], cfg["dim"], 1000 + h)


class ClockSampler:
    """SM clock and throttle-reason sampling DURING the timed region: NVML
    polled every 2 ms from a thread (so even a 20-ms region gets samples);
    nvidia-smi -lms 100 when NVML is unavailable."""

    _NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
              "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.proc = None
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            dev = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(dev, pynvml.NVML_CLOCK_SM)

            def poll():
                while True:
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(dev, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(dev)
                        self.samples.append((float(sm), float(mx), int(rs)))
                    except Exception:  # noqa: BLE001
                        pass
                    if self.stop.wait(0.002):
                        return
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
            except (ValueError, IndexError):
                pass

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self.thread is not None:
            self.thread.join(timeout=1)
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({n for _, _, r in self.samples for n, bit in self._NAMES.items() if r & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "sampler": "nvml 2 ms" if self.proc is None
                else "nvidia-smi 100 ms"}


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def roofline_peak(clocks: dict):
    """Burst bf16 peak when the timed region ran at max SM clock (the burst
    figure was measured at max clock), else the sustained one."""
    pk, kind = peaks()
    sm, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    if sm and mx and sm >= 0.97 * mx and "bf16_tflops" in pk:
        return float(pk["bf16_tflops"]), f"{kind} burst bf16 (kernel ran at {sm:.0f} of {mx:.0f} MHz)"
    return float(pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1400.0))), \
        f"{kind} sustained bf16 (SM clock {sm} of {mx} MHz)"


# ---------------------------------------------------------------------------
# host facts for the CPU baselines
# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def blas_info() -> str:
    try:
        from threadpoolctl import threadpool_info
        inf = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if inf:
            i = inf[0]
            return f"{i.get('internal_api')} {i.get('version')} ({i.get('architecture')}), " \
                   f"{i.get('num_threads')} threads"
    except Exception:  # noqa: BLE001
        pass
    return f"numpy {np.__version__}"


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
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import adacluster
    return adacluster


def ref_warm_step(q, k, v, kc, qc, cfg, threads: int):
    """One warm denoising step of one head through the reference's public
    adacluster_attention (or the oracle port when the reference is absent),
    from carried centres kc/qc.  Returns (seconds, out, labels/selection, kind)."""
    R = _reference_pkg()
    if R is not None:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(threads):
            p = R.PipelineParams(q_clusters=65, topk=cfg["topk"], m0=100, n_max=1000,
                                 full_layer_quota=0.0)
            pol = R.LayerPolicy(mode="sparse", topk=cfg["topk"])
            st = R.StepState(step=1, key_centers=kc, query_centers=qc)
            t0 = time.perf_counter()
            out, hs = R.adacluster_attention(q, k, v, pol, st, 0, p)
            dt = time.perf_counter() - t0
        return dt, out, (hs.q_model.assignments, hs.key_model.assignments,
                         hs.selection.selected), "reference"
    from oracle import oracle as O  # checker only (reference not installed)
    st = O.HeadState()
    st.step, st.key_centers, st.query_centers = 1, kc, qc
    p = O.Params(q_clusters=65, topk=cfg["topk"], m0=100, n_max=1000, full_layer_quota=0.0)
    t0 = time.perf_counter()
    r = O.head_step(q, k, v, "sparse", st, 0, p)
    dt = time.perf_counter() - t0
    return dt, r.out, (r.q_model.assignments, r.key_model.assignments, r.selection.selected), "port"


def run_reference(args, cfg, rank):
    """Reference arm: the reference's own CPU implementation of the path on
    the host cores (all threads), through its public API
    (adacluster_attention, pipeline.py:237).  Bounded sample: head 0's warm
    denoising steps (layer 0), extrapolated over the heads (and layers)."""
    if rank != 0:
        return
    R = _reference_pkg()
    steps = gen_head(cfg, 0)
    if cfg["dtype"] == "bf16":
        steps = [[tuple(bf16_host(a) for a in steps[t][0])] for t in range(2)]
    (q0, k0, v0), (q1, k1, v1) = steps[0][0], steps[1][0]
    inputs = [(q1, k1, v1), (q0, k0, v0)]
    times = []
    cores = os.cpu_count() or 1
    if R is not None:
        from threadpoolctl import threadpool_limits
        kind = "reference"
        with threadpool_limits(cores):
            p = R.PipelineParams(q_clusters=65, topk=cfg["topk"], m0=100, n_max=1000,
                                 full_layer_quota=0.0)
            pol, st = R.LayerPolicy(topk=cfg["topk"]), R.StepState()
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
        p = O.Params(q_clusters=65, topk=cfg["topk"], m0=100, n_max=1000, full_layer_quota=0.0)
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
    units = cfg["heads"] * cfg["layers"]
    layer_s = head_s * units
    value = cfg["seq"] / layer_s
    out = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": layer_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (bf16-valued inputs)" if cfg["dtype"] == "bf16" else "f32",
        "data": data_desc(cfg), "impl": "reference",
        "config": config_block(cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "cpu": cpu_model(), "blas": blas_info(),
                         "sample": f"head 0 of {cfg['heads']} (layer 0), warm step at "
                                   f"L={cfg['seq']}, mean of {args.steps} steps "
                                   f"({head_s:.2f}s/head), x{units} head-steps extrapolated; "
                                   f"cold step-0 plan {cold:.1f}s/head"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cold_step_ms": cold * units * 1e3,
    }
    print(json.dumps(out), flush=True)


def data_desc(cfg) -> str:
    specs = "/".join(cfg["specs"])
    s = f"synthetic (reference generator, {specs} spec, per-head seed 1000+h, drift {DRIFT})"
    if cfg["layers"] > 1:
        s += f"; stack inputs tile a pool of {cfg['pool']} distinct heads per spec over layers x heads"
    return s


def config_block(cfg, n):
    esz = 2 if cfg["dtype"] == "bf16" else 4
    qkv = 3 * cfg["heads"] * cfg["seq"] * cfg["dim"] * esz / 1e6
    return {"workload": f"{cfg['name']}: {cfg['layers']} layer(s) x {cfg['heads']} heads x "
                        f"{cfg['dim']}, L={cfg['seq']}, {cfg['dtype']}, topk {cfg['topk']}, "
                        f"quota {cfg['quota']}, warm denoising step",
            "layers": cfg["layers"], "heads": cfg["heads"], "seq_len": cfg["seq"],
            "head_dim": cfg["dim"], "q_clusters": 65, "topk": cfg["topk"], "drift_sigma": DRIFT,
            "specs": cfg["specs"],
            "parallelism": f"head-sharded x{n} (balanced blocks) + NCCL all-gather of outputs",
            "l2_policy": f"inputs larger than L2 ({qkv:.0f} MB of Q/K/V per layer step, "
                         f"alternating step inputs)"}


# ---------------------------------------------------------------------------
# dense baselines (timed on the same box; never on the product path)
# ---------------------------------------------------------------------------
def _time_cuda(fn, reps=3):
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def dense_baselines(trip, tdt, with_flashinfer=True) -> dict:
    """Dense attention over the same [H, L, D] Q/K/V: cuDNN/torch SDPA,
    flash_attn (FA2) and flashinfer (in a subprocess with a time limit: it
    JIT-compiles on a fresh box).  ms per layer; 'fastest' names the winner."""
    import torch
    import torch.nn.functional as F
    res = {}
    q, k, v = (x.unsqueeze(0) for x in trip)  # [1, H, L, D]
    try:
        res["sdpa_cudnn"] = _time_cuda(lambda: F.scaled_dot_product_attention(q, k, v))
    except RuntimeError as exc:
        res["sdpa_cudnn"] = f"failed: {exc}"[:200]
    if tdt == torch.bfloat16:
        try:
            from flash_attn import flash_attn_func
            qf, kf, vf = (x.transpose(1, 2).contiguous() for x in (q, k, v))  # [1, L, H, D]
            res["flash_attn2"] = _time_cuda(lambda: flash_attn_func(qf, kf, vf))
            del qf, kf, vf
        except Exception as exc:  # noqa: BLE001
            res["flash_attn2"] = f"failed: {exc!r}"[:200]
        if with_flashinfer:
            H, Ln, D = trip[0].shape
            try:
                r = subprocess.run([sys.executable, str(ROOT / "tools" / "dense_flashinfer.py"),
                                    str(H), str(Ln), str(D)], capture_output=True, text=True,
                                   timeout=240)
                line = [x for x in r.stdout.splitlines() if x.startswith("{")]
                res["flashinfer"] = json.loads(line[-1])["ms"] if line else \
                    f"failed: {(r.stderr or r.stdout)[-200:]}"
            except subprocess.TimeoutExpired:
                res["flashinfer"] = "failed: timed out (JIT compile)"
    nums = {k2: v2 for k2, v2 in res.items() if isinstance(v2, float)}
    res["fastest"] = min(nums, key=nums.get) if nums else None
    res["fastest_ms"] = nums[res["fastest"]] if nums else None
    return res


def dense_e2e_ms(host_trip, tdt, chunks: int = 4, reps: int = 3) -> float:
    """The fastest dense kernel (cuDNN SDPA) end to end from the same pinned
    host Q/K/V into a pinned host result: head chunks pipelined over three
    streams (H2D of chunk c+1 and D2H of chunk c-1 overlap the attention of
    chunk c), so the dense baseline gets the same copy overlap as ours."""
    import torch
    import torch.nn.functional as F
    hq, hk, hv = host_trip
    H = hq.shape[0]
    out_h = torch.empty(hq.shape, dtype=tdt).pin_memory()
    dq, dk, dv = (torch.empty(hq.shape, dtype=tdt, device="cuda") for _ in range(3))
    do = torch.empty(hq.shape, dtype=tdt, device="cuda")
    s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    bounds = [(H * c) // chunks for c in range(chunks + 1)]

    def run():
        main = torch.cuda.current_stream()
        s_in.wait_stream(main)
        s_c.wait_stream(main)
        s_out.wait_stream(main)
        for c in range(chunks):
            h0, h1 = bounds[c], bounds[c + 1]
            if h1 <= h0:
                continue
            with torch.cuda.stream(s_in):
                for src, dst in ((hq, dq), (hk, dk), (hv, dv)):
                    dst[h0:h1].copy_(src[h0:h1], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            s_c.wait_event(ev_in)
            with torch.cuda.stream(s_c):
                do[h0:h1] = F.scaled_dot_product_attention(
                    dq[h0:h1].unsqueeze(0), dk[h0:h1].unsqueeze(0), dv[h0:h1].unsqueeze(0))[0]
                ev_c = torch.cuda.Event()
                ev_c.record(s_c)
            s_out.wait_event(ev_c)
            with torch.cuda.stream(s_out):
                out_h[h0:h1].copy_(do[h0:h1], non_blocking=True)
        main.wait_stream(s_out)
        main.synchronize()  # result ready on the host, as for LayerSession.step

    return _time_cuda(run, reps)


def count_launches(step_fn) -> int:
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step_fn()
        torch.cuda.synchronize()
    n = 0
    for e in prof.events():
        if e.device_type.name == "CUDA" and ("ac::" in e.name or e.name.startswith("k_")
                                             or "fa::" in e.name or "asg::" in e.name):
            n += 1
    return n


def attn_traffic(dim: int):
    """DRAM bytes (read + write) per launch of the attention kernel from the
    committed ncu --set full capture, or None."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            t = json.loads((ROOT / "profiles" / name).read_text())
        except (OSError, ValueError):
            continue
        key = "k_attn_fa4" if dim == 64 else "k_attn_fa4_d128"
        if key in t:
            return t[key]["dram_bytes_per_launch"]
    return None


def rel_l2(ref, x) -> float:
    ref = np.asarray(ref, np.float64)
    x = np.asarray(x, np.float64)
    return float(np.linalg.norm(ref - x) / max(np.linalg.norm(ref), 1e-30))


def dense_f32_head(q, k, v):
    """Dense attention of one head in f32 on the device (evaluation only)."""
    import torch
    import torch.nn.functional as F
    tq, tk, tv = (torch.as_tensor(a).float().cuda()[None, None] for a in (q, k, v))
    with torch.nn.attention.sdpa_kernel([torch.nn.attention.SDPBackend.EFFICIENT_ATTENTION,
                                         torch.nn.attention.SDPBackend.MATH]):
        return F.scaled_dot_product_attention(tq, tk, tv)[0, 0].cpu().numpy()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# GPU arm: one layer (c1-c4)
# ---------------------------------------------------------------------------
def run_layer(args, cfg, world, rank, local):
    import torch
    import torch.distributed as dist
    import paper_2604_18348_b200 as P
    from paper_2604_18348_b200.profiling import PhaseTimer
    from paper_2604_18348_b200.sharding import ShardedLayerSession, head_block

    H, Ln, D = cfg["heads"], cfg["seq"], cfg["dim"]
    h0, h1 = head_block(H, world, rank)
    my = list(range(h0, h1))
    tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32

    # ---- inputs: two consecutive denoising steps per head ----
    steps = [[], []]
    for h in my:
        s = gen_head(cfg, h)
        for t in range(2):
            steps[t].append(s[t][0])
    host, dev_in = [], []
    for t in range(2):
        trip = []
        for j in range(3):
            arr = np.stack([steps[t][i][j] for i in range(len(my))]) if my else \
                np.zeros((0, Ln, D), np.float32)
            trip.append(torch.from_numpy(arr).to(tdt).pin_memory())
        host.append(trip)
        dev_in.append([x.cuda() for x in trip])
    del steps
    params = _params(P, cfg)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # process warm-up: the first step-0 of a process also pays one-off costs
    first = ShardedLayerSession(H, params, seed=0, layer=0, out_dtype=tdt)
    barrier()
    tf = time.perf_counter()
    first.step_local(*dev_in[0])
    barrier()
    cold_first_ms = (time.perf_counter() - tf) * 1e3
    # (the first session's buffers go back to the caching allocator: the
    # timed cold step is a new layer's step 0 in a running process)
    del first
    shard = ShardedLayerSession(H, params, seed=0, layer=0, out_dtype=tdt)
    sess = shard.session

    def step(i):
        return shard.step(*dev_in[i % 2])

    # ---- cold step (step 0 planning + sparse step + consolidation) ----
    barrier()
    cold_timer = PhaseTimer()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with cold_timer:
        t0.record()
        step(0)
        t1.record()
    barrier()
    cold_ms = t0.elapsed_time(t1)
    cold_breakdown = cold_timer.summary()
    for i in range(args.warmup):
        step(i + 1)
    barrier()

    # ---- timed warm steps (device-resident inputs; one CUDA graph per step) ----
    with ClockSampler(local) as clocks:
        barrier()
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for i in range(args.steps):
            step(args.warmup + i + 1)
        stop.record()
        barrier()
    ms = max_over_ranks(start.elapsed_time(stop) / max(args.steps, 1), world)
    attn_ms = sess.steady.last_times_ms()["attention"] if sess.steady is not None else 0.0
    useful = sess.useful_attention_flops() if my else 0.0
    launches = count_launches(lambda: step(0)) * args.steps

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        esz = 2 if tdt == torch.bfloat16 else 4
        if world == 1:
            host_out = [torch.empty(host[0][0].shape, dtype=tdt).pin_memory() for _ in range(2)]

            def e2e_step(i):
                j = i % 2
                return sess.step(*host[j], host_out=host_out[j])  # ready on return
            d2h = len(my) * Ln * D * esz
        else:
            full_out = [torch.empty((H, Ln, D), dtype=tdt).pin_memory() for _ in range(2)]

            def e2e_step(i):  # H2D of this rank's heads, step, all-gather, D2H of all heads
                j = i % 2
                ins = [x.to("cuda", non_blocking=True) for x in host[j]]
                full_out[j].copy_(shard.step(*ins), non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return full_out[j]
            d2h = H * Ln * D * esz
        for i in range(args.warmup):
            e2e_step(i + 1)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.steps):
            e2e_step(args.warmup + i + 1)
        b.record()
        barrier()
        e_ms = max_over_ranks(a.elapsed_time(b) / max(args.steps, 1), world)
        e2e = {"value": Ln / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": 3 * len(my) * Ln * D * esz, "d2h_bytes_per_step": d2h,
               "api": "LayerSession.step(host pinned Q/K/V) -> host result (N=1); "
                      "ShardedLayerSession.step + D2H of the gathered layer (N>1)"}

    phases = {}
    if args.breakdown and my:  # eager replica of one warm step with per-phase events
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
    dense = None
    if not args.no_dense and rank == 0 and my:
        dense = dense_baselines(dev_in[0], tdt)
        if not args.no_e2e and world == 1:
            try:
                dense["sdpa_cudnn_e2e_ms"] = dense_e2e_ms(host[0], tdt)
            except RuntimeError as exc:
                dense["sdpa_cudnn_e2e_ms"] = f"failed: {exc}"[:200]

    # ---- parity block + CPU baseline (rank 0, N = 1) ----
    parity, cpu = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            parity, cpu = parity_and_cpu(sess, host, dev_in, args, cfg)
        except Exception as exc:  # noqa: BLE001 -- baseline failures must not hide the GPU number
            cpu = {"value": None, "unit": "tokens/s", "cores": None, "kind": "port",
                   "sample": f"failed: {exc!r}"[:300]}

    if rank == 0:
        clk = clocks.summary()
        if cfg["dtype"] == "bf16":
            peak, peak_kind = roofline_peak(clk)
        else:  # f32 inputs run the CUDA-core kernel (the 1e-4 parity bar needs f32 math)
            mhz = clk.get("sm_max_mhz") or 1965.0
            peak = 148 * 128 * 2 * mhz / 1e6
            peak_kind = f"nominal FP32 FFMA peak (148 SMs x 128 lanes x 2 x {mhz:.0f} MHz)"
        achieved = useful / (attn_ms / 1e3) / 1e12 if attn_ms > 0 else 0.0
        kname = ("k_attn_fa4" if D == 64 else "k_attn_fa4_d128") if cfg["dtype"] == "bf16" \
            else "k_attn_simt (f32)"
        line = {
            "metric": METRIC, "value": Ln / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": data_desc(cfg),
            "config": config_block(cfg, world),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": attn_traffic(D),
                         "kernel": f"ac_sparse_attention ({kname})", "peak_kind": peak_kind,
                         "useful_flops_per_step": useful, "kernel_ms_per_step": attn_ms},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "parity": parity,
            "cold_step_ms": cold_ms, "cold_step_first_in_process_ms": cold_first_ms,
            "phases_ms_eager_step": phases, "dense_ms": dense,
            "density": sess.density() if my else None,
            "key_clusters_rank0": [int(c.shape[0]) for c in sess.key_centers] if my else [],
        }
        if dense and dense.get("fastest_ms"):
            line["speedup_vs_fastest_dense"] = dense["fastest_ms"] / ms
            if e2e and isinstance(dense.get("sdpa_cudnn_e2e_ms"), float):
                # both from the same pinned host buffers into a host result
                line["e2e_speedup_vs_dense_e2e"] = dense["sdpa_cudnn_e2e_ms"] / e2e["ms_per_step"]
        if args.breakdown:
            line["cold_phases_ms"] = cold_breakdown
        print(json.dumps(line), flush=True)


def parity_and_cpu(sess, host, dev_in, args, cfg):
    """One more warm step of the GPU session on input ``idx`` and the
    reference's warm step of heads 0 (and 1) from the SAME carried centres on
    the same (bf16-rounded) input: label / selection agreement, rel-L2 of the
    GPU output against the reference's, both against dense attention; the
    reference's times give the CPU baseline (all threads, heads 0-1; one
    thread, head 0)."""
    idx = (args.warmup + args.steps + 1) % 2
    nh = min(2, host[idx][0].shape[0])
    kcs = [sess.key_centers[h].cpu().numpy() for h in range(nh)]
    qcs = [sess.query_centers[h].cpu().numpy() for h in range(nh)]
    out = sess.step(*dev_in[idx]).float().cpu().numpy()
    st = sess.steady
    gq = [st.qmodels[h].labels.cpu().numpy() for h in range(nh)]
    gk = [st.kmodels[h].labels.cpu().numpy() for h in range(nh)]
    gs = [st.selected[h].cpu().numpy() for h in range(nh)]
    cores = os.cpu_count() or 1
    times, par = [], []
    kind = "reference"
    for h in range(nh):
        q, k, v = (host[idx][j][h].float().numpy() for j in range(3))
        dt, rout, (rq, rk, rsel), kind = ref_warm_step(q, k, v, kcs[h], qcs[h], cfg, cores)
        times.append(dt)
        dense = dense_f32_head(q, k, v)
        par.append({"head": h, "q_label_agreement": float(np.mean(gq[h] == np.asarray(rq))),
                    "k_label_agreement": float(np.mean(gk[h] == np.asarray(rk))),
                    "selected_equal_frac": float(np.mean(np.all(gs[h] == np.asarray(rsel), axis=1))),
                    "rel_l2_vs_reference": rel_l2(rout, out[h]),
                    "rel_l2_vs_dense": rel_l2(dense, out[h]),
                    "reference_rel_l2_vs_dense": rel_l2(dense, rout)})
    q, k, v = (host[idx][j][0].float().numpy() for j in range(3))
    dt1, _, _, _ = ref_warm_step(q, k, v, kcs[0], qcs[0], cfg, 1)
    head_s = statistics.mean(times)
    units = cfg["heads"] * cfg["layers"]
    layer = head_s * units
    cpu = {"value": cfg["seq"] / layer, "unit": "tokens/s", "cores": cores, "kind": kind,
           "cpu": cpu_model(), "blas": blas_info(),
           "one_thread": {"value": cfg["seq"] / (dt1 * units), "unit": "tokens/s", "cores": 1,
                          "head_s": dt1},
           "sample": f"heads 0..{nh - 1} of {cfg['heads']}: one warm step each at L={cfg['seq']} "
                     f"({', '.join(f'{t:.1f}s' for t in times)}) with all {cores} threads, "
                     f"mean x{units} extrapolated; 1 thread: head 0 ({dt1:.1f}s)"}
    parity = {"heads": par,
              "q_label_agreement": min(p["q_label_agreement"] for p in par),
              "k_label_agreement": min(p["k_label_agreement"] for p in par),
              "selected_equal_frac": min(p["selected_equal_frac"] for p in par),
              "rel_l2_vs_reference": max(p["rel_l2_vs_reference"] for p in par),
              "rel_l2_vs_dense": max(p["rel_l2_vs_dense"] for p in par),
              "reference_rel_l2_vs_dense": max(p["reference_rel_l2_vs_dense"] for p in par),
              "against": f"{kind} (same carried centres, same bf16-rounded inputs)"}
    return parity, cpu


# ---------------------------------------------------------------------------
# GPU arm: the C5 layer stack
# ---------------------------------------------------------------------------
def run_stack(args, cfg, world, rank, local):
    import torch
    import torch.distributed as dist
    import paper_2604_18348_b200 as P
    from paper_2604_18348_b200.sharding import head_block

    H, Ln, D, NL = cfg["heads"], cfg["seq"], cfg["dim"], cfg["layers"]
    h0, h1 = head_block(H, world, rank)
    tdt = torch.bfloat16
    # pool of distinct heads per spec (2 steps each), on the device
    names = cfg["specs"]
    pool = {}
    for si, nm in enumerate(names):
        for j in range(cfg["pool"]):
            s = gen_spec(_specs()[nm], Ln, D, 5000 + 100 * si + j)
            pool[(nm, j)] = [[torch.from_numpy(s[t][0][x]).to(tdt).cuda() for x in range(3)]
                             for t in range(2)]

    def layer_inputs(l, t):
        nm = names[l % len(names)]
        heads = [pool[(nm, (7 * l + h) % cfg["pool"])][t] for h in range(h0, h1)]
        return [torch.stack([hd[x] for hd in heads]) if heads else
                torch.empty((0, Ln, D), dtype=tdt, device="cuda") for x in range(3)]

    params = _params(P, cfg)
    stack = P.StackSession(NL, H, params, seed=0, out_dtype=tdt)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    tp0 = time.perf_counter()
    modes = stack.plan([tuple(layer_inputs(l, 0)[:2]) for l in range(NL)])
    barrier()
    plan_ms = (time.perf_counter() - tp0) * 1e3
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for l in range(NL):
        p = stack.step_layer(l, *layer_inputs(l, 0))
        if hasattr(p, "wait"):
            p.wait()
    a1.record()
    barrier()
    step0_ms = a0.elapsed_time(a1)

    def warm_step(t, ev=None):
        pend = []
        for l in range(NL):
            if ev is not None:
                ev[l].record()
            pend.append(stack.step_layer(l, *layer_inputs(l, t)))
        if ev is not None:
            ev[NL].record()
        for p in pend:
            if hasattr(p, "wait"):
                p.wait()

    for i in range(args.warmup):
        warm_step((i + 1) % 2)
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(NL + 1)]
    with ClockSampler(local) as clocks:
        barrier()
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for i in range(args.steps):
            warm_step((args.warmup + i + 1) % 2, ev if i == args.steps - 1 else None)
        stop.record()
        barrier()
    ms = max_over_ranks(start.elapsed_time(stop) / max(args.steps, 1), world)
    layer_ms = [ev[l].elapsed_time(ev[l + 1]) for l in range(NL)]
    if rank == 0:
        clk = clocks.summary()
        sparse_ms = [m for m, md in zip(layer_ms, modes) if md == "sparse"]
        full_ms = [m for m, md in zip(layer_ms, modes) if md == "full"]
        line = {
            "metric": METRIC, "value": Ln / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": data_desc(cfg), "config": config_block(cfg, world),
            "stack": {"modes": modes, "full_layers": modes.count("full"),
                      "layer_ms_last_step": layer_ms,
                      "sparse_layer_ms_mean": statistics.mean(sparse_ms) if sparse_ms else None,
                      "full_layer_ms_mean": statistics.mean(full_ms) if full_ms else None,
                      "mse_layer": stack.mse_layer, "plan_ms": plan_ms,
                      "step0_ms": step0_ms,
                      "input_assembly": "each layer's [H, L, D] Q/K/V stacked from the device "
                                        "pool inside the timed region"},
            "clocks": clk, "gpu_launches": None, "cpu_baseline": None, "e2e": None,
            "roofline": None,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--breakdown", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    stack = cfg["layers"] > 1
    if args.steps is None:
        args.steps = 3 if stack else 20
    if args.warmup is None:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if stack:
            run_stack(args, cfg, world, rank, local)
        else:
            run_layer(args, cfg, world, rank, local)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
