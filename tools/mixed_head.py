"""Step-0 multi-stage key planning of one hard-to-compress "mixed" head
(LayerSpec(kind="mixed") keys at L = 32,760, D = 128,
where the reference runs ~66 rounds and flags the layer full).

Times the device planner through the drop-in API (kmeans -> compute_tau ->
multi_stage_cluster_keys, numpy in / numpy out), then the unmodified
reference package (baseline/_ref) on the same keys with all host threads,
and checks the two results bit for bit (rounds, flag, Lloyd iterations,
stage MSEs, centres, assignments).

    python tools/mixed_head.py [--seq 32760] [--dim 128] [--seed 0] [--out f.json]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_18348_b200 as ac  # noqa: E402
from workload.synthetic import LayerSpec, gen_synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=32760)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--no-ref", action="store_true")
ap.add_argument("--out", default="")
args = ap.parse_args()

steps = gen_synthetic(LayerSpec(kind="mixed"), args.seq, args.dim, 1, 1, args.seed)
k = np.ascontiguousarray(steps[0][0][1], dtype=np.float32)
seed = args.seed


def plan(mod):
    s0 = mod.kmeans(k, 100, seed)
    tau = mod.compute_tau(k, s0)
    return s0, tau, mod.multi_stage_cluster_keys(k, tau, 1000, 100, seed, stage0=s0)


res = {"workload": f"one LayerSpec(kind='mixed') key head, L={args.seq}, D={args.dim}, f32, "
                   f"seed {seed}: kmeans(m0=100) -> compute_tau -> multi_stage_cluster_keys"}
times = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s0, tau, m = plan(ac)
    torch.cuda.synchronize()
    times.append((time.perf_counter() - t0) * 1e3)
res["gpu_ms"] = times
res["gpu"] = dict(rounds=int(m.stage_count), flag_full=bool(m.flag_full), clusters=int(m.num_clusters),
                  lloyd_iterations=int(m.n_iter), tau=float(tau))
print(json.dumps(res), flush=True)

ref = None
if not args.no_ref:
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    try:
        import adacluster as ref  # the unmodified reference package
    except ImportError as e:
        res["reference"] = f"unavailable: {e}"
if ref is not None:
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=os.cpu_count()):
        t0 = time.perf_counter()
        r0, rtau, rm = plan(ref)
        res["reference_s"] = time.perf_counter() - t0
    res["reference_threads"] = os.cpu_count()
    res["reference"] = dict(rounds=int(rm.stage_count), flag_full=bool(rm.flag_full),
                            clusters=int(rm.num_clusters), lloyd_iterations=int(rm.n_iter),
                            tau=float(rtau))
    res["parity"] = dict(
        tau_equal=bool(np.float64(tau) == np.float64(rtau)),
        stage_mse_equal=bool(list(m.stage_mse) == list(rm.stage_mse)),
        centers_equal=bool(np.array_equal(m.centers, rm.centers)),
        assignments_equal=bool(np.array_equal(m.assignments, rm.assignments)),
        counts_equal=bool(np.array_equal(m.counts, rm.counts)),
        rounds_equal=int(m.stage_count) == int(rm.stage_count),
        flag_equal=bool(m.flag_full) == bool(rm.flag_full),
        iterations_equal=int(m.n_iter) == int(rm.n_iter))
    res["speedup_vs_reference"] = res["reference_s"] * 1e3 / min(times)
print(json.dumps(res), flush=True)
if args.out:
    Path(args.out).write_text(json.dumps(res, indent=1) + "\n")
