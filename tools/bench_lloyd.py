"""Micro-benchmark of the warm-step query Lloyd chain of one C2 head block
(15 heads x 70000 x 64, normalised f32 queries, 25 iterations): kernel
breakdown and wall time, with the queries in token order or physically
sorted by the previous step's clustering, for both centroid-update modes.

    python tools/bench_lloyd.py [--heads 15] [--config c2]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402
from paper_2604_18348_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--heads", type=int, default=15)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
cfg["heads"] = args.heads
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
dev = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).to(tdt).cuda() for j in range(3)]
       for t in range(2)]
sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
sess.step(*dev[0])
sess.step(*dev[1])  # builds the steady step (split = 2 blocks by default)
st = sess.steady
H, Ln, D = st.H, st.L, st.D
qc0 = st.qb.centers.clone()
perm = st.qb.perm.view(H, Ln).long().clone()  # previous step's member order per head
Q = dev[0][0]
Qs = torch.stack([Q[h][perm[h]] for h in range(H)]).contiguous()
p = st.p


def run(src, mode):
    L.lib().ac_set_update_mode(mode)
    st.qb.centers.copy_(qc0)
    r0 = 0
    L.call("ac_l2norm_ex", src.data_ptr(), st.dt, H * Ln, D, st.qn.data_ptr(), st.qb.xx.data_ptr(),
           st.qdeg.data_ptr(), st.qb.planes.data_ptr() if st.qb.planes is not None else 0, Ln,
           L.stream_ptr())
    st.qb.lloyd_range(0, H, p.max_iter, p.tol, inertia=False, prepared=True)


from torch.profiler import ProfilerActivity, profile  # noqa: E402

for name, src, mode in [("token-order, member-order update", Q, 1),
                        ("token-order, split-chain update", Q, 0),
                        ("sorted, member-order update", Qs, 1),
                        ("sorted, split-chain update", Qs, 0),
                        ("token-order, streamed update", Q, 2)]:
    run(src, mode)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        run(src, mode)
    b.record()
    torch.cuda.synchronize()
    iters = int(st.qb.status.view(H, -1)[:, L.ST_NITER].max().item())
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run(src, mode)
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            k = e.name.split("(")[0][:40]
            t, c = agg.get(k, (0.0, 0))
            agg[k] = (t + e.device_time_total / 1e3 if hasattr(e, "device_time_total") else t, c + 1)
    stv = st.qb.status.view(H, -1).cpu()
    print(f"== {name}: {a.elapsed_time(b) / args.reps:.3f} ms per chain ({iters} iterations)"
          f"  fix-up rows/launch {int(stv[:, L.ST_FIXUPS].sum()) / 26:.0f}, >2 cand "
          f"{int(stv[:, L.ST_WIDE].sum()) / 26:.0f} of {H * Ln}; split-chain fallback dims "
          f"{int((stv[:, L.ST_FLAGS] >> 8).sum())} over {iters} iterations")
    for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:8]:
        print(f"   {t:8.3f} ms  {c:4d}  {k}")
L.lib().ac_set_update_mode(1)
