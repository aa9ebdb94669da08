"""Kernel timeline of one graph-replayed warm step (torch profiler / CUPTI):
per stream, the sum of kernel durations vs the span and the gaps between
consecutive kernels -- the launch / dependency latency a PDL or persistent
design would hide."""
import sys
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = dict(bench.CONFIGS[name])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
dev = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).to(tdt).cuda() for j in range(3)]
       for t in range(2)]
sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
for i in range(4):
    sess.step(*dev[i % 2])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sess.step(*dev[0])
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
by = defaultdict(list)
for e in ev:
    by[getattr(e, "device_resource_id", 0)].append(e)
t0 = min(e.time_range.start for e in ev)
t1 = max(e.time_range.end for e in ev)
print(f"{name}: step span {(t1 - t0) / 1e3:.3f} ms, {len(ev)} kernels")
for sid, es in sorted(by.items()):
    es.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in es)
    gaps = [b.time_range.start - a.time_range.end for a, b in zip(es, es[1:])]
    span = es[-1].time_range.end - es[0].time_range.start
    gp = sorted(gaps)
    print(f"  stream {sid}: {len(es)} kernels, busy {busy / 1e3:.3f} ms of span {span / 1e3:.3f} ms, "
          f"gap median {gp[len(gp) // 2] if gp else 0:.1f} us, sum {sum(g for g in gaps if g > 0) / 1e3:.3f} ms")
