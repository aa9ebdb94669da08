"""Per-stream timeline of one cold (step-0) layer step (torch profiler):
for each stream, the span and busy time, and per kernel name the first
start / last end (ms from the step's first kernel) -- which chain is the
critical path of the cold step."""
import sys
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [bench.gen_head(cfg, h)[0][0] for h in range(cfg["heads"])]
dev = [torch.stack([torch.from_numpy(x[j]) for x in ins]).to(tdt).cuda() for j in range(3)]
P.LayerSession(bench._params(P, cfg), out_dtype=tdt).step(*dev)
torch.cuda.synchronize()
sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sess.step(*dev)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
by = defaultdict(list)
for e in ev:
    by[getattr(e, "device_resource_id", 0)].append(e)
print(f"step span {(max(e.time_range.end for e in ev) - t0) / 1e3:.2f} ms, {len(ev)} device events")
for sid, es in sorted(by.items()):
    es.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in es)
    print(f"stream {sid}: {len(es)} events, {(es[0].time_range.start - t0) / 1e3:.2f} .. "
          f"{(es[-1].time_range.end - t0) / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms")
    names = defaultdict(lambda: [1e18, 0, 0, 0.0])
    for e in es:
        n = names[e.name[:60]]
        n[0] = min(n[0], e.time_range.start)
        n[1] = max(n[1], e.time_range.end)
        n[2] += 1
        n[3] += e.time_range.end - e.time_range.start
    for nm, (a, b, c, d) in sorted(names.items(), key=lambda kv: kv[1][0]):
        print(f"    {(a - t0) / 1e3:8.2f} .. {(b - t0) / 1e3:8.2f}  x{c:4d} busy {d / 1e3:7.2f}  {nm}")
