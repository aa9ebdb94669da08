"""Kernel-time summary of one cold (step-0) C2 layer step via torch.profiler
(second cold step of a fresh session, after a warm-up cold step)."""
import sys
from pathlib import Path
import collections
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = []
for h in range(cfg["heads"]):
    ins.append(bench.gen_head(cfg, h)[0][0])
dev = [torch.stack([torch.from_numpy(x[j]) for x in ins]).to(tdt).cuda() for j in range(3)]
P.LayerSession(bench._params(P, cfg), out_dtype=tdt).step(*dev)
torch.cuda.synchronize()
sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    sess.step(*dev)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
tot = collections.Counter(); cnt = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name] += 1
print(f"wall {wall:.1f} ms, kernel sum {sum(tot.values())/1e3:.1f} ms, launches {sum(cnt.values())}")
for k, v in tot.most_common(30):
    print(f"{v/1e3:9.3f} ms {cnt[k]:6d}  {k[:90]}")
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
