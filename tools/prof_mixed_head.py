import cProfile, pstats, sys, time, io
sys.argv = ["x", "--no-ref"]
sys.path.insert(0, "tools")
import runpy
import torch
pr = cProfile.Profile()
g = runpy.run_path("tools/mixed_head.py", run_name="__main__")
plan = g["plan"]; ac = g["ac"]
torch.cuda.synchronize()
pr.enable()
plan(ac)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue())
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    plan(ac); torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.split("(")[0][:50]
        t, c = agg.get(k, (0.0, 0))
        agg[k] = (t + e.device_time_total / 1e3, c + 1)
tot = sum(t for t, c in agg.values()); n = sum(c for t, c in agg.values())
print(f"device total {tot:.1f} ms, {n} launches")
for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"{t:9.3f} ms {c:6d} {k}")
