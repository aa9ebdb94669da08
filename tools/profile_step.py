"""One profiled warm layer step (for ncu --profile-from-start off).

Runs the C2 layer's cold step and warm-up steps unprofiled, then brackets a
single warm step with cudaProfilerStart/Stop so `ncu --profile-from-start off`
captures exactly one steady-state step's launches.
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--heads", type=int, default=0)
ap.add_argument("--warmup", type=int, default=2)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
if args.heads:
    cfg["heads"] = args.heads
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
dev = []
for t in range(2):
    dev.append([torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).to(tdt).cuda()
                for j in range(3)])
sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
sess.step(*dev[0])
for i in range(args.warmup):
    sess.step(*dev[(i + 1) % 2])
torch.cuda.synchronize()
torch.cuda.profiler.start()
sess.step(*dev[(args.warmup + 1) % 2])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one warm step")
