"""Phase timeline of one warm C2 step (device-resident and pinned-host paths)."""
import os
import sys
from pathlib import Path
os.environ["AC_STEADY_TRACE"] = "1"
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
host = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).to(tdt).pin_memory() for j in range(3)]
        for t in range(2)]
dev = [[x.cuda() for x in host[t]] for t in range(2)]
sess = P.LayerSession(bench._params(P), out_dtype=tdt)
sess.step(*dev[0])
for i in range(3):
    sess.step(*dev[(i + 1) % 2])
torch.cuda.synchronize()
print("device step:", sess.steady.trace())
hout = torch.empty(dev[0][0].shape, dtype=tdt).pin_memory()
for i in range(4):
    sess.step(*host[i % 2], host_out=hout)
torch.cuda.synchronize()
print("host step:", sess.steady.trace())
