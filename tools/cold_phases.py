"""Cold (step-0) layer step by phase: device time between each phase's CUDA
events and host time spent inside the phase, for a fresh session."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402
from paper_2604_18348_b200.profiling import PhaseTimer  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [bench.gen_head(cfg, h)[0][0] for h in range(cfg["heads"])]
dev = [torch.stack([torch.from_numpy(x[j]) for x in ins]).to(tdt).cuda() for j in range(3)]
for rep in range(3):
    sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
    torch.cuda.synchronize()
    with PhaseTimer() as pt:
        t0 = time.perf_counter()
        sess.step(*dev)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    dm, hm = pt.summary(), pt.host_ms()
    print(f"cold step {rep}: wall {wall:.1f} ms; " + ", ".join(
        f"{k} dev {dm[k]:.1f} host {hm[k]:.1f}" for k in dm))
