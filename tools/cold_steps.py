"""Wall time of the cold (step-0) layer step of fresh sessions, plus the
time of its phases (AC_COLD_TRACE-free: host perf_counter around step)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [bench.gen_head(cfg, h)[0][0] for h in range(cfg["heads"])]
dev = [torch.stack([torch.from_numpy(x[j]) for x in ins]).to(tdt).cuda() for j in range(3)]
for i in range(6):
    sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess.step(*dev)
    torch.cuda.synchronize()
    print(f"cold step {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms")
    del sess
