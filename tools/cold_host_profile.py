"""cProfile of the host side of one cold (step-0) layer step (after two
warm-up cold steps): where the Python/ctypes enqueue time goes."""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [bench.gen_head(cfg, h)[0][0] for h in range(cfg["heads"])]
dev = [torch.stack([torch.from_numpy(x[j]) for x in ins]).to(tdt).cuda() for j in range(3)]
for _ in range(2):
    P.LayerSession(bench._params(P, cfg), out_dtype=tdt).step(*dev)
torch.cuda.synchronize()
sess = P.LayerSession(bench._params(P, cfg), out_dtype=tdt)
pr = cProfile.Profile()
pr.enable()
sess.step(*dev)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
