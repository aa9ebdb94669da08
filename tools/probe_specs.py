"""Key-cluster counts / rounds / flag of the multi-stage planner for
candidate outlier-cloud heads at a config's size (GPU), to pick the C3/C5
spec mix that exercises adaptive key-cluster counts without flagging."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_18348_b200 as P  # noqa: E402
from paper_2604_18348_b200.pipeline import LayerRunner  # noqa: E402
from workload.synthetic import outlier_cloud_head  # noqa: E402

L, D = int(sys.argv[1]), int(sys.argv[2])
params = P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
for frac in (0.0003, 0.001, 0.002, 0.005):
    for tail in (1.0, 6.0):
        q, k, v = outlier_cloud_head(np.random.default_rng(7), L=L, D=D, g=32, frac_tail=frac,
                                     sep=15.0, sigma=0.5, tail_sigma=tail)
        K = torch.from_numpy(k).bfloat16().cuda()[None]
        Q = torch.from_numpy(q).bfloat16().cuda()[None]
        t0 = time.perf_counter()
        plan = LayerRunner(params).plan(Q, K, [0])
        torch.cuda.synchronize()
        m = plan.key_models[0]
        print(f"frac {frac:5.2f} tail {tail:4.1f}: C={m.k:5d} rounds={m.stage_count:3d} "
              f"flag={m.flag_full} plan {time.perf_counter() - t0:.2f}s", flush=True)
