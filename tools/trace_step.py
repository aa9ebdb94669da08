"""Phase timeline of one graph-captured warm step (AC_STEADY_TRACE marks):
when each clustering chain (keys / queries x head blocks) ends, when the
selection + layout ends and when the attention ends (ms from step start)."""
import os
import sys
from pathlib import Path

os.environ["AC_STEADY_TRACE"] = "1"
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
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
    print(name, sess.steady.trace())
    from paper_2604_18348_b200 import _lib as L
    st = sess.steady
    ki = st.kb.status.view(st.H, -1)[:, L.ST_NITER].tolist()
    qi = st.qb.status.view(st.H, -1)[:, L.ST_NITER].tolist()
    print(name, "key Lloyd iterations per head", ki, "query", qi)
    del sess, dev
    torch.cuda.empty_cache()
