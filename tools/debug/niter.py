"""n_iter / repairs / fix-ups of the query and key Lloyd runs of a warm C2 step."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402
from paper_2604_18348_b200 import _lib as L  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
dev = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).to(tdt).cuda() for j in range(3)]
       for t in range(2)]
sess = P.LayerSession(bench._params(P), out_dtype=tdt)
sess.step(*dev[0])
for i in range(3):
    sess.step(*dev[(i + 1) % 2])
torch.cuda.synchronize()
st = sess.steady
for name, b in (("query", st.qb), ("key", st.kb)):
    s = b.status.view(b.P, L.STATUS_WORDS).cpu().numpy()
    print(name, "k", b.ks[:4], "n_iter", list(s[:, L.ST_NITER]), "repairs", list(s[:, L.ST_REPAIRS]),
          "fixups", list(s[:, L.ST_FIXUPS])[:6], "wide", list(s[:, L.ST_WIDE])[:6])
    print(name, "counts max/min", [(int(b.counts[o:o + k].max()), int(b.counts[o:o + k].min()))
                                   for o, k in zip([sum(b.kcaps[:i]) for i in range(4)], b.ks[:4])])
