import sys, torch
sys.path.insert(0, '.')
import bench
import paper_2604_18348_b200 as P
from paper_2604_18348_b200 import _lib as L
cfg = dict(bench.CONFIGS["c2"]); cfg["heads"] = 4
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
dev = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).bfloat16().cuda() for j in range(3)] for t in range(2)]
sess = P.LayerSession(bench._params(P), out_dtype=torch.bfloat16)
sess.step(*dev[0]); sess.step(*dev[1])
qm, km, _ = sess.last
for name, ms in (("queries", qm), ("keys", km)):
    for h, m in enumerate(ms):
        st = m.status.cpu().tolist()
        print(name, h, "k", m.k, "n_iter", st[L.ST_NITER], "fixups", st[L.ST_FIXUPS], "wide", st[L.ST_WIDE], "n", m.n)
