import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2604_18348_b200 as P
from workload.synthetic import CRIT7_SPEC, gen_synthetic
q, k, v = gen_synthetic(CRIT7_SPEC, 8192, 64, 1, 1, 0)[0][0]
Q, K, V = (torch.from_numpy(a).bfloat16().cuda()[None] for a in (q, k, v))
params = P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
outs = {}
for impl in ("simt", "auto"):
    s = P.LayerSession(params, attn_impl=impl, graph=False, out_dtype=torch.float32)
    outs[impl] = s.step(Q, K, V)[0]
    qm = s.last[0][0]
a, b = outs["simt"], outs["auto"]
err = (a - b).norm(dim=1) / a.norm(dim=1).clamp_min(1e-9)
bad = (err > 0.05).nonzero().flatten()
print("bad rows", bad.numel(), "of", a.shape[0])
lab = qm.labels.cpu().numpy(); cnt = qm.counts.cpu().numpy(); starts = qm.starts.cpu().numpy(); perm = qm.perm.cpu().numpy()
pos = np.empty_like(perm); pos[perm] = np.arange(len(perm))
for r in bad[:10].tolist():
    g = lab[r]; local = pos[r] - starts[g]
    print("row", r, "cluster", g, "count", cnt[g], "local", local, "tile", local // 128, "pair-item", local // 256, "err", float(err[r]))
