"""Standalone tcgen05 attention probe (dev tool): one tiny dense case."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2604_18348_b200 import engine as E
from oracle import oracle as O
for (H, L, D) in [(1, 128, 64), (1, 300, 64), (2, 1000, 64), (1, 256, 128)]:
    rng = np.random.default_rng(0)
    q, k, v = (rng.normal(size=(H, L, D)).astype(np.float32) for _ in range(3))
    qb, kb, vb = (torch.from_numpy(a).bfloat16().cuda() for a in (q, k, v))
    t = time.time()
    out = E.dense_attention_heads(qb, kb, vb, out_dtype=torch.float32)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    up = lambda a: torch.from_numpy(a).bfloat16().float().numpy()
    rel = max(np.linalg.norm(out[h] - O.full_attention(up(q[h]), up(k[h]), up(v[h]))) /
              np.linalg.norm(O.full_attention(up(q[h]), up(k[h]), up(v[h]))) for h in range(H))
    print((H, L, D), 'rel', rel, 'nan', np.isnan(out).any(), '%.3fs' % (time.time() - t), flush=True)
# sparse case through the pipeline (multiple runs, partial tiles, partial q tiles)
import paper_2604_18348_b200 as P
from paper_2604_18348_b200.synthetic import CRIT7_SPEC, gen_synthetic
q, k, v = gen_synthetic(CRIT7_SPEC, 8192, 64, 1, 1, 0)[0][0]
qb, kb, vb = (torch.from_numpy(a).bfloat16().cuda() for a in (q, k, v))
p = P.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
t = time.time()
out, hs = P.adacluster_attention(qb, kb, vb, P.LayerPolicy(topk=25), P.StepState(), 0, p)
torch.cuda.synchronize()
up = lambda a: torch.from_numpy(a).bfloat16().float().numpy()
r = O.head_step(up(q), up(k), up(v), None, O.HeadState(), 0,
                O.Params(q_clusters=65, topk=25, full_layer_quota=0.0))
o = out.float().cpu().numpy()
print('sparse 8192 rel', np.linalg.norm(o - r.out) / np.linalg.norm(r.out), '%.2fs' % (time.time() - t))
