"""Assignment launches on the real C2 warm-step state (for ncu
--profile-from-start off): key side (bf16, k=100) then query side (f32
planes, k=65), labels-only, all 30 heads per launch."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402
from paper_2604_18348_b200 import _lib as L  # noqa: E402

cfg = dict(bench.CONFIGS["c2"])
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
dev = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).bfloat16().cuda() for j in range(3)]
       for t in range(2)]
sess = P.LayerSession(bench._params(P, cfg), out_dtype=torch.bfloat16)
for i in range(3):
    sess.step(*dev[i % 2])
torch.cuda.synchronize()
st = sess.steady
flags = L.ASSIGN_ALL | L.ASSIGN_LABELS_ONLY
for b in (st.kb, st.qb):
    b.assign(0, flags)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for b in (st.kb, st.qb):
    b.assign(0, flags)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record(); st.kb.assign(0, flags); ev[1].record(); st.qb.assign(0, flags); ev[2].record()
torch.cuda.synchronize()
print(f"key assign {ev[0].elapsed_time(ev[1]):.3f} ms, query assign {ev[1].elapsed_time(ev[2]):.3f} ms (30 heads)")
