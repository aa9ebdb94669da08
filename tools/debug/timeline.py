import sys, os, torch
sys.path.insert(0, '.')
import bench
import paper_2604_18348_b200 as P
from paper_2604_18348_b200 import steady as S
cfg = dict(bench.CONFIGS["c2"])
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
dev = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).bfloat16().cuda() for j in range(3)] for t in range(2)]
# monkeypatch: timing events at block boundaries
orig = S.SteadyStep._enqueue
def enq(self, host=None):
    if not hasattr(self, "tev"):
        nb = len(self.blocks)
        self.tev = {k: [torch.cuda.Event(enable_timing=True, external=True) for _ in range(nb)] for k in ("k", "q", "t0", "t1")}
    # wrap tail to record events
    orig_tail = self._tail
    def tail(b, h0, h1):
        self.tev["t0"][b].record()
        orig_tail(b, h0, h1)
        self.tev["t1"][b].record()
    self._tail = tail
    orig_lr_k = self.kb.lloyd_range
    orig_lr_q = self.qb.lloyd_range
    def lrk(h0, h1, *a, **k):
        orig_lr_k(h0, h1, *a, **k); self.tev["k"][self.blocks.index((h0, h1))].record()
    def lrq(h0, h1, *a, **k):
        orig_lr_q(h0, h1, *a, **k); self.tev["q"][self.blocks.index((h0, h1))].record()
    self.kb.lloyd_range = lrk; self.qb.lloyd_range = lrq
    try:
        orig(self, host)
    finally:
        self._tail = orig_tail; self.kb.lloyd_range = orig_lr_k; self.qb.lloyd_range = orig_lr_q
S.SteadyStep._enqueue = enq
sess = P.LayerSession(bench._params(P), out_dtype=torch.bfloat16)
for i in range(5):
    sess.step(*dev[i % 2])
torch.cuda.synchronize()
st = sess.steady
e0 = st.ev[0]
for b in range(len(st.blocks)):
    f = lambda k: e0.elapsed_time(st.tev[k][b])
    print(f"block {b}: keys done {f('k'):.2f}  queries done {f('q'):.2f}  tail {f('t0'):.2f} -> {f('t1'):.2f}")
print("attention alone (all heads):", st.time_attention())
