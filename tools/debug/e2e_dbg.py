import sys, torch
sys.path.insert(0, '.')
import bench
import paper_2604_18348_b200 as P
cfg = dict(bench.CONFIGS["c2"])
ins = [[], []]
for h in range(cfg["heads"]):
    s = bench.gen_head(cfg, h)
    for t in range(2):
        ins[t].append(s[t][0])
host = [[torch.stack([torch.from_numpy(x[j]) for x in ins[t]]).bfloat16().pin_memory() for j in range(3)] for t in range(2)]
dev = [[x.cuda() for x in trip] for trip in host]
sess = P.LayerSession(bench._params(P), out_dtype=torch.bfloat16)
sess.step(*dev[0]); sess.step(*dev[1]); sess.step(*dev[0])
outs = [torch.empty(host[0][0].shape, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
for i in range(3):
    sess.step(*host[i % 2], host_out=outs[i % 2])
torch.cuda.synchronize()
st = sess.steady
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for trial in range(2):
    e[0].record(); sess.step(*dev[0]); e[1].record(); sess.step(*host[1], host_out=outs[0]); e[2].record()
    torch.cuda.synchronize()
    print("device step", e[0].elapsed_time(e[1]), "host step", e[1].elapsed_time(e[2]), st.last_times_ms())
