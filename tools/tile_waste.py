"""Tile padding of the sparse attention: useful FLOPs (4·D·Σ|Q_g|·|S_g|)
vs the FLOPs the 128x128 tiles execute (partial query tiles, run tails),
from the work items and key runs of a warm graph step."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2604_18348_b200 as P  # noqa: E402
from paper_2604_18348_b200 import _lib as L  # noqa: E402

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
    for i in range(3):
        sess.step(*dev[i % 2])
    torch.cuda.synchronize()
    st = sess.steady
    D = dev[0][0].shape[-1]
    items = np.frombuffer(st.items.cpu().numpy().tobytes(), dtype=L.ITEM_DTYPE)
    items = items[items["q_rows"] > 0]
    runs = st.runs.cpu().numpy().reshape(-1, 2)
    useful = sess.useful_attention_flops()
    tiles = 0
    run_lens = []
    for it in items:
        r = runs[it["run0"]:it["run0"] + it["nruns"]]
        ln = r[:, 1] - r[:, 0]
        run_lens.append(ln)
        kt = int(np.sum((ln + 127) // 128))
        tiles += ((int(it["q_rows"]) + 127) // 128) * kt
    rl = np.concatenate(run_lens)
    tile_flops = tiles * 128 * 128 * 4 * D
    qr = items["q_rows"]
    print(f"{name}: items {len(items)}, q_rows mean {qr.mean():.1f} (<=128: {np.mean(qr <= 128):.2f}), "
          f"runs/item {np.mean([len(x) for x in run_lens]):.1f}, run len mean {rl.mean():.0f} "
          f"median {np.median(rl):.0f}, useful {useful:.3e} tile {tile_flops:.3e} "
          f"ratio {useful / tile_flops:.3f}; q-tile util {qr.sum() / (np.sum((qr + 127) // 128) * 128):.3f}, "
          f"k-tile util {rl.sum() / (np.sum((rl + 127) // 128) * 128):.3f}")
    del sess, dev
    torch.cuda.empty_cache()
