"""Micro-benchmark of the assignment kernels on a C2-shaped batch
(30 heads x 70000 x 64): tensor-core vs exact FFMA, f32 (queries, k=65)
and bf16 (keys, k=100)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2604_18348_b200 import _lib as L
from paper_2604_18348_b200 import engine as E

H, N, D = int(sys.argv[1]) if len(sys.argv) > 1 else 30, 70000, 64
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tc", "exact"]
g = torch.Generator(device="cuda").manual_seed(0)
for dtype, k in (("f32", 65), ("bf16", 100)):
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    X = (torch.randn(H, N, D, device="cuda", generator=g) * 20).to(tdt)
    if dtype == "f32":
        X = X / X.norm(dim=-1, keepdim=True)
    xs = [X[h] for h in range(H)]
    b = E.Batch(xs, [k] * H, 1)
    for h in range(H):
        b.centers_of(h).copy_(X[h, torch.randint(0, N, (k,), device="cuda", generator=g)].float())
    b.prepare()
    for mode in modes:
        L.call("ac_set_assign_mode", L.ASSIGN_MODE_TC if mode == "tc" else L.ASSIGN_MODE_EXACT)
        for _ in range(2):
            b.assign(0, L.ASSIGN_ALL)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        R = 5
        for _ in range(R):
            b.assign(0, L.ASSIGN_ALL)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        byts = H * N * D * (4 if dtype == "f32" else 2)
        fl = 2.0 * H * N * k * D
        fix = b.status.view(b.P, L.STATUS_WORDS)[:, L.ST_FIXUPS].sum().item()
        print(f"{dtype} k={k} {mode}: {ms:.3f} ms  {byts/ms/1e6:.0f} GB/s  {fl/ms/1e9:.1f} TFLOP/s  fixup rows so far {fix}")
L.call("ac_set_assign_mode", L.ASSIGN_MODE_AUTO)
