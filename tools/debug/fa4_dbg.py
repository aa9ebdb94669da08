import sys, torch, math
sys.path.insert(0, '.')
from paper_2604_18348_b200 import engine as E
torch.manual_seed(0)
for Ln in (128, 200, 256, 384, 1024):
    q = torch.randn(1, Ln, 64, device="cuda").bfloat16()
    k = torch.randn(1, Ln, 64, device="cuda").bfloat16()
    v = torch.randn(1, Ln, 64, device="cuda").bfloat16()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float()[None], k.float()[None], v.float()[None])[0]
    for impl in ("auto", "simt"):
        o = E.dense_attention_heads(q, k, v, out_dtype=torch.float32, impl=impl)
        torch.cuda.synchronize()
        nan = torch.isnan(o).sum().item()
        err = ((o - ref).norm() / ref.norm()).item() if nan == 0 else float('nan')
        rows_bad = torch.isnan(o).any(-1)[0].nonzero().flatten()
        print(Ln, impl, "nan", nan, "rel", err, "bad rows", rows_bad[:8].tolist(), rows_bad.numel())
