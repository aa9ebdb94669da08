"""flashinfer dense prefill attention time for an [H, L, D] bf16 layer
(baseline only; run by bench.py in a subprocess with a time limit because
flashinfer JIT-compiles its kernels on a fresh box).  Prints {"ms": ...}."""
import json
import sys

import torch

H, L, D = (int(x) for x in sys.argv[1:4])
import flashinfer  # noqa: E402

q, k, v = (torch.randn(L, H, D, dtype=torch.bfloat16, device="cuda") for _ in range(3))
f = lambda: flashinfer.single_prefill_with_kv_cache(q, k, v)  # noqa: E731
for _ in range(2):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    f()
b.record()
torch.cuda.synchronize()
print(json.dumps({"ms": a.elapsed_time(b) / 3, "backend": "flashinfer.single_prefill_with_kv_cache"}))
