import sys, torch, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from test_assign_tc import _run
from paper_2604_18348_b200 import _lib as L
for dtype in ["f32", "bf16"]:
    n, k = 200, 16
    g = torch.Generator().manual_seed(n * 131 + k)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    x = (torch.randn(n, 64, generator=g) * 20).to(tdt).cuda()
    idx = torch.randint(0, n, (k,), generator=g)
    c = (x.float().cpu()[idx] + torch.randn(k, 64, generator=g) * 0.5).cuda()
    a = _run([x], [c], L.ASSIGN_MODE_TC)
    e = _run([x], [c], L.ASSIGN_MODE_EXACT)
    bad = (a[0] != e[0]).nonzero().flatten().tolist()
    print(dtype, "bad rows", bad, "fixups", a[3].tolist())
    xd = x.double(); cd = c.double()
    dd = ((xd[:, None, :] - cd[None]) ** 2).sum(-1)
    for r in bad[:10]:
        print(r, "tc", a[0][r].item(), a[1][r].item(), "ex", e[0][r].item(), e[1][r].item(),
              "true", dd[r].argmin().item(), sorted(dd[r].tolist())[:3])
    bb = (a[1].view(torch.int32) != e[1].view(torch.int32)).nonzero().flatten().tolist()
    print("best differs rows", bb[:20])
