"""ac_order_items: the attention work items are reordered in place, longest
first (Q tiles x (K/V tiles of the runs + 2)), as a permutation of the input
(empty items last).  Results do not depend on the order: every config-scale
parity test runs the steady step with the ordering on."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cost(it, runs):
    if it["q_rows"] <= 0:
        return 0
    r = runs[2 * it["run0"]: 2 * (it["run0"] + it["nruns"])].reshape(-1, 2)
    tiles = int(((r[:, 1] - r[:, 0] + 127) // 128).sum())
    return ((int(it["q_rows"]) + 127) // 128) * (tiles + 2)


@pytest.mark.parametrize("n", [1, 7, 1000, 20000])
def test_order_items_is_a_longest_first_permutation(gpu, n):
    from paper_2604_18348_b200 import _lib as L
    rng = np.random.default_rng(n)
    nruns_tot = 4 * n + 4
    starts = rng.integers(0, 100000, size=nruns_tot)
    lens = rng.integers(1, 2000, size=nruns_tot)
    runs = np.stack([starts, starts + lens], 1).reshape(-1).astype(np.int32)
    items = np.zeros(n, dtype=L.ITEM_DTYPE)
    items["q_row0"] = np.arange(n) * 256
    items["q_rows"] = np.where(rng.random(n) < 0.3, 0, rng.integers(1, 257, size=n))
    items["head"] = rng.integers(0, 30, size=n)
    items["run0"] = rng.integers(0, nruns_tot - 4, size=n)
    items["nruns"] = rng.integers(0, 5, size=n)
    dev = torch.from_numpy(items.view(np.uint8).copy()).cuda()
    scratch = torch.empty_like(dev)
    druns = torch.from_numpy(runs).cuda()
    L.call("ac_order_items", dev.data_ptr(), n, druns.data_ptr(), scratch.data_ptr(), L.stream_ptr())
    out = dev.cpu().numpy().view(L.ITEM_DTYPE)
    # a permutation of the input (q_row0 is unique)
    assert sorted(out["q_row0"].tolist()) == sorted(items["q_row0"].tolist())
    by_row = {int(r): i for i, r in enumerate(items["q_row0"])}
    for o in out:
        assert o.tobytes() == items[by_row[int(o["q_row0"])]].tobytes()
    costs = [min(_cost(o, runs), 4095) for o in out]
    assert all(a >= b for a, b in zip(costs, costs[1:]))
