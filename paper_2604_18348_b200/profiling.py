"""CUDA-event phase timing on the launching (current) stream.

``with phase("attention"):`` records a start/stop event pair when a
PhaseTimer is active; ``PhaseTimer.summary()`` synchronises once and returns
milliseconds per phase.  No-op (and sync-free) when no timer is active.
"""

from __future__ import annotations

import contextlib
import time
from collections import defaultdict

import torch

_ACTIVE: "PhaseTimer | None" = None


class PhaseTimer:
    def __init__(self):
        self.events = defaultdict(list)
        self.host = defaultdict(float)  # host seconds inside each phase

    def __enter__(self):
        global _ACTIVE
        self._prev = _ACTIVE
        _ACTIVE = self
        return self

    def __exit__(self, *exc):
        global _ACTIVE
        _ACTIVE = self._prev
        return False

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for name, pairs in self.events.items():
            out[name] = sum(a.elapsed_time(b) for a, b in pairs)
        return out

    def host_ms(self) -> dict:
        return {k: v * 1e3 for k, v in self.host.items()}

    def counts(self) -> dict:
        return {k: len(v) for k, v in self.events.items()}


@contextlib.contextmanager
def phase(name: str):
    t = _ACTIVE
    if t is None:
        yield
        return
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    h0 = time.perf_counter()
    try:
        yield
    finally:
        b.record()
        t.host[name] += time.perf_counter() - h0
        t.events[name].append((a, b))
