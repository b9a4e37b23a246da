#!/usr/bin/env python
"""Dev probe: pinned host <-> device copy bandwidth, one direction and both at once
(the bound of bench.py's e2e leg)."""
import json

import torch

n = 1 << 30  # 1 GiB
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, k=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    s1.synchronize(); s2.synchronize()
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / k / 1e3


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


a, b, c = t(h2d), t(d2h), t(both)
print(json.dumps({"h2d_gbs": n / a / 1e9, "d2h_gbs": n / b / 1e9, "bidir_each_gbs": n / c / 1e9,
                  "e2e_bound_gbs": n / c / 1e9}))
