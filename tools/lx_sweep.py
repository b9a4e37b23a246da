#!/usr/bin/env python
"""Dev timing of compress / decompress for the cfg4 polynomial-order sweep
(spectral fields, 262,144 elements, lx = 6/8/10/12, eps 1e-2..1e-5): field GB/s."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_20731_b200 as PK  # noqa: E402

import os
res = {}
PS = [int(x) for x in os.environ.get("LXS", "6,8,10,12").split(",")]
for P in PS:
    n = 262144
    plan = PK.LossyPlan(P, 1, 0)
    f = torch.empty(n * P ** 3, dtype=torch.float64, device="cuda")
    amp = np.array([10.0 ** (-0.5 * np.sqrt(kx * kx + ky * ky + kz * kz)) for kz in range(P) for ky in range(P)
                    for kx in range(P)])
    plan.generate_spectral(f, n, 0, 0x240720731, amp)
    st = torch.empty(plan.capacity(n), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(f)
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    for eps in (1e-2, 1e-5):
        for _ in range(2):
            plan.compress_async(f, n, eps, st, stats)
        torch.cuda.synchronize()
        nb = int(stats.view(torch.int64)[8].item())
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        K = 5
        e0.record()
        for _ in range(K):
            plan.compress_async(f, n, eps, st, stats)
        e1.record()
        for _ in range(K):
            plan.decompress_async(st, nb, n, out, stats)
        e2.record()
        torch.cuda.synchronize()
        tc, td = e0.elapsed_time(e1) / K, e1.elapsed_time(e2) / K
        F = n * P ** 3 * 8
        res[f"lx{P}_eps{eps:g}"] = {"compress_gbs": F / tc / 1e6, "decompress_gbs": F / td / 1e6,
                                    "field_gbs": F / (tc + td) / 1e6, "C_over_F": nb / F}
    del f, st, out
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
