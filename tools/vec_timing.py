#!/usr/bin/env python
"""Dev timing: the lx = 8 vector-field path (components = 3, AoS) against the same data
as three scalar fields (TGV u, v, p at cfg2 size), compress and decompress GB/s."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_20731_b200 as PK  # noqa: E402

E = 64
n = E ** 3
ps = PK.LossyPlan(8, 1, 0)
pv = PK.LossyPlan(8, 3, 0)
comps = []
for w in (0, 1, 3):
    t = torch.empty(n * 512, dtype=torch.float64, device="cuda")
    ps.generate_tgv(t, E, w)
    comps.append(t)
vec = torch.stack(comps, dim=-1).reshape(-1).contiguous()
F = 3 * n * 4096


def run(plan, fields, nel, K=10):
    st = torch.empty(plan.capacity(nel), dtype=torch.uint8, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    out = torch.empty_like(fields[0])
    tc = td = 0.0
    for f in fields:
        for _ in range(2):
            plan.compress_async(f, nel, 1e-3, st, stats)
        torch.cuda.synchronize()
        nb = int(stats.view(torch.int64)[8].item())
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(K):
            plan.compress_async(f, nel, 1e-3, st, stats)
        e[1].record()
        for _ in range(K):
            plan.decompress_async(st, nb, nel, out, stats)
        e[2].record()
        torch.cuda.synchronize()
        tc += e[0].elapsed_time(e[1]) / K
        td += e[1].elapsed_time(e[2]) / K
    return {"compress_gbs": F / tc / 1e6, "decompress_gbs": F / td / 1e6, "field_gbs": F / (tc + td) / 1e6,
            "launches": plan.last_launches()}


print(json.dumps({"scalar_x3": run(ps, comps, n), "vector": run(pv, [vec], n)}))
