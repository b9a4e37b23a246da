#!/usr/bin/env python
"""Small driver for ncu captures: cfg2 TGV field `which` (default u), lx=8, one warm
compress + decompress, then one more of each (capture with -k / --launch-skip)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_20731_b200 as PK  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 0
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
n = 64 ** 3
plan = PK.LossyPlan(P, 1, 0)
f = torch.empty(n * P ** 3, dtype=torch.float64, device="cuda")
if P == 8 and which < 4:
    plan.generate_tgv(f, 64, which)
else:
    from oracle import oracle as O
    plan.generate_spectral(f, n, 0, O.SPECTRAL_SEED, O.spectral_amplitudes(P))
cap = plan.capacity(n)
st = torch.empty(cap, dtype=torch.uint8, device="cuda")
stats = torch.zeros(12, dtype=torch.float64, device="cuda")
out = torch.empty_like(f)
for _ in range(2):
    plan.compress_async(f, n, eps, st, stats)
    torch.cuda.synchronize()
    nb = int(stats.view(torch.int64)[8].item())
    plan.decompress_async(st, nb, n, out, stats)
    torch.cuda.synchronize()
print("ok", nb)
