#!/usr/bin/env python
"""Dev timing of decompress with the error report (decompress8_kernel<true>) on TGV u at
cfg2 size; the library is taken from ISF_LOSSY_LIB when set."""
import sys, json, torch
sys.path.insert(0, ".")
import paper_2407_20731_b200 as PK
E = 64; n = E ** 3
plan = PK.LossyPlan(8, 1, 0)
f = torch.empty(n * 512, dtype=torch.float64, device="cuda")
st = torch.empty(plan.capacity(n), dtype=torch.uint8, device="cuda")
stats = torch.zeros(12, dtype=torch.float64, device="cuda")
out = torch.empty_like(f)
plan.generate_tgv(f, E, 0)
plan.compress_async(f, n, 1e-3, st, stats); torch.cuda.synchronize()
nb = int(stats.view(torch.int64)[8].item())
for _ in range(3): plan.decompress_async(st, nb, n, out, stats, original=f)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): plan.decompress_async(st, nb, n, out, stats, original=f)
e1.record(); torch.cuda.synchronize()
print("decompress+error GB/s", n * 4096 / (e0.elapsed_time(e1) / 10) / 1e6)
