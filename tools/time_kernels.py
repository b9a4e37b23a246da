#!/usr/bin/env python
"""Dev timing of compress / decompress on TGV u,v,w,p (cfg2 sizes) for a list of
library builds (ISF_LOSSY_LIB per subprocess); no parity gates, for A/B of
experimental variants.  Usage: tools/time_kernels.py LIB [LIB ...]"""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, torch
sys.path.insert(0, ".")
import paper_2407_20731_b200 as PK
E = 64; n = E ** 3; P = 8
plan = PK.LossyPlan(P, 1, 0)
f = torch.empty(n * 512, dtype=torch.float64, device="cuda")
cap = plan.capacity(n)
st = torch.empty(cap, dtype=torch.uint8, device="cuda")
stats = torch.zeros(12, dtype=torch.float64, device="cuda")
out = torch.empty_like(f)
res = {}
tc = td = 0.0
import os
for which in (range(1) if os.environ.get("TK_ONLY_U") else range(4)):
    plan.generate_tgv(f, E, which)
    for _ in range(3):
        plan.compress_async(f, n, 1e-3, st, stats)
    torch.cuda.synchronize()
    nb = int(stats.view(torch.int64)[8].item())
    if nb == 0:  # variant without the finalize (compress-only timing)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            plan.compress_async(f, n, 1e-3, st, stats)
        e1.record()
        torch.cuda.synchronize()
        tc += e0.elapsed_time(e1) / 10
        td += 1e-9
        continue
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    K = 10
    e0.record()
    for _ in range(K):
        plan.compress_async(f, n, 1e-3, st, stats)
    e1.record()
    for _ in range(K):
        plan.decompress_async(st, nb, n, out, stats)
    e2.record()
    torch.cuda.synchronize()
    tc += e0.elapsed_time(e1) / K
    td += e1.elapsed_time(e2) / K
    res["uvwp"[which]] = [round(e0.elapsed_time(e1) / K, 4), round(e1.elapsed_time(e2) / K, 4)]
F = (1 if os.environ.get("TK_ONLY_U") else 4) * n * 4096
print(json.dumps({"compress_gbs": F / tc / 1e6, "decompress_gbs": F / td / 1e6, "field_gbs": F / (tc + td) / 1e6,
                  "ms_c_d": res}))
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, ISF_LOSSY_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip().splitlines()[-1]
    print(lib, line, flush=True)
