#!/usr/bin/env python
"""Dev tool: selection-path histogram of compress8 per TGV field (needs a library
built with -DISF_PATHSTATS, given as ISF_LOSSY_LIB)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20731_b200 as PK  # noqa: E402
from paper_2407_20731_b200 import _native  # noqa: E402

E = 64
n = E ** 3
plan = PK.LossyPlan(8, 1, 0)
f = torch.empty(n * 512, dtype=torch.float64, device="cuda")
st = torch.empty(plan.capacity(n), dtype=torch.uint8, device="cuda")
stats = torch.zeros(12, dtype=torch.float64, device="cuda")
lib = _native.lib()
buf = (ctypes.c_ulonglong * 16)()
names = ["zero", "H", "one-move", "radix"] + [f"k={k}" for k in range(8)] + ["k8-15", "k16-63", "k64+", "-"]
for eps in (1e-3, 1e-2):
    for which in range(4):
        plan.generate_tgv(f, E, which)
        lib.isf_debug_pathstats(buf, 1)
        plan.compress_async(f, n, eps, st, stats)
        torch.cuda.synchronize()
        lib.isf_debug_pathstats(buf, 1)
        print(eps, "uvwp"[which], {names[i]: buf[i] for i in range(15) if buf[i]})
