#!/usr/bin/env python
"""Dev tool: selection-path histogram of compress8 on cfg4 spectral lx=8 fields
(library built with -DISF_PATHSTATS, given as ISF_LOSSY_LIB)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20731_b200 as PK  # noqa: E402
from paper_2407_20731_b200 import _native  # noqa: E402

n = 262144
P = 8
plan = PK.LossyPlan(P, 1, 0)
f = torch.empty(n * 512, dtype=torch.float64, device="cuda")
amp = np.array([10.0 ** (-0.5 * np.sqrt(kx * kx + ky * ky + kz * kz)) for kz in range(P) for ky in range(P)
                for kx in range(P)])
plan.generate_spectral(f, n, 0, 0x240720731, amp)
st = torch.empty(plan.capacity(n), dtype=torch.uint8, device="cuda")
stats = torch.zeros(12, dtype=torch.float64, device="cuda")
lib = _native.lib()
buf = (ctypes.c_ulonglong * 16)()
names = ["zero", "H", "moves", "general"] + [f"k={k}" for k in range(8)] + ["k8-15", "k16-63", "k64+", "bins-fallback"]
for eps in (1e-2, 1e-3, 1e-5):
    lib.isf_debug_pathstats(buf, 1)
    plan.compress_async(f, n, eps, st, stats)
    torch.cuda.synchronize()
    lib.isf_debug_pathstats(buf, 1)
    print(eps, {names[i]: buf[i] for i in range(16) if buf[i]})
