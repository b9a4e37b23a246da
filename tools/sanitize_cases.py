#!/usr/bin/env python
"""Small compress / decompress(+error report) cases for compute-sanitizer runs (dev tool):
  compute-sanitizer --tool racecheck|memcheck|synccheck python tools/sanitize_cases.py [lx ...]"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2407_20731_b200 as PK
from oracle import oracle
Ps = [int(a) for a in sys.argv[1:]] or [4, 6, 12]
for P in Ps:
    nb = 512
    u = oracle.gen_spectral(P, nb)
    f = PK.Field(8, P, 1, torch.from_numpy(u).cuda())
    for eps in (1e-2, 1e-5):
        blk = PK.lossy_compress(f, PK.LossyConfig(eps))
        back, rep = PK.decompress_with_error(blk, f.shape, f)
        back2 = PK.lossy_decompress(blk, f.shape)
        torch.cuda.synchronize()
        print(P, eps, blk.kept_total, rep.rel_l2)
