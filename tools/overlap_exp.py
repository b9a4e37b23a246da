#!/usr/bin/env python
"""Co-scheduling experiment (cfg2): the bench step (compress + decompress of TGV u, v,
w, p, one stream) against a pipelined step where decompress(field i) runs on a second
stream / plan next to compress(field i + 1).  Prints ms per step for both."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_20731_b200 as PK  # noqa: E402

E, LX, eps = 64, 8, 1e-3
n_el = E ** 3
nv = n_el * LX ** 3
pa, pb = PK.LossyPlan(LX, 1, 0), PK.LossyPlan(LX, 1, 0)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
fields = []
with torch.cuda.stream(sa):
    for w in range(4):
        t = torch.empty(nv, dtype=torch.float64, device="cuda")
        pa.generate_tgv(t, E, w, cuda_stream=sa)
        fields.append(t)
    cap = pa.capacity(n_el)
    strs = [torch.empty(cap, dtype=torch.uint8, device="cuda") for _ in range(4)]
    out = torch.empty(nv, dtype=torch.float64, device="cuda")
    sc = torch.zeros(4, 12, dtype=torch.float64, device="cuda")
    sd = torch.zeros(4, 12, dtype=torch.float64, device="cuda")
sa.synchronize()
for i in range(4):
    pa.compress_async(fields[i], n_el, eps, strs[i], sc[i], cuda_stream=sa)
sa.synchronize()
sizes = [int(x) for x in sc.view(torch.int64)[:, 8].cpu()]


def seq():
    for i in range(4):
        pa.compress_async(fields[i], n_el, eps, strs[i], sc[i], cuda_stream=sa)
        pa.decompress_async(strs[i], sizes[i], n_el, out, sd[i], cuda_stream=sa)


def pipe():
    for i in range(4):
        pa.compress_async(fields[i], n_el, eps, strs[i], sc[i], cuda_stream=sa)
        e = torch.cuda.Event()
        e.record(sa)
        sb.wait_event(e)
        pb.decompress_async(strs[i], sizes[i], n_el, out, sd[i], cuda_stream=sb)
    sa.wait_stream(sb)


res = {}
for name, fn in (("seq", seq), ("pipe", pipe), ("seq2", seq), ("pipe2", pipe)):
    for _ in range(3):
        fn()
    sa.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record(sa)
    for _ in range(K):
        fn()
    e1.record(sa)
    e1.synchronize()
    res[name] = e0.elapsed_time(e1) / K
ok = all(int(x) == 0 for x in sd.view(torch.int64)[:, 10].cpu())
alg = 4 * (2 * nv * 8 + 2 * sum(sizes) / 4)
res["step_frac_seq"] = alg / (res["seq"] * 1e-3) / 6463.3e9
res["step_frac_pipe"] = alg / (res["pipe"] * 1e-3) / 6463.3e9
res["ok"] = ok
print(json.dumps(res))
