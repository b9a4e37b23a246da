"""World-size-2 check of the element-sharded path on CPU with gloo:
each rank compresses its z-slab (CPU oracle standing in for the device), the
per-rank isf_lossy_stats are reduced with paper_2407_20731_b200.dist, and the
global scalars must equal those of the concatenated single-rank field."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stats_tensor(stc, std):
    t = torch.zeros(12, dtype=torch.float64)
    t[0], t[1], t[2], t[3], t[4], t[5] = std.err2, std.nrm2, std.err_inf, std.u_inf, stc.disc2, stc.tot2
    iv = t.view(torch.int64)
    iv[6], iv[7], iv[8], iv[9], iv[10] = stc.kept, stc.blocks, stc.stream_bytes, stc.field_bytes, stc.status | std.status
    return t


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from paper_2407_20731_b200 import dist as D
    E = 4
    ez0, nz = D.slab_for_rank(E, rank, world)
    u = O.gen_tgv(E, 8, 0, ez0, nz)
    rc, s, stc = O.compress(u, 8, 1, 1e-3, nthreads=1)
    rc2, _, std = O.decompress(s, 8, 1, E * E * nz, original=u, nthreads=1)
    t = _stats_tensor(stc, std)
    if rank == 1:
        t.view(torch.int64)[10] = 2  # a shape flag on one rank must survive the reduction
    D.allreduce_stats(t)
    if rank == 0:
        out.put((t.numpy().tobytes()))
    dist.destroy_process_group()


def test_two_rank_stats_reduction(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    raw = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = torch.frombuffer(bytearray(raw), dtype=torch.float64)
    from paper_2407_20731_b200 import dist as D
    rep = D.global_report(t)
    # single-rank reference over the concatenated 4 x 4 x 8 mesh
    u = oracle.gen_tgv(4, 8, 0, 0, 8)
    rc, s, stc = oracle.compress(u, 8, 1, 1e-3, nthreads=1)
    rc2, _, std = oracle.decompress(s, 8, 1, 128, original=u, nthreads=1)
    assert rep.kept == stc.kept
    hdr_single = oracle.stream_header_bytes(8, 128)
    hdr_ranks = 2 * oracle.stream_header_bytes(8, 64)
    assert rep.stream_bytes - hdr_ranks == stc.stream_bytes - hdr_single  # same values, rank-local headers
    assert rep.field_bytes == stc.field_bytes
    assert abs(rep.rel_l2 - math.sqrt(std.err2 / std.nrm2)) <= 1e-12
    assert rep.rel_linf == std.err_inf / std.u_inf
    assert t.view(torch.int64)[10].item() == 2


def test_slab_partition():
    from paper_2407_20731_b200 import dist as D
    assert [D.slab_for_rank(64, r, 8) for r in range(3)] == [(0, 64), (64, 64), (128, 64)]
