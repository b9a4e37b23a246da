"""World-size-2 run of the DEVICE path (SPEC.md:279-280 element-parallel
over disjoint ranges with a deterministic merge): each rank runs the sm_100a kernels
on its element z-slab (both ranks on cuda:0; gloo carries the scalars, since one GPU
cannot host two NCCL ranks), the per-rank statistics are reduced with
paper_2407_20731_b200.dist, and

  * every rank's stream equals the single-rank GPU stream of the same slab,
  * the concatenation of the slabs' streams' blocks equals the single-rank stream of
    the whole mesh (counts, masks, values), and
  * the global report equals the concatenated single-rank run (integers exactly,
    energies to rounding)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

E, P, EPS = 16, 8, 1e-3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, which, tmp):
    import sys
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_2407_20731_b200 as PK
    from paper_2407_20731_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    plan = PK.LossyPlan(P, 1, 0)
    ez0, nz = D.slab_for_rank(E, rank, world)
    n_el = E * E * nz
    vals = torch.empty(n_el * P ** 3, dtype=torch.float64, device="cuda")
    plan.generate_tgv(vals, E, which, ez0=ez0, nz=nz)
    cap = plan.capacity(n_el)
    sbuf = torch.empty(cap, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(vals)
    st = torch.zeros(2, 12, dtype=torch.float64, device="cuda")
    plan.compress_async(vals, n_el, EPS, sbuf, st[0])
    torch.cuda.synchronize()
    nb = int(st[0].view(torch.int64)[8].item())
    plan.decompress_async(sbuf, nb, n_el, out, st[1], original=vals)
    torch.cuda.synchronize()
    np.save(os.path.join(tmp, f"stream{rank}.npy"), sbuf[:nb].cpu().numpy())
    np.save(os.path.join(tmp, f"field{rank}.npy"), vals.cpu().numpy())
    # one record: compress scalars + decompress error scalars
    rec = st[0].clone()
    rec[0:4] = st[1][0:4]
    g = rec.cpu()
    D.allreduce_stats(g)
    if rank == 0:
        np.save(os.path.join(tmp, "global.npy"), g.numpy())
    dist.destroy_process_group()
    plan.close()


@pytest.mark.parametrize("which", [0, 3])
def test_two_rank_device_slabs(native, oracle, which, tmp_path):
    import torch.multiprocessing as mp
    import paper_2407_20731_b200 as PK
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, which, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    # single-rank GPU reference: the whole 16 x 16 x 32 mesh and each slab alone
    plan = PK.get_plan(P, 1, 0)
    n_el = E * E * 2 * E
    whole = torch.empty(n_el * P ** 3, dtype=torch.float64, device="cuda")
    plan.generate_tgv(whole, E, which, ez0=0, nz=2 * E)
    cap = plan.capacity(n_el)
    sb = torch.empty(cap, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(whole)
    st = torch.zeros(2, 12, dtype=torch.float64, device="cuda")
    plan.compress_async(whole, n_el, EPS, sb, st[0])
    torch.cuda.synchronize()
    nbw = int(st[0].view(torch.int64)[8].item())
    plan.decompress_async(sb, nbw, n_el, out, st[1], original=whole)
    torch.cuda.synchronize()
    ws = sb[:nbw].cpu().numpy()
    wc, wm, wv = oracle.parse_stream(ws, P, n_el)
    half = n_el // 2
    off = 0
    for r in range(2):
        srank = np.load(tmp_path / f"stream{r}.npy")
        frank = np.load(tmp_path / f"field{r}.npy")
        # the slab's field is the whole mesh's slab, bit for bit
        assert np.array_equal(frank.view(np.uint64), whole[r * half * 512:(r + 1) * half * 512].cpu().numpy().view(np.uint64))
        # per-rank stream == single-rank GPU stream of the same slab
        x = torch.from_numpy(frank).cuda()
        s1 = torch.empty(plan.capacity(half), dtype=torch.uint8, device="cuda")
        st1 = torch.zeros(12, dtype=torch.float64, device="cuda")
        plan.compress_async(x, half, EPS, s1, st1)
        torch.cuda.synchronize()
        n1 = int(st1.view(torch.int64)[8].item())
        assert np.array_equal(s1[:n1].cpu().numpy(), srank)
        # ... and its blocks are the whole-mesh stream's blocks of that slab
        rc_, rm, rv = oracle.parse_stream(srank, P, half)
        assert np.array_equal(wc[r * half:(r + 1) * half], rc_)
        assert np.array_equal(wm[r * half:(r + 1) * half], rm)
        k = int(rc_.astype(np.int64).sum())
        assert np.array_equal(np.asarray(wv[off:off + k]).view(np.uint64), np.asarray(rv).view(np.uint64))
        off += k
    g = np.load(tmp_path / "global.npy")
    gi = g.view(np.int64)
    w = torch.cat([st[1][0:4], st[0][4:]]).cpu().numpy()
    wi = w.view(np.int64)
    assert gi[6] == wi[6] and gi[7] == wi[7] and gi[9] == wi[9]          # kept, blocks, field bytes
    assert gi[8] == wi[8]                                                # stream bytes (16-B aligned counts)
    assert gi[10] == 0 and wi[10] == 0
    for j in (0, 1, 4, 5):                                               # energies: to rounding
        assert abs(g[j] - w[j]) <= 1e-12 * abs(w[j]) + 1e-300, (j, g[j], w[j])
    assert g[2] == w[2] and g[3] == w[3]                                 # Linf terms: exact max
