"""Multi-rank plumbing for the element-sharded hot path.

Elements are independent under the per-element transform, so
ranks own contiguous z-slabs of the element mesh and exchange no field data.
The only exchange step is the global reduction of the per-rank scalars
(isf_lossy_stats): sums of the energies and byte / coefficient counts and the
max of the Linf terms.  With torch.distributed (NCCL on GPUs, gloo on CPU) this is
three tiny all-reduces; C++ users call isf_lossy_allreduce with an ncclComm_t.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

# isf_lossy_stats field order (include/isf_lossy.h)
F_ERR2, F_NRM2, F_ERRINF, F_UINF, F_DISC2, F_TOT2 = range(6)
I_KEPT, I_BLOCKS, I_STREAM, I_FIELD, I_STATUS = range(6, 11)


def slab_for_rank(E_ax: int, rank: int, world: int):
    """Element z-layers [ez0, ez0 + nz) of rank `rank` when an E_ax^2 x (E_ax*world)
    mesh is split into equal slabs (weak scaling: E_ax^3 elements per rank)."""
    return rank * E_ax, E_ax


def allreduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Global reduction of a [..., 12] float64 stats tensor (bit layout of
    isf_lossy_stats; integer fields reinterpreted as int64).  In place; returns it."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return stats
    flat = stats.reshape(-1, 12)
    sums_f = flat[:, [F_ERR2, F_NRM2, F_DISC2, F_TOT2]].contiguous()
    maxs_f = flat[:, [F_ERRINF, F_UINF]].contiguous()
    ints = flat.view(torch.int64)[:, I_KEPT:I_STATUS + 1].contiguous()
    sums_i = ints[:, :4].contiguous()
    status = ints[:, 4:5].contiguous()
    dist.all_reduce(sums_f, group=group)
    dist.all_reduce(maxs_f, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(sums_i, group=group)
    # status is a bit set: OR over ranks == per-bit MAX
    bits = torch.stack([(status >> b) & 1 for b in range(3)], dim=-1)
    dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
    status = (bits * torch.tensor([1, 2, 4], dtype=bits.dtype, device=bits.device)).sum(-1)
    flat[:, [F_ERR2, F_NRM2, F_DISC2, F_TOT2]] = sums_f
    flat[:, [F_ERRINF, F_UINF]] = maxs_f
    iv = flat.view(torch.int64)
    iv[:, I_KEPT:I_FIELD + 1] = sums_i
    iv[:, I_STATUS:I_STATUS + 1] = status
    return stats


@dataclass
class GlobalReport:
    rel_l2: float           # measured (decompress with original) GLL-weighted relative L2
    rel_linf: float         # measured relative Linf
    rel_l2_estimate: float  # coefficient-space (Parseval) estimate from compress
    cr: float               # Eq. 1 over all ranks
    kept: int
    stream_bytes: int
    field_bytes: int


def global_report(stats: torch.Tensor) -> GlobalReport:
    s = stats.reshape(12).detach().cpu()
    f = s.tolist()
    i = s.view(torch.int64).tolist()
    rl2 = 0.0 if f[F_NRM2] == 0 else math.sqrt(f[F_ERR2] / f[F_NRM2])
    rli = 0.0 if f[F_UINF] == 0 else f[F_ERRINF] / f[F_UINF]
    est = 0.0 if f[F_TOT2] == 0 else math.sqrt(f[F_DISC2] / f[F_TOT2])
    cr = (float(i[I_FIELD]) - float(i[I_STREAM])) / float(i[I_FIELD]) if i[I_FIELD] else 0.0
    return GlobalReport(rl2, rli, est, cr, i[I_KEPT], i[I_STREAM], i[I_FIELD])


def nccl_comm_ptr(group=None, device=None) -> int:
    """The ncclComm_t of torch.distributed's NCCL backend for `device` (0 if the group
    is not NCCL): handed to the C ABI's isf_lossy_allreduce_n."""
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    try:
        be = pg._get_backend(dev)
        return int(be._comm_ptr())
    except Exception:
        return 0


def allreduce_stats_nccl(stats: torch.Tensor, comm: int, cuda_stream) -> None:
    """In-place global reduction of n consecutive isf_lossy_stats records (a [n, 12]
    float64 CUDA tensor) through the C ABI (isf_lossy_allreduce_n: one NCCL group of
    three all-reduces), asynchronous on `cuda_stream`."""
    import ctypes
    from . import _native
    from .lossy import _check
    n = stats.numel() // 12
    _check(_native.lib().isf_lossy_allreduce_n(ctypes.c_void_p(stats.data_ptr()), n, ctypes.c_void_p(comm),
                                               ctypes.c_void_p(cuda_stream.cuda_stream)))
