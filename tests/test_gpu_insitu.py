"""Async in-situ mode (BASELINE.json configs[4]; SPEC.md:104 handoff rule,
proj/include/isf/staging/staging.hpp:5-9): the streams compressed on the side stream,
concurrently with the solver stand-in, must be byte-identical to a synchronous
compress of the same solver state -- i.e. the event handoff lets the side stream read
each state before the solver overwrites that buffer, and never a torn one."""
import ctypes

import pytest
import torch

import paper_2407_20731_b200 as PK
from paper_2407_20731_b200 import _native
from paper_2407_20731_b200.insitu import AsyncInSitu

pytestmark = pytest.mark.gpu


def _solver_ref(L, dst, src, aux, stream):
    assert L.isf_lossy_solver_standin(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                      ctypes.c_void_p(aux.data_ptr()), dst.numel(), 1e-3,
                                      ctypes.c_void_p(stream.cuda_stream)) == 0


@pytest.mark.parametrize("every", [1, 2, 3])
def test_async_streams_equal_sync(every):
    torch.cuda.set_device(0)
    E = 16
    n_el = E ** 3
    plan = PK.LossyPlan(8, 1, 0)
    fields = []
    for w in range(4):
        t = torch.empty(n_el * 512, dtype=torch.float64, device="cuda")
        plan.generate_tgv(t, E, w)
        fields.append(t)
    torch.cuda.synchronize()
    init = torch.stack(fields).clone()
    ai = AsyncInSitu(plan, fields, n_el, 1e-3)
    steps = 7
    snaps = []
    ai.run(steps, every, True, keep=snaps)
    torch.cuda.synchronize()
    assert [n for n, _, _ in snaps] == [n for n in range(steps) if (n + 1) % every == 0]

    # synchronous replay of the same solver steps, compressing the same states
    L = _native.lib()
    s = torch.cuda.Stream()
    aux = torch.flip(init, dims=[1]).contiguous()
    state = [init.clone(), torch.empty_like(init)]
    cap = plan.capacity(n_el)
    st = torch.empty(cap, dtype=torch.uint8, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    k = 0
    for n in range(steps):
        _solver_ref(L, state[(n + 1) % 2], state[n % 2], aux, s)
        s.synchronize()
        if (n + 1) % every:
            continue
        sn, sstreams, sstats = snaps[k]
        k += 1
        for f in range(4):
            plan.compress_async(state[(n + 1) % 2][f], n_el, 1e-3, st, stats, cuda_stream=s)
            s.synchronize()
            nb = int(stats.view(torch.int64)[8].item())
            assert int(sstats.view(torch.int64)[f, 8].item()) == nb, (n, f)
            assert int(sstats.view(torch.int64)[f, 10].item()) == 0
            assert torch.equal(sstreams[f][:nb], st[:nb]), (n, f)
    # the run really overlapped: the side stream is a separate, lower-priority stream
    assert ai.side.priority >= ai.solver.priority
