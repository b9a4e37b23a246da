"""Asynchronous in-situ mode (SPEC.md:104,300-321 async semantics; BASELINE cfg5).

The solver stand-in runs on a high-priority CUDA stream and double-buffers its
state; every `every` steps the freshly written buffer is compressed on a
low-priority side stream.  The handoff rule of the reference
(proj/include/isf/staging/staging.hpp:5-9: the producer may mutate
its buffer only after the handoff completed) becomes two CUDA events:

    solver stream:  step n writes buf[(n+1)%2]; if compressed: record ready(n)
    side stream:    wait ready(n) -> compress all fields of buf[(n+1)%2] -> record done(n)
    solver stream:  step n+2 overwrites buf[(n+1)%2] -> first wait done(n)

Reported: solver time per step with and without the concurrent compression and
the slowdown (T_with - T_alone) / T_alone, all from CUDA events on the solver
stream.
"""
from __future__ import annotations

import ctypes

import torch

from . import _native
from .lossy import IsfError, ErrorCode, LossyPlan


class AsyncInSitu:
    def __init__(self, plan: LossyPlan, fields: list[torch.Tensor], n_elements: int, max_error: float):
        self.plan = plan
        self.n_el = n_elements
        self.eps = float(max_error)
        dev = fields[0].device
        self.dev = dev
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        self.solver = torch.cuda.Stream(dev, priority=-1)   # high priority
        self.side = torch.cuda.Stream(dev, priority=0)      # low priority
        self.nf = len(fields)
        n = fields[0].numel()
        self.n = n
        # double-buffered solver state (all fields stacked) + an auxiliary operand
        self.buf = [torch.stack(fields).contiguous(), torch.empty(self.nf, n, dtype=torch.float64, device=dev)]
        self.aux = torch.flip(self.buf[0], dims=[1]).contiguous()
        cap = plan.capacity(n_elements)
        self.streams = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in range(self.nf)]
        self.stats = torch.zeros(self.nf, 12, dtype=torch.float64, device=dev)
        self.L = _native.lib()

    def _solver_step(self, n: int):
        src, dst = self.buf[n % 2], self.buf[(n + 1) % 2]
        rc = self.L.isf_lossy_solver_standin(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                             ctypes.c_void_p(self.aux.data_ptr()), dst.numel(), 1e-3,
                                             ctypes.c_void_p(self.solver.cuda_stream))
        if rc:
            raise IsfError(ErrorCode(rc - 1), _native.last_error())

    def run(self, steps: int, every: int, compress: bool, keep: list | None = None):
        """`steps` solver steps, compressing every `every`-th state on the side stream.
        keep: optional list that receives (step, [stream copy per field], stats copy) of
        every compression, copied on the side stream (tests)."""
        ev = lambda: torch.cuda.Event(enable_timing=True)
        done = [None, None]
        t0, t1 = ev(), ev()
        torch.cuda.synchronize(self.dev)
        t0.record(self.solver)
        for n in range(steps):
            target = (n + 1) % 2
            if done[target] is not None:          # handoff: compress must have read it
                self.solver.wait_event(done[target])
                done[target] = None
            self._solver_step(n)
            if compress and (n + 1) % every == 0:
                ready = torch.cuda.Event()
                ready.record(self.solver)
                self.side.wait_event(ready)
                for f in range(self.nf):
                    self.plan.compress_async(self.buf[target][f], self.n_el, self.eps, self.streams[f],
                                             self.stats[f], cuda_stream=self.side)
                if keep is not None:
                    with torch.cuda.stream(self.side):
                        keep.append((n, [t.clone() for t in self.streams], self.stats.clone()))
                d = torch.cuda.Event()
                d.record(self.side)
                done[target] = d
        t1.record(self.solver)
        torch.cuda.synchronize(self.dev)
        return t0.elapsed_time(t1) / steps

    def measure(self, steps: int = 40, every: int = 10):
        self.run(4, every, False)                  # warm-up
        self.run(every, every, True)
        alone = self.run(steps, every, False)
        withc = self.run(steps, every, True)
        st = self.stats.view(torch.int64).cpu()
        assert int(st[:, 10].max()) == 0, "compression status flags set"
        return {"solver_ms_per_step_alone": alone, "solver_ms_per_step_with": withc,
                "slowdown": (withc - alone) / alone, "steps": steps, "compress_every": every,
                "fields": self.nf, "solver_bytes_per_step": 3 * self.buf[0].numel() * 8}
