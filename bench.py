#!/usr/bin/env python
"""Benchmark of the in-situ lossy-compression hot path (BASELINE.json metric:
"Field GB/s compressed+decompressed at 1/2/4/8 B200; % of HBM roofline").

Workload (BASELINE.json configs[1]): per GPU a 64^3 = 262,144
element mesh, lx = 8, fp64, four scalar fields u/v/w/p of the t=0 Taylor-Green
vortex (4 x 1 GiB = 4.29 GB), RelativeL2 max_error 1e-3.  One step = compress +
decompress of all four fields plus the global all-reduce of error / ratio scalars
(NCCL, N > 1).  Multi-GPU = weak scaling: rank r owns the element slab
ez in [64 r, 64 r + 64) of a 64 x 64 x 64N mesh (cfg3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints one JSON line (rank 0).  `value` = sum over ranks of field bytes / max over
ranks of the device time (CUDA events, inputs resident in HBM, inputs 4.3 GB >> L2
so no flush is needed); `e2e` = the same metric through the host-buffer C ABI
(isf_lossy_compress_host / isf_lossy_decompress_host: H2D, kernels, D2H inside the
timed region).  `--impl reference` times the reference CPU path (the oracle port of
SPEC.md:222-239; the reference ships no implementation) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import queue
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E_AX = 64
LX = 8
EPS = 1e-3
FIELDS = ("u", "v", "w", "p")
METRIC = "Field GB/s compressed+decompressed (TGV u/v/w/p, 262144 elements lx=8 fp64 per GPU, RelativeL2 1e-3)"
UNIT = "GB/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 20 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else None
        sm = sorted(v for v in (num(s[0]) for s in self.samples) if v is not None)
        mx = max((v for v in (num(s[1]) for s in self.samples) if v is not None), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        pw = [v for v in (num(s[6]) for s in self.samples) if v is not None]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples), "power_w_max": max(pw) if pw else None}


def cpu_reference(n_samples_el: int, steps: int, warmup: int, threads: int):
    """The reference CPU path (oracle port) on a bounded sample of the workload:
    the first `n_samples_el` elements (z-layers) of each of the four TGV fields."""
    import numpy as np
    from oracle import oracle as O
    O.build()
    nz = max(1, n_samples_el // (E_AX * E_AX))
    fields = [O.gen_tgv(E_AX, LX, w, 0, nz, nthreads=threads) for w in range(4)]
    n_el = E_AX * E_AX * nz
    fbytes = sum(f.nbytes for f in fields)

    def one():
        for f in fields:
            rc, s, st = O.compress(f, LX, 1, EPS, nthreads=threads)
            assert rc == 0
            rc, out, st2 = O.decompress(s, LX, 1, n_el, nthreads=threads)
            assert rc == 0

    for _ in range(warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    return fbytes / dt / 1e9, dt, n_el, fbytes


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    gbs, dt, n_el, fbytes = cpu_reference(args.cpu_sample_elements, args.steps, args.warmup, threads)
    sample = (f"first {n_el} elements ({n_el // (E_AX * E_AX)} z-layers) of each of u,v,w,p "
              f"({fbytes / 1e9:.3f} GB/step), OpenMP {threads} threads")
    line = {
        "metric": METRIC, "value": gbs, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (TGV t=0 at GLL nodes)",
        "config": {"workload": "cfg2 sample: TGV u/v/w/p lx=8 eps=1e-3", "elements_per_gpu": E_AX ** 3,
                   "lx": LX, "fields": 4, "max_error": EPS, "parallelism": "cpu"},
        "impl": "reference",
        "cpu_baseline": {"value": gbs, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": gbs, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--cpu-sample-elements", type=int, default=8 * 64 * 64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--eps", type=float, default=EPS)
    ap.add_argument("--no-async", action="store_true")
    ap.add_argument("--async-steps", type=int, default=20)
    ap.add_argument("--async-every", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "native" else args.warmup
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2407_20731_b200 as PK

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    eps = args.eps
    plan = PK.LossyPlan(LX, 1, local)
    n_el = E_AX ** 3
    nvals = n_el * LX ** 3
    fbytes_field = nvals * 8
    cap = plan.capacity(n_el)
    hdr = plan.header_bytes(n_el)
    stream = torch.cuda.Stream(dev)
    # in-situ producer stand-in: TGV u/v/w/p on device for this rank's slab
    fields = []
    with torch.cuda.stream(stream):
        for w in range(4):
            t = torch.empty(nvals, dtype=torch.float64, device=dev)
            plan.generate_tgv(t, E_AX, w, ez0=rank * E_AX, nz=E_AX, cuda_stream=stream)
            fields.append(t)
        streams = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in range(4)]
        out = torch.empty(nvals, dtype=torch.float64, device=dev)
        stats_c = torch.zeros(4, 12, dtype=torch.float64, device=dev)
        stats_d = torch.zeros(4, 12, dtype=torch.float64, device=dev)
    stream.synchronize()

    # first pass: stream sizes (needed by decompress) + correctness gates
    sizes = []
    for i in range(4):
        plan.compress_async(fields[i], n_el, eps, streams[i], stats_c[i], cuda_stream=stream)
    stream.synchronize()
    ci = stats_c.view(torch.int64).cpu().numpy()
    cf = stats_c.cpu().numpy()
    for i in range(4):
        assert ci[i, 10] == 0, f"compress status {ci[i, 10]}"
        sizes.append(int(ci[i, 8]))
    for i in range(4):
        plan.decompress_async(streams[i], sizes[i], n_el, out, stats_d[i], original=fields[i], cuda_stream=stream)
    stream.synchronize()
    df = stats_d.cpu().numpy()
    di = stats_d.view(torch.int64).cpu().numpy()
    rel_l2 = [math.sqrt(df[i, 0] / df[i, 1]) if df[i, 1] > 0 else 0.0 for i in range(4)]
    rel_linf = [df[i, 2] / df[i, 3] if df[i, 3] > 0 else 0.0 for i in range(4)]
    for i in range(4):
        assert di[i, 10] == 0, f"decompress status {di[i, 10]}"
        assert rel_l2[i] <= eps * (1 + 1e-9), (FIELDS[i], rel_l2[i])
    kept = [int(ci[i, 6]) for i in range(4)]

    ev = lambda: torch.cuda.Event(enable_timing=True)

    glob = {}

    def step(timers=None):
        for i in range(4):
            if timers is not None:
                timers[i][0].record(stream)
            plan.compress_async(fields[i], n_el, eps, streams[i], stats_c[i], cuda_stream=stream)
            if timers is not None:
                timers[i][1].record(stream)
            plan.decompress_async(streams[i], sizes[i], n_el, out, stats_d[i], cuda_stream=stream)
            if timers is not None:
                timers[i][2].record(stream)
        if world > 1:
            with torch.cuda.stream(stream):
                a = stats_c[:, 4:6].contiguous()                      # disc2, tot2
                b = stats_c.view(torch.int64)[:, 6:10].contiguous()   # kept, blocks, bytes, field bytes
                c = stats_d[:, 2:4].contiguous()                      # err_inf, u_inf
                dist.all_reduce(a)
                dist.all_reduce(b)
                dist.all_reduce(c, op=dist.ReduceOp.MAX)
                glob["c"], glob["b"], glob["d"] = a, b, c

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    timers = [[[ev(), ev(), ev()] for _ in range(4)] for _ in range(args.steps)]
    t_start, t_end = ev(), ev()
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for s in range(args.steps):
            step(timers[s])
        t_end.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    comp_ms = sum(timers[s][i][0].elapsed_time(timers[s][i][1]) for s in range(args.steps) for i in range(4))
    deco_ms = sum(timers[s][i][1].elapsed_time(timers[s][i][2]) for s in range(args.steps) for i in range(4))
    t = torch.tensor([total_ms, comp_ms, deco_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    total_ms, comp_ms, deco_ms = t.tolist()
    ms_per_step = total_ms / args.steps
    field_bytes_step = 4 * fbytes_field
    value = world * field_bytes_step / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant kernel (per launch: one field)
    hbm, peak_src = peaks()
    C = sum(sizes) / 4.0
    comp_launch_ms = comp_ms / (4 * args.steps)
    deco_launch_ms = deco_ms / (4 * args.steps)
    comp_bytes = fbytes_field + C                    # read field, write stream
    deco_bytes = C + fbytes_field                    # read stream, write field
    comp_gbs = comp_bytes / (comp_launch_ms * 1e-3) / 1e9
    deco_gbs = deco_bytes / (deco_launch_ms * 1e-3) / 1e9
    dom = "compress8_kernel" if comp_launch_ms >= deco_launch_ms else "decompress8_kernel"
    achieved = comp_gbs if dom == "compress8_kernel" else deco_gbs
    step_alg_bytes = 4 * (comp_bytes + deco_bytes)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(dom)
        except Exception:
            traffic = None

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (TGV t=0 at GLL nodes, generated on device)",
        "config": {"workload": "cfg2: TGV u/v/w/p, 262144 elements/GPU, lx=8, fp64, RelativeL2 1e-3",
                   "elements_per_gpu": n_el, "lx": LX, "fields": 4, "max_error": eps,
                   "field_bytes_per_gpu": field_bytes_step, "parallelism": f"elements sharded x{world} (z-slabs)",
                   "l2": "inputs 4.3 GB/GPU >> 126 MB L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": comp_bytes if dom == "compress8_kernel" else deco_bytes,
                     "compress_gbs": comp_gbs, "decompress_gbs": deco_gbs,
                     "compress_frac": comp_gbs / hbm, "decompress_frac": deco_gbs / hbm,
                     "step_frac": step_alg_bytes / (ms_per_step * 1e-3) / 1e9 / hbm,
                     "compress_ms_per_field": comp_launch_ms, "decompress_ms_per_field": deco_launch_ms},
        "quality": {"fields": list(FIELDS), "kept_fraction": [k / nvals for k in kept],
                    "C_over_F": [s / fbytes_field for s in sizes],
                    "cr": [PK.CompressionReport.from_sizes(fbytes_field, s).cr for s in sizes],
                    "rel_l2": rel_l2, "rel_linf": rel_linf},
        "gpu_launches": 4 * 4 * args.steps,
        "clocks": clk.summary(),
    }

    # cfg5: async in-situ mode -- compression on a low-priority side stream next to a
    # memory-bound solver stand-in (double-buffered state of the four fields)
    if not args.no_async:
        from paper_2407_20731_b200.insitu import AsyncInSitu
        ai = AsyncInSitu(plan, fields, n_el, eps)
        result["async_insitu"] = ai.measure(steps=args.async_steps, every=args.async_every)
        del ai
        torch.cuda.empty_cache()

    # e2e through the host-buffer C ABI (rank-local; H2D + kernels + D2H per call)
    if not args.no_e2e:
        hf = [f.cpu().pin_memory().numpy() for f in fields]
        hs = [torch.empty(cap, dtype=torch.uint8).pin_memory().numpy() for _ in range(4)]
        ho = torch.empty(nvals, dtype=torch.float64).pin_memory().numpy()

        # Two plans driven from two host threads: the compress calls are H2D-bound and the
        # decompress calls D2H-bound, so running field i+1's compress next to field i's
        # decompress keeps both PCIe directions busy.  Every call is the blocking
        # host-buffer C ABI; a ring of 4 host stream buffers hands fields over.
        plan2 = PK.LossyPlan(LX, 1, local)
        nbs = [0] * 4

        def e2e_run(nsteps):
            q: "queue.Queue" = queue.Queue(maxsize=2)
            err = []

            def producer():
                try:
                    for j in range(4 * nsteps):
                        nbs[j % 4], _ = plan.compress_host(hf[j % 4], n_el, eps, hs[j % 4])
                        q.put(j)
                except BaseException as e:  # noqa: BLE001
                    err.append(e)
                    q.put(None)

            th = threading.Thread(target=producer)
            th.start()
            for _ in range(4 * nsteps):
                j = q.get()
                if j is None:
                    break
                plan2.decompress_host(hs[j % 4], nbs[j % 4], n_el, ho)
            th.join()
            if err:
                raise err[0]
            h2d = sum(fbytes_field + n for n in nbs)
            return h2d, h2d

        e2e_run(1)
        if world > 1:
            dist.barrier()
        k = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        h2d, d2h = e2e_run(k)
        dt = (time.perf_counter() - t0) / k
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        result["e2e"] = {"value": world * field_bytes_step / dt / 1e9, "unit": UNIT,
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "api": "isf_lossy_compress_host + isf_lossy_decompress_host (pinned host buffers; compress of field i+1 overlaps decompress of field i on a second plan)",
                         "steps": k}

    if rank == 0 and not args.no_cpu:
        threads = os.cpu_count() or 1
        gbs, dt, n_s, fb = cpu_reference(args.cpu_sample_elements, 1, 1, threads)
        result["cpu_baseline"] = {"value": gbs, "unit": UNIT, "cores": threads, "kind": "port",
                                  "sample": f"first {n_s} elements of each of u,v,w,p ({fb / 1e9:.3f} GB), "
                                            f"compress+decompress, OpenMP {threads} threads"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    plan.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
