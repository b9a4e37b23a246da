#!/usr/bin/env python
"""Benchmark of the in-situ lossy-compression hot path (BASELINE.json metric:
"Field GB/s compressed+decompressed at 1/2/4/8 B200; % of HBM roofline").

Workload (BASELINE.json configs[1]): per GPU a 64^3 = 262,144
element mesh, lx = 8, fp64, four scalar fields u/v/w/p of the t=0 Taylor-Green
vortex (4 x 1 GiB = 4.29 GB), RelativeL2 max_error 1e-3.  One step = compress +
decompress of all four fields plus, for N > 1, the global all-reduce of the four
fields' statistics (error energies, kept counts, bytes, status) through the C ABI
(isf_lossy_allreduce_n on torch's NCCL communicator).  Multi-GPU = weak scaling
(configs[2]): rank r owns the element slab ez in [64 r, 64 r + 64) of a
64 x 64 x 64N mesh.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Without torchrun, --gpus N > 1 re-launches itself under torch.distributed.run
(N ranks, 127.0.0.1).  Prints one JSON line (rank 0).  `value` = sum over ranks of
field bytes / max over ranks of the device time (CUDA events on the launching
stream, inputs resident in HBM; 4.3 GB of inputs >> 126 MB L2, so no flush);
`e2e` = the same metric through the host-buffer C ABI (H2D, kernels, D2H inside
the timed region).  Extra keys: `roofline.error_report` (decompress re-reading the
original for the L2/Linf report: 3F + 2C bytes), `cfg4` (BASELINE.json configs[3]:
lx 6/8/10/12 spectral sweep), `quality.near_threshold` (blocks whose mask differs
from the SPEC-literal rule, all inside SURVEY 8c's band), `async_insitu`
(configs[4]), `cpu_baseline`.  `--impl reference` times the reference CPU path (the
oracle port of SPEC.md:222-239 -- the reference ships no implementation) on the
host cores over the full cfg2 workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import queue
import socket
import subprocess
import sys
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
WORKLOAD = "cfg2: TGV u/v/w/p, 262144 elements/GPU, lx=8, fp64, RelativeL2 1e-3"


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


# ------------------------------------------------------------------ CPU side
def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    cpu_max = None
    for p in ("/sys/fs/cgroup/cpu.max", "/sys/fs/cgroup/cpu/cpu.cfs_quota_us"):
        try:
            with open(p) as f:
                cpu_max = f.read().strip()
            break
        except Exception:
            continue
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count()
    return {"model": model, "nproc": os.cpu_count(), "affinity": aff, "cgroup_cpu_max": cpu_max}


def oracle_native():
    """The CPU oracle built on this host with -O3 -march=native, falling
    back to the portable -O2 build that travels with the repo."""
    lib = os.path.join(ROOT, "oracle", "_build", "libisf_oracle_native.so")
    build = "-O3 -march=native (built on this host)"
    try:
        subprocess.run(["make", "-s", "-B", "-C", os.path.join(ROOT, "oracle"), "native"], check=True,
                       capture_output=True, timeout=120)
        os.environ["ISF_ORACLE_LIB"] = lib
    except Exception:
        build = "-O2 -march=x86-64-v2 (portable build)"
    from oracle import oracle as O
    O.build()
    return O, build


def cpu_reference(O, nz: int, steps: int, warmup: int, threads: int):
    """The reference CPU path (oracle port) on the first `nz` element z-layers of each of
    the four TGV fields (nz = 64: the whole cfg2 workload)."""
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
    O, build = oracle_native()
    nz = max(1, min(E_AX, args.ref_elements // (E_AX * E_AX)))
    # warm-up: first touch of the buffers and the thread pool; capped at 2 full steps
    gbs, dt, n_el, fbytes = cpu_reference(O, nz, args.steps, min(args.warmup, 2), threads)
    sample = (f"{'all' if nz == E_AX else 'first'} {n_el} elements ({nz} of 64 z-layers) of each of u,v,w,p "
              f"({fbytes / 1e9:.3f} GB per step), compress+decompress, OpenMP {threads} threads")
    line = {
        "metric": METRIC, "value": gbs, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (TGV t=0 at GLL nodes)",
        "config": {"workload": WORKLOAD if nz == E_AX else WORKLOAD + f" (sample: {nz} z-layers)",
                   "elements_per_gpu": n_el, "lx": LX, "fields": 4, "max_error": EPS, "parallelism": "cpu",
                   "warmup_steps_run": min(args.warmup, 2)},
        "impl": "reference",
        "cpu_baseline": {"value": gbs, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "build": build, "cpu": cpu_info()},
        "e2e": {"value": gbs, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(n: int):
    """--gpus N > 1 without torchrun: run N ranks of this script under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------ GPU side
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--ref-elements", type=int, default=E_AX ** 3, help="reference arm: elements per field")
    ap.add_argument("--cpu-sample-layers", type=int, default=16, help="native arm cpu_baseline: z-layers per field")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-async", action="store_true")
    ap.add_argument("--no-cfg4", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--eps", type=float, default=EPS)
    ap.add_argument("--async-steps", type=int, default=20)
    ap.add_argument("--async-every", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "native" else args.warmup
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args.gpus)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2407_20731_b200 as PK
    from paper_2407_20731_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    oversub = world > ndev  # test mode: several ranks share a GPU (gloo for the scalars)
    local_dev = local % ndev
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    comm = 0
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
            comm = D.nccl_comm_ptr(device=dev)
    eps = args.eps
    plan = PK.LossyPlan(LX, 1, local_dev)
    n_el = E_AX ** 3
    nvals = n_el * LX ** 3
    fbytes_field = nvals * 8
    cap = plan.capacity(n_el)
    stream = torch.cuda.Stream(dev)
    # in-situ producer stand-in: TGV u/v/w/p on device for this rank's slab
    fields = []
    with torch.cuda.stream(stream):
        ez0, nz = D.slab_for_rank(E_AX, rank, world)
        for w in range(4):
            t = torch.empty(nvals, dtype=torch.float64, device=dev)
            plan.generate_tgv(t, E_AX, w, ez0=ez0, nz=nz, cuda_stream=stream)
            fields.append(t)
        streams = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in range(4)]
        out = torch.empty(nvals, dtype=torch.float64, device=dev)
        stats_c = torch.zeros(4, 12, dtype=torch.float64, device=dev)
        stats_d = torch.zeros(4, 12, dtype=torch.float64, device=dev)
        stats_e = torch.zeros(8, 12, dtype=torch.float64, device=dev)  # error variant: compress + decompress
    stream.synchronize()

    def reduce(st):
        """Global reduction of the step's statistics (N > 1)."""
        if world == 1:
            return
        if comm:
            D.allreduce_stats_nccl(st, comm, stream)
        else:
            stream.synchronize()
            D.allreduce_stats(st)

    # first pass: stream sizes (needed by decompress) + correctness gates
    sizes = []
    for i in range(4):
        plan.compress_async(fields[i], n_el, eps, streams[i], stats_c[i], cuda_stream=stream)
    stream.synchronize()
    ci = stats_c.view(torch.int64).cpu().numpy()
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
    launches_per_step = 16 + (2 if world > 1 and comm else 0)

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
        reduce(stats_c)

    def step_err():
        # decompress with the error report: re-reads the original (3F + 2C per field)
        for i in range(4):
            plan.compress_async(fields[i], n_el, eps, streams[i], stats_e[i], cuda_stream=stream)
            plan.decompress_async(streams[i], sizes[i], n_el, out, stats_e[4 + i], original=fields[i],
                                  cuda_stream=stream)
        reduce(stats_e)

    def timed(fn, steps, warmup, sample_clocks=False):
        for _ in range(warmup):
            fn()
        stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = ev(), ev()
        clk = ClockSampler(local_dev) if sample_clocks else None
        if clk:
            clk.__enter__()
        t0.record(stream)
        for s in range(steps):
            fn(s)
        t1.record(stream)
        stream.synchronize()
        if clk:
            clk.__exit__(None, None, None)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1), clk

    timers = [[[ev(), ev(), ev()] for _ in range(4)] for _ in range(args.steps)]
    total_ms, clk = timed(lambda s=None: step(timers[s] if s is not None else None), args.steps, args.warmup, True)
    comp_ms = sum(timers[s][i][0].elapsed_time(timers[s][i][1]) for s in range(args.steps) for i in range(4))
    deco_ms = sum(timers[s][i][1].elapsed_time(timers[s][i][2]) for s in range(args.steps) for i in range(4))
    ksteps_err = max(3, min(args.steps, 10))
    err_ms, _ = timed(lambda s=None: step_err(), ksteps_err, 2)
    t = torch.tensor([total_ms, comp_ms, deco_ms, err_ms], dtype=torch.float64, device=dev)
    if world > 1:
        if oversub:
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    total_ms, comp_ms, deco_ms, err_ms = t.tolist()
    ms_per_step = total_ms / args.steps
    field_bytes_step = 4 * fbytes_field
    value = world * field_bytes_step / (ms_per_step * 1e-3) / 1e9
    if world > 1:  # global statistics of the last timed step must be clean
        assert int(stats_c.view(torch.int64)[:, 10].max().item()) == 0
        assert int(stats_c.view(torch.int64)[:, 7].sum().item()) == 4 * world * n_el

    # roofline of the dominant call (per launch: one field)
    hbm, peak_src = peaks()
    C = sum(sizes) / 4.0
    comp_launch_ms = comp_ms / (4 * args.steps)
    deco_launch_ms = deco_ms / (4 * args.steps)
    comp_bytes = fbytes_field + C                    # read field, write stream
    deco_bytes = C + fbytes_field                    # read stream, write field
    comp_gbs = comp_bytes / (comp_launch_ms * 1e-3) / 1e9
    deco_gbs = deco_bytes / (deco_launch_ms * 1e-3) / 1e9
    dom_is_comp = comp_launch_ms >= deco_launch_ms
    dom = ("compress call (compress8_kernel + compact8_kernel)" if dom_is_comp
           else "decompress call (block_offsets8_kernel + decompress8_kernel)")
    achieved = comp_gbs if dom_is_comp else deco_gbs
    step_alg_bytes = 4 * (comp_bytes + deco_bytes)
    err_step_ms = err_ms / ksteps_err
    err_alg_bytes = 4 * (comp_bytes + deco_bytes + fbytes_field)
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tj = json.load(f)
            traffic = tj.get("compress_call" if dom_is_comp else "decompress_call")
            traffic_src = f"profiles/ncu_traffic.json ({tj.get('source', '')})"
        except Exception:
            traffic = None

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (TGV t=0 at GLL nodes, generated on device)",
        "config": {"workload": WORKLOAD,
                   "elements_per_gpu": n_el, "lx": LX, "fields": 4, "max_error": eps,
                   "field_bytes_per_gpu": field_bytes_step,
                   "parallelism": f"elements sharded x{world} (z-slabs)" + (" [oversubscribed: ranks share GPUs, gloo scalars]" if oversub else ""),
                   "collective": ("isf_lossy_allreduce_n over NCCL (4 stats records per step)" if comm else
                                  ("gloo all-reduce (oversubscribed test mode)" if world > 1 else "none (1 rank)")),
                   "l2": "inputs 4.3 GB/GPU >> 126 MB L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "alg_bytes_per_launch": comp_bytes if dom_is_comp else deco_bytes,
                     "compress_gbs": comp_gbs, "decompress_gbs": deco_gbs,
                     "compress_frac": comp_gbs / hbm, "decompress_frac": deco_gbs / hbm,
                     "step_frac": step_alg_bytes / (ms_per_step * 1e-3) / 1e9 / hbm,
                     "compress_ms_per_field": comp_launch_ms, "decompress_ms_per_field": deco_launch_ms,
                     "error_report": {"ms_per_step": err_step_ms,
                                      "field_gbs": world * field_bytes_step / (err_step_ms * 1e-3) / 1e9,
                                      "alg_bytes_per_step": err_alg_bytes,
                                      "step_frac": err_alg_bytes / (err_step_ms * 1e-3) / 1e9 / hbm,
                                      "steps": ksteps_err,
                                      "what": "compress + decompress re-reading the original for the L2/Linf report (3F+2C per field)"}},
        "quality": {"fields": list(FIELDS), "kept_fraction": [k / nvals for k in kept],
                    "C_over_F": [s / fbytes_field for s in sizes],
                    "cr": [PK.CompressionReport.from_sizes(fbytes_field, s).cr for s in sizes],
                    "rel_l2": rel_l2, "rel_linf": rel_linf,
                    "norm": "GLL-weighted relative L2 (the norm the truncation guarantees, DESIGN.md 3.8)"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }

    O = None
    if rank == 0 and not (args.no_parity and args.no_cpu):
        O, obuild = oracle_native()

    # SPEC-literal parity of the timed streams (rank 0's slab): byte parity with the
    # oracle and the near-threshold count (north_star "counted and reported")
    if rank == 0 and not args.no_parity:
        par = {"streams_equal_oracle": [], "near_threshold": [], "far": [], "kept_literal": [], "kept": []}
        for i in range(4):
            host = fields[i].cpu().numpy()
            got = streams[i][: sizes[i]].cpu().numpy()
            rc, ref, _ = O.compress(host, LX, 1, eps)
            par["streams_equal_oracle"].append(bool(rc == 0 and ref.size == got.size and np.array_equal(ref, got)))
            lit = O.literal_check(host, LX, 1, eps, got)
            par["near_threshold"].append(lit["near_threshold"])
            par["far"].append(lit["far"])
            par["kept_literal"].append(lit["kept_literal"])
            par["kept"].append(lit["kept_stream"])
            del host
        result["quality"]["near_threshold"] = int(sum(par["near_threshold"]))
        result["quality"]["parity"] = par

    # cfg4 (BASELINE.json configs[3]): lx 6/8/10/12 spectral sweep, 262,144 elements
    if world == 1 and not args.no_cfg4:
        del out
        torch.cuda.empty_cache()
        result["cfg4"] = cfg4_sweep(PK, torch, dev, stream, ev, hbm)
        out = torch.empty(nvals, dtype=torch.float64, device=dev)

    # cfg5: async in-situ mode -- compression on a low-priority side stream next to a
    # memory-bound solver stand-in (double-buffered state of the four fields)
    if not args.no_async:
        from paper_2407_20731_b200.insitu import AsyncInSitu
        ai = AsyncInSitu(plan, fields, n_el, eps)
        r = ai.measure(steps=args.async_steps, every=args.async_every)
        if world > 1:
            sd = torch.tensor([r["slowdown"]], dtype=torch.float64, device=dev)
            if oversub:
                sd = sd.cpu()
            dist.all_reduce(sd, op=dist.ReduceOp.MAX)
            r["slowdown_max_over_ranks"] = float(sd.item())
        result["async_insitu"] = r
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
        plan2 = PK.LossyPlan(LX, 1, local_dev)
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
            if oversub:
                tt = tt.cpu()
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        result["e2e"] = {"value": world * field_bytes_step / dt / 1e9, "unit": UNIT,
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "api": "isf_lossy_compress_host + isf_lossy_decompress_host (pinned host buffers; compress of field i+1 overlaps decompress of field i on a second plan)",
                         "steps": k}
        # the bound of this leg: every step moves the fields both ways over PCIe at once
        pb = pcie_bidir_gbs(torch, dev)
        result["e2e"]["pcie"] = pb
        result["e2e"]["frac_of_pcie_bound"] = result["e2e"]["value"] / world / pb["bidir_each_gbs"]
        plan2.close()

    if rank == 0 and not args.no_cpu and world == 1:
        threads = os.cpu_count() or 1
        nzs = max(1, min(E_AX, args.cpu_sample_layers))
        gbs, dt, n_s, fb = cpu_reference(O, nzs, 1, 1, threads)
        gbs1, dt1, n_s1, fb1 = cpu_reference(O, max(1, nzs // 8), 1, 0, 1)
        result["cpu_baseline"] = {"value": gbs, "unit": UNIT, "cores": threads, "kind": "port",
                                  "sample": f"first {n_s} elements ({nzs} of 64 z-layers) of each of u,v,w,p "
                                            f"({fb / 1e9:.3f} GB), compress+decompress, OpenMP {threads} threads",
                                  "single_thread": {"value": gbs1, "unit": UNIT, "cores": 1,
                                                    "sample": f"first {n_s1} elements of each field ({fb1 / 1e9:.3f} GB)"},
                                  "build": obuild, "cpu": cpu_info()}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    plan.close()
    return 0


def pcie_bidir_gbs(torch, dev, nbytes=256 << 20, reps=4):
    """Pinned host <-> device copy bandwidth on this box: each direction alone and both
    at once (per direction).  The e2e leg moves every field H2D and back D2H with the
    two directions overlapped, so bidir_each_gbs is its bound (field GB/s)."""
    h1 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(up, down):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            if up:
                with torch.cuda.stream(s1):
                    d1.copy_(h1, non_blocking=True)
            if down:
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            s1.synchronize()
            s2.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return nbytes / best / 1e9

    return {"h2d_gbs": timed(True, False), "d2h_gbs": timed(False, True), "bidir_each_gbs": timed(True, True),
            "bytes": nbytes, "how": "best of 4 pinned copies of 256 MiB, wall clock around the stream syncs"}


def cfg4_sweep(PK, torch, dev, stream, ev, hbm, n_el=262144, lxs=(6, 8, 10, 12), epss=(1e-2, 1e-5),
               steps=5, warmup=3):
    """BASELINE.json configs[3]: turbulent-like spectral fields of
    262,144 elements at lx = 6/8/10/12, eps 1e-2 and 1e-5; compress + decompress."""
    from oracle import oracle as O  # amplitudes table only (the field is generated on the device)
    rows = []
    for lx in lxs:
        plan = PK.LossyPlan(lx, 1, dev.index)
        nv = n_el * lx ** 3
        f = torch.empty(nv, dtype=torch.float64, device=dev)
        plan.generate_spectral(f, n_el, 0, O.SPECTRAL_SEED, O.spectral_amplitudes(lx), cuda_stream=stream)
        cap = plan.capacity(n_el)
        sbuf = torch.empty(cap, dtype=torch.uint8, device=dev)
        o = torch.empty(nv, dtype=torch.float64, device=dev)
        st = torch.zeros(2, 12, dtype=torch.float64, device=dev)
        F = nv * 8
        for eps in epss:
            plan.compress_async(f, n_el, eps, sbuf, st[0], cuda_stream=stream)
            stream.synchronize()
            si = st.view(torch.int64)
            assert int(si[0, 10].item()) == 0
            nb = int(si[0, 8].item())
            for _ in range(warmup):
                plan.compress_async(f, n_el, eps, sbuf, st[0], cuda_stream=stream)
                plan.decompress_async(sbuf, nb, n_el, o, st[1], cuda_stream=stream)
            tm = [[ev(), ev(), ev()] for _ in range(steps)]
            stream.synchronize()
            for s in range(steps):
                tm[s][0].record(stream)
                plan.compress_async(f, n_el, eps, sbuf, st[0], cuda_stream=stream)
                tm[s][1].record(stream)
                plan.decompress_async(sbuf, nb, n_el, o, st[1], cuda_stream=stream)
                tm[s][2].record(stream)
            stream.synchronize()
            cms = sum(x[0].elapsed_time(x[1]) for x in tm) / steps
            dms = sum(x[1].elapsed_time(x[2]) for x in tm) / steps
            rows.append({"lx": lx, "eps": eps, "field_bytes": F, "C_over_F": nb / F,
                         "compress_gbs": (F + nb) / (cms * 1e-3) / 1e9, "decompress_gbs": (F + nb) / (dms * 1e-3) / 1e9,
                         "field_gbs": F / ((cms + dms) * 1e-3) / 1e9,
                         "step_frac": 2 * (F + nb) / ((cms + dms) * 1e-3) / 1e9 / hbm,
                         "compress_ms": cms, "decompress_ms": dms})
        del f, sbuf, o
        plan.close()
        torch.cuda.empty_cache()
    return rows


if __name__ == "__main__":
    sys.exit(main())
