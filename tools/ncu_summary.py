#!/usr/bin/env python
"""Summarise an ncu report: per kernel duration, DRAM bytes, pipe utilisation,
issue activity and the top stall reasons (used to write profiles/*.md)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg"]


def main(rep, blocks=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    hdr = next(r)
    units = next(r)
    for row in r:
        d = dict(zip(hdr, row))
        print(f"== {d['Kernel Name'][:70]}")
        for k in KEYS:
            if k in d:
                print(f"   {k} = {d[k]} {units[hdr.index(k)]}")
        if blocks:
            n = float(d["smsp__inst_executed.sum"].replace(",", ""))
            print(f"   warp-instructions per block = {n / blocks:.1f}")
        st = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("   stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
