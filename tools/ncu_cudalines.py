#!/usr/bin/env python
"""Executed warp-instructions and stall samples per CUDA source line of one kernel in an
ncu report (ncu's own `cuda,sass` source correlation).
usage: ncu_cudalines.py REPORT KERNEL_REGEX BLOCKS [TOP]"""
import collections
import csv
import subprocess
import sys


def _f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(rep, kern, blocks, top=40):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", "regex:" + kern, "--launch-count", "1"], capture_output=True, text=True).stdout
    agg, st = collections.Counter(), collections.Counter()
    fl, line, hdr, src = None, None, None, {}
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fl = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            line = int(r[0])
            src[(fl, line)] = r[1].strip()[:80]
        if r[2]:
            n = _f(r[7])
            s = _f(r[4])
            agg[(fl, line)] += n
            st[(fl, line)] += s
    tot, tots = sum(agg.values()), sum(st.values()) or 1
    print(f"total per block {tot / blocks:.1f}")
    for k, v in agg.most_common(top):
        print(f"{v / blocks:8.1f}/blk {st[k] / tots * 100:5.1f}%stall {k[0]}:{k[1]}  {src.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 40)
