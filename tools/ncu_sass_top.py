#!/usr/bin/env python
"""Top SASS instructions of one kernel by stall samples (with the dominant reasons)."""
import csv
import subprocess
import sys


def main(rep, kernel, top=40, ctx=0):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    i0 = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and ("::" + kernel + "(") in r[1]][0]
    hdr = rows[i0 + 1]
    data = []
    for r in rows[i0 + 2:]:
        if r and r[0] == "Kernel Name":
            break
        data.append(r)
    col = {h: k for k, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_")]
    tot = sum(float(r[col["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    order = sorted(range(len(data)), key=lambda k: -float(data[k][col["Warp Stall Sampling (All Samples)"]] or 0))
    for k in sorted(order[:top]):
        r = data[k]
        s = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        reasons = sorted(((float(r[col[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
        rs = " ".join(f"{n}={v / max(s, 1) * 100:.0f}%" for v, n in reasons if v)
        print(f"{k:5d} {s / tot * 100:5.2f}% ex={r[col['Instructions Executed']]:>9s} {r[col['Source']][:60]:60s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
