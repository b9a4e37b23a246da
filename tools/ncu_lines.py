#!/usr/bin/env python
"""Per-source-line executed instructions and stall samples of one kernel in an ncu
report (joins the SASS page with nvdisasm -g line info of the built library)."""
import collections
import csv
import re
import subprocess
import sys


def main(rep, kernel, so, blocks, top=40, mangled=None):
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(sass.splitlines()))
    i0 = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and (("::" + kernel + "(") in r[1] or ("::" + kernel + "<") in r[1] or ("::" + kernel + ">(") in r[1])][0]
    hdr = rows[i0 + 1]
    data = []
    for r in rows[i0 + 2:]:
        if r and r[0] == "Kernel Name":
            break
        data.append(r)
    ad, ex = hdr.index("Address"), hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    import os
    import tempfile
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    cub = [l for l in os.listdir(tmp) if l.endswith(".cubin")]
    key = mangled or (str(len(kernel.split("<")[0])) + kernel.split("<")[0])
    for c in cub:  # the cubin that holds the kernel
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, c)], capture_output=True, text=True).stdout.split("\n")
        if any(l.startswith(".text.") and key in l for l in dis):
            break
    start = [i for i, l in enumerate(dis) if l.startswith(".text.") and key in l][0]
    fl, offmap = None, {}
    for l in dis[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            fl = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            offmap[int(m.group(1), 16)] = fl
    base = int(data[0][ad], 16)
    agg, st = collections.Counter(), collections.Counter()
    tot = tots = 0.0
    for r in data:
        k = offmap.get(int(r[ad], 16) - base)
        n, s = float(r[ex] or 0), float(r[si] or 0)
        agg[k] += n
        st[k] += s
        tot += n
        tots += s
    print(f"total per block {tot / blocks:.1f}")
    for k, v in agg.most_common(top):
        print(f"{v / blocks:7.1f}/blk {st[k] / tots * 100:5.1f}%stall {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), mangled=sys.argv[5] if len(sys.argv) > 5 else None)
