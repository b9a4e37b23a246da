#!/usr/bin/env python
"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each
kernel in an `ncu --set full` report (the `traffic` field of bench.py's roofline).
Usage: tools/ncu_traffic.py REPORT [REPORT ...]; later reports override earlier."""
import csv
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(reps):
    out = {}
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        r = csv.reader(txt.splitlines())
        hdr, units = next(r), next(r)
        ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        for row in r:
            name = row[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
            # decompress8_kernel<0> is the plain decode bench.py times; <1> adds the error report
            name = name.replace("void ", "").replace("<0>", "").replace("<1>", "_with_error")
            b = float(row[ir]) * SCALE[units[ir]] + float(row[iw]) * SCALE[units[iw]]
            out.setdefault(name, []).append(b)
    res = {k: sum(v) / len(v) for k, v in out.items()}
    res["_source"] = [os.path.basename(x) for x in reps]
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
