#!/usr/bin/env python
"""Executed warp-instructions per block of compress8_kernel grouped by source region
(dev tool; regions keyed on the current dlt_fast8.cuh / dlt_common.cuh line ranges)."""
import collections
import contextlib
import io
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import ncu_lines  # noqa: E402


def main(rep, so, kernel="compress8_kernel", blocks=262144):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        ncu_lines.main(rep, kernel, so, blocks, top=100000)
    src = open(__file__.rsplit("/", 2)[0] + "/paper_2407_20731_b200/csrc/dlt_fast8.cuh").read().split("\n")
    # region markers: the nearest preceding comment line starting with '// --' or a function head
    reg = collections.Counter()
    lines = collections.Counter()
    for l in buf.getvalue().split("\n")[1:]:
        m = re.search(r"([\d.]+)/blk.*\('(\S+)', (\d+)\)", l)
        if not m:
            if "None" in l:
                reg["(no line)"] += float(l.split("/")[0])
            continue
        v, f, n = float(m.group(1)), m.group(2), int(m.group(3))
        lines[(f, n)] += v
        if f == "dlt_fast8.cuh":
            head = "?"
            for k in range(n - 1, -1, -1):
                t = src[k]
                if re.match(r"^(__global__|__device__|template|struct)", t) or re.match(r"^\s*// ", t) and k < n - 1 and src[k].strip().startswith("// ") and len(t) - len(t.lstrip()) <= 4:
                    head = f"{k + 1}: {t.strip()[:70]}"
                    break
            reg[head] += v
        else:
            reg[f] += v
    for k, v in reg.most_common(40):
        print(f"{v:7.1f}  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
