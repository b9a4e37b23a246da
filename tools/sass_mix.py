#!/usr/bin/env python
"""Static SASS opcode mix of one kernel (nvdisasm output): tools/sass_mix.py k.sass name"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().split('\n')
name = sys.argv[2]
st = [i for i, l in enumerate(lines) if l.startswith('.text.') and name in l][0]
ins = []
for l in lines[st + 1:]:
    if l.startswith('.text.'):
        break
    m = re.match(r'\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', l)
    if m:
        ins.append(m.group(2))
c = collections.Counter(i.split('.')[0] for i in ins)
print(len(ins), c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 40))
