"""Opcode mix and stall share from an ncu --page source --csv SASS dump.
    python tools/src_mix.py FILE.src.csv [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 22
hdr = next(r for r in rows if r and r[0] == "Address")
ie = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
ops, st = collections.Counter(), collections.Counter()
tot = tots = 0
for r in rows:
    if len(r) <= ie or not r[0].startswith("0x"):
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
    if not m:
        continue
    n, s = int(r[ie] or 0), int(r[ss] or 0)
    ops[m.group(2)] += n
    st[m.group(2)] += s
    tot += n
    tots += s
print("warp instructions:", tot)
for op, n in ops.most_common(top):
    print(f"  {op:10s} {n / tot * 100:5.1f}% inst  {st[op] / max(tots, 1) * 100:5.1f}% stall")
