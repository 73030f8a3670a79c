"""Instruction mix of an ncu source-page CSV (SASS view): executed warp
instructions and stall samples per opcode.  python tools/sass_mix.py F.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iI, iSmp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ins = collections.Counter(); smp = collections.Counter(); tot = 0
for r in rows[2:]:
    if len(r) <= iI or not r[iI].strip():
        continue
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    n = int(r[iI] or 0); ins[o] += n; tot += n; smp[o] += int(r[iSmp] or 0)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
st = sum(smp.values()) or 1
print(f"total warp instructions {tot}")
for o, n in ins.most_common(top):
    print(f"{o:10s} {n:12d} {100*n/tot:5.1f}%   stall samples {100*smp[o]/st:5.1f}%")
