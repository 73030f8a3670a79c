"""Compare two bench_suite.py jsonl files case by case (frac of memcpy)."""
import json
import statistics
import sys


def load(p):
    d = {}
    for line in open(p):
        line = line.strip()
        if line.startswith("{"):
            j = json.loads(line)
            if "case" in j:
                d[j["case"]] = j
    return d


a, b = load(sys.argv[1]), load(sys.argv[2])
common = [k for k in a if k in b]
groups = {}
for k in common:
    g = k.split("_")[0]
    key = (g, a[k]["kernel"], a[k]["esize"])
    groups.setdefault(key, []).append((a[k]["frac_memcpy"], b[k]["frac_memcpy"], k))
for key in sorted(groups):
    v = groups[key]
    ra = statistics.median(x[0] for x in v)
    rb = statistics.median(x[1] for x in v)
    win = sum(1 for x in v if x[1] > x[0] * 1.01)
    loss = sum(1 for x in v if x[1] < x[0] * 0.99)
    print(f"{key[0]:5s} {key[1]:8s} E{key[2]} n={len(v):3d}  {ra:.4f} -> {rb:.4f}  win {win} loss {loss}")
for g in sorted({k[0] for k in groups}):
    va = [a[k]["frac_memcpy"] for k in common if k.split("_")[0] == g]
    vb = [b[k]["frac_memcpy"] for k in common if k.split("_")[0] == g]
    print(f"{g:5s} all n={len(va)} median {statistics.median(va):.4f} -> {statistics.median(vb):.4f}")
bad = [k for k in b if b[k].get("verified") is False]
print("unverified:", bad)
