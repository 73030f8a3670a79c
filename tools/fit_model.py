"""Fit the generic-tile model constants (planner.cpp namespace model) to a
calibration sweep (tools/sweep.py calib).  Objective: mean regret of the
model's pick per case (measured time of the argmin-predicted config over
the best measured config), tie-broken by log-time error."""
import json
import math
import random
import sys
from collections import defaultdict

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
cases = defaultdict(list)
hdr = {}
for j in rows:
    if "auto" in j:
        hdr[j["case"]] = j
        a = j["auto"]
        if a.get("model"):
            cases[j["case"]].append(dict(a, auto=True))
    elif j.get("ok") and j.get("model"):
        cases[j["case"]].append(j)
NSM, CLK = 148, 1800.0


def predict(r, P):
    m = r["model"]
    E = r["word"]
    V, nT, T, R = r["V"], r["nTiles"], r["threads"], r["nreg"]
    dense = V * E
    per = (P["wIn"] * m["sec_in"] * 32 + (1 - P["wIn"]) * dense +
           P["wOut"] * m["sec_out"] * 32 + (1 - P["wOut"]) * dense +
           V * (P["cIn"] / max(1, m["run_in"]) + P["cOut"] / max(1, m["run_out"])))
    mlp = min(1.0, m["inflight"] / P["I0"]) ** P["g"]
    tmem = nT * per / (P["bw"] * mlp)
    tiss = nT * (T / 32.0) * (P["kTile"] + R * P["kSlot"] * (1.25 if E > 4 else 1.0)) / (4 * NSM * CLK)
    return max(tmem, tiss) + 0.25 * min(tmem, tiss) + 3.0


def score(P):
    reg, err = [], []
    for c, rs in cases.items():
        if len(rs) < 4:
            continue
        preds = [predict(r, P) for r in rs]
        best = min(r["ms"] for r in rs)
        pick = rs[min(range(len(rs)), key=lambda i: preds[i])]
        reg.append(pick["ms"] / best)
        err += [abs(math.log(p / (r["ms"] * 1000))) for p, r in zip(preds, rs)]
    return sum(reg) / len(reg), sum(err) / len(err), reg


P0 = dict(wIn=0.5, wOut=1.0, cIn=12.0, cOut=12.0, I0=49152.0, g=1.0, kTile=90.0, kSlot=11.0, bw=6.3e6)
s0 = score(P0)
print("current constants: mean regret %.3f  log-err %.3f" % s0[:2])
rng = random.Random(0)
best, bs = dict(P0), s0
space = dict(wIn=(0, 1), wOut=(0, 1), cIn=(0, 256), cOut=(0, 256), I0=(8192, 131072), g=(0.3, 1.5),
             kTile=(20, 600), kSlot=(3, 40))
for it in range(6000):
    P = dict(best)
    for k in rng.sample(list(space), rng.randint(1, 3)):
        lo, hi = space[k]
        P[k] = min(hi, max(lo, P[k] + rng.gauss(0, (hi - lo) * 0.15)))
    s = score(P)
    if (s[0], s[1]) < (bs[0], bs[1]):
        best, bs = P, s
print("fitted: mean regret %.3f  log-err %.3f" % bs[:2])
print(json.dumps({k: round(v, 3) for k, v in best.items()}))
print("per-case regret:", [round(x, 2) for x in bs[2]])
