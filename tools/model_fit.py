import json, math, subprocess, sys, collections, random, os
FIT = "/tmp/prof/fit/fit"

def load(paths):
    rows = []
    for p in paths:
        rows += [json.loads(l) for l in open(p)]
    return rows

def rows_file(rows, path):
    with open(path, "w") as f:
        for r in rows:
            if r["cand"] == "heur":
                ri, ro = r["model"]["run_in"], r["model"]["run_out"]
            else:
                ri, ro = r["opts"]["run_in"], r["opts"]["run_out"]
            f.write(f"{len(r['dims'])} {r['esize']} " + " ".join(map(str, r["dims"])) + " " +
                    " ".join(map(str, r["perm"])) + f" {ri} {ro}\n")

def heur_file(rows, path):
    cases = collections.OrderedDict()
    for r in rows:
        cases.setdefault(r["case"], r)
    with open(path, "w") as f:
        for r in cases.values():
            f.write(f"{len(r['dims'])} {r['esize']} " + " ".join(map(str, r["dims"])) + " " +
                    " ".join(map(str, r["perm"])) + " 0 0\n")
    return list(cases)

def run(path, params):
    args = [FIT, path] + [f"{k}={v}" for k, v in params.items()]
    out = subprocess.run(args, capture_output=True, text=True).stdout.split("\n")
    res = []
    for l in out:
        if not l.strip():
            continue
        a = l.split()
        res.append((float(a[0]), a[1], int(a[2]) if len(a) > 2 else -1, int(a[3]) if len(a) > 3 else -1))
    return res

def score(rows, preds):
    by = collections.defaultdict(list)
    for r, p in zip(rows, preds):
        if math.isnan(p[0]):
            continue
        by[r["case"]].append((p[0], r["ms"], r))
    tot, n, heur_tot = 0.0, 0, 0.0
    for c, v in by.items():
        best = min(x[1] for x in v)
        pick = min(v, key=lambda x: x[0])
        tot += math.log(pick[1] / best)
        h = [x for x in v if x[2]["cand"] == "heur"]
        if h:
            heur_tot += math.log(h[0][1] / best)
        n += 1
    return tot / n, heur_tot / n, n

if __name__ == "__main__":
    rows = load(sys.argv[1:])
    rows_file(rows, "/tmp/prof/fit/rows.txt")
    base = {}
    preds = run("/tmp/prof/fit/rows.txt", base)
    s, h, n = score(rows, preds)
    print(f"cases {n}  base-param pick loss {math.exp(s):.4f}  heuristic loss {math.exp(h):.4f}")

def fit(rows, iters=3):
    rows_file(rows, "/tmp/prof/fit/rows_fit.txt")
    p = {"slot": 11.0, "slotsd": 9.0, "tile": 90.0, "run": 12.0, "inflight": 49152.0, "lat": 1.5,
         "readw": 0.5, "restw": 0.25}
    def loss(q):
        return score(rows, run("/tmp/prof/fit/rows_fit.txt", q))[0]
    best = loss(p)
    print("start", math.exp(best), flush=True)
    for it in range(iters):
        for k in list(p):
            for f in (0.25, 0.5, 0.7, 1.4, 2.0, 4.0):
                q = dict(p)
                q[k] = p[k] * f
                if k in ("readw",) and q[k] > 1: continue
                l = loss(q)
                if l < best - 1e-6:
                    best, p = l, q
                    print(f"  {k}={q[k]:.4g} -> {math.exp(l):.4f}", flush=True)
    return p, best
