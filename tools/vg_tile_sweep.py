"""For the worst suite cases: the heuristic plan vs forced tiles (run targets)
with and without the vector-gather load phase, timed interleaved (CUDA events,
inputs > L2).  Prints the best few per case.
    python tools/vg_tile_sweep.py CASES.jsonl [n_worst]"""
import itertools, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1705_01598_b200 as tt

rows = [json.loads(l) for l in open(sys.argv[1])]
rows.sort(key=lambda r: r["frac_memcpy"])
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for r in rows[:nw]:
    dims, perm, E = tuple(r["dims"]), tuple(r["perm"]), r["esize"]
    n = 1
    for d in dims:
        n *= d
    x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32 if E == 4 else torch.int64, device="cuda")
    y = torch.empty_like(x)
    W = E
    opts = [{}]
    for a, b in itertools.product([32, 64, 128, 256, 512, 1024, 2048], repeat=2):
        base = dict(run_in=max(2, a // W), run_out=max(2, b // W))
        opts.append(dict(base))
        opts.append(dict(base, vector_gather=1, stages=3))
        opts.append(dict(base, vector_gather=1, stages=3, sd_vmax=8192 if E == 4 else 6144))
    res = []
    for o in opts:
        try:
            p = tt.Plan(dims, perm, E, **o)
        except tt.TTError:
            continue
        d = p.describe()
        key = json.dumps(d.get("tile", {}).get("ext")) + ("vg" if "vg" in d.get("tile", {}) else "")
        s = torch.cuda.current_stream()
        for _ in range(2):
            p.execute(x, y)
        ts = []
        for _ in range(5):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(s); p.execute(x, y); b_.record(s); b_.synchronize(); ts.append(a_.elapsed_time(b_))
        res.append((statistics.median(ts), o, key, d["kernel"], d["threads"]))
        p.destroy()
    res.sort(key=lambda t: t[0])
    h = [t for t in res if t[1] == {}][0]
    print(json.dumps({"case": r["case"], "suite_frac": r["frac_memcpy"], "heur_ms": round(h[0], 4),
                      "best": [(round(t[0], 4), round(h[0] / t[0], 3), t[1], t[2]) for t in res[:5]]}), flush=True)
    del x, y
    torch.cuda.empty_cache()
