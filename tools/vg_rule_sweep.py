"""Fixed vector-gather tile targets vs the heuristic plan on a spread of
suite cases (timed interleaved, CUDA events, inputs > L2).
    python tools/vg_rule_sweep.py [n_cases] [out.jsonl]"""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1705_01598_b200 as tt
import tt_workloads as wl

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
out = open(sys.argv[2], "w") if len(sys.argv) > 2 else None
cases = [c for c in wl.s3_random(per_cell=2, set2_random=10) if c.tags[0] in ("S3", "SET2")] + wl.s2_ttc()
rng = np.random.default_rng(5)
pick = [cases[i] for i in sorted(rng.choice(len(cases), size=min(n_cases, len(cases)), replace=False))]
PAIRS = [(64, 512), (64, 1024), (128, 1024), (128, 2048), (256, 2048), (512, 512)]
agg = {}
for c in pick:
    h = tt.Plan(c.dims, c.perm, c.esize)
    hd = h.describe()
    if hd["kernel"] != "tile":
        h.destroy()
        continue
    x = torch.from_numpy(wl.random_words(c.vol, c.esize, 3).view(np.int32 if c.esize == 4 else np.int64)).cuda()
    y = torch.empty_like(x)
    plans = {"heur": h}
    try:
        plans["heur_vg"] = tt.Plan(c.dims, c.perm, c.esize, vector_gather=1, stages=3)
    except tt.TTError:
        pass
    for a, b in PAIRS:
        try:
            plans[f"vg_{a}_{b}"] = tt.Plan(c.dims, c.perm, c.esize, run_in=max(2, a // c.esize),
                                           run_out=max(2, b // c.esize), vector_gather=1, stages=3)
        except tt.TTError:
            pass
    s = torch.cuda.current_stream()
    times = {k: [] for k in plans}
    for rep in range(7):
        for k, p in plans.items():
            if rep == 0:
                p.execute(x, y)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(s); p.execute(x, y); b_.record(s); b_.synchronize()
            times[k].append(a_.elapsed_time(b_))
    med = {k: statistics.median(v) for k, v in times.items()}
    row = {"case": c.name, "esize": c.esize, "perm0": c.perm[0], "heur_ms": round(med["heur"], 4),
           "heur_kind": ("vg" if "vg" in hd["tile"] else "sd" if "sd" in hd["tile"] else "classic") + str(hd["stages"])}
    for k, v in med.items():
        if k != "heur":
            row[k] = round(med["heur"] / v, 3)
            agg.setdefault(k, []).append(med["heur"] / v)
    print(json.dumps(row), flush=True)
    if out:
        out.write(json.dumps(row) + "\n")
    for p in plans.values():
        p.destroy()
    del x, y
    torch.cuda.empty_cache()
for k, v in agg.items():
    sm = {"variant": k, "n": len(v), "median_x": round(statistics.median(v), 3), "min": round(min(v), 3),
          "max": round(max(v), 3), "wins": sum(t > 1.03 for t in v), "losses": sum(t < 0.97 for t in v)}
    print(json.dumps(sm))
    if out:
        out.write(json.dumps(sm) + "\n")
