"""A/B: the TMA-staged 2-D kernel (tma=1) vs the planner's 2-D plan on the
suites' 16-byte-aligned Tiled-class cases; outputs checked against the oracle
in full.  python tools/ab_tma.py [out.jsonl]"""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1705_01598_b200 as tt
import tt_workloads as wl
from oracle import oracle as orc

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
cases = [wl.s1()] + wl.s2_ttc() + wl.s3_random(per_cell=2, set2_random=0) + wl.s4_alignment()
agg = {}
for c in cases:
    try:
        tt.Plan(c.dims, c.perm, c.esize, tma=1).destroy()
    except tt.TTError:
        continue
    words = c.words()
    x = torch.from_numpy(words.view(np.int32 if c.esize == 4 else np.int64)).cuda()
    y = torch.empty_like(x)
    want = orc.permute_threaded(c.dims, c.perm, words)
    plans = {"heur": tt.Plan(c.dims, c.perm, c.esize)}
    for cps in (1, 2, 3):
        try:
            plans[f"tma_c{cps}"] = tt.Plan(c.dims, c.perm, c.esize, tma=1, ctas_per_sm=cps)
        except tt.TTError:
            pass
    s = torch.cuda.current_stream()
    times = {k: [] for k in plans}
    ok = {}
    for k, p in plans.items():
        y.zero_(); p.execute(x, y); torch.cuda.synchronize()
        ok[k] = bool(np.array_equal(y.cpu().numpy().view(words.dtype), want))
    for rep in range(9):
        for k, p in plans.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); p.execute(x, y); b.record(s); b.synchronize()
            times[k].append(a.elapsed_time(b))
    med = {k: statistics.median(v) for k, v in times.items()}
    hd = plans["heur"].describe()
    row = {"case": c.name, "dims": list(c.dims), "esize": c.esize, "heur_kernel": hd["kernel"], "heur_vec": hd.get("vec"),
           "heur_ms": round(med["heur"], 4), "ok": ok,
           "gbs": {k: round(2 * c.nbytes / v / 1e6, 1) for k, v in med.items()}}
    for k in med:
        if k != "heur":
            row[k + "_x"] = round(med["heur"] / med[k], 3)
            agg.setdefault(k, []).append(med["heur"] / med[k])
    print(json.dumps(row), flush=True)
    if out:
        out.write(json.dumps(row) + "\n")
    for p in plans.values():
        p.destroy()
    del x, y
    torch.cuda.empty_cache()
for k, v in agg.items():
    sm = {"variant": k, "n": len(v), "median_x": round(statistics.median(v), 3), "min": round(min(v), 3),
          "max": round(max(v), 3)}
    print(json.dumps(sm))
    if out:
        out.write(json.dumps(sm) + "\n")
