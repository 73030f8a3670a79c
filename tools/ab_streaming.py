"""A/B: evict-first (.cs) global accesses in the vector 2-D kernel vs the
default, interleaved, on the aligned 2-D suite cases and S1."""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1705_01598_b200 as tt
import tt_workloads as wl
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
cases = [wl.s1()] + wl.s2_ttc() + wl.s3_random(per_cell=2, set2_random=0) + wl.s4_alignment()
agg = []
for c in cases:
    d = tt.plan_offline(c.dims, c.perm, c.esize)
    if d["kernel"] != "tiled2d" or d["vec"] == 1:
        continue
    x = torch.from_numpy(wl.random_words(c.vol, c.esize, 3).view(np.int32 if c.esize == 4 else np.int64)).cuda()
    y = torch.empty_like(x)
    a = tt.Plan(c.dims, c.perm, c.esize)
    b = tt.Plan(c.dims, c.perm, c.esize, t2d_streaming=1)
    s = torch.cuda.current_stream()
    t = {"def": [], "cs": []}
    for rep in range(15):
        for k, p in (("def", a), ("cs", b)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); p.execute(x, y); e1.record(s); e1.synchronize()
            if rep >= 3:
                t[k].append(e0.elapsed_time(e1))
    r = {"case": c.name, "def_gbs": round(2 * c.nbytes / statistics.median(t["def"]) / 1e6, 1),
         "cs_gbs": round(2 * c.nbytes / statistics.median(t["cs"]) / 1e6, 1)}
    r["x"] = round(r["cs_gbs"] / r["def_gbs"], 4)
    agg.append(r["x"])
    print(json.dumps(r), flush=True)
    if out:
        out.write(json.dumps(r) + "\n")
print(json.dumps({"n": len(agg), "median_x": statistics.median(agg), "min": min(agg), "max": max(agg)}))
