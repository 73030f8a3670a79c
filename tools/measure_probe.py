"""Time every tt_plan_measure candidate of one problem (one launch each,
after a warm-up), print the slow ones with their launch shape.
    python tools/measure_probe.py dims perm esize"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1705_01598_b200 as tt
import tt_workloads as wl
dims = tuple(int(x) for x in sys.argv[1].split(","))
perm = tuple(int(x) for x in sys.argv[2].split(","))
E = int(sys.argv[3])
W = E
n = int(np.prod(dims))
x = torch.from_numpy(wl.random_words(n, E, 3).view(np.int32 if E == 4 else np.int64)).cuda()
y = torch.empty_like(x)
cands = [{}]
for ta, tb in [(64, 128), (128, 64), (128, 128), (64, 64)] if E == 4 else [(64, 64), (64, 32), (32, 64), (32, 32)]:
    for cps in (1, 2, 3, 4):
        for st in (0, 4):
            cands.append(dict(kernel=4, run_in=ta, run_out=tb, ctas_per_sm=cps, grid_order=2, stages=st))
for cps in (2, 4, 8):
    cands.append(dict(kernel=3, ctas_per_sm=cps))
for bi in (128, 256, 512, 1024):
    for bo in (128, 256, 512, 1024):
        cands.append(dict(kernel=2, run_in=max(2, bi // W), run_out=max(2, bo // W)))
for bi in (64, 128, 256, 512):
    for bo in (64, 128, 256, 512):
        cands.append(dict(kernel=2, run_in=max(2, bi // W), run_out=max(2, bo // W), sd_vmax=8192 if E == 4 else 6144))
for st in (3, 4):
    cands.append(dict(kernel=2, slot_dims=1, stages=st))
for st in (4, 3):
    cands.append(dict(kernel=2, vector_gather=1, stages=st))
for bi in (64, 128, 256):
    for bo in (256, 512, 1024, 2048):
        cands.append(dict(kernel=2, run_in=max(2, bi // W), run_out=max(2, bo // W), vector_gather=1, stages=3))
for cps in (0, 2):
    cands.append(dict(tma=1, ctas_per_sm=cps))
s = torch.cuda.current_stream()
for o in cands:
    try:
        p = tt.Plan(dims, perm, E, **o)
    except tt.TTError:
        continue
    p.execute(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); p.execute(x, y); b.record(s); b.synchronize()
    ms = a.elapsed_time(b)
    d = p.describe()
    print(json.dumps({"ms": round(ms, 3), "opts": o, "kernel": d["kernel"], "grid": d["grid"], "threads": d["threads"],
                      "smem": d["smem"], "tile": d.get("tile", {}).get("ext"), "vg": "vg" in d.get("tile", {}),
                      "sd": "sd" in d.get("tile", {}), "stages": d["stages"]}), flush=True)
    p.destroy()
t0 = time.perf_counter()
mp = tt.Plan(dims, perm, E, measure=(x, y))
print("tt_plan_measure s", round(time.perf_counter() - t0, 2), mp.describe().get("measured"))
