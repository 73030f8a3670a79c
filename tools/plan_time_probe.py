"""Plan-creation time on the GPU box: first plan of the process (cold: CUDA
occupancy queries load kernels), then other problems, then repeats."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1705_01598_b200 as tt
import tt_workloads as wl
torch.cuda.init(); torch.empty(1, device="cuda"); torch.cuda.synchronize()
out = []
def t(c, tag):
    t0 = time.perf_counter(); p = tt.Plan(c.dims, c.perm, c.esize); dt = (time.perf_counter() - t0) * 1e6
    out.append({"tag": tag, "case": c.name, "us": round(dt, 1), "kernel": p.describe()["kernel"]}); p.destroy()
cs = [wl.s1()] + wl.s2_ttc()[::10] + [c for c in wl.s3_random(per_cell=1, set2_random=2)][::7]
for i, c in enumerate(cs): t(c, "first" if i == 0 else "cold-problem")
for c in cs: t(c, "repeat")
for r in out: print(json.dumps(r))
