"""Run one permutation a few times (for ncu captures).
    python tools/run_case.py "5,5,5,5" "0,2,1,3" 4 [reps] [key=value opts...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

dims = tuple(int(x) for x in sys.argv[1].split(","))
perm = tuple(int(x) for x in sys.argv[2].split(","))
E = int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
opts = {k: int(v) for k, v in (a.split("=") for a in sys.argv[5:])}
n = 1
for d in dims:
    n *= d
td = torch.int32 if E == 4 else torch.int64
import tt_workloads as wl
import numpy as np
x = torch.from_numpy(wl.random_words(n, E, 7).view(np.int32 if E == 4 else np.int64)).cuda()
y = torch.empty_like(x)
p = tt.Plan(dims, perm, E, **opts)
for _ in range(reps):
    p.execute(x, y)
torch.cuda.synchronize()
d = p.describe()
print({k: d.get(k) for k in ("kernel", "threads", "grid", "smem", "nreg", "widen")}, d.get("tile", {}).get("ext"))
