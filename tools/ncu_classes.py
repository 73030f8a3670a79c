"""Pick one suite case per kernel class as the planner chooses it on this
device (for ncu captures); prints 'class dims perm esize' lines."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: F401
import paper_1705_01598_b200 as tt
import tt_workloads as wl


def klass(d):
    k = d["kernel"]
    t = d.get("tile", {})
    if k == "tiled2d":
        return f"tiled2d_vec{d['vec']}" + ("_ring" if d["stages"] else "") + f"_e{d['word_size']}"
    if k == "tile":
        v = "vg" if "vg" in t else ("sd_async" if "sd" in t and d["stages"] else "sd" if "sd" in t else "classic")
        return f"tile_{v}_e{d['word_size']}"
    return f"{k}_e{d['word_size']}"


want = sys.argv[1:]
cases = [wl.s1()] + wl.s2_ttc() + wl.s3_random(per_cell=2, set2_random=10) + wl.s4_alignment()
seen = set()
for c in cases:
    d = tt.Plan(c.dims, c.perm, c.esize).describe()
    k = klass(d)
    if k in seen or (want and k not in want):
        continue
    seen.add(k)
    print(k, ",".join(map(str, c.dims)), ",".join(map(str, c.perm)), c.esize, c.name, flush=True)
