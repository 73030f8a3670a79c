"""Snapshot of the planner's offline choices (tt_plan_offline, the default
B200 description) for a fixed problem set: kernel, launch shape and tile.
A regression guard for planner refactors that must not change plans (the
round-2 speed-ups were checked this way); regenerate deliberately when a
planner rule changes:  python tools/plan_time/write_golden_plans.py"""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1705_01598_b200 as tt  # noqa: E402
import tt_workloads as wl  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "planner_offline_plans.jsonl")


def problems():
    cs = [wl.s1()] + wl.s2_ttc()[::3] + wl.s3_random(per_cell=1)[::2] + wl.s4_alignment()[::4]
    out = [(list(c.dims), list(c.perm), c.esize) for c in cs]
    rng = random.Random(20261018)
    for _ in range(120):
        r = rng.randint(2, 12)
        while True:
            dims = [rng.choice([1, 2, 3, 5, 7, 8, 13, 16, 31, 32, 33, 64, 100, 127, 128, 255, 256, 1000, 1024])
                    for _ in range(r)]
            v = 1
            for d in dims:
                v *= d
            if 1000 < v < (1 << 31):
                break
        perm = list(range(r))
        rng.shuffle(perm)
        out.append((dims, perm, rng.choice([4, 8])))
    return out


def summary(d):
    t = d.get("tile") or {}
    keep = {k: d.get(k) for k in ("kernel", "threads", "grid", "smem", "nreg", "vec", "stages", "widen", "idx64")}
    keep["tile"] = {k: t.get(k) for k in ("ext", "sm", "V", "nTiles", "sd", "vg")} if t else None
    if "tiled2d" in d:
        keep["tiled2d"] = {k: d["tiled2d"].get(k) for k in ("TA", "TB", "nTiles")}
    if "rowcopy" in d:
        keep["rowcopy"] = d["rowcopy"]
    return keep


def main():
    with open(OUT, "w") as f:
        for dims, perm, e in problems():
            d = tt.plan_offline(dims, perm, e)
            f.write(json.dumps({"dims": dims, "perm": perm, "esize": e, "plan": summary(d)}, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
