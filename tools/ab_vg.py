"""A/B of the vector-gather load phase (tile_vg_kernel) against the
heuristic plan on suite cases, timed interleaved on one box (CUDA events,
inputs > L2).  Every timed output is checked against the oracle in full.
    python tools/ab_vg.py [--suite s3,set2,s2] [--per-cell 1] [--out F.jsonl]"""
import argparse, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1705_01598_b200 as tt
import tt_workloads as wl
from oracle import oracle as orc
sys.path.insert(0, os.path.join(ROOT))
from bench_suite import cases_for


def timeit(plan, x, y, reps=10):
    s = torch.cuda.current_stream()
    for _ in range(3):
        plan.execute(x, y)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); plan.execute(x, y); b.record(s); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", default="s3,set2")
    ap.add_argument("--per-cell", type=int, default=1)
    ap.add_argument("--out", default="")
    ap.add_argument("--variants", default="vg4,vg3")
    ap.add_argument("--only-tile", action="store_true", default=True)
    ap.add_argument("--esize", type=int, default=0)
    ap.add_argument("--perm0", default="", choices=["", "zero", "nonzero"])
    ap.add_argument("--kind", default="", choices=["", "classic", "sd", "vg"])
    a = ap.parse_args()
    variants = {}
    for st in (3, 4):
        for pol in range(4):
            variants[f"vg{st}" + (f"p{pol}" if pol else "")] = dict(vector_gather=1, stages=st, vg_policy=pol)
    # slot-dim map on the heuristic tile, synchronous and cp.async ring
    variants["sd"] = dict(slot_dims=1)
    variants["sd3"] = dict(slot_dims=1, stages=3)
    f = open(a.out, "w") if a.out else None
    ratios = {v: [] for v in a.variants.split(",")}
    for c in cases_for(a.suite.split(","), a.per_cell):
        base = tt.plan_offline(c.dims, c.perm, c.esize)
        if a.only_tile and base["kernel"] != "tile":
            continue
        if a.esize and c.esize != a.esize:
            continue
        if a.perm0 and (base["fused"]["perm"][0] == 0) != (a.perm0 == "zero"):
            continue
        kind = "vg" if "vg" in base.get("tile", {}) else "sd" if "sd" in base.get("tile", {}) else "classic"
        if a.kind and kind != a.kind:
            continue
        words = c.words()
        nd = np.int32 if c.esize == 4 else np.int64
        x = torch.from_numpy(words.view(nd)).cuda()
        y = torch.empty_like(x)
        want = orc.permute_threaded(c.dims, c.perm, words)
        row = {"case": c.name, "esize": c.esize, "rank": c.rank}
        h = tt.Plan(c.dims, c.perm, c.esize)
        t_h = timeit(h, x, y)
        row["heur_ms"] = round(t_h, 4)
        row["heur_ok"] = bool(np.array_equal(y.cpu().numpy().view(words.dtype), want))
        h.destroy()
        for v in ratios:
            try:
                p = tt.Plan(c.dims, c.perm, c.esize, **variants[v])
            except tt.TTError:
                continue
            d = p.describe()
            want_key = "sd" if v.startswith("sd") else "vg"
            if want_key not in d.get("tile", {}):
                p.destroy(); continue
            y.zero_()
            t = timeit(p, x, y)
            ok = bool(np.array_equal(y.cpu().numpy().view(words.dtype), want))
            p.destroy()
            row[v + "_ms"] = round(t, 4)
            row[v + "_ok"] = ok
            row[v + "_x"] = round(t_h / t, 3)
            ratios[v].append(t_h / t)
        line = json.dumps(row)
        print(line, flush=True)
        if f:
            f.write(line + "\n")
        del x, y
        torch.cuda.empty_cache()
    for v, r in ratios.items():
        if r:
            s = {"variant": v, "n": len(r), "median_x": round(statistics.median(r), 3),
                 "min_x": round(min(r), 3), "max_x": round(max(r), 3), "wins": sum(x > 1.02 for x in r),
                 "losses": sum(x < 0.98 for x in r)}
            print(json.dumps(s))
            if f:
                f.write(json.dumps(s) + "\n")


if __name__ == "__main__":
    main()
