"""Calibration data for the tile model (GPU box): for every suite case whose
heuristic plan is an un-widened generic tile, time the tiles of a grid of
forced run targets (and the heuristic's own) and record each candidate's
plan description, model prediction and measured time.  Offline fitting:
tools/model_fit.py.

    python tools/model_data.py --suite s2,s3,set2 --per-cell 2 --out data.jsonl"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402
from bench_suite import cases_for  # noqa: E402


def prefixes(dims, order, cap):
    out, P = [], 1
    for i in order:
        if P * dims[i] > cap:
            break
        P *= dims[i]
        if P >= 8:
            out.append(P)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", default="s2,s3,set2")
    ap.add_argument("--per-cell", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    s = torch.cuda.current_stream()
    f = open(a.out, "w")
    for c in cases_for(a.suite.split(","), a.per_cell):
        h = tt.Plan(c.dims, c.perm, c.esize)
        dh = h.describe()
        if dh["kernel"] != "tile" or dh.get("widen", 1) != 1 or (dh.get("tile") or {}).get("vg"):
            h.destroy()
            continue
        fused = dh["fused"]
        fd, fp = fused["dims"], fused["perm"]
        E = c.esize
        tin = [max(2, b // E) for b in (128, 256, 512, 1024, 2048)]
        tout = list(tin)
        tin += prefixes(fd, range(len(fd)), 4096)
        tout += prefixes(fd, fp, 4096)
        cands = [("heur", {})]
        for ri in sorted(set(tin)):
            for ro in sorted(set(tout)):
                cands.append((f"{ri}x{ro}", {"run_in": ri, "run_out": ro}))
        x = torch.from_numpy(c.words().view(np.int32 if E == 4 else np.int64)).cuda()
        y = torch.empty_like(x)
        seen = {}
        for tag, o in cands:
            try:
                p = h if tag == "heur" else tt.Plan(c.dims, c.perm, E, **o)
            except tt.TTError:
                continue
            d = p.describe()
            t = d.get("tile") or {}
            key = json.dumps([d["kernel"], t.get("ext"), t.get("sd"), d["threads"], d["nreg"], d["grid"],
                              d["stages"]])
            if key in seen:
                if tag != "heur":
                    p.destroy()
                continue
            times = []
            for _ in range(a.reps):
                for _ in range(2):
                    p.execute(x, y)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(a.iters):
                    p.execute(x, y)
                e1.record(s)
                e1.synchronize()
                times.append(e0.elapsed_time(e1) / a.iters)
            ms = statistics.median(times)
            seen[key] = ms
            row = {"case": c.name, "dims": list(c.dims), "perm": list(c.perm), "esize": E, "cand": tag,
                   "opts": o, "ms": round(ms, 5), "kernel": d["kernel"], "threads": d["threads"],
                   "nreg": d["nreg"], "grid": d["grid"], "stages": d["stages"], "predicted_us": d["predicted_us"],
                   "model": d.get("model"), "ext": t.get("ext"), "sd": t.get("sd"), "V": t.get("V"),
                   "nTiles": t.get("nTiles")}
            f.write(json.dumps(row) + "\n")
            if tag != "heur":
                p.destroy()
        h.destroy()
        f.flush()
        best = min(seen.values())
        print(f"{c.name:16s} cands {len(seen):3d} heur {seen[next(iter(seen))]*1e3:8.1f}us best {best*1e3:8.1f}us "
              f"ratio {seen[next(iter(seen))] / best:.3f}", flush=True)
        del x, y


if __name__ == "__main__":
    main()
