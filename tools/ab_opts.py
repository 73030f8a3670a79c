"""A/B planner options on the same build and GPU, case by case, interleaved:
arm A = the default plan, arm B = the plan with the given options.

    python tools/ab_opts.py --suite s3,set2 [--kernel-filter tile] slots=8 [key=value ...]
Ratio = time(B) / time(A) (< 1: the options are faster)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402
from bench_suite import cases_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("opts", nargs="*")
    ap.add_argument("--suite", default="s2,s3,set2")
    ap.add_argument("--per-cell", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--kernel-filter", default="")
    ap.add_argument("--esize", type=int, default=0)
    ap.add_argument("--env", action="append", default=[],
                    help="KEY=VAL planner knob set for arm B only; cases whose plans agree are skipped")
    a = ap.parse_args()
    opts = {k: int(v) for k, v in (o.split("=") for o in a.opts)}
    s = torch.cuda.current_stream()
    groups = {}
    for c in cases_for(a.suite.split(","), a.per_cell):
        if a.esize and c.esize != a.esize:
            continue
        pa = tt.Plan(c.dims, c.perm, c.esize)
        da = pa.describe()
        if a.kernel_filter and da["kernel"] != a.kernel_filter:
            pa.destroy()
            continue
        env = dict(kv.split("=", 1) for kv in a.env)
        os.environ.update(env)
        try:
            pb = tt.Plan(c.dims, c.perm, c.esize, **opts)
        except tt.TTError as e:
            print(f"{c.name:14s} B plan failed: {e}")
            pa.destroy()
            continue
        finally:
            for k in env:
                os.environ.pop(k, None)
        db = pb.describe()
        if env and json.dumps(da, sort_keys=True) == json.dumps(db, sort_keys=True):
            pa.destroy()
            pb.destroy()
            continue
        td = torch.int32 if c.esize == 4 else torch.int64
        x = torch.randint(-2**31, 2**31 - 1, (c.vol,), dtype=td, device="cuda")
        ya, yb = torch.empty_like(x), torch.empty_like(x)
        t = {0: [], 1: []}
        for _ in range(a.reps):
            for i, (p, y) in enumerate(((pa, ya), (pb, yb))):
                for _ in range(2):
                    p.execute(x, y)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(a.iters):
                    p.execute(x, y)
                e1.record(s)
                e1.synchronize()
                t[i].append(e0.elapsed_time(e1) / a.iters)
        same = bool(torch.equal(ya, yb))
        ma, mb = statistics.median(t[0]), statistics.median(t[1])
        key = (c.name.split("_")[0], da["kernel"], c.esize)
        groups.setdefault(key, []).append(mb / ma)

        def shape(d):
            t = d.get("tile") or {}
            fl = ("/vg" if t.get("vg") else "") + ("/sd" if "sd" in t and not t.get("vg") else "")
            return (f"{d['kernel']}/T{d.get('threads')}/R{d.get('nreg')}/G{d.get('grid')}"
                    f"/S{d.get('stages')}/W{d.get('widen')}{fl}")
        print(f"{c.name:14s} E{c.esize} A {shape(da):34s} {ma*1e3:8.1f}us  B {shape(db):34s} {mb*1e3:8.1f}us"
              f"  ratio {mb/ma:.4f}{'' if same else '  OUTPUT DIFFERS'}", flush=True)
        pa.destroy()
        pb.destroy()
        del x, ya, yb
    print("group medians (B/A time):")
    for k in sorted(groups):
        v = groups[k]
        print(f"  {k[0]:5s} {k[1]:8s} E{k[2]} n={len(v):3d} {statistics.median(v):.4f}"
              f"  B wins {sum(r < 0.99 for r in v)} B losses {sum(r > 1.01 for r in v)}")
    allv = [r for v in groups.values() for r in v]
    if allv:
        print(f"  all n={len(allv)} median {statistics.median(allv):.4f}")


if __name__ == "__main__":
    main()
