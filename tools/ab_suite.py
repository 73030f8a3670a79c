"""A/B the current libtt.so against another build on the same GPU, case by
case over bench_suite's cases, measurements interleaved (box-to-box noise of
a few % makes separate suite runs useless for small changes).

    python tools/ab_suite.py OTHER.so --suite s2,s3,set2 [--per-cell 1] [--reps 5]
Prints one line per case and per-group medians of new/old time ratios
(< 1 = the current build is faster)."""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402
from bench_suite import cases_for  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    vp, i64p, ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)
    L.tt_plan.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t, vp]
    L.tt_execute.argtypes = [vp, vp, vp]
    L.tt_destroy.argtypes = [vp]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("other")
    ap.add_argument("--suite", default="s2,s3,set2")
    ap.add_argument("--per-cell", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    libs = [tt.lib, load(a.other)]
    s = torch.cuda.current_stream()
    groups = {}
    for c in cases_for(a.suite.split(","), a.per_cell):
        td = torch.int32 if c.esize == 4 else torch.int64
        x = torch.randint(-2**31, 2**31 - 1, (c.vol,), dtype=td, device="cuda")
        y0, y1 = torch.empty_like(x), torch.empty_like(x)
        hs = []
        for L in libs:
            h = ctypes.c_void_p()
            r = L.tt_plan(ctypes.byref(h), len(c.dims), (ctypes.c_int64 * len(c.dims))(*c.dims),
                          (ctypes.c_int * len(c.perm))(*c.perm), c.esize, s.cuda_stream)
            assert r == 0, (c.name, r)
            hs.append(h)
        t = {0: [], 1: []}
        for _ in range(a.reps):
            for i, (L, h, y) in enumerate(zip(libs, hs, (y0, y1))):
                for _ in range(2):
                    L.tt_execute(h, x.data_ptr(), y.data_ptr())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(a.iters):
                    L.tt_execute(h, x.data_ptr(), y.data_ptr())
                e1.record(s)
                e1.synchronize()
                t[i].append(e0.elapsed_time(e1) / a.iters)
        same = bool(torch.equal(y0, y1))
        for L, h in zip(libs, hs):
            L.tt_destroy(h)
        m0, m1 = statistics.median(t[0]), statistics.median(t[1])
        kern = tt.Plan(c.dims, c.perm, c.esize).describe()["kernel"]
        key = (c.name.split("_")[0], kern, c.esize)
        groups.setdefault(key, []).append(m0 / m1)
        print(f"{c.name:12s} {kern:8s} E{c.esize} new {m0*1e3:8.1f}us old {m1*1e3:8.1f}us ratio {m0/m1:.4f}"
              f"{'' if same else '  OUTPUT DIFFERS'}", flush=True)
        del x, y0, y1
    print("group medians (new/old time):")
    for k in sorted(groups):
        v = groups[k]
        print(f"  {k[0]:5s} {k[1]:8s} E{k[2]} n={len(v):3d} {statistics.median(v):.4f}"
              f"  wins {sum(r < 0.99 for r in v)} losses {sum(r > 1.01 for r in v)}")
    allv = [r for v in groups.values() for r in v]
    print(f"  all n={len(allv)} median {statistics.median(allv):.4f}")


if __name__ == "__main__":
    main()
