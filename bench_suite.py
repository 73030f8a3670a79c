#!/usr/bin/env python
"""Suite benchmark: the paper's benchmark sets on one B200.

    python bench_suite.py [--suite s2,s3,s4,set2] [--per-cell K] [--reps R]
                          [--verify sampled|full|none] [--out FILE.jsonl]

Per case: the seeded words of tt_workloads uploaded to HBM, plan time (host), median of
R CUDA-event-timed tt_execute calls (inputs > L2: no flush needed), the
same-bytes device copy (torch copy_) as the memcpy roofline (the paper's
GPU-STREAM analogue), and bit-exact verification against the CPU
oracle: by default every output element against the threaded oracle
(`--verify sampled` = sampled positions + multiset sum, a quick look only).  Summary: worst / median / best per suite,
per-rank medians and their max/min ratio (the "independent of rank" check).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402
import tt_workloads as wl  # noqa: E402


def cases_for(suites, per_cell):
    out = []
    for s in suites:
        if s == "s1":
            out.append(wl.s1())
        elif s == "s2":
            out += wl.s2_ttc()
        elif s == "s3":
            out += [c for c in wl.s3_random(per_cell=per_cell, set2_random=0) if c.tags[0] == "S3"]
        elif s == "set2":
            out += [c for c in wl.s3_random(per_cell=0, set2_random=per_cell * 3) if c.tags[0] == "SET2"]
        elif s == "s4":
            out += wl.s4_alignment()
        elif s == "s5":
            out += wl.s5_sharded()[:4]
    return out


def event_ms(fn, reps):
    s = torch.cuda.current_stream()
    times = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        times.append(a.elapsed_time(b))
    return statistics.median(times), min(times), max(times)


def verify(case, x, y, mode):
    if mode == "none":
        return None
    from oracle import oracle as orc
    words = x.cpu().numpy().view(np.uint32 if case.esize == 4 else np.uint64)
    got = y.cpu().numpy().view(words.dtype)
    if mode == "full":
        return bool(np.array_equal(got, orc.permute_threaded(case.dims, case.perm, words)))
    # sampled (quick look only; the default is full)
    rng = np.random.default_rng(case.seed & 0xFFFFFFFF)
    pos = np.concatenate([rng.integers(0, case.vol, 1 << 16), np.arange(min(case.vol, 2048)),
                          np.arange(max(0, case.vol - 2048), case.vol)])
    ok = np.array_equal(got[pos], orc.permute_sample(case.dims, case.perm, words, pos))
    ok = ok and int(got.sum(dtype=np.uint64)) == int(words.sum(dtype=np.uint64))
    return bool(ok)


def verify_scaled(case, x, y0, y1, alpha, beta):
    """Sampled check of out = alpha*perm(in) + beta*out: the oracle gives
    in[src(q)] one position at a time; numpy's float ops (pinned equal to the
    oracle's scaled form in tests/test_accumulate.py) finish the sample."""
    from oracle import oracle as orc
    wt, ft = (np.uint32, np.float32) if case.esize == 4 else (np.uint64, np.float64)
    words = x.cpu().numpy().view(wt)
    rng = np.random.default_rng(case.seed & 0xFFFFFFFF)
    pos = rng.integers(0, case.vol, 1 << 16)
    src = orc.permute_sample(case.dims, case.perm, words, pos).view(ft)
    before = y0.cpu().numpy().view(ft)[pos]
    want = (ft(alpha) * src + ft(beta) * before).astype(ft).view(wt)
    got = y1.cpu().numpy().view(wt)[pos]
    ok_nan = np.isnan(want.view(ft)) == np.isnan(got.view(ft))
    fin = ~np.isnan(want.view(ft))
    return bool(ok_nan.all() and np.array_equal(want[fin], got[fin]))


def run_case(case, reps, vmode, memcpy_cache, opts, measured=False):
    nd = np.int32 if case.esize == 4 else np.int64
    x = torch.from_numpy(case.words().view(nd)).cuda()   # the seeded words the oracle also gets
    y = torch.empty_like(x)
    if opts.get("accumulate"):
        g = torch.Generator(device="cuda")
        g.manual_seed(case.seed & 0x7FFFFFFFFFFFFFFF)
        ft = torch.float32 if case.esize == 4 else torch.float64
        x.view(ft).uniform_(-1.0, 1.0, generator=g)
        y.view(ft).uniform_(-1.0, 1.0, generator=g)
        plan = tt.Plan(case.dims, case.perm, case.esize, **opts)
        y0 = y.clone()
        plan.execute_scaled(x, y, 1.5, 0.5)
        torch.cuda.synchronize()
        ok = verify_scaled(case, x, y0, y, 1.5, 0.5) if vmode != "none" else None
        ms, mn, mx = event_ms(lambda: plan.execute_scaled(x, y, 1.5, 0.5), reps)
        d = plan.describe()
        plan.destroy()
        gbs = 3 * case.nbytes / ms / 1e6      # read in, read out, write out
        return {"case": case.name, "rank": case.rank, "esize": case.esize, "dims": list(case.dims),
                "perm": list(case.perm), "kernel": "tile+acc", "ms": round(ms, 5),
                "gbs": round(gbs, 1), "gibs": round(3 * case.nbytes / (ms * 1e-3) / 2**30, 1),
                "frac_memcpy": None, "verified": ok, "tile": d.get("tile", {}).get("ext"),
                "threads": d["threads"], "grid": d["grid"], "plan": "accumulate"}
    t0 = time.perf_counter()
    if measured:
        plan = tt.Plan(case.dims, case.perm, case.esize, measure=(x, y))
    else:
        plan = tt.Plan(case.dims, case.perm, case.esize, **opts)
    plan_us = (time.perf_counter() - t0) * 1e6
    ms, mn, mx = event_ms(lambda: plan.execute(x, y), reps)
    torch.cuda.synchronize()
    ok = verify(case, x, y, vmode)
    key = case.nbytes
    if key not in memcpy_cache:
        z = torch.empty_like(x)
        memcpy_cache[key] = event_ms(lambda: z.copy_(x), reps)[0]
        del z
    mc = memcpy_cache[key]
    d = plan.describe()
    plan.destroy()
    gbs = 2 * case.nbytes / ms / 1e6
    return {"case": case.name, "rank": case.rank, "esize": case.esize, "dims": list(case.dims),
            "perm": list(case.perm), "fused_rank": len(d["fused"]["dims"]), "kernel": d["kernel"],
            "ms": round(ms, 5), "ms_min": round(mn, 5), "ms_max": round(mx, 5),
            "gbs": round(gbs, 1), "memcpy_gbs": round(2 * case.nbytes / mc / 1e6, 1),
            "frac_memcpy": round(mc / ms, 4), "plan_us": round(plan_us, 1),
            "pred_us": round(d["predicted_us"], 1), "verified": ok,
            "tile": d.get("tile", {}).get("ext"), "threads": d["threads"], "grid": d["grid"],
            "plan": "measured" if measured else "heuristic", "measured": d.get("measured")}


def summarize(rows):
    out = {}
    by_suite = {}
    for r in rows:
        key = r["case"].split("_")[0] + ("@measured" if r["case"].endswith("@measured") else "")
        by_suite.setdefault(key, []).append(r)
    for s, rs in by_suite.items():
        if rs[0]["frac_memcpy"] is None:  # accumulate form: GB/s and GiB/s only
            g = sorted(r["gbs"] for r in rs)
            out[s] = {"n": len(rs), "worst_gbs": g[0], "median_gbs": statistics.median(g),
                      "best_gbs": g[-1], "median_gibs": statistics.median(r["gibs"] for r in rs),
                      "all_verified": all(r["verified"] in (True, None) for r in rs)}
            continue
        f = sorted(r["frac_memcpy"] for r in rs)
        g = sorted(r["gbs"] for r in rs)
        per_rank = {}
        for r in rs:
            per_rank.setdefault(r["rank"], []).append(r["frac_memcpy"])
        med = {k: round(statistics.median(v), 4) for k, v in sorted(per_rank.items())}
        out[s] = {"n": len(rs), "worst_frac": f[0], "median_frac": round(statistics.median(f), 4),
                  "best_frac": f[-1], "worst_gbs": g[0], "median_gbs": statistics.median(g),
                  "best_gbs": g[-1], "per_rank_median_frac": med,
                  "rank_max_over_min": round(max(med.values()) / max(1e-9, min(med.values())), 3),
                  "all_verified": all(r["verified"] in (True, None) for r in rs)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", default="s2,s3,set2,s4")
    ap.add_argument("--per-cell", type=int, default=1)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--verify", default="full", choices=["sampled", "full", "none"])
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--grid-order", type=int, default=0)
    ap.add_argument("--accumulate", action="store_true",
                    help="TTC-style accumulate form, bandwidth 3*vol*E/D (P:L303)")
    ap.add_argument("--out", default="")
    ap.add_argument("--plan", default="heuristic", choices=["heuristic", "measured", "both"])
    a = ap.parse_args()
    cases = cases_for(a.suite.split(","), a.per_cell)
    if a.limit:
        cases = cases[:a.limit]
    opts = {}
    if a.kernel:
        opts["kernel"] = a.kernel
    if a.ctas_per_sm:
        opts["ctas_per_sm"] = a.ctas_per_sm
    if a.stages:
        opts["stages"] = a.stages
    if a.slots:
        opts["slots"] = a.slots
    if a.grid_order:
        opts["grid_order"] = a.grid_order
    if a.accumulate:
        opts["accumulate"] = True
    rows, cache = [], {}
    f = open(a.out, "w") if a.out else None
    modes = {"heuristic": [False], "measured": [True], "both": [False, True]}[a.plan]
    for c in cases:
        for m in modes:
            r = run_case(c, a.reps, a.verify, cache, opts, measured=m)
            if m:
                r["case"] = r["case"] + "@measured"
            rows.append(r)
            line = json.dumps(r)
            print(line, flush=True)
            if f:
                f.write(line + "\n")
        torch.cuda.empty_cache()
    summ = summarize(rows)
    print(json.dumps({"summary": summ}), flush=True)
    if f:
        f.write(json.dumps({"summary": summ}) + "\n")
        f.close()
    return 0 if all(s["all_verified"] for s in summ.values()) else 1


if __name__ == "__main__":
    sys.exit(main())
