"""GPU parameter sweeps for the B200 model calibration (row a-4).

    python tools/sweep.py t2d            # 2-D kernel tiles x CTAs/SM on S1 (+ fp64 square)
    python tools/sweep.py tile [N]       # generic tile run targets on N suite cases
Prints one JSON object per measurement.  Every configuration is checked
against the auto plan's output (bit-exact) before its time counts.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402
import tt_workloads as wl  # noqa: E402


def timeit(fn, reps=20, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def setup(case):
    td = torch.int32 if case.esize == 4 else torch.int64
    g = torch.Generator(device="cuda")
    g.manual_seed(case.seed)
    x = torch.randint(-2**31, 2**31 - 1, (case.vol,), dtype=td, device="cuda", generator=g)
    ref = torch.empty_like(x)
    p = tt.Plan(case.dims, case.perm, case.esize)
    p.execute(x, ref)
    torch.cuda.synchronize()
    return x, ref, p


def measure(case, x, ref, **opts):
    y = torch.empty_like(x)
    try:
        p = tt.Plan(case.dims, case.perm, case.esize, **opts)
    except tt.TTError as e:
        return {"err": str(e)}
    p.execute(x, y)
    torch.cuda.synchronize()
    ok = bool(torch.equal(y, ref))
    ms = timeit(lambda: p.execute(x, y))
    d = p.describe()
    p.destroy()
    return {"ok": ok, "ms": round(ms, 5), "gbs": round(2 * case.nbytes / ms / 1e6, 1),
            "kernel": d["kernel"], "grid": d["grid"], "threads": d["threads"],
            "ext": d.get("tile", {}).get("ext"), "V": d.get("tile", {}).get("V"),
            "nTiles": d.get("tile", {}).get("nTiles"), "nreg": d.get("nreg"),
            "model": d.get("model"), "word": d.get("word_size"),
            "pred_us": d["predicted_us"]}


def memcpy_gbs(x):
    z = torch.empty_like(x)
    ms = timeit(lambda: z.copy_(x))
    return round(2 * x.numel() * x.element_size() / ms / 1e6, 1)


def sweep_t2d():
    cases = [wl.s1(), wl.Case("sq8", (11584, 11584), (1, 0), 8, 3),
             wl.Case("s5_2301", (12544, 11648), (1, 0), 8, 4)]
    for c in cases:
        x, ref, p0 = setup(c)
        print(json.dumps({"case": c.name, "memcpy_gbs": memcpy_gbs(x), "auto": measure(c, x, ref)}), flush=True)
        tiles = [(64, 64), (128, 64), (64, 128), (128, 128)] if c.esize == 4 else \
                [(32, 32), (64, 32), (32, 64), (64, 64)]
        for order in (1, 2):
            for ta, tb in tiles:
                for cps in (1, 2, 3, 4, 6, 8):
                    r = measure(c, x, ref, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb,
                                ctas_per_sm=cps, grid_order=order)
                    print(json.dumps({"case": c.name, "order": order, "ta": ta, "tb": tb, "cps": cps,
                                      **r}), flush=True)
        ident = tt.Plan((c.vol,), (0,), c.esize)
        y = torch.empty_like(x)
        ms = timeit(lambda: ident.execute(x, y))
        print(json.dumps({"case": c.name, "own_copy_gbs": round(2 * c.nbytes / ms / 1e6, 1)}), flush=True)
        del x, ref
        torch.cuda.empty_cache()


def sweep_tile(n):
    cases = wl.s2_ttc()[::max(1, 57 // n)][:n]
    for c in cases:
        x, ref, p0 = setup(c)
        auto = measure(c, x, ref)
        print(json.dumps({"case": c.name, "dims": c.dims, "perm": c.perm, "memcpy_gbs": memcpy_gbs(x),
                          "auto": auto}), flush=True)
        E = c.esize
        for rb_in in (128, 256, 512, 1024, 2048):
            for rb_out in (128, 256, 512, 1024, 2048):
                r = measure(c, x, ref, kernel=tt.KERNEL_TILE, run_in=rb_in // E, run_out=rb_out // E)
                print(json.dumps({"case": c.name, "rin": rb_in, "rout": rb_out, **r}), flush=True)
        del x, ref
        torch.cuda.empty_cache()


def sweep_t2ds():
    """Scalar 2-D kernel (odd extents): tiles x CTAs/SM x order."""
    cases = [wl.Case("o4", (12953, 12953), (1, 0), 4, 3), wl.Case("o8", (9159, 9161), (1, 0), 8, 4),
             wl.Case("o8b", (119, 119, 119, 119), (3, 2, 1, 0), 8, 5)]
    for c in cases:
        x, ref, p0 = setup(c)
        print(json.dumps({"case": c.name, "memcpy_gbs": memcpy_gbs(x), "auto": measure(c, x, ref)}), flush=True)
        tiles = [(64, 64), (128, 64), (64, 128)] if c.esize == 4 else [(64, 64), (32, 64), (64, 32)]
        for order in (1, 2):
            for ta, tb in tiles:
                for cps in (1, 2, 3, 4, 6):
                    r = measure(c, x, ref, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb,
                                ctas_per_sm=cps, grid_order=order)
                    print(json.dumps({"case": c.name, "order": order, "ta": ta, "tb": tb, "cps": cps,
                                      "gbs": r.get("gbs"), "ok": r.get("ok")}), flush=True)
        r = measure(c, x, ref, kernel=tt.KERNEL_TILE)
        print(json.dumps({"case": c.name, "generic": r.get("gbs")}), flush=True)
        del x, ref
        torch.cuda.empty_cache()


def sweep_cps(n):
    """Auto tile geometry at different persistent-grid sizes (CTAs per SM)."""
    cases = wl.s2_ttc()[::max(1, 57 // n)][:n] + \
        [c for c in wl.s3_random(per_cell=1, set2_random=0) if c.rank >= 6][::7]
    for c in cases:
        x, ref, p0 = setup(c)
        print(json.dumps({"case": c.name, "dims": c.dims, "perm": c.perm, "esize": c.esize,
                          "memcpy_gbs": memcpy_gbs(x), "auto": measure(c, x, ref)}), flush=True)
        for cps in (1, 2, 3, 4, 6, 8):
            r = measure(c, x, ref, ctas_per_sm=cps)
            print(json.dumps({"case": c.name, "cps": cps, **r}), flush=True)
        del x, ref
        torch.cuda.empty_cache()


def calib_cases():
    cs = wl.s2_ttc()[2::5]
    s3 = [c for c in wl.s3_random(per_cell=1, set2_random=0)]
    cs += [c for c in s3 if c.rank >= 4][::5]
    cs += [c for c in wl.s3_random(per_cell=0, set2_random=2) if c.tags[0] == "SET2"][::2]
    return cs


def sweep_calib():
    """Forced generic-tile geometries (run targets x threads) per case, for
    fitting the planner's model."""
    for c in calib_cases():
        j0 = tt.plan_offline(c.dims, c.perm, c.esize)
        if j0["kernel"] != "tile":
            continue
        x, ref, p0 = setup(c)
        print(json.dumps({"case": c.name, "dims": c.dims, "perm": c.perm, "esize": c.esize,
                          "memcpy_gbs": memcpy_gbs(x), "auto": measure(c, x, ref)}), flush=True)
        E = c.esize
        seen = set()
        for rb_in in (64, 128, 256, 512, 1024):
            for rb_out in (64, 128, 256, 512, 1024):
                for thr in (0, 64, 128, 256, 512):
                    try:
                        j = tt.plan_offline(c.dims, c.perm, E, kernel=tt.KERNEL_TILE,
                                            run_in=max(2, rb_in // E), run_out=max(2, rb_out // E),
                                            threads=thr)
                    except tt.TTError:
                        continue
                    key = (tuple(j["tile"]["ext"]), j["threads"], j["nreg"])
                    if key in seen:
                        continue
                    seen.add(key)
                    r = measure(c, x, ref, kernel=tt.KERNEL_TILE, run_in=max(2, rb_in // E),
                                run_out=max(2, rb_out // E), threads=thr)
                    print(json.dumps({"case": c.name, "rin": rb_in, "rout": rb_out, "thr": thr,
                                      "nreg": j["nreg"], **r}), flush=True)
        del x, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "t2d":
        sweep_t2d()
    elif mode == "t2ds":
        sweep_t2ds()
    elif mode == "calib":
        sweep_calib()
    elif mode == "cps":
        sweep_cps(int(sys.argv[2]) if len(sys.argv) > 2 else 8)
    else:
        sweep_tile(int(sys.argv[2]) if len(sys.argv) > 2 else 6)
