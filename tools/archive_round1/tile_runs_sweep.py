"""Generic tile: forced (run_in, run_out) targets with and without the
larger slot-dim tiles (TT_KNOB_SD_VMAX), on the weakest generic-tile cases.
GB/s = 2*vol*E/t; sanity-compared with the default plan's output."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

CASES = [((7,) * 10, (0, 2, 1, 3, 5, 4, 8, 7, 9, 6), 4),
         ((7, 4, 11, 14, 12, 3, 12, 5, 5, 3), (0, 6, 8, 1, 3, 5, 4, 9, 2, 7), 4),
         ((5, 7, 7, 7, 7, 7, 7, 7, 7, 7), (0, 8, 3, 1, 5, 7, 4, 6, 2, 9), 8),
         ((1, 2, 25, 2, 3, 2, 6, 4, 23, 19, 2, 19), (0, 8, 11, 4, 10, 3, 2, 6, 1, 7, 5, 9), 8),
         ((5,) * 12, (0, 11, 3, 10, 6, 8, 4, 7, 2, 9, 5, 1), 8),
((5, 3, 2, 4, 35, 33, 37, 40), (7, 6, 5, 4, 3, 2, 1, 0), 4),
         ((5,) * 12, (0, 8, 4, 10, 1, 3, 9, 5, 7, 2, 6, 11), 4),
         ((2, 3, 4, 3, 2, 2, 3, 2, 20, 18, 22, 24), tuple(range(11, -1, -1)), 4),
         ((5, 3, 2, 4, 35, 33, 37, 40), (6, 4, 1, 7, 5, 3, 0, 2), 4),
         ((3, 6, 6, 6, 6, 6, 6, 6, 6, 6, 6), (0, 7, 2, 3, 6, 9, 10, 8, 5, 1, 4), 4),
         ((7,) * 10, (0, 2, 1, 3, 5, 4, 8, 7, 9, 6), 4)]


def timed(p, x, y, reps=10):
    for _ in range(2):
        p.execute(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        p.execute(x, y)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    torch.cuda.set_device(0)
    for dims, perm, E in CASES:
        n = 1
        for d in dims:
            n *= d
        td = torch.int32 if E == 4 else torch.int64
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=td, device="cuda")
        y = torch.empty_like(x)
        ref = torch.empty_like(x)
        p0 = tt.Plan(dims, perm, E)
        t0 = timed(p0, x, ref)
        res = {"dims": dims, "perm": perm, "default": round(2 * n * E / t0 / 1e6, 1),
               "default_tile": p0.describe()["tile"]["ext"], "v": []}
        # run targets: powers of two and whole-dimension prefix products
        pin, pout, acc = [], [], 1
        for d in dims:
            acc *= d
            if 2 <= acc <= 8192:
                pin.append(acc)
        acc = 1
        for j in perm:
            acc *= dims[j]
            if 2 <= acc <= 8192:
                pout.append(acc)
        tin = sorted(set([16, 32, 64, 128, 256, 512] + pin))
        tout = sorted(set([16, 32, 64, 128, 256, 512, 1024] + pout))
        for vmax in ("0", "8192"):
            os.environ["TT_KNOB_SD_VMAX"] = vmax
            for ri in tin:
                for ro in tout:
                    try:
                        p = tt.Plan(dims, perm, E, run_in=ri, run_out=ro)
                    except tt.TTError:
                        continue
                    t = timed(p, x, y)
                    if not torch.equal(y, ref):
                        res["v"].append((vmax, ri, ro, "MISMATCH"))
                        continue
                    d = p.describe()
                    res["v"].append((vmax, ri, ro, round(2 * n * E / t / 1e6, 1), d["tile"]["ext"],
                                     d["threads"], d["grid"], "sd" in d["tile"]))
        os.environ["TT_KNOB_SD_VMAX"] = "0"
        res["v"].sort(key=lambda r: -r[3] if isinstance(r[3], float) else 0)
        res["v"] = res["v"][:6]
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
