"""Scalar 2-D kernel: register double buffer vs cp.async ring (stages 3/4),
tiles x CTAs/SM, on odd-extent 2-D-class cases (S2/S4 shapes).  GB/s by
2*vol*E/t; outputs compared with the default plan's (sanity only; parity is
in tests/)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

CASES_BIG = [((31623, 6325), (1, 0), 8), ((35897, 7179), (1, 0), 8), ((64807, 4320), (1, 0), 8),
             ((585, 342225), (1, 0), 8), ((181, 1107981), (1, 0), 8), ((76475, 2619), (1, 0), 8),
             ((5881, 29403), (1, 0), 4), ((12953, 12953), (1, 0), 4), ((585, 585, 585), (1, 0, 2), 8),
             ((585, 585, 585), (2, 1, 0), 8)]
CASES = [((585, 585, 585), (1, 0, 2), 8), ((119,) * 4, (3, 2, 1, 0), 8), ((36, 77, 15, 5, 51, 19), (4, 3, 2, 5, 0, 1), 8),
         ((1304, 101, 1517), (1, 0, 2), 8), ((585, 585, 585), (2, 1, 0), 8), ((181, 2709, 409), (1, 2, 0), 8),
         ((13953, 13953), (1, 0), 4), ((13955, 13955), (1, 0), 4), ((11585, 11585), (1, 0), 8)]
TILES = {8: [(32, 64), (64, 64), (64, 32)], 4: [(64, 64), (128, 64), (64, 128)]}


def timed(p, x, y, reps=15):
    for _ in range(3):
        p.execute(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        p.execute(x, y)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


CPS = (2, 3, 4, 6)


def main():
    global CPS
    torch.cuda.set_device(0)
    cases = CASES
    if len(sys.argv) > 1 and sys.argv[1] == "big":
        cases, CPS = CASES_BIG, (1, 2, 3, 4)
    for dims, perm, E in cases:
        n = 1
        for d in dims:
            n *= d
        td = torch.int32 if E == 4 else torch.int64
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=td, device="cuda")
        y = torch.empty_like(x)
        ref = torch.empty_like(x)
        p0 = tt.Plan(dims, perm, E)
        t0 = timed(p0, x, ref)
        z = torch.empty_like(x)
        z.copy_(x)
        tc = timed(type("C", (), {"execute": lambda self, a, b: b.copy_(a)})(), x, z)
        res = {"dims": dims, "perm": perm, "E": E, "default_kernel": p0.describe()["kernel"],
               "default_gbs": round(2 * n * E / t0 / 1e6, 1), "memcpy_gbs": round(2 * n * E / tc / 1e6, 1), "v": {}}
        for ta, tb in (TILES[E] if cases is CASES else [(64, 64)]):
            for st in (0, 3, 4):
                for cps in CPS:
                    try:
                        p = tt.Plan(dims, perm, E, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb,
                                    stages=st, ctas_per_sm=cps)
                    except tt.TTError:
                        continue
                    if p.describe().get("vec", 1) != 1:
                        continue
                    t = timed(p, x, y)
                    ok = bool(torch.equal(y, ref))
                    res["v"][f"{ta}x{tb}_s{st}_c{cps}"] = round(2 * n * E / t / 1e6, 1) if ok else "MISMATCH"
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
