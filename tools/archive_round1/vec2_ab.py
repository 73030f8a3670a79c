"""A/B: vectorised 2-D kernel with 2-element vectors vs the scalar 2-D kernel
(TT_KNOB_T2D_VEC2 / _VEC8 = 0), 2-D-class cases whose rows allow only
2-element vectors.  Each variant planned in a subprocess-free way by setting
the knob before planning (the planner reads it per plan)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

CASES = [((13954, 13954), (1, 0), 4), ((13958, 13958), (1, 0), 4), ((13962, 13962), (1, 0), 4),
         ((13966, 13966), (1, 0), 4), ((2 * 4099, 3 * 4099), (1, 0), 4), ((586, 586, 586), (2, 1, 0), 4),
         ((586, 586, 586), (1, 0, 2), 4),
         ((11584, 11584), (1, 0), 8), ((11586, 11586), (1, 0), 8), ((14142, 14142), (1, 0), 8),
         ((584, 584, 584), (2, 1, 0), 8), ((584, 584, 584), (1, 0, 2), 8), ((186, 50, 250, 86), (2, 3, 0, 1), 8),
         ((120, 120, 120, 120), (3, 2, 1, 0), 8)]


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
        z = torch.empty_like(x)
        res = {"dims": dims, "perm": perm, "E": E}
        tc = timed(type("C", (), {"execute": lambda self, a, b: b.copy_(a)})(), x, z)
        res["memcpy"] = round(2 * n * E / tc / 1e6, 1)
        knob = "TT_KNOB_T2D_VEC2" if E == 4 else "TT_KNOB_T2D_VEC8"
        for val in ("1", "0", "1", "0"):
            os.environ[knob] = val
            p = tt.Plan(dims, perm, E)
            d = p.describe()
            t = timed(p, x, y if val == "0" else ref)
            key = f"{'vec' if val == '1' else 'scalar'}:{d['kernel']}:v{d.get('vec')}"
            res.setdefault(key, []).append(round(2 * n * E / t / 1e6, 1))
            p.destroy()
        os.environ[knob] = "1"
        res["equal"] = bool(torch.equal(y, ref))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
