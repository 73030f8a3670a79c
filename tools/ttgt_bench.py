"""TTGT contraction benchmark (SURVEY f-4; Section 3.4).

A seeded sample of TAL-SH-style random contractions: tensors up to
rank 8, contracted and free labels at random positions, up to 4 leading
"large" dimensions per tensor, the others of extent <= 8, large dimensions
scaled so that the largest tensor holds ~150 M fp64 (or 300 M fp32)
elements (the M40/P100 setting).  Each contraction D = L . R runs through
tt_contract_execute; time from the first transpose to the end of the last
operation (CUDA events on the plan's stream), GFLOP/s = 2 m n k / t,
arithmetic intensity AI = 2 sqrt(vol D vol L vol R) / (vol D + vol L + vol R)
(P:L321), and the share of time in the transposes.  Sanity: a few sampled
outputs against torch.einsum in fp64 (parity proper is tests/test_contract.py).
    python tools/ttgt_bench.py [count] [esize] > out.jsonl"""
import json
import math
import os
import string
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402


def gen(rng, esize):
    target = 150_000_000 if esize == 8 else 300_000_000
    while True:
        rl, rr = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        c = int(rng.integers(1, min(rl, rr) + 1))
        fl, fr = rl - c, rr - c
        if fl + fr >= 1 and fl + fr <= 8:
            break
    labels = list(range(fl + fr + c))
    rng.shuffle(labels)
    K, FL, FR = labels[:c], labels[c:c + fl], labels[c + fl:]
    ml = [int(x) for x in rng.permutation(K + FL)]
    mr = [int(x) for x in rng.permutation(K + FR)]
    md = [int(x) for x in rng.permutation(FL + FR)]
    large = set()
    for ms in (ml, mr, md):
        for m in ms[:int(rng.integers(1, 5))]:
            large.add(m)
    small = {m: int(rng.integers(2, 9)) for m in labels}
    base = {m: float(rng.uniform(1.0, 2.0)) for m in labels}

    def ext(s):
        return {m: (max(2, int(round(base[m] * s))) if m in large else small[m]) for m in labels}

    def vmax(e):
        return max(math.prod(e[m] for m in ms) for ms in (ml, mr, md))
    lo, hi = 1.0, 1e6
    for _ in range(60):
        mid = math.sqrt(lo * hi)
        if vmax(ext(mid)) <= target:
            lo = mid
        else:
            hi = mid
    e = ext(lo)
    return md, [e[m] for m in ml], ml, [e[m] for m in mr], mr


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    esize = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    rng = np.random.default_rng(1705)
    dt = torch.float64 if esize == 8 else torch.float32
    for i in range(count):
        md, dl, ml, dr, mr = gen(rng, esize)
        c = tt.Contraction(md, dl, ml, dr, mr, esize, stream=stream)
        g = torch.Generator(device=dev)
        g.manual_seed(i)
        L = torch.randn(math.prod(dl), dtype=dt, device=dev, generator=g)
        R = torch.randn(math.prod(dr), dtype=dt, device=dev, generator=g)
        vd = math.prod(c.dims_d) if c.dims_d else 1
        D = torch.empty(vd, dtype=dt, device=dev)
        for _ in range(2):
            c.execute(L, R, D)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(stream)
        for _ in range(reps):
            c.execute(L, R, D)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        steps = c.timings()
        # sanity: sampled outputs vs torch.einsum (fp64) on the column-major views
        labels = sorted(set(ml) | set(mr))
        ch = {m: string.ascii_letters[j] for j, m in enumerate(labels)}
        sub = lambda ms_: "".join(ch[m] for m in reversed(ms_))  # noqa: E731
        ok = None
        if 2 * c.m * c.n * c.k < 2e12:
            want = torch.einsum(f"{sub(ml)},{sub(mr)}->{sub(md)}",
                                L.double().reshape(tuple(reversed(dl))),
                                R.double().reshape(tuple(reversed(dr)))).reshape(-1)
            idx = torch.randint(0, vd, (4096,), device=dev, generator=g)
            err = (D.double()[idx] - want[idx]).abs().max().item()
            scale = want[idx].abs().max().item() + 1e-300
            ok = err <= (1e-10 if esize == 8 else 1e-3) * scale * max(1.0, math.sqrt(c.k))
            del want
        vl, vr = math.prod(dl), math.prod(dr)
        ai = 2 * math.sqrt(vd * vl * vr) / (vd + vl + vr)
        print(json.dumps({"i": i, "modes_d": md, "dims_l": dl, "modes_l": ml, "dims_r": dr, "modes_r": mr,
                          "m": c.m, "n": c.n, "k": c.k, "ai": round(ai, 1), "ms": round(ms, 4),
                          "gflops": round(2 * c.m * c.n * c.k / ms / 1e6, 1),
                          "steps_ms": [round(x, 4) for x in steps],
                          "transpose_share": round((steps[0] + steps[1] + steps[3]) / max(1e-9, sum(steps)), 4),
                          "launches": c.describe()["launches"], "ok": ok}), flush=True)
        c.destroy()
        del L, R, D
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
