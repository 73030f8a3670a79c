"""Time one permutation under several plan-option sets, interleaved on the
same buffers, and report GB/s (2*vol*E/D) per option set.

    python tools/case_sweep.py "5,5,5,5" "0,2,1,3" 4 "run_in=125,run_out=125" "slots=4" ...
The first row is always the default plan."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402


def main():
    dims = tuple(int(x) for x in sys.argv[1].split(","))
    perm = tuple(int(x) for x in sys.argv[2].split(","))
    E = int(sys.argv[3])
    sets = [{}] + [{k: int(v) for k, v in (kv.split("=") for kv in s.split(",") if kv)}
                   for s in sys.argv[4:]]
    n = 1
    for d in dims:
        n *= d
    td = torch.int32 if E == 4 else torch.int64
    x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=td, device="cuda")
    ys = []
    plans = []
    for o in sets:
        try:
            plans.append(tt.Plan(dims, perm, E, **o))
            ys.append(torch.empty_like(x))
        except tt.TTError as e:
            plans.append(None)
            ys.append(None)
            print(f"{o}: plan failed: {e}")
    s = torch.cuda.current_stream()
    times = [[] for _ in sets]
    for _ in range(5):
        for i, p in enumerate(plans):
            if p is None:
                continue
            for _ in range(2):
                p.execute(x, ys[i])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                p.execute(x, ys[i])
            e1.record(s)
            e1.synchronize()
            times[i].append(e0.elapsed_time(e1) / 10)
    ref = None
    for i, p in enumerate(plans):
        if p is None:
            continue
        ms = statistics.median(times[i])
        same = ref is None or bool(torch.equal(ys[0], ys[i]))
        ref = ref or ms
        d = p.describe()
        t = d.get("tile", {})
        print(f"{str(sets[i]):40s} {2 * n * E / (ms * 1e-3) / 1e9:8.1f} GB/s  x{ref / ms:.3f}  "
              f"{d['kernel']}/T{d.get('threads')}/R{d.get('nreg')}/G{d.get('grid')} ext={t.get('ext')} "
              f"chunks={t.get('split_chunk')} sd={'sd' in t} model={d.get('model')}"
              f"{'' if same else '  OUTPUT DIFFERS'}", flush=True)


if __name__ == "__main__":
    main()
