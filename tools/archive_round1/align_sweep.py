"""S1 throughput vs buffer base alignment x tile config (robustness sweep)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

n = 16384 * 16384
MB = 1 << 20
big = torch.empty((4096 * MB) // 4, dtype=torch.int32, device="cuda")
print("big at", hex(big.data_ptr()), flush=True)
big[: 2 * n].random_()
s = torch.cuda.current_stream()
configs = [dict(kernel=4, run_in=ta, run_out=tb, grid_order=o, ctas_per_sm=c)
           for (ta, tb) in ((64, 128), (128, 64), (128, 128), (64, 64))
           for o in (1, 2) for c in (1, 2, 3)]
for xoff_mb, yoff_mb in ((0, 1024), (512, 1536), (256, 1280), (2, 1026), (0, 1536), (512, 2048)):
    base = big.data_ptr()
    # align the big buffer's start to 1 GB inside the allocation
    pad = ((base + (1 << 30) - 1) & ~((1 << 30) - 1)) - base
    x = big[(pad + xoff_mb * MB) // 4:(pad + xoff_mb * MB) // 4 + n]
    y = big[(pad + yoff_mb * MB) // 4:(pad + yoff_mb * MB) // 4 + n]
    res = []
    for cfg in configs:
        try:
            p = tt.Plan((16384, 16384), (1, 0), 4, **cfg)
        except tt.TTError:
            continue
        for _ in range(3):
            p.execute(x, y)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(30):
            p.execute(x, y)
        b.record(s)
        b.synchronize()
        res.append((round(2 * n * 4 / (a.elapsed_time(b) / 30) / 1e6), cfg["run_in"], cfg["run_out"],
                    cfg["grid_order"], cfg["ctas_per_sm"]))
        p.destroy()
    res.sort(reverse=True)
    print("x@%s y@%s" % (hex(x.data_ptr() % (1 << 32)), hex(y.data_ptr() % (1 << 32))), res, flush=True)
