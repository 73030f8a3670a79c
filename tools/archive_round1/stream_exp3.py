"""bench.py's setup order (stream first) vs tile configs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

mode = sys.argv[1]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n = 16384 * 16384
if mode == "stream_first":
    s = torch.cuda.Stream(device=dev)
g = torch.Generator(device=dev)
g.manual_seed(1)
x = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device=dev, generator=g)
y = torch.empty_like(x)
torch.cuda.synchronize()
if mode == "stream_after":
    s = torch.cuda.Stream(device=dev)
out = []
for cfg in [dict(), dict(kernel=4, run_in=128, run_out=128, ctas_per_sm=1), dict(kernel=4, run_in=128, run_out=128, ctas_per_sm=2),
            dict(kernel=4, run_in=64, run_out=128, ctas_per_sm=2), dict(kernel=4, run_in=128, run_out=64, ctas_per_sm=2)]:
    p = tt.Plan((16384, 16384), (1, 0), 4, stream=s, **cfg)
    with torch.cuda.stream(s):
        for _ in range(5):
            p.execute(x, y)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(100):
            p.execute(x, y)
        b.record(s)
    b.synchronize()
    out.append((cfg.get("run_in"), cfg.get("run_out"), cfg.get("ctas_per_sm"), round(2 * n * 4 / (a.elapsed_time(b) / 100) / 1e6)))
    p.destroy()
print(mode, hex(x.data_ptr()), out, flush=True)
