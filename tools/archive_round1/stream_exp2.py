"""Reproduce bench.py's setup order: stream created before the inputs."""
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
if mode == "default":
    s = torch.cuda.current_stream(dev)
p = tt.Plan((16384, 16384), (1, 0), 4, stream=s)
with torch.cuda.stream(s):
    for _ in range(10):
        p.execute(x, y)
s.synchronize()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    a.record(s)
    for _ in range(200):
        p.execute(x, y)
    b.record(s)
b.synchronize()
print(mode, round(2 * n * 4 / (a.elapsed_time(b) / 200) / 1e6), hex(x.data_ptr()), hex(y.data_ptr()), flush=True)
