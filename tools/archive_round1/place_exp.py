"""Does the relative placement of input and output buffers change S1 throughput?"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

n = 16384 * 16384
big = torch.empty(3 * n + (64 << 20) // 4, dtype=torch.int32, device="cuda")
big.random_()
p = tt.Plan((16384, 16384), (1, 0), 4)
s = torch.cuda.current_stream()
for off_mb in [0, 1, 2, 4, 8, 16, 32, 64, 0.5, 0.25, 3, 5, 7, 13]:
    off = int(off_mb * (1 << 20)) // 4
    x = big[:n]
    y = big[n + off: 2 * n + off]
    for _ in range(3):
        p.execute(x, y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(50):
        p.execute(x, y)
    b.record(s)
    b.synchronize()
    z = big[2 * n + off: 3 * n + off]
    c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c.record(s)
    for _ in range(20):
        z.copy_(x)
    d.record(s)
    d.synchronize()
    print("y offset %6.2f MB after x: transpose %d GB/s, copy %d GB/s" % (
        off_mb, 2 * n * 4 / (a.elapsed_time(b) / 50) / 1e6, 2 * n * 4 / (c.elapsed_time(d) / 20) / 1e6), flush=True)
