"""S1 back-to-back on different streams (legacy default, created, high priority)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402

n = 16384 * 16384
x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
streams = {"legacy": torch.cuda.default_stream(), "created": torch.cuda.Stream(),
           "created_hi": torch.cuda.Stream(priority=-1), "external0": torch.cuda.ExternalStream(0)}
for rnd in range(2):
    for name, s in streams.items():
        p = tt.Plan((16384, 16384), (1, 0), 4, stream=s)
        with torch.cuda.stream(s):
            for _ in range(5):
                p.execute(x, y)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(100):
                p.execute(x, y)
            b.record(s)
        b.synchronize()
        print(rnd, name, s.cuda_stream, round(2 * n * 4 / (a.elapsed_time(b) / 100) / 1e6), flush=True)
        p.destroy()
