"""Is the S1 headline sensitive to where its buffers land in device memory?
For k = 0..K-1: reserve k x 2 MiB (or k x 64 MiB) before allocating the
1 GiB input and output, plan and time the S1 transpose (CUDA events, 20
launches after 5 warm-up), release everything (empty_cache) and repeat.
Also the same with a stream created before the first allocation."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1705_01598_b200 as tt  # noqa: E402

N = 16384
dev = torch.device("cuda", 0)


def timed(pre_bytes, stream_first):
    s0 = torch.cuda.Stream() if stream_first else None
    pad = torch.empty(max(1, pre_bytes // 4), dtype=torch.int32, device=dev) if pre_bytes else None
    x = torch.randint(-2**31, 2**31 - 1, (N * N,), dtype=torch.int32, device=dev)
    y = torch.empty_like(x)
    s = s0 if s0 is not None else torch.cuda.Stream()
    p = tt.Plan((N, N), (1, 0), 4, stream=s)
    with torch.cuda.stream(s):
        for _ in range(5):
            p.execute(x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            p.execute(x, y)
        e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    r = {"pre_MiB": pre_bytes >> 20, "stream_first": stream_first, "gbs": round(2 * N * N * 4 / ms / 1e6, 1),
         "x_addr_mod_2MiB": x.data_ptr() % (2 << 20), "x_addr_GiB": round(x.data_ptr() / 2**30, 3),
         "y_minus_x_MiB": (y.data_ptr() - x.data_ptr()) >> 20}
    p.destroy()
    del x, y, pad, s, s0
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return r


torch.empty(1, device=dev)
for stream_first in (False, True):
    for k in list(range(0, 8)) + [16, 31, 32, 33, 64, 100, 127]:
        print(json.dumps(timed(k * (2 << 20), stream_first)), flush=True)
