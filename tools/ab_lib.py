"""A/B two builds of libtt.so on the same GPU in one process (same input).
    python tools/ab_lib.py OTHER.so "dims" "perm" esize [rounds]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    vp, i64p, ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)
    L.tt_plan.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t, vp]
    L.tt_execute.argtypes = [vp, vp, vp]
    return L


other = load(sys.argv[1])
cur = tt.lib
dims = [int(x) for x in sys.argv[2].split(",")]
perm = [int(x) for x in sys.argv[3].split(",")]
E = int(sys.argv[4])
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 5
n = 1
for d in dims:
    n *= d
td = torch.int32 if E == 4 else torch.int64
x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=td, device="cuda")
ys = [torch.empty_like(x), torch.empty_like(x)]
s = torch.cuda.current_stream()
plans = []
for L in (cur, other):
    h = ctypes.c_void_p()
    r = L.tt_plan(ctypes.byref(h), len(dims), (ctypes.c_int64 * len(dims))(*dims),
                  (ctypes.c_int * len(perm))(*perm), E, s.cuda_stream)
    assert r == 0, r
    plans.append((L, h))
    vp = ctypes.c_void_p
    buf = ctypes.create_string_buffer(1 << 16)
    L.tt_plan_describe.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    L.tt_plan_describe(h, buf, 1 << 16)
    import json
    dj = json.loads(buf.value.decode())
    print({k: dj.get(k) for k in ("kernel", "threads", "grid", "smem", "vec")}, dj.get("tiled2d", {}).get("TA"),
          dj.get("tiled2d", {}).get("TB"), dj.get("tiled2d", {}).get("lanes"))
res = {0: [], 1: []}
for _ in range(rounds):
    for i, (L, h) in enumerate(plans):
        for _ in range(3):
            L.tt_execute(h, x.data_ptr(), ys[i].data_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(20):
            L.tt_execute(h, x.data_ptr(), ys[i].data_ptr())
        b.record(s)
        b.synchronize()
        res[i].append(2 * n * E / (a.elapsed_time(b) / 20) / 1e6)
assert torch.equal(ys[0], ys[1])
print("current GB/s", [round(v) for v in res[0]], "max", round(max(res[0])))
print("other   GB/s", [round(v) for v in res[1]], "max", round(max(res[1])))
