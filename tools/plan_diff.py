"""Offline plan of a case from two libtt builds: python tools/plan_diff.py OTHER.so CASE..."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1705_01598_b200 as tt  # noqa: E402
import tt_workloads as wl  # noqa: E402


def offline(L, c):
    vp = ctypes.c_void_p
    h = vp()
    props = tt.DeviceProps(148, 232448, 233472, 2048, 65536)
    o = tt.PlanOptions()
    L.tt_plan_offline.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_int), ctypes.c_size_t,
                                  ctypes.POINTER(tt.DeviceProps), ctypes.POINTER(tt.PlanOptions)]
    r = L.tt_plan_offline(ctypes.byref(h), len(c.dims), (ctypes.c_int64 * len(c.dims))(*c.dims),
                          (ctypes.c_int * len(c.perm))(*c.perm), c.esize, ctypes.byref(props), ctypes.byref(o))
    assert r == 0, r
    buf = ctypes.create_string_buffer(1 << 16)
    L.tt_plan_describe.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    L.tt_plan_describe(h, buf, 1 << 16)
    return json.loads(buf.value.decode())


other = ctypes.CDLL(sys.argv[1])
cs = {c.name: c for c in wl.s2_ttc() + wl.s3_random(per_cell=1) + wl.s4_alignment()}
for nm in sys.argv[2:]:
    c = cs[nm]
    for tag, L in (("new", tt.lib), ("old", other)):
        j = offline(L, c)
        t = j.get("tile", {})
        print(nm, tag, j["kernel"], "T", j["threads"], "G", j["grid"], "V", t.get("V"), t.get("ext"),
              "sd", (t.get("sd") or {}).get("R"), "pred", round(j["predicted_us"], 1),
              "runs", j.get("model", {}).get("run_in"), j.get("model", {}).get("run_out"))
