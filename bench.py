#!/usr/bin/env python
"""Benchmark of the B200 tensor-permutation hot path (arXiv 1705.01598, cuTT).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config s1|s2|s5local|s5batch|s5redist|s5p2p]
                    [--suites default|full|none] [--verify full|none]

One step = one pass of the whole hot path (plan already built: one
tt_execute, or one tt_execute_sharded) over one tensor.  The default workload
is BASELINE.json configs[1] (16384x16384 fp32, perm (1,0)); the metric is the
paper's bandwidth 2*vol*E/D in GB/s (10^9), whole job.

Inputs are the seeded words of tt_workloads (host), uploaded to HBM before
the timed region; after it the timed output is copied back and compared with
the CPU oracle element by element (memcmp; "verified" in the JSON line).

Multi-GPU (one process per GPU; `--gpus N` outside torchrun spawns its own N
ranks through torch.distributed.run):
  s1        every rank permutes its own tensor (independent units, weak scaling)
  s5local   BASELINE configs[4], local case: the global tensor block-sharded
            along its outermost dim, a 1/N slab per rank (strong scaling)
  s5batch   8 independent S5 tensors, 8/N per rank (strong scaling)
  s5redist  redistribution case: pack -> ncclAlltoAll -> unpack, with the
            pack / all-to-all / unpack split and the NVLink fraction
  s5p2p     the fused NVLink-P2P redistribution (f-1)

At N = 1 the JSON line also carries `suites`: the rank 2-12 suites of
BASELINE.json configs[2-3] (a fixed seeded set; `--suites full` = every case
of S2 / S3 / Set 2 / S4), each case verified in full against the oracle,
reported as worst / median / best fraction of a same-bytes device copy
(P:L281), per-rank medians and plan time.

``--impl reference`` times the CPU oracle (oracle/) on the same workload
(bounded sample per step) -- the deliberately slow baseline, not a target.
``--dry-run`` runs the multi-process plumbing (spawn, gloo process group,
offline sharded plans, max-over-ranks timing) without a GPU, for CPU tests.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import queue
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import tt_workloads as wl  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
DTYPE_NAME = {4: "u32", 8: "u64"}
NVLINK_GBS = 900.0        # NVLink 5 per direction per GPU (nominal)
NVLINK_MEASURED = 770.0   # B200_PROFILING.md: measured peer copy per direction
CONFIGS = ["s1", "s2", "s5local", "s5batch", "s5redist", "s5p2p"]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="s1", choices=CONFIGS)
    ap.add_argument("--suites", default="default", choices=["default", "full", "none"])
    ap.add_argument("--suites-out", default="", help="per-case JSONL of the suites")
    ap.add_argument("--suites-plan", default="both-all", choices=["heuristic", "both", "both-all"],
                    help="both-all: also the measurement-based plan (tt_plan_measure) of every suite case; "
                         "both: only on Set 2 and S3 ranks 10-12")
    ap.add_argument("--verify", default="full", choices=["full", "none"])
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps (capped at 20)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--stream-first", action="store_true",
                    help="create the plan's stream before the first device allocation (order check)")
    ap.add_argument("--no-order-check", action="store_true",
                    help="skip the stream-first re-measurement of the S1 headline")
    return ap.parse_args(argv)


def workload(name: str):
    if name == "s1":
        c = wl.s1()
        return c, f"S1: {c.dims[0]}x{c.dims[1]} fp32 transpose, perm (1,0) (BASELINE.json configs[1])"
    if name == "s2":
        c = wl.s2_ttc()[30]
        return c, f"S2 TTC-style rank-{c.rank} fp64 case {c.name} dims {c.dims} perm {c.perm}"
    if name in ("s5local", "s5batch"):
        c = wl.s5_sharded()[0]
        return c, (f"S5 {name[2:]} 112x112x112x104 fp64 perm {c.perm} (BASELINE.json configs[4])"
                   + (", 8 independent tensors" if name == "s5batch" else ""))
    if name in ("s5redist", "s5p2p"):
        c = wl.s5_sharded()[5]
        return c, f"S5 {name[2:]} 112x112x112x104 fp64 perm {c.perm} (BASELINE.json configs[4])"
    raise ValueError(name)


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args, argv) -> int:
    """`--gpus N` outside torchrun: relaunch this script as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML every few ms."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples = []
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self, t0: float, t1: float):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        if not inside:  # region shorter than one sample: take the nearest ones
            inside = sorted(self.samples, key=lambda s: abs(s[0] - (t0 + t1) / 2))[:3]
        reasons = set()
        for _, _, rs in inside:
            for bit, name in self.REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[1] for s in inside), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(inside)}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(kernel_key: str):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(kernel_key)
    return None


# ---------------------------------------------------------------------------
# Verification leg: the timed output against the CPU oracle, in full.
# (Test infrastructure inside the bench: never on the product path.)
# ---------------------------------------------------------------------------

_libc = ctypes.CDLL(None)
_libc.memcmp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
_libc.memcmp.restype = ctypes.c_int


def memcmp_equal(a: np.ndarray, b: np.ndarray) -> bool:
    if a.nbytes != b.nbytes:
        return False
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return _libc.memcmp(a.ctypes.data, b.ctypes.data, a.nbytes) == 0


def oracle_expected(case, words, threads=None):
    from oracle import oracle as orc
    return orc.permute_threaded(case.dims, case.perm, words, threads=threads)


# ---------------------------------------------------------------------------
# CPU oracle baseline (bounded sample)
# ---------------------------------------------------------------------------

def _oracle_range_threaded(orc, case, words, out, begin, end, threads):
    bounds = [begin + (end - begin) * t // threads for t in range(threads + 1)]
    ts = [threading.Thread(target=orc.permute_range,
                           args=(case.dims, case.perm, words, out, bounds[t], bounds[t + 1]))
          for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def oracle_sample_time(case, words, budget_s: float, threads: int):
    """Time the oracle on output ranges until ~budget_s of CPU work; returns
    (GB/s, elements, seconds)."""
    from oracle import oracle as orc
    out = np.empty(case.vol, dtype=words.dtype)
    probe = min(case.vol, 1 << 20)
    t0 = time.perf_counter()
    _oracle_range_threaded(orc, case, words, out, 0, probe, threads)
    dt = max(1e-6, time.perf_counter() - t0)
    n = int(min(case.vol, max(probe, probe * budget_s / dt)))
    t0 = time.perf_counter()
    _oracle_range_threaded(orc, case, words, out, 0, n, threads)
    dt = time.perf_counter() - t0
    return 2.0 * n * case.esize / dt / 1e9, n, dt


def cpu_baseline(case, words):
    """The oracle on all host threads (bounded sample) and on one thread
    (smaller sample), as it stands."""
    threads = len(os.sched_getaffinity(0))
    gbs, n, dt = oracle_sample_time(case, words, 10.0, threads)
    g1, n1, d1 = oracle_sample_time(case, words, 4.0, 1)
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"output elements [0, {n}) of {case.vol} ({dt:.1f} s, {threads} threads, "
                      f"C gather odometer)",
            "single_thread": {"value": round(g1, 3), "unit": "GB/s", "cores": 1,
                              "sample": f"output elements [0, {n1}) ({d1:.1f} s, 1 thread)"}}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    case, desc = workload(args.config)
    threads = len(os.sched_getaffinity(0))
    words = case.words()
    from oracle import oracle as orc
    out = np.empty(case.vol, dtype=words.dtype)
    # one step = a bounded sample: ~ (budget / steps) seconds of CPU work
    probe = min(case.vol, 1 << 20)
    t0 = time.perf_counter()
    _oracle_range_threaded(orc, case, words, out, 0, probe, threads)
    rate = probe / max(1e-6, time.perf_counter() - t0)
    total_budget = 60.0
    per_step = max(1 << 16, int(min(case.vol, rate * total_budget / max(1, args.steps + args.warmup))))
    for _ in range(args.warmup):
        _oracle_range_threaded(orc, case, words, out, 0, per_step, threads)
    t0 = time.perf_counter()
    for s in range(args.steps):
        b = (s * per_step) % max(1, case.vol - per_step + 1)
        _oracle_range_threaded(orc, case, words, out, b, b + per_step, threads)
    dt = time.perf_counter() - t0
    ms = dt / args.steps * 1e3
    gbs = 2.0 * per_step * case.esize * args.steps / dt / 1e9
    sample = (f"{per_step} output elements per step (of {case.vol}; contiguous output range, "
              f"{threads} host threads, C gather odometer)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE_NAME[case.esize], "data": "synthetic",
        "config": config_dict(args, case, desc, args.gpus, sharded=False),
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, case, desc, world, sharded, plan_desc=None):
    c = {"workload": desc, "dims": list(case.dims), "perm": list(case.perm), "elem_bytes": case.esize,
         "global_batch": (8 if args.config == "s5batch" else (1 if sharded else world)),
         "parallelism": {"s1": "independent tensor per GPU" if world > 1 else "single GPU",
                         "s2": "independent tensor per GPU" if world > 1 else "single GPU",
                         "s5local": f"sharded along the outermost dim, 1/{world} slab per GPU",
                         "s5batch": f"8 independent tensors, {8 // max(1, world)} per GPU",
                         "s5redist": "sharded, pack -> ncclAlltoAll -> unpack",
                         "s5p2p": "sharded, fused NVLink-P2P redistribution"}[args.config],
         "l2": "inputs larger than L2 (126 MB); no flush"}
    if plan_desc:
        c["plan"] = {k: plan_desc.get(k) for k in ("kernel", "threads", "grid", "smem", "nreg", "stages")}
        c["tile"] = {k: plan_desc.get("tile", {}).get(k) for k in ("ext", "V", "sm")}
    return c


# ---------------------------------------------------------------------------
# suites (rank 2-12, BASELINE.json configs[2-3]), N = 1
# ---------------------------------------------------------------------------

def suite_cases(which: str):
    if which == "full":
        s2 = wl.s2_ttc()
        s3 = [c for c in wl.s3_random(per_cell=20, set2_random=0) if c.tags[0] == "S3"]
        st = [c for c in wl.s3_random(per_cell=0, set2_random=50) if c.tags[0] == "SET2"]
    else:
        s2 = wl.s2_ttc()
        s3 = [c for c in wl.s3_random(per_cell=2, set2_random=0) if c.tags[0] == "S3"]
        st = [c for c in wl.s3_random(per_cell=0, set2_random=10) if c.tags[0] == "SET2"]
    return {"S2": s2, "S3": s3, "SET2": st, "S4": wl.s4_alignment()}


def _event_median(fn, reps, stream):
    import torch
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def _plan_key(d):
    return json.dumps({k: v for k, v in d.items() if k not in ("measured",)}, sort_keys=True)


def run_suites(tt, dev, which, reps, out_path="", measured=False):
    """Every case: seeded words uploaded to HBM, plan time, median of `reps`
    event-timed executes, same-bytes device copy, full memcmp against the
    oracle.  Words and oracle output of the next cases are prepared on host
    threads while the GPU works."""
    import torch
    groups = suite_cases(which)
    cases = [(g, c) for g, cs in groups.items() for c in cs]
    q: "queue.Queue" = queue.Queue(maxsize=2)

    def producer():
        for g, c in cases:
            w = c.words()
            q.put((g, c, w, oracle_expected(c, w)))
        q.put(None)

    th = threading.Thread(target=producer, daemon=True)
    t_start = time.perf_counter()
    th.start()
    # one pinned host buffer for the outputs copied back for verification
    # (pageable copies of 1-2 GB cost ~0.5 s each under the oracle's threads)
    pin = torch.empty(max(c.nbytes for _, c in cases), dtype=torch.uint8).pin_memory()

    def fetch(y, dtype):
        h = pin[:y.numel() * y.element_size()]
        h.copy_(y.view(torch.uint8))
        return h.numpy().view(dtype)
    stream = torch.cuda.Stream(device=dev)
    memcpy_ms = {}
    rows = []
    fout = open(out_path, "w") if out_path else None
    while True:
        item = q.get()
        if item is None:
            break
        g, c, words, want = item
        nd = np.int32 if c.esize == 4 else np.int64
        x = torch.from_numpy(words.view(nd)).to(dev)
        y = torch.empty_like(x)
        t0 = time.perf_counter()
        plan = tt.Plan(c.dims, c.perm, c.esize, stream=stream)
        plan_first = (time.perf_counter() - t0) * 1e6
        warm = []
        for _ in range(5):
            t0 = time.perf_counter()
            p2 = tt.Plan(c.dims, c.perm, c.esize, stream=stream)
            warm.append((time.perf_counter() - t0) * 1e6)
            p2.destroy()
        with torch.cuda.stream(stream):
            ms = _event_median(lambda: plan.execute(x, y), reps, stream)
            if c.nbytes not in memcpy_ms:
                z = torch.empty_like(x)
                memcpy_ms[c.nbytes] = _event_median(lambda: z.copy_(x), reps, stream)
                del z
        stream.synchronize()
        ok = memcmp_equal(fetch(y, words.dtype), want)
        d = plan.describe()
        plan.destroy()
        mrow = {}
        # measurement-based plans: by default on the cases the round-1 review
        # targets (Set 2, and S3 ranks 10-12); --suites-plan both-all = every case
        if measured and (measured == "all" or g == "SET2" or (g == "S3" and c.rank >= 10)):
            # measurement-based plan selection (tt_plan_measure):
            # the candidates run on these buffers, the fastest is kept
            t0 = time.perf_counter()
            mp = tt.Plan(c.dims, c.perm, c.esize, stream=stream, measure=(x, y))
            m_us = (time.perf_counter() - t0) * 1e6
            md = mp.describe()
            with torch.cuda.stream(stream):
                m_ms = _event_median(lambda: mp.execute(x, y), reps, stream)
            stream.synchronize()
            if _plan_key(md) == _plan_key(d):
                m_ok = ok        # the heuristic plan won: same kernel, same output (verified above)
            else:
                m_ok = memcmp_equal(fetch(y, words.dtype), want)
            mp.destroy()
            mt = md.get("tile", {})
            mrow = {"m_ms": round(m_ms, 5), "m_frac_memcpy": round(memcpy_ms[c.nbytes] / m_ms, 4),
                    "m_plan_us": round(m_us, 1), "m_kernel": md["kernel"], "m_vg": "vg" in mt,
                    "m_sd": "sd" in mt, "m_stages": md.get("stages"), "m_tile": mt.get("ext"),
                    "m_run": [md.get("model", {}).get("run_in"), md.get("model", {}).get("run_out")],
                    "m_candidates": md.get("measured", {}).get("candidates"), "m_verified": m_ok}
        r = {"suite": g, "case": c.name, "rank": c.rank, "esize": c.esize, "dims": list(c.dims),
             "perm": list(c.perm), "kernel": d["kernel"], "vg": "vg" in d.get("tile", {}),
             "tile": d.get("tile", {}).get("ext"),
             "run": [d.get("model", {}).get("run_in"), d.get("model", {}).get("run_out")],
             "sd": "sd" in d.get("tile", {}), "ms": round(ms, 5),
             "gbs": round(2 * c.nbytes / ms / 1e6, 1), "frac_memcpy": round(memcpy_ms[c.nbytes] / ms, 4),
             "plan_us": round(statistics.median(warm), 1), "plan_us_first": round(plan_first, 1),
             "plan_us_lib": round(float(d.get("plan_us", 0.0)), 1),
             "verified": ok, "elements": c.vol}
        r.update(mrow)
        rows.append(r)
        if fout:
            fout.write(json.dumps(r) + "\n")
            fout.flush()
        del x, y, want, words
        torch.cuda.empty_cache()
    th.join()
    if fout:
        fout.close()
    out = {}
    for g in groups:
        rs = [r for r in rows if r["suite"] == g]
        if not rs:
            continue
        f = sorted(r["frac_memcpy"] for r in rs)
        gb = sorted(r["gbs"] for r in rs)
        per_rank = {}
        for r in rs:
            per_rank.setdefault(r["rank"], []).append(r["frac_memcpy"])
        med = {str(k): round(statistics.median(v), 4) for k, v in sorted(per_rank.items())}
        pu = sorted(r["plan_us"] for r in rs)
        out[g] = {"n": len(rs), "worst_frac": f[0], "median_frac": round(statistics.median(f), 4),
                  "best_frac": f[-1], "worst_gbs": gb[0], "median_gbs": statistics.median(gb),
                  "best_gbs": gb[-1], "per_rank_median_frac": med,
                  "rank_max_over_min": round(max(med.values()) / max(1e-9, min(med.values())), 3),
                  "plan_us_median": statistics.median(pu), "plan_us_max": pu[-1],
                  "plan_us_first_median": statistics.median(r["plan_us_first"] for r in rs),
                  "plan_us_first_max": max(r["plan_us_first"] for r in rs),
                  # the library's own planning time of that first plan (tt_plan
                  # internal clock: no Python / ctypes; the oracle's host
                  # threads run concurrently in this loop)
                  "plan_us_lib_median": statistics.median(r["plan_us_lib"] for r in rs),
                  "plan_us_lib_max": max(r["plan_us_lib"] for r in rs),
                  "verified": f"{sum(r['verified'] for r in rs)}/{len(rs)} cases, full memcmp vs oracle, "
                              f"{sum(r['elements'] for r in rs)} elements",
                  "all_verified": all(r["verified"] for r in rs)}
        mrs = [r for r in rs if "m_frac_memcpy" in r]
        if measured and mrs:
            rs = mrs
            mf = sorted(r["m_frac_memcpy"] for r in rs)
            mper = {}
            for r in rs:
                mper.setdefault(r["rank"], []).append(r["m_frac_memcpy"])
            out[g]["measured"] = {
                "n": len(rs), "cases": "every case" if len(rs) == out[g]["n"] else "ranks 10-12",
                "heuristic_median_frac_same_cases": round(statistics.median(r["frac_memcpy"] for r in rs), 4),
                "worst_frac": mf[0], "median_frac": round(statistics.median(mf), 4), "best_frac": mf[-1],
                "per_rank_median_frac": {str(k): round(statistics.median(v), 4) for k, v in sorted(mper.items())},
                "plan_us_median": statistics.median(r["m_plan_us"] for r in rs),
                "all_verified": all(r["m_verified"] for r in rs)}
    allr = [r for r in rows if r["suite"] in ("S2", "S3", "SET2")]
    if allr:
        f = sorted(r["frac_memcpy"] for r in allr)
        out["rank2_12"] = {"n": len(allr), "worst_frac": f[0], "median_frac": round(statistics.median(f), 4),
                           "best_frac": f[-1], "all_verified": all(r["verified"] for r in allr)}
        mall = [r for r in allr if "m_frac_memcpy" in r]
        if measured and mall:
            mf = sorted(r["m_frac_memcpy"] for r in mall)
            out["rank2_12"]["measured"] = {"n": len(mall), "worst_frac": mf[0],
                                           "median_frac": round(statistics.median(mf), 4), "best_frac": mf[-1],
                                           "all_verified": all(r["m_verified"] for r in mall)}
    out["wall_s"] = round(time.perf_counter() - t_start, 1)
    out["reps"] = reps
    out["which"] = which
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_dry(args):
    """Multi-process plumbing on CPU: gloo group, offline sharded plans of
    this rank, max-over-ranks reduction and the JSON line -- no kernels."""
    import torch
    import torch.distributed as dist
    import paper_1705_01598_b200 as tt
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    case, desc = workload(args.config)
    if args.config in ("s5local", "s5redist"):
        d = tt.plan_sharded_offline(world, rank, case.dims, case.perm, case.esize)
    elif args.config == "s5p2p":
        d = tt.plan_sharded_p2p_offline(world, rank, case.dims, case.perm, case.esize)
    else:
        d = tt.plan_offline(case.dims, case.perm, case.esize)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "config": args.config,
                          "max_over_ranks": float(t.item()), "mode": d.get("mode", d.get("kernel")),
                          "plan": d}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1705_01598_b200 as tt

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    case, desc = workload(args.config)
    E = case.esize
    nd = np.int32 if E == 4 else np.int64
    p2p = args.config == "s5p2p"
    redist = args.config in ("s5redist", "s5p2p")
    sharded = args.config in ("s5local", "s5redist", "s5p2p")
    batch = args.config == "s5batch"

    # seeded input, uploaded before timing.  Allocated BEFORE the plan's
    # stream is created (tools/stream_exp3.py: ~4 % on S1 otherwise; the
    # default run re-measures the headline with the other order in a child
    # process and reports both, "order_check").
    early_stream = torch.cuda.Stream(device=dev) if args.stream_first else None
    if sharded:
        words_all = case.words()
        slab = case.vol // world
        words = words_all[rank * slab:(rank + 1) * slab]   # input slab r (outermost dim)
        nbatch = 1
    elif batch:
        nbatch = max(1, 8 // world)
        words_all = None
        words = None
    else:
        words = wl.random_words(case.vol, E, case.seed + rank)
        nbatch = 1
    if batch:
        xs = [torch.from_numpy(wl.random_words(case.vol, E, case.seed + 8 * rank + b).view(nd)).to(dev)
              for b in range(nbatch)]
        ys = [torch.empty_like(x) for x in xs]
        x, y = xs[0], ys[0]
    else:
        x = torch.from_numpy(np.ascontiguousarray(words).view(nd)).to(dev)
        y = torch.empty_like(x)
    local_vol = x.numel()
    torch.cuda.synchronize()
    stream = early_stream if early_stream is not None else torch.cuda.Stream(device=dev)

    if p2p:
        comm = tt.Comm.from_process_group() if world > 1 else tt.Comm(tt.unique_id(), 1, 0)
        # one rank: force the fused path (registration + both barriers run)
        plan = tt.P2PShardedPlan(comm, case.dims, case.perm, E, stream=stream, force_redistribute=world == 1)
        plan.register_output(y)
        execute = plan.execute
        units_all = case.vol
    elif sharded:
        comm = tt.Comm.from_process_group() if world > 1 else tt.Comm(tt.unique_id(), 1, 0)
        plan = tt.ShardedPlan(comm, case.dims, case.perm, E, stream=stream)
        execute = plan.execute
        units_all = case.vol
    else:
        t0 = time.perf_counter()
        plan = tt.Plan(case.dims, case.perm, E, stream=stream)
        plan_us = (time.perf_counter() - t0) * 1e6   # first plan of the process: includes the CUDA module load
        t0 = time.perf_counter()
        tt.Plan(case.dims, case.perm, E, stream=stream).destroy()
        plan_us_cached = (time.perf_counter() - t0) * 1e6
        if batch:
            def execute(_x, _y):
                for xb, yb in zip(xs, ys):
                    plan.execute(xb, yb)
            units_all = case.vol * nbatch * world
        else:
            execute = plan.execute
            units_all = case.vol * world
    desc_plan = plan.describe()
    if desc_plan.get("sharded"):  # report the dominant sub-plan (fused / local / pack)
        for key in ("fused", "local", "pack"):
            if key in desc_plan:
                desc_plan = dict(desc_plan[key], sharded_mode=desc_plan["mode"])
                break

    sampler = ClockSampler(local)
    sampler.start()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            execute(x, y)
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            execute(x, y)
        ev1.record(stream)
    ev1.synchronize()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler.stop()
    ms_local = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = 2.0 * units_all * E / (ms_step * 1e-3) / 1e9
    clocks = sampler.summary(h0, h1)

    # sharded split (pack / all-to-all / unpack, or barriers / fused / barrier)
    split = None
    if sharded:
        with torch.cuda.stream(stream):
            execute(x, y)
        sp = torch.tensor(list(plan.timings()), dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(sp, op=dist.ReduceOp.MAX)
        sp = [float(v) for v in sp.tolist()]
        shard_bytes = local_vol * E
        nv_bytes = (world - 1) / world * shard_bytes
        keys = ("entry_barrier_ms", "fused_ms", "exit_barrier_ms") if p2p else ("pack_ms", "alltoall_ms", "unpack_ms")
        split = dict(zip(keys, [round(v, 4) for v in sp]))
        if not p2p and redist:
            split["a2a_chunks"] = int(plan.describe().get("chunks", 1))
            if split["a2a_chunks"] > 1:
                split["split_note"] = ("chunked exchange: each value is that step's span (first chunk's "
                                       "start to last chunk's end); the spans overlap")
        split["nvlink_bytes_per_gpu_per_direction"] = int(nv_bytes)
        if redist and world > 1:
            t_x = sp[1] if not p2p else ms_step
            split["nvlink_frac"] = round(nv_bytes / (t_x * 1e-3) / 1e9 / NVLINK_GBS, 4)
            split["nvlink_frac_of_measured"] = round(nv_bytes / (t_x * 1e-3) / 1e9 / NVLINK_MEASURED, 4)
            split["nvlink_note"] = ("(P-1)/P * shard bytes over the " + ("all-to-all" if not p2p else "whole step")
                                    + f" time, vs {NVLINK_GBS:.0f} GB/s nominal / {NVLINK_MEASURED:.0f} measured")

    # verification leg: the timed output, in full, against the oracle
    verified = None
    if args.verify == "full" and not batch:
        stream.synchronize()
        got = y.cpu().numpy().view(np.uint32 if E == 4 else np.uint64)
        if sharded:
            # the global output, block-sharded along its outermost output dim
            threads = max(1, len(os.sched_getaffinity(0)) // world)
            want = oracle_expected(case, words_all, threads)
            slab = case.vol // world
            ok = memcmp_equal(got, want[rank * slab:(rank + 1) * slab])
        else:
            threads = max(1, len(os.sched_getaffinity(0)) // world)
            ok = memcmp_equal(got, oracle_expected(case, words, threads))
        okt = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        if world > 1:
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        verified = {"ok": bool(okt.item()), "how": f"full memcmp of every rank's timed output vs the CPU oracle",
                    "elements": int(case.vol if sharded else case.vol * world)}
        del got

    # memcpy roofline of the same bytes on the same stream (P:L252 GPU-STREAM
    # analogue).  It runs after the host-side verification leg, when the GPU
    # has idled and its clocks may still be ramping: 10 warm-up copies, then
    # the best of three timed batches
    z = torch.empty_like(x)
    with torch.cuda.stream(stream):
        for _ in range(10):
            z.copy_(x)
    reps = max(10, min(50, args.steps))
    best_ms = None
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(reps):
                z.copy_(x)
        e1.record(stream)
        e1.synchronize()
        t = e0.elapsed_time(e1) / reps
        best_ms = t if best_ms is None else min(best_ms, t)
    memcpy_gbs = 2.0 * local_vol * E / (best_ms * 1e-3) / 1e9
    del z

    # end-to-end through the C ABI with pinned host buffers (H2D + kernel + D2H)
    e2e = None
    if not sharded and not batch and not args.no_e2e:
        e2e_steps = args.e2e_steps or min(args.steps, 20)
        hin = torch.empty(local_vol, dtype=x.dtype).pin_memory()
        hin.copy_(torch.from_numpy(words.view(nd)))
        hout = torch.empty_like(hin).pin_memory()
        plan.execute_host(hin, hout, x, y)
        stream.synchronize()
        if world > 1:
            dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(e2e_steps):
            plan.execute_host(hin, hout, x, y)
        f1.record(stream)
        f1.synchronize()
        te = torch.tensor([f0.elapsed_time(f1) / e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(2.0 * local_vol * E * world / (float(te.item()) * 1e-3) / 1e9, 3),
               "unit": "GB/s", "h2d_bytes_per_step": local_vol * E, "d2h_bytes_per_step": local_vol * E,
               "ms_per_step": round(float(te.item()), 4), "steps": e2e_steps,
               "note": "tt_execute_host: pinned H2D + permute + D2H on the plan stream",
               "verified": bool(memcmp_equal(hout.numpy().view(np.uint32 if E == 4 else np.uint64),
                                             oracle_expected(case, words)))
               if args.verify == "full" and rank == 0 else None}
        del hin, hout

    cpu = None
    suites = None
    if rank == 0 and world == 1:
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(case, words if words is not None else case.words())
        if args.suites != "none":
            plan.destroy()
            del x, y
            torch.cuda.empty_cache()
            suites = run_suites(tt, dev, args.suites, 10 if args.suites == "full" else 20, args.suites_out,
                                measured={"heuristic": False, "both": True, "both-all": "all"}[args.suites_plan])
            plan = None

    if rank == 0:
        peak, peak_src = peak_hbm()
        achieved = 2.0 * local_vol * E * nbatch / (ms_step * 1e-3) / 1e9  # per GPU
        kernel_key = f"{args.config}:{desc_plan.get('kernel')}"
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True,
            "scaling": "strong" if args.config in ("s5local", "s5batch", "s5redist", "s5p2p") else "weak",
            "vs_baseline": None, "dtype": DTYPE_NAME[E], "data": "synthetic",
            "config": config_dict(args, case, desc, world, sharded, desc_plan),
            "verified": verified,
            "memcpy_gbs_per_gpu": round(memcpy_gbs, 2),
            "frac_of_memcpy": round(achieved / memcpy_gbs, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic_from_profiles(kernel_key),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": 2 * local_vol * E,
                         "kernel": desc_plan.get("kernel")},
            "clocks": clocks,
            "gpu_launches": args.steps * (plan.launches if plan is not None else 1) * nbatch,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if (args.config == "s1" and world == 1 and not args.stream_first and not args.no_order_check
                and not args.dry_run):
            # the same headline in a child process whose stream exists before
            # its first allocation (the order a caller may well use)
            cmd =[sys.executable, os.path.abspath(__file__), "--steps", str(args.steps), "--warmup",
                   str(args.warmup), "--suites", "none", "--no-e2e", "--no-cpu-baseline", "--verify", "none",
                   "--stream-first", "--no-order-check"]
            try:
                r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
                alt = json.loads(r.stdout.strip().splitlines()[-1])
                line["order_check"] = {
                    "stream_first_value": alt["value"], "unit": alt["unit"],
                    "stream_first_frac": alt["roofline"]["frac"],
                    "note": "same workload, plan and timing in a child process that creates its CUDA stream "
                            "before the first device allocation; `value` allocates first (DESIGN.md, "
                            "'A measured environment effect')"}
            except Exception as ex:  # noqa: BLE001 -- reported, not fatal
                line["order_check"] = {"error": str(ex)[:200]}
        if not sharded:
            line["plan_us"] = round(plan_us, 1)
            line["plan_us_cached"] = round(plan_us_cached, 1)
            line["plan_note"] = ("plan_us: the process's first tt_plan (includes the CUDA module load); "
                                 "plan_us_cached: the same problem again (plan cache); cold per-problem "
                                 "plan times of the suites: suites.*.plan_us_first")
        if split:
            line["sharded"] = split
        if suites:
            line["suites"] = suites
        print(json.dumps(line), flush=True)
    if plan is not None:
        plan.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    world, _, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args, argv)
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
