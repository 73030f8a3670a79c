#!/usr/bin/env python
"""Benchmark of the B200 tensor-permutation hot path (arXiv 1705.01598, cuTT).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config s1|s2|s5local|s5redist]

One step = one pass of the whole hot path (plan already built: one
tt_execute) over one tensor.  The default workload is BASELINE.json
configs[1] (16384x16384 fp32, perm (1,0)); the metric is the paper's
bandwidth 2*vol*E/D in GB/s (10^9), whole job.  At N > 1 every rank
permutes its own tensor (independent units, weak scaling, no collective);
``--config s5redist`` times the sharded NCCL redistribution instead.

``--impl reference`` times the CPU oracle (oracle/) on the same workload
(bounded sample per step) -- the deliberately slow baseline, not a target.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import tt_workloads as wl  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
DTYPE_NAME = {4: "u32", 8: "u64"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="s1", choices=["s1", "s2", "s5local", "s5redist", "s5p2p"])
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps (capped at 20)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload(name: str):
    if name == "s1":
        c = wl.s1()
        return c, f"S1: {c.dims[0]}x{c.dims[1]} fp32 transpose, perm (1,0) (BASELINE.json configs[1])"
    if name == "s2":
        c = wl.s2_ttc()[30]
        return c, f"S2 TTC-style rank-{c.rank} fp64 case {c.name} dims {c.dims} perm {c.perm}"
    if name in ("s5local", "s5redist", "s5p2p"):
        c = wl.s5_sharded()[0 if name == "s5local" else 5]
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
# CPU oracle baseline (the only bench leg that executes oracle/)
# ---------------------------------------------------------------------------

def oracle_sample_time(case, words, budget_s: float, threads: int):
    """Time the oracle on output ranges until ~budget_s of CPU work; returns
    (GB/s, elements, seconds, description)."""
    from oracle import oracle as orc
    out = np.empty(case.vol, dtype=words.dtype)
    # probe the rate on a small range, then size the sample
    probe = min(case.vol, 1 << 20)
    t0 = time.perf_counter()
    _oracle_range_threaded(orc, case, words, out, 0, probe, threads)
    dt = max(1e-6, time.perf_counter() - t0)
    n = int(min(case.vol, max(probe, probe * budget_s / dt)))
    t0 = time.perf_counter()
    _oracle_range_threaded(orc, case, words, out, 0, n, threads)
    dt = time.perf_counter() - t0
    gbs = 2.0 * n * case.esize / dt / 1e9
    return gbs, n, dt


def _oracle_range_threaded(orc, case, words, out, begin, end, threads):
    bounds = [begin + (end - begin) * t // threads for t in range(threads + 1)]
    ts = [threading.Thread(target=orc.permute_range,
                           args=(case.dims, case.perm, words, out, bounds[t], bounds[t + 1]))
          for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    case, desc = workload(args.config)
    threads = len(os.sched_getaffinity(0))
    words = case.words()
    from oracle import oracle as orc
    out = np.empty(case.vol, dtype=words.dtype)
    # size one step as a bounded sample: ~ (budget / steps) seconds of CPU work
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
        "config": {"workload": desc, "dims": list(case.dims), "perm": list(case.perm),
                   "elem_bytes": case.esize, "parallelism": "host threads"},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1705_01598_b200 as tt

    world, rank, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus > 1 must be launched with torch.distributed.run (one rank per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    case, desc = workload(args.config)
    E = case.esize
    tdt = torch.int32 if E == 4 else torch.int64
    # s5p2p: the fused redistribution (f-1); on one GPU the redistribution is
    # forced with a one-rank communicator (registration + both barriers run)
    p2p = args.config == "s5p2p"
    if p2p and world == 1:
        os.environ["TT_SHARD_FORCE_REDIST"] = "1"
    sharded = (args.config == "s5redist" and world > 1) or p2p
    local_vol = case.vol // world if sharded else case.vol

    # seeded input, resident in HBM before timing (rank-specific seed).
    # Allocated BEFORE the plan's stream is created: creating a stream before
    # the first device allocation measured ~4 % slower for S1 with the same
    # kernel (tools/stream_exp3.py; profiles/round1_summary.md).
    g = torch.Generator(device=dev)
    g.manual_seed(case.seed + rank)
    x = torch.randint(-(2 ** 31), 2 ** 31 - 1, (local_vol,), dtype=tdt, device=dev, generator=g)
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=dev)

    if p2p:
        comm = tt.Comm.from_process_group() if world > 1 else tt.Comm(tt.unique_id(), 1, 0)
        plan = tt.P2PShardedPlan(comm, case.dims, case.perm, E, stream=stream)
        plan.register_output(y)
        execute = plan.execute
        units_per_step_all = case.vol  # global tensor per step
    elif sharded:
        comm = tt.Comm.from_process_group()
        plan = tt.ShardedPlan(comm, case.dims, case.perm, E, stream=stream)
        execute = plan.execute
        units_per_step_all = case.vol  # global tensor per step
    else:
        plan = tt.Plan(case.dims, case.perm, E, stream=stream)
        execute = plan.execute
        units_per_step_all = case.vol * world
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
    bytes_step_all = 2.0 * units_per_step_all * E
    value = bytes_step_all / (ms_step * 1e-3) / 1e9
    clocks = sampler.summary(h0, h1)

    # memcpy roofline of the same bytes on the same stream (P:L252 GPU-STREAM analogue)
    z = torch.empty_like(x)
    with torch.cuda.stream(stream):
        for _ in range(3):
            z.copy_(x)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = max(10, min(50, args.steps))
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(reps):
            z.copy_(x)
    e1.record(stream)
    e1.synchronize()
    memcpy_gbs = 2.0 * local_vol * E / (e0.elapsed_time(e1) / reps * 1e-3) / 1e9
    del z

    # end-to-end through the C ABI with pinned host buffers (H2D + kernel + D2H)
    e2e = None
    if not sharded and not args.no_e2e:
        e2e_steps = args.e2e_steps or min(args.steps, 20)
        hin = torch.empty(local_vol, dtype=tdt).pin_memory()
        hin.copy_(x.cpu())
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
               "note": "tt_execute_host: pinned H2D + permute + D2H on the plan stream"}
        del hin, hout

    # CPU oracle baseline (rank 0, N=1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        words = case.words()
        gbs, n, dt = oracle_sample_time(case, words, 15.0, threads)
        cpu = {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "oracle",
               "sample": f"output elements [0, {n}) of {case.vol} ({dt:.1f} s, {threads} threads, "
                         f"C gather odometer)"}
        del words

    if rank == 0:
        peak, peak_src = peak_hbm()
        achieved = 2.0 * local_vol * E / (ms_step * 1e-3) / 1e9  # per GPU, dominant kernel
        kernel_key = f"{args.config}:{desc_plan.get('kernel')}"
        traffic = traffic_from_profiles(kernel_key)
        launches_per_step = plan.launches
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": DTYPE_NAME[E], "data": "synthetic",
            "config": {
                "workload": desc, "dims": list(case.dims), "perm": list(case.perm),
                "elem_bytes": E, "global_batch": world if not sharded else 1,
                "parallelism": ("sharded, fused P2P redistribution" if p2p else
                                "sharded all-to-all" if sharded else
                                ("independent tensor per GPU" if world > 1 else "single GPU")),
                "l2": "inputs larger than L2 (%.0f MB per tensor > 126 MB L2); no flush" % (local_vol * E / 1e6),
                "plan": {k: desc_plan.get(k) for k in ("kernel", "threads", "grid", "smem", "nreg")},
                "tile": {k: desc_plan.get("tile", {}).get(k) for k in ("ext", "V", "sm")},
            },
            "memcpy_gbs_per_gpu": round(memcpy_gbs, 2),
            "frac_of_memcpy": round(achieved / memcpy_gbs, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": 2 * local_vol * E,
                         "kernel": desc_plan.get("kernel")},
            "clocks": clocks,
            "gpu_launches": args.steps * launches_per_step,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    plan.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
