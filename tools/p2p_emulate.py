"""Fused redistribution (f-1) vs the pack / all-to-all / unpack form, one GPU,
emulated ranks: the S5 redistribution permutations (BJ configs[4]) for
P = 2, 4, 8.  Rank 0's work is timed (all ranks are symmetric):
  fused : the P sub-box launches of tt_plan_sharded_p2p into P slabs in HBM
          (on a real box (P-1)/P of these stores go over NVLink)
  nccl  : pack + unpack kernels of tt_plan_sharded (the all-to-all itself is
          not emulated; it adds ~2S of HBM traffic and the NVLink transfer)
Prints one JSON line per (perm, P): ms and GB/s by 2*S/t (S = shard bytes)."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_01598_b200 as tt  # noqa: E402
import tt_workloads as wl  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    for c in [c for c in wl.s5_sharded() if c.tags[1] == "redist"]:
        vol = c.vol
        for P in (2, 4, 8):
            slab = vol // P
            x = torch.randint(-2**62, 2**62, (slab,), dtype=torch.int64, device=dev)
            outs = [torch.empty(slab, dtype=torch.int64, device=dev) for _ in range(P)]
            sp = tt.P2PShardedPlan(None, c.dims, c.perm, 8, nranks=P, proc=0,
                                   stream=torch.cuda.current_stream())
            fused_ms = timed(lambda: sp.execute_slabs(x, outs))
            kern = sp.describe()["fused"]["kernel"]
            d = tt.plan_sharded_offline(P, 0, c.dims, c.perm, 8)
            pk = tt.Plan(d["pack"]["dims"], d["pack"]["perm"], 8)
            up = tt.Plan(d["unpack"]["dims"], d["unpack"]["perm"], 8)
            tmp = torch.empty_like(x)
            pack_ms = timed(lambda: pk.execute(x, tmp))
            unpack_ms = timed(lambda: up.execute(tmp, outs[0]))
            S = slab * 8
            copy_ms = timed(lambda: tmp.copy_(x))
            print(json.dumps({"perm": c.perm, "P": P, "shard_bytes": S, "fused_kernel": kern,
                              "fused_ms": round(fused_ms, 5),
                              "fused_gbs": round(2 * S / fused_ms / 1e6, 1),
                              "pack_ms": round(pack_ms, 5), "unpack_ms": round(unpack_ms, 5),
                              "pack_unpack_gbs": round(2 * S / (pack_ms + unpack_ms) / 1e6, 1),
                              "memcpy_gbs": round(2 * S / copy_ms / 1e6, 1)}), flush=True)
            sp.destroy()
            pk.destroy()
            up.destroy()


if __name__ == "__main__":
    main()
