"""Sharded path host logic with a real 2-process exchange on CPU (gloo).

Each process builds the library's sharded plan for its rank offline
(tt_plan_sharded_offline: same geometry and sub-plans tt_plan_sharded
builds), replays its pack plan on its input slab, exchanges blocks with
torch.distributed.all_to_all_single over gloo (standing in for
ncclAlltoAll), replays the unpack plan, and rank 0 checks the gathered
output slabs against the oracle of the global tensor."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CASES = [
    ((6, 4, 5, 8), (3, 2, 1, 0), 8),   # redistribute
    ((6, 4, 5, 8), (2, 3, 0, 1), 4),   # redistribute, fuses to rank 2
    ((6, 4, 6, 8), (1, 0, 3, 2), 8),   # redistribute
    ((6, 4, 6, 8), (0, 3, 1, 2), 4),   # redistribute
    ((6, 4, 5, 8), (1, 0, 2, 3), 8),   # local
    ((6, 4, 5, 8), (2, 1, 0, 3), 4),   # local
    ((7, 4, 10), (2, 0, 1), 8),        # redistribute, rank 3
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    sys.path[:0] = [ROOT, HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1705_01598_b200 as tt
    from oracle import oracle as orc
    import tt_workloads as wl
    from plan_interp import interpret_plan
    ok = []
    for gdims, perm, esize in CASES:
        j = tt.plan_sharded_offline(world, rank, gdims, perm, esize)
        n = len(gdims)
        vol = int(np.prod(gdims))
        words = wl.random_words(vol, esize, 31)           # the global tensor
        slab = vol // world
        local_in = words[rank * slab:(rank + 1) * slab]   # outermost-dim block
        if j["mode"] == "local":
            local_out = interpret_plan(j["local"], local_in)
        else:
            packed = interpret_plan(j["pack"], local_in)
            td = torch.int64 if esize == 8 else torch.int32
            nd = np.int64 if esize == 8 else np.int32
            send = torch.from_numpy(packed.view(nd).copy())
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send)
            local_out = interpret_plan(j["unpack"], recv.numpy().view(words.dtype))
        assert list(j["local_out_dims"]) == [gdims[perm[k]] // (world if k == n - 1 else 1)
                                             for k in range(n)]
        gathered = [torch.empty(slab, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(local_out.astype(np.int64)))
        if rank == 0:
            got = np.concatenate([g.numpy() for g in gathered]).astype(words.dtype)
            want = orc.permute(gdims, perm, words)
            ok.append(bool(np.array_equal(got, want)))
    if rank == 0:
        results.extend(ok)
    dist.destroy_process_group()


def test_sharded_two_ranks_gloo():
    mgr = mp.Manager()
    results = mgr.list()
    mp.spawn(_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    assert list(results) == [True] * len(CASES)


def test_sharded_offline_geometry_and_errors():
    sys.path[:0] = [ROOT, HERE]
    import paper_1705_01598_b200 as tt
    j = tt.plan_sharded_offline(8, 3, (112, 112, 112, 104), (1, 0, 2, 3), 8)
    assert j["mode"] == "local" and j["local_in_dims"] == [112, 112, 112, 13]
    assert j["launches"] == 1
    j = tt.plan_sharded_offline(8, 3, (112, 112, 112, 104), (3, 2, 1, 0), 8)
    assert j["mode"] == "redistribute" and j["launches"] == 3
    assert j["local_out_dims"] == [104, 112, 112, 14]
    assert j["a2a_count"] * 8 == j["shard_bytes"] // 8
    with pytest.raises(tt.TTError):   # shard dim not divisible
        tt.plan_sharded_offline(3, 0, (112, 112, 112, 104), (3, 2, 1, 0), 8)
    with pytest.raises(tt.TTError):   # redistributed dim not divisible
        tt.plan_sharded_offline(8, 0, (6, 4, 5, 8), (0, 1, 3, 2), 8)


def _replay_fused(j, inbuf, outbuf):
    """Host replay of the fused sub-box plan (strided geometry) into outbuf."""
    from plan_interp import interpret_tile_plan, interpret_tiled2d_plan
    fj = dict(j)
    fj["dims"] = j["fused"]["dims"]
    if j["kernel"] == "tiled2d":
        return interpret_tiled2d_plan(fj, inbuf, out=outbuf)
    return interpret_tile_plan(fj, inbuf, out=outbuf)


P2P_CASES = [
    ((6, 4, 5, 8), (3, 2, 1, 0), 8, 2),
    ((6, 4, 6, 8), (2, 3, 0, 1), 4, 2),
    ((8, 4, 8, 8), (1, 0, 3, 2), 8, 4),
    ((6, 4, 8, 8), (0, 3, 1, 2), 4, 4),
    ((7, 4, 10), (2, 0, 1), 8, 2),
    ((8, 8, 4, 8), (2, 3, 0, 1), 4, 8),
    ((6, 4, 5, 8), (1, 0, 2, 3), 8, 4),     # local case: one launch into the own slab
]


@pytest.mark.parametrize("gdims,perm,esize,P", P2P_CASES)
def test_p2p_fused_geometry_emulated_ranks(gdims, perm, esize, P):
    """Fused redistribution (f-1) geometry: every emulated rank replays its
    sub-box plan once per destination into the destination's output slab at
    the plan's offsets; the slabs must tile the oracle's output exactly once."""
    sys.path[:0] = [ROOT, HERE]
    import paper_1705_01598_b200 as tt
    from oracle import oracle as orc
    import tt_workloads as wl
    from plan_interp import interpret_plan
    n = len(gdims)
    vol = int(np.prod(gdims))
    words = wl.random_words(vol, esize, 77)
    slab = vol // P
    outs = [np.zeros(slab, dtype=words.dtype) for _ in range(P)]
    hits = [np.zeros(slab, dtype=np.int64) for _ in range(P)]
    for r in range(P):
        j = tt.plan_sharded_p2p_offline(P, r, gdims, perm, esize)
        local_in = words[r * slab:(r + 1) * slab]
        if j["mode"] == "local":
            assert j["launches"] == 1
            outs[r][:] = interpret_plan(j["local"], local_in)
            hits[r] += 1
            continue
        assert j["mode"] == "p2p" and j["launches"] == P
        assert j["dest_order"][-1] == r and sorted(j["dest_order"]) == list(range(P))
        fused = j["fused"]
        assert fused["fused"]["dims"] and int(np.prod(fused["dims"])) == slab // P
        for q in j["dest_order"]:
            src = local_in[q * j["in_step"]:]
            before = outs[q].copy()
            _replay_fused(fused, src, outs[q][j["out_offset"]:])
            hits[q] += outs[q] != before   # positions this sub-box wrote (random words)
    want = orc.permute(gdims, perm, words)
    got = np.concatenate(outs)
    np.testing.assert_array_equal(got, want)
    assert list(j["local_out_dims"]) == [gdims[perm[k]] // (P if k == n - 1 else 1) for k in range(n)]


def test_p2p_offline_errors():
    sys.path[:0] = [ROOT, HERE]
    import paper_1705_01598_b200 as tt
    with pytest.raises(tt.TTError):   # redistributed dim not divisible
        tt.plan_sharded_p2p_offline(8, 0, (6, 4, 5, 8), (0, 1, 3, 2), 8)
    with pytest.raises(tt.TTError):   # more than 64 ranks
        tt.plan_sharded_p2p_offline(128, 0, (6, 4, 5, 128), (0, 1, 3, 2), 8)
    j = tt.plan_sharded_p2p_offline(8, 3, (112, 112, 112, 104), (3, 2, 1, 0), 8)
    assert j["mode"] == "p2p" and j["local_out_dims"] == [104, 112, 112, 14]
    assert j["in_step"] == 14 and j["out_offset"] == 3 * 13   # input dim 3 is output dim 0
