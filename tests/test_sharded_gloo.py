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
