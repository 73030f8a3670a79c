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
    # 146 MB shards: the exchange is chunked by default, 14 = 4 + 4 + 4 + 2 along t
    assert j["mode"] == "redistribute" and j["chunks"] == 4 and j["launches"] == 3 * 4
    assert (j["chunk_t"], j["chunk_tail"]) == (4, 2) and "pack_tail" in j and "unpack_tail" in j
    j1 = tt.plan_sharded_offline(8, 3, (112, 112, 112, 104), (3, 2, 1, 0), 8, a2a_chunks=1)
    assert j1["chunks"] == 1 and j1["launches"] == 3
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


CHUNK_CASES = [
    ((6, 4, 5, 8), (3, 2, 1, 0), 8, 2, 2),    # c = 3: chunks 2 + 1 (ragged tail)
    ((6, 4, 6, 8), (2, 3, 0, 1), 4, 2, 3),    # c = 3: three chunks of 1
    ((8, 4, 8, 8), (1, 0, 3, 2), 8, 4, 2),    # c = 2: two chunks of 1
    ((8, 4, 8, 8), (1, 0, 3, 2), 8, 4, 5),    # c = 2: asked for 5, clamped to 2
    ((12, 4, 8, 8), (0, 3, 2, 1), 4, 2, 4),   # t = 0 (c = 6): chunks 2 + 2 + 2
    ((7, 4, 10), (2, 0, 1), 8, 2, 3),         # rank 3, c = 2 -> 2 chunks
    ((10, 3, 6, 6), (3, 1, 0, 2), 4, 3, 2),   # P = 3, t = 2 (c = 2): two chunks
]


@pytest.mark.parametrize("gdims,perm,esize,P,K", CHUNK_CASES)
def test_chunked_exchange_geometry_emulated_ranks(gdims, perm, esize, P, K):
    """Chunked redistribution: every emulated rank replays its chunk pack
    plans (strided sub-boxes at the plan's input offsets) into its send
    buffer, the all-to-all of each chunk is emulated block by block, and the
    chunk unpack plans write the output slabs at the chunk offsets; the slabs
    must equal the oracle's output."""
    sys.path[:0] = [ROOT, HERE]
    import paper_1705_01598_b200 as tt
    from oracle import oracle as orc
    import tt_workloads as wl
    from plan_interp import interpret_plan, interpret_tile_plan, interpret_tiled2d_plan
    n = len(gdims)
    if gdims[perm[-1]] % P or gdims[-1] % P:
        pytest.skip("not divisible")
    vol = int(np.prod(gdims))
    words = wl.random_words(vol, esize, 91)
    slab = vol // P
    js = [tt.plan_sharded_offline(P, r, gdims, perm, esize, a2a_chunks=K) for r in range(P)]
    j0 = js[0]
    assert j0["mode"] == "redistribute"
    c = gdims[perm[-1]] // P
    Kc = j0["chunks"]
    assert Kc == -(-c // j0["chunk_t"]) and j0["chunk_tail"] == c - (Kc - 1) * j0["chunk_t"]
    assert j0["launches"] == Kc * (3 if P > 1 else 2)
    w = j0["chunk_w"]
    sends = [np.zeros(slab, dtype=words.dtype) for _ in range(P)]

    def replay(pj, src, dst):
        fj = dict(pj)
        fj["dims"] = pj["fused"]["dims"]
        if pj["kernel"] == "tiled2d":
            interpret_tiled2d_plan(fj, src, out=dst)
        else:
            interpret_tile_plan(fj, src, out=dst)

    chunk_of = lambda k: (j0["chunk_tail"] if k == Kc - 1 else j0["chunk_t"])
    for r, j in enumerate(js):
        local_in = words[r * slab:(r + 1) * slab]
        for k in range(Kc):
            off = k * j["chunk_t"] * w * P
            e = chunk_of(k)
            pj = j["pack_tail"] if (k == Kc - 1 and "pack_tail" in j) else j["pack"]
            assert int(np.prod(pj["dims"])) == P * w * e
            if Kc == 1:
                sends[r][:] = interpret_plan(pj, local_in)
            else:
                replay(pj, local_in[k * j["chunk_t"] * j["chunk_in_step"]:], sends[r][off:off + P * w * e])
    outs = [np.zeros(slab, dtype=words.dtype) for _ in range(P)]
    for r, j in enumerate(js):
        for k in range(Kc):
            off = k * j["chunk_t"] * w * P
            e = chunk_of(k)
            recv = np.concatenate([sends[q][off + r * w * e:off + (r + 1) * w * e] for q in range(P)])
            uj = j["unpack_tail"] if (k == Kc - 1 and "unpack_tail" in j) else j["unpack"]
            outs[r][off:off + P * w * e] = interpret_plan(uj, recv)
    want = orc.permute(gdims, perm, words)
    np.testing.assert_array_equal(np.concatenate(outs), want)
