"""Sharded path on one GPU.

* Emulated P ranks: the pack and unpack sub-plans of every virtual rank
  (tt_plan_sharded_offline geometry) run on the GPU through tt_plan/
  tt_execute; the all-to-all is emulated with device copies.  Compared with
  the oracle of the global tensor.
* A real single-rank NCCL communicator through tt_comm_init /
  tt_plan_sharded / tt_execute_sharded.
(Multi-rank NCCL needs several GPUs; its host logic is covered by
test_sharded_gloo.py.)
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1705_01598_b200 as tt
from oracle import oracle as orc
import tt_workloads as wl

pytestmark = pytest.mark.gpu

_ND = {4: np.int32, 8: np.int64}


def _dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch.device("cuda", 0)


def _gpu_plan(desc, x):
    y = torch.empty_like(x)
    p = tt.Plan(desc["dims"], desc["perm"], desc["elem_size"])
    p.execute(x, y)
    p.destroy()
    return y


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("perm", [(3, 2, 1, 0), (2, 3, 0, 1), (1, 0, 3, 2), (0, 3, 1, 2),
                                  (1, 0, 2, 3), (2, 1, 0, 3)])
def test_emulated_ranks(P, perm):
    gdims, esize = (16, 24, 8, 40), 8
    vol = int(np.prod(gdims))
    words = wl.random_words(vol, esize, 5)
    x = torch.from_numpy(words.view(_ND[esize]).copy()).to(_dev())
    slab = vol // P
    descs = [tt.plan_sharded_offline(P, r, gdims, perm, esize) for r in range(P)]
    outs = []
    if descs[0]["mode"] == "local":
        for r in range(P):
            outs.append(_gpu_plan(descs[r]["local"], x[r * slab:(r + 1) * slab]))
    else:
        packed = [_gpu_plan(descs[r]["pack"], x[r * slab:(r + 1) * slab]) for r in range(P)]
        cnt = descs[0]["a2a_count"]
        for q in range(P):
            recv = torch.cat([packed[r][q * cnt:(q + 1) * cnt] for r in range(P)])
            outs.append(_gpu_plan(descs[q]["unpack"], recv))
    torch.cuda.synchronize()
    got = torch.cat(outs).cpu().numpy().view(words.dtype)
    np.testing.assert_array_equal(got, orc.permute(gdims, perm, words))


def test_single_rank_nccl():
    _dev()
    comm = tt.Comm(tt.unique_id(), 1, 0)
    for perm in [(3, 2, 1, 0), (1, 0, 2, 3)]:
        gdims = (16, 24, 8, 40)
        words = wl.random_words(int(np.prod(gdims)), 4, 6)
        x = torch.from_numpy(words.view(np.int32).copy()).to(_dev())
        y = torch.empty_like(x)
        sp = tt.ShardedPlan(comm, gdims, perm, 4)
        assert sp.local_in_dims == gdims
        sp.execute(x, y)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy().view(np.uint32), orc.permute(gdims, perm, words))
        sp.destroy()
    comm.destroy()


def test_single_rank_nccl_redistribution_path(monkeypatch):
    """pack -> ncclAlltoAll -> unpack with one rank (forced), so the NCCL
    exchange and the staging buffers run on a single-GPU box."""
    _dev()
    comm = tt.Comm(tt.unique_id(), 1, 0)
    for perm, esize in [((3, 2, 1, 0), 8), ((2, 3, 0, 1), 4), ((0, 3, 1, 2), 8)]:
        gdims = (16, 24, 8, 40)
        words = wl.random_words(int(np.prod(gdims)), esize, 7)
        x = torch.from_numpy(words.view(_ND[esize]).copy()).to(_dev())
        y = torch.empty_like(x)
        sp = tt.ShardedPlan(comm, gdims, perm, esize, force_redistribute=True)
        d = sp.describe()
        assert d["mode"] == "redistribute" and d["launches"] == 2
        sp.execute(x, y)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy().view(words.dtype), orc.permute(gdims, perm, words))
        pack_ms, a2a_ms, unpack_ms = sp.timings()
        assert pack_ms > 0 and unpack_ms > 0 and a2a_ms >= 0
        sp.destroy()
    comm.destroy()


@pytest.mark.parametrize("K", [2, 3, 5])
def test_single_rank_nccl_chunked_exchange(K):
    """The chunked, overlapped exchange (a2a_chunks) with one rank (forced):
    per chunk a strided pack on the plan stream, ncclAlltoAll on the
    high-priority stream, the unpack on the second stream; repeated executes
    reuse the staging buffers."""
    _dev()
    comm = tt.Comm(tt.unique_id(), 1, 0)
    for perm, esize in [((3, 2, 1, 0), 8), ((2, 3, 0, 1), 4), ((0, 3, 1, 2), 8), ((1, 3, 2, 0), 4)]:
        gdims = (14, 24, 9, 40)
        words = wl.random_words(int(np.prod(gdims)), esize, 8)
        x = torch.from_numpy(words.view(_ND[esize]).copy()).to(_dev())
        y = torch.empty_like(x)
        s = torch.cuda.Stream()
        sp = tt.ShardedPlan(comm, gdims, perm, esize, stream=s, force_redistribute=True, a2a_chunks=K)
        d = sp.describe()
        c = gdims[perm[-1]]
        assert d["mode"] == "redistribute" and d["chunks"] == -(-c // d["chunk_t"]) and d["chunks"] > 1
        assert d["launches"] == 2 * d["chunks"]
        want = orc.permute(gdims, perm, words)
        for _ in range(3):
            y.fill_(-1)
            with torch.cuda.stream(s):
                sp.execute(x, y)
            s.synchronize()
            np.testing.assert_array_equal(y.cpu().numpy().view(words.dtype), want)
        pack_ms, a2a_ms, unpack_ms = sp.timings()
        assert pack_ms > 0 and unpack_ms > 0 and a2a_ms >= 0
        sp.destroy()
    comm.destroy()


# ---- fused redistribution (SURVEY f-1): tt_plan_sharded_p2p ----------------

@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("perm,esize", [((3, 2, 1, 0), 8), ((2, 3, 0, 1), 4), ((1, 0, 3, 2), 8),
                                        ((0, 3, 1, 2), 4), ((2, 0, 3, 1), 8), ((1, 0, 2, 3), 4)])
def test_p2p_emulated_ranks(P, perm, esize):
    """Single-process form: P emulated ranks on one GPU, each storing its P
    sub-boxes straight into the P output slabs (tt_execute_sharded_p2p);
    the slabs together equal the oracle's output of the global tensor.
    Extents leave ragged tiles (24*7 = 168 etc.)."""
    gdims = (24, 56, 16, 40)
    vol = int(np.prod(gdims))
    words = wl.random_words(vol, esize, 11)
    x = torch.from_numpy(words.view(_ND[esize]).copy()).to(_dev())
    slab = vol // P
    outs = [torch.full((slab,), -1, dtype=x.dtype, device=x.device) for _ in range(P)]
    plans = [tt.P2PShardedPlan(None, gdims, perm, esize, nranks=P, proc=r) for r in range(P)]
    want_mode = "local" if perm[-1] == 3 else "p2p"
    for r, sp in enumerate(plans):
        assert sp.describe()["mode"] == want_mode
        sp.execute_slabs(x[r * slab:(r + 1) * slab], outs)
    torch.cuda.synchronize()
    got = torch.cat(outs).cpu().numpy().view(words.dtype)
    np.testing.assert_array_equal(got, orc.permute(gdims, perm, words))
    for sp in plans:
        sp.destroy()


def test_p2p_emulated_full_size_s5():
    """BJ configs[4] at full size (112x112x112x104 fp64, 1.17 GB), 8 emulated
    ranks in the launch configuration the plans choose; every output element
    against the oracle."""
    c = [c for c in wl.s5_sharded() if tuple(c.perm) == (3, 2, 1, 0)][0]
    P, gdims, perm = 8, c.dims, c.perm
    vol = int(np.prod(gdims))
    words = c.words()
    x = torch.from_numpy(words.view(np.int64)).to(_dev())
    slab = vol // P
    out = torch.empty_like(x)
    outs = [out[q * slab:(q + 1) * slab] for q in range(P)]
    for r in range(P):
        sp = tt.P2PShardedPlan(None, gdims, perm, 8, nranks=P, proc=r)
        sp.execute_slabs(x[r * slab:(r + 1) * slab], outs)
        sp.destroy()
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(words.dtype)
    np.testing.assert_array_equal(got, orc.permute_threaded(gdims, perm, words))


def test_p2p_single_rank_comm_barriers(monkeypatch):
    """Multi-process form with one rank (forced redistribution): IPC
    registration through the NCCL all-gather, entry/exit barrier kernels
    over the signal words, repeated executes (epochs), timings."""
    _dev()
    comm = tt.Comm(tt.unique_id(), 1, 0)
    for perm, esize in [((3, 2, 1, 0), 8), ((2, 3, 0, 1), 4)]:
        gdims = (16, 24, 8, 40)
        words = wl.random_words(int(np.prod(gdims)), esize, 8)
        x = torch.from_numpy(words.view(_ND[esize]).copy()).to(_dev())
        big = torch.empty(x.numel() + 64, dtype=x.dtype, device=x.device)
        y = big[32:32 + x.numel()]          # inside an allocation: IPC base + offset
        sp = tt.P2PShardedPlan(comm, gdims, perm, esize, force_redistribute=True)
        d = sp.describe()
        assert d["mode"] == "p2p" and d["launches"] == 3
        with pytest.raises(tt.TTError):      # not registered yet
            sp.execute(x, y)
        sp.register_output(y)
        with pytest.raises(tt.TTError):      # not the registered buffer
            sp.execute(x, torch.empty_like(x))
        for _ in range(3):
            y.fill_(-1)
            sp.execute(x, y)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(y.cpu().numpy().view(words.dtype), orc.permute(gdims, perm, words))
        bar_in, fused_ms, bar_out = sp.timings()
        assert fused_ms > 0 and bar_in >= 0 and bar_out >= 0
        sp.destroy()
    comm.destroy()


def _ipc_worker(rank, port, gdims, perm, result_q):
    """One of two processes sharing cuda:0: the fused redistribution with its
    peer registered through exported / imported IPC records (gloo carries the
    records), entry/exit barriers across the processes, remote stores into the
    other process's output slab."""
    import torch.distributed as dist
    import paper_1705_01598_b200 as tt_
    import tt_workloads as wl_
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    try:
        vol = int(np.prod(gdims))
        words = wl_.random_words(vol, 8, 31)
        slab = vol // 2
        x = torch.from_numpy(words[rank * slab:(rank + 1) * slab].view(np.int64).copy()).cuda()
        y = torch.zeros(slab, dtype=torch.int64, device="cuda")
        plan = tt_.P2PShardedPlan(None, gdims, perm, 8, nranks=2, proc=rank)
        rec = plan.export_record(y)
        recs = [None, None]
        dist.all_gather_object(recs, rec)
        plan.import_records(recs)
        outs = []
        for it in range(3):                       # epochs advance across executes
            y.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            plan.execute(x, y)
            torch.cuda.synchronize()
            dist.barrier()                        # both exit barriers passed
            outs.append(y.cpu().numpy().view(np.uint64).copy())
        t = plan.timings()
        result_q.put((rank, outs, t, plan.describe()["mode"]))
        dist.barrier()
        plan.destroy()
    finally:
        dist.destroy_process_group()


def test_p2p_two_processes_one_gpu_ipc():
    """Two processes on one GPU run the multi-process fused path end to end:
    IPC open of the peer's output slab and signal words, cross-process
    release/acquire barriers, remote stores; the gathered output equals the
    oracle's, on every one of three executes."""
    _dev()
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    gdims, perm = (16, 24, 8, 40), (3, 2, 1, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, gdims, perm, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, outs, t, mode = q.get(timeout=300)
        res[r] = (outs, t, mode)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    words = wl.random_words(int(np.prod(gdims)), 8, 31)
    want = orc.permute(gdims, perm, words)
    for it in range(3):
        got = np.concatenate([res[0][0][it], res[1][0][it]])
        np.testing.assert_array_equal(got, want, err_msg=f"execute {it}")
    for r in range(2):
        assert res[r][2] == "p2p"
        assert all(v >= 0 for v in res[r][1])
