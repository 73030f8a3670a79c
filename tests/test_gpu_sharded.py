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
    monkeypatch.setenv("TT_SHARD_FORCE_REDIST", "1")
    comm = tt.Comm(tt.unique_id(), 1, 0)
    for perm, esize in [((3, 2, 1, 0), 8), ((2, 3, 0, 1), 4), ((0, 3, 1, 2), 8)]:
        gdims = (16, 24, 8, 40)
        words = wl.random_words(int(np.prod(gdims)), esize, 7)
        x = torch.from_numpy(words.view(_ND[esize]).copy()).to(_dev())
        y = torch.empty_like(x)
        sp = tt.ShardedPlan(comm, gdims, perm, esize)
        d = sp.describe()
        assert d["mode"] == "redistribute" and d["launches"] == 2
        sp.execute(x, y)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy().view(words.dtype), orc.permute(gdims, perm, words))
        pack_ms, a2a_ms, unpack_ms = sp.timings()
        assert pack_ms > 0 and unpack_ms > 0 and a2a_ms >= 0
        sp.destroy()
    comm.destroy()
