"""Sharded (multi-GPU, one box) permutation: binding of tt_comm_* / tt_*_sharded.

One process per GPU.  The NCCL unique id is created by rank 0 through the
library and broadcast with ``torch.distributed`` (plumbing only); the
exchange itself is the library's ncclAlltoAll on the plan's stream
(``ShardedPlan``), or the fused form (``P2PShardedPlan``, SURVEY f-1) whose
permute kernels store straight into the peers' output slabs.
"""
from __future__ import annotations

import ctypes

from . import lib, _check, _arrays, _stream_handle, _describe, _ptr, _options, NCCL_UNIQUE_ID_BYTES

SHARD_RECORD_BYTES = 256


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    _check(lib.tt_comm_unique_id(buf), "tt_comm_unique_id")
    return buf.raw


class Comm:
    """NCCL communicator on the current CUDA device."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        if len(uid) != NCCL_UNIQUE_ID_BYTES:
            raise ValueError("unique id must be 128 bytes")
        self.nranks, self.rank = int(nranks), int(rank)
        h = ctypes.c_void_p()
        _check(lib.tt_comm_init(ctypes.byref(h), ctypes.create_string_buffer(uid, len(uid)),
                                self.nranks, self.rank), "tt_comm_init")
        self._h = h

    @classmethod
    def from_process_group(cls, group=None):
        """Rank 0 makes the id, torch.distributed broadcasts it."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], world, rank)

    def destroy(self):
        if self._h is not None:
            _check(lib.tt_comm_destroy(self._h), "tt_comm_destroy")
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class ShardedPlan:
    """Permutation of a tensor block-sharded along its outermost input dim
    (slab ``rank`` of ``global_dims[-1] / nranks``) into the output
    block-sharded along its outermost output dim."""

    def __init__(self, comm: Comm, global_dims, perm, elem_size: int, stream=None,
                 force_redistribute: bool = False, a2a_chunks: int = 0):
        """``force_redistribute``: the pack / all-to-all / unpack path even
        with one rank (single-GPU tests); ``a2a_chunks``: chunks of the
        overlapped exchange (0 = planner, 1 = serial)."""
        n, d, p = _arrays(global_dims, perm)
        self.comm = comm
        self.global_dims, self.perm, self.elem_size = tuple(global_dims), tuple(perm), int(elem_size)
        h = ctypes.c_void_p()
        o = _options(force_redistribute=force_redistribute, a2a_chunks=a2a_chunks)
        _check(lib.tt_plan_sharded_ex(ctypes.byref(h), comm._h, n, d, p, self.elem_size,
                                      _stream_handle(stream), ctypes.byref(o)), "tt_plan_sharded")
        self._h = h
        a = (ctypes.c_int64 * n)()
        b = (ctypes.c_int64 * n)()
        _check(lib.tt_plan_shard_dims(h, a, b), "tt_plan_shard_dims")
        self.local_in_dims = tuple(a)
        self.local_out_dims = tuple(b)

    def execute(self, in_local, out_local) -> None:
        _check(lib.tt_execute_sharded(self._h, _ptr(in_local), _ptr(out_local)),
               "tt_execute_sharded")

    __call__ = execute

    def describe(self) -> dict:
        return _describe(self._h)

    def timings(self):
        """(pack, all-to-all, unpack) milliseconds of the last execute."""
        ms = (ctypes.c_float * 3)()
        _check(lib.tt_sharded_timings(self._h, ms), "tt_sharded_timings")
        return tuple(float(x) for x in ms)

    @property
    def launches(self) -> int:
        return lib.tt_plan_launches(self._h)

    def destroy(self):
        if self._h is not None:
            _check(lib.tt_destroy(self._h), "tt_destroy")
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class P2PShardedPlan(ShardedPlan):
    """Fused redistribution (tt_plan_sharded_p2p): the permutation kernels
    write every destination sub-box straight into its rank's output slab.

    ``comm`` given: multi-process form -- ``register_output(buf)`` once
    (collective), then ``execute(in_local, buf)`` (collective; device-side
    entry/exit barriers).  ``comm=None``: single-process form for process
    ``proc`` of ``nranks`` -- ``execute_slabs(in_local, [out_0, ...])`` with
    every rank's output slab as a device tensor (no barriers)."""

    def __init__(self, comm, global_dims, perm, elem_size: int, stream=None, nranks=None,
                 proc=None, force_redistribute: bool = False):
        n, d, p = _arrays(global_dims, perm)
        self.comm = comm
        if comm is not None:
            nranks, proc = comm.nranks, comm.rank
        if nranks is None or proc is None:
            raise ValueError("nranks and proc are required without a communicator")
        self.nranks, self.proc = int(nranks), int(proc)
        self.global_dims, self.perm, self.elem_size = tuple(global_dims), tuple(perm), int(elem_size)
        h = ctypes.c_void_p()
        o = _options(force_redistribute=force_redistribute)
        _check(lib.tt_plan_sharded_p2p_ex(ctypes.byref(h), comm._h if comm is not None else None,
                                          self.nranks, self.proc, n, d, p, self.elem_size,
                                          _stream_handle(stream), ctypes.byref(o)), "tt_plan_sharded_p2p")
        self._h = h
        a = (ctypes.c_int64 * n)()
        b = (ctypes.c_int64 * n)()
        _check(lib.tt_plan_shard_dims(h, a, b), "tt_plan_shard_dims")
        self.local_in_dims = tuple(a)
        self.local_out_dims = tuple(b)
        self._registered = None

    def register_output(self, out_local) -> None:
        _check(lib.tt_sharded_register_output(self._h, _ptr(out_local)),
               "tt_sharded_register_output")
        self._registered = out_local   # keep the buffer alive with the plan

    def export_record(self, out_local) -> bytes:
        """This rank's registration record (tt_sharded_export_record)."""
        buf = ctypes.create_string_buffer(SHARD_RECORD_BYTES)
        _check(lib.tt_sharded_export_record(self._h, _ptr(out_local), buf), "tt_sharded_export_record")
        self._registered = out_local
        return buf.raw

    def import_records(self, records) -> None:
        """Every rank's record, rank order (tt_sharded_import_records)."""
        blob = b"".join(records)
        if len(blob) != SHARD_RECORD_BYTES * self.nranks:
            raise ValueError("need one record per rank")
        _check(lib.tt_sharded_import_records(self._h, ctypes.create_string_buffer(blob, len(blob))),
               "tt_sharded_import_records")

    def execute_slabs(self, in_local, out_slabs) -> None:
        if len(out_slabs) != self.nranks:
            raise ValueError(f"need {self.nranks} output slabs")
        arr = (ctypes.c_void_p * self.nranks)(*[_ptr(o) for o in out_slabs])
        _check(lib.tt_execute_sharded_p2p(self._h, _ptr(in_local), arr), "tt_execute_sharded_p2p")


def plan_sharded_p2p_offline(nranks: int, proc: int, global_dims, perm, elem_size: int) -> dict:
    """Fused-redistribution geometry for process ``proc`` of ``nranks``
    without a GPU (JSON description: "fused", "in_step", "out_offset")."""
    n, d, p = _arrays(global_dims, perm)
    h = ctypes.c_void_p()
    _check(lib.tt_plan_sharded_p2p_offline(ctypes.byref(h), int(nranks), int(proc), n, d, p,
                                           int(elem_size)), "tt_plan_sharded_p2p_offline")
    try:
        return _describe(h)
    finally:
        lib.tt_destroy(h)


def plan_sharded_offline(nranks: int, proc: int, global_dims, perm, elem_size: int,
                         a2a_chunks: int = 0) -> dict:
    """Sharded geometry and sub-plans for process ``proc`` of ``nranks``,
    without a communicator or GPU (JSON description); ``a2a_chunks`` as
    for ShardedPlan."""
    n, d, p = _arrays(global_dims, perm)
    h = ctypes.c_void_p()
    o = _options(a2a_chunks=a2a_chunks)
    _check(lib.tt_plan_sharded_offline_ex(ctypes.byref(h), int(nranks), int(proc), n, d, p,
                                          int(elem_size), ctypes.byref(o)), "tt_plan_sharded_offline")
    try:
        return _describe(h)
    finally:
        lib.tt_destroy(h)
