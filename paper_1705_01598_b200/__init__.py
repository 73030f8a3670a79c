"""B200-native tensor permutation (the hot path of arXiv 1705.01598, cuTT).

Thin ctypes binding over ``libtt.so`` (C ABI in ``include/tt.h``).  Argument
marshalling only: every step of the permutation runs in the library's CUDA
kernels.  There is no CPU fallback -- importing this package without a built
``libtt.so`` raises, and executing without a CUDA device raises.

Conventions (readings R1, R5, R6): ``dims[0]`` is the stride-1
dimension, ``perm[j]`` is the input dimension that becomes output dimension
j.  :func:`permute_torch` maps torch's row-major ``permute(axes)`` onto this.
"""
from __future__ import annotations

import ctypes
import json
import os

__all__ = [
    "TTError", "Plan", "plan_offline", "permute_torch", "lib", "library_path",
    "KERNEL_AUTO", "KERNEL_COPY", "KERNEL_TILE", "KERNEL_ROWCOPY", "KERNEL_TILED2D",
    "Comm", "ShardedPlan", "unique_id", "plan_sharded_offline",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "libtt.so")

KERNEL_AUTO, KERNEL_COPY, KERNEL_TILE, KERNEL_ROWCOPY, KERNEL_TILED2D = range(5)
NCCL_UNIQUE_ID_BYTES = 128

_STATUS = {
    0: "TT_SUCCESS", 1: "TT_INVALID_PLAN", 2: "TT_INVALID_PARAMETER", 3: "TT_INVALID_DEVICE",
    4: "TT_UNSUPPORTED", 5: "TT_CUDA_ERROR", 6: "TT_NCCL_ERROR", 7: "TT_INTERNAL_ERROR",
    8: "TT_BUFFER_TOO_SMALL",
}


class TTError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_STATUS.get(status, status)}")


class PlanOptions(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int), ("run_in", ctypes.c_int), ("run_out", ctypes.c_int),
                ("threads", ctypes.c_int), ("ctas_per_sm", ctypes.c_int),
                ("no_fusion", ctypes.c_int), ("grid_order", ctypes.c_int),
                ("no_widen", ctypes.c_int), ("stages", ctypes.c_int),
                ("accumulate", ctypes.c_int), ("slots", ctypes.c_int),
                ("slot_dims", ctypes.c_int), ("sd_vmax", ctypes.c_int),
                ("vector_gather", ctypes.c_int), ("t2d_vec2", ctypes.c_int),
                ("force_redistribute", ctypes.c_int), ("vg_policy", ctypes.c_int),
                ("tma", ctypes.c_int), ("a2a_chunks", ctypes.c_int)]


class DeviceProps(ctypes.Structure):
    _fields_ = [("num_sms", ctypes.c_int), ("max_smem_per_block", ctypes.c_int),
                ("max_smem_per_sm", ctypes.c_int), ("max_threads_per_sm", ctypes.c_int),
                ("regs_per_sm", ctypes.c_int)]


def _load():
    if not os.path.exists(library_path):
        raise ImportError(
            f"{library_path} is missing: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback")
    L = ctypes.CDLL(library_path)
    vp, i64p, ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)
    sig = {
        "tt_plan": [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t, vp],
        "tt_plan_ex": [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t, vp,
                       ctypes.POINTER(PlanOptions)],
        "tt_plan_strided": [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t, i64p, i64p, vp],
        "tt_plan_strided_offline": [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t,
                                    i64p, i64p, ctypes.POINTER(DeviceProps),
                                    ctypes.POINTER(PlanOptions)],
        "tt_plan_offline": [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t,
                            ctypes.POINTER(DeviceProps), ctypes.POINTER(PlanOptions)],
        "tt_plan_measure": [ctypes.POINTER(vp), ctypes.c_int, i64p, ip, ctypes.c_size_t, vp, vp, vp,
                            ctypes.c_int],
        "tt_execute": [vp, vp, vp],
        "tt_execute_scaled": [vp, vp, vp, ctypes.c_double, ctypes.c_double],
        "tt_execute_host": [vp, vp, vp, vp, vp],
        "tt_destroy": [vp],
        "tt_plan_describe": [vp, ctypes.c_char_p, ctypes.c_size_t],
        "tt_comm_unique_id": [vp],
        "tt_comm_init": [ctypes.POINTER(vp), vp, ctypes.c_int, ctypes.c_int],
        "tt_comm_destroy": [vp],
        "tt_plan_sharded": [ctypes.POINTER(vp), vp, ctypes.c_int, i64p, ip, ctypes.c_size_t, vp],
        "tt_plan_sharded_ex": [ctypes.POINTER(vp), vp, ctypes.c_int, i64p, ip, ctypes.c_size_t, vp,
                               ctypes.POINTER(PlanOptions)],
        "tt_plan_sharded_offline": [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    i64p, ip, ctypes.c_size_t],
        "tt_plan_sharded_offline_ex": [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       i64p, ip, ctypes.c_size_t, ctypes.POINTER(PlanOptions)],
        "tt_sharded_timings": [vp, ctypes.POINTER(ctypes.c_float)],
        "tt_execute_sharded": [vp, vp, vp],
        "tt_plan_shard_dims": [vp, i64p, i64p],
        "tt_plan_sharded_p2p": [ctypes.POINTER(vp), vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                i64p, ip, ctypes.c_size_t, vp],
        "tt_plan_sharded_p2p_ex": [ctypes.POINTER(vp), vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   i64p, ip, ctypes.c_size_t, vp, ctypes.POINTER(PlanOptions)],
        "tt_plan_sharded_p2p_offline": [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        i64p, ip, ctypes.c_size_t],
        "tt_sharded_register_output": [vp, vp],
        "tt_sharded_export_record": [vp, vp, vp],
        "tt_sharded_import_records": [vp, vp],
        "tt_execute_sharded_p2p": [vp, vp, ctypes.POINTER(vp)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.tt_plan_launches.argtypes = [vp]
    L.tt_plan_launches.restype = ctypes.c_int
    L.tt_status_string.argtypes = [ctypes.c_int]
    L.tt_status_string.restype = ctypes.c_char_p
    L.tt_version.argtypes = []
    L.tt_version.restype = ctypes.c_int
    L.tt_set_log_level.argtypes = [ctypes.c_int]
    L.tt_set_log_level.restype = ctypes.c_int
    if os.environ.get("TT_LOG"):
        L.tt_set_log_level(int(os.environ["TT_LOG"]))
    return L


lib = _load()


def _check(status: int, where: str) -> None:
    if status != 0:
        raise TTError(status, where)


def _arrays(dims, perm):
    dims = [int(x) for x in dims]
    perm = [int(x) for x in perm]
    if len(dims) != len(perm):
        raise ValueError("dims and perm must have the same length")
    return len(dims), (ctypes.c_int64 * len(dims))(*dims), (ctypes.c_int * len(perm))(*perm)


def _options(kernel=0, run_in=0, run_out=0, threads=0, ctas_per_sm=0, no_fusion=False,
             grid_order=0, no_widen=False, stages=0, accumulate=False, slots=0, slot_dims=0,
             sd_vmax=0, vector_gather=0, t2d_vec2=0, force_redistribute=False,
             vg_policy=0, tma=0, a2a_chunks=0):
    return PlanOptions(int(kernel), int(run_in), int(run_out), int(threads), int(ctas_per_sm),
                       1 if no_fusion else 0, int(grid_order), 1 if no_widen else 0, int(stages),
                       1 if accumulate else 0, int(slots), int(slot_dims), int(sd_vmax),
                       int(vector_gather), int(t2d_vec2), 1 if force_redistribute else 0, int(vg_policy),
                       int(tma), int(a2a_chunks))


def _ptr(x) -> int:
    """Device pointer of a torch tensor, or an int address."""
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _stream_handle(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """plan -> execute -> destroy.  ``dims`` stride-1 first,
    ``perm[j]`` = input dim of output dim j, ``elem_size`` 4 or 8."""

    def __init__(self, dims, perm, elem_size: int, stream=None, measure=None,
                 max_candidates: int = 0, in_strides=None, out_strides=None, **opts):
        """``measure=(inp, out)``: measurement-based selection on those device
        buffers (tt_plan_measure) instead of the heuristic.  ``in_strides``
        (per input dim) / ``out_strides`` (per output dim), in elements:
        a strided plan (tt_plan_strided)."""
        n, d, p = _arrays(dims, perm)
        self.dims, self.perm, self.elem_size = tuple(dims), tuple(perm), int(elem_size)
        self.vol = 1
        for x in self.dims:
            self.vol *= int(x)
        h = ctypes.c_void_p()
        if in_strides is not None or out_strides is not None:
            if measure is not None or opts:
                raise ValueError("strided plans take no measurement or planner overrides")
            _check(lib.tt_plan_strided(ctypes.byref(h), n, d, p, self.elem_size,
                                       _strides(in_strides, n), _strides(out_strides, n),
                                       _stream_handle(stream)), "tt_plan_strided")
        elif measure is not None:
            if opts:
                raise ValueError("measured planning takes no planner overrides")
            _check(lib.tt_plan_measure(ctypes.byref(h), n, d, p, self.elem_size,
                                       _stream_handle(stream), _ptr(measure[0]), _ptr(measure[1]),
                                       int(max_candidates)), "tt_plan_measure")
        else:
            o = _options(**opts)
            _check(lib.tt_plan_ex(ctypes.byref(h), n, d, p, self.elem_size,
                                  _stream_handle(stream), ctypes.byref(o)), "tt_plan")
        self._h = h

    @property
    def out_dims(self):
        return tuple(self.dims[j] for j in self.perm)

    @property
    def nbytes(self) -> int:
        return self.vol * self.elem_size

    def execute(self, inp, out) -> None:
        """Enqueue out = permute(inp) on the plan's stream (device buffers)."""
        if self._h is None:
            raise TTError(1, "tt_execute")
        _check(lib.tt_execute(self._h, _ptr(inp), _ptr(out)), "tt_execute")

    __call__ = execute

    def execute_scaled(self, inp, out, alpha: float, beta: float) -> None:
        """out = alpha * permute(inp) + beta * out (plan made with accumulate=True)."""
        _check(lib.tt_execute_scaled(self._h, _ptr(inp), _ptr(out), float(alpha), float(beta)),
               "tt_execute_scaled")

    def execute_host(self, host_in, host_out, dev_in, dev_out) -> None:
        """Enqueue H2D(host_in -> dev_in), permute, D2H(dev_out -> host_out)."""
        _check(lib.tt_execute_host(self._h, _ptr(host_in), _ptr(host_out), _ptr(dev_in),
                                   _ptr(dev_out)), "tt_execute_host")

    def describe(self) -> dict:
        return _describe(self._h)

    @property
    def launches(self) -> int:
        return lib.tt_plan_launches(self._h)

    def destroy(self) -> None:
        if self._h is not None:
            _check(lib.tt_destroy(self._h), "tt_destroy")
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def _describe(h) -> dict:
    size = 1 << 14
    while True:
        buf = ctypes.create_string_buffer(size)
        st = lib.tt_plan_describe(h, buf, size)
        if st == 8:
            size *= 4
            continue
        _check(st, "tt_plan_describe")
        return json.loads(buf.value.decode())


def _strides(st, n):
    if st is None:
        return None
    if len(st) != n:
        raise ValueError("one stride per dimension")
    return (ctypes.c_int64 * n)(*[int(x) for x in st])


def plan_offline(dims, perm, elem_size: int, num_sms: int = 148, in_strides=None,
                 out_strides=None, **opts) -> dict:
    """Plan for a described B200 without touching CUDA; returns the JSON plan."""
    n, d, p = _arrays(dims, perm)
    h = ctypes.c_void_p()
    props = DeviceProps(int(num_sms), 0, 0, 0, 0)
    o = _options(**opts)
    if in_strides is not None or out_strides is not None:
        _check(lib.tt_plan_strided_offline(ctypes.byref(h), n, d, p, int(elem_size),
                                           _strides(in_strides, n), _strides(out_strides, n),
                                           ctypes.byref(props), ctypes.byref(o)),
               "tt_plan_strided_offline")
    else:
        _check(lib.tt_plan_offline(ctypes.byref(h), n, d, p, int(elem_size), ctypes.byref(props),
                                   ctypes.byref(o)), "tt_plan_offline")
    try:
        return _describe(h)
    finally:
        lib.tt_destroy(h)


def torch_axes_to_perm(axes) -> tuple:
    """torch row-major ``x.permute(axes)`` == this library's perm on the reversed shape."""
    n = len(axes)
    return tuple(n - 1 - int(axes[n - 1 - j]) for j in range(n))


def permute_torch(x, axes, out=None, stream=None, **opts):
    """``x.permute(axes).contiguous()`` computed by the library's kernels.

    ``x`` must be a contiguous CUDA tensor with a 4- or 8-byte dtype.
    """
    import torch
    if not x.is_cuda or not x.is_contiguous():
        raise ValueError("x must be a contiguous CUDA tensor")
    if x.element_size() not in (4, 8):
        raise ValueError("element size must be 4 or 8 bytes")
    dims = tuple(reversed(x.shape))
    perm = torch_axes_to_perm(axes)
    shape_out = tuple(x.shape[a] for a in axes)
    if out is None:
        out = torch.empty(shape_out, dtype=x.dtype, device=x.device)
    plan = Plan(dims if dims else (1,), perm if perm else (0,), x.element_size(), stream=stream,
                **opts)
    plan.execute(x, out)
    plan.destroy()
    return out


from ._dist import (Comm, ShardedPlan, P2PShardedPlan, unique_id, plan_sharded_offline,  # noqa: E402
                    plan_sharded_p2p_offline)
from ._contract import Contraction, contract_offline  # noqa: E402
