"""TTGT tensor contraction (SURVEY f-4): binding of
tt_contract_*.  D = alpha * L . R + beta * D with labelled modes (dim 0
stride-1); the transposes are libtt plans, the GEMM is cuBLAS.  Argument
marshalling only."""
from __future__ import annotations

import ctypes
import json

from . import lib, _check, _stream_handle, _ptr

_vp, _i64p, _ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)
for _name, _args in {
    "tt_contract_plan": [ctypes.POINTER(_vp), ctypes.c_int, _ip, ctypes.c_int, _i64p, _ip, ctypes.c_int,
                         _i64p, _ip, ctypes.c_size_t, _vp],
    "tt_contract_plan_offline": [ctypes.POINTER(_vp), ctypes.c_int, _ip, ctypes.c_int, _i64p, _ip,
                                 ctypes.c_int, _i64p, _ip, ctypes.c_size_t],
    "tt_contract_execute": [_vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_double],
    "tt_contract_timings": [_vp, ctypes.POINTER(ctypes.c_float)],
    "tt_contract_describe": [_vp, ctypes.c_char_p, ctypes.c_size_t],
    "tt_contract_destroy": [_vp],
}.items():
    getattr(lib, _name).argtypes = _args
    getattr(lib, _name).restype = ctypes.c_int


def _marshal(modes_d, dims_l, modes_l, dims_r, modes_r):
    a32 = lambda v: (ctypes.c_int * max(1, len(v)))(*[int(x) for x in v])  # noqa: E731
    a64 = lambda v: (ctypes.c_int64 * max(1, len(v)))(*[int(x) for x in v])  # noqa: E731
    if len(dims_l) != len(modes_l) or len(dims_r) != len(modes_r):
        raise ValueError("dims and modes differ in length")
    return (len(modes_d), a32(modes_d), len(modes_l), a64(dims_l), a32(modes_l), len(modes_r),
            a64(dims_r), a32(modes_r))


def _describe_c(h) -> dict:
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib.tt_contract_describe(h, buf, len(buf)), "tt_contract_describe")
    return json.loads(buf.value.decode())


class Contraction:
    """plan -> execute -> destroy for D = alpha * L . R + beta * D."""

    def __init__(self, modes_d, dims_l, modes_l, dims_r, modes_r, elem_size: int, stream=None):
        self.elem_size = int(elem_size)
        h = ctypes.c_void_p()
        _check(lib.tt_contract_plan(ctypes.byref(h), *_marshal(modes_d, dims_l, modes_l, dims_r, modes_r),
                                    self.elem_size, _stream_handle(stream)), "tt_contract_plan")
        self._h = h
        d = self.describe()
        self.m, self.n, self.k = d["m"], d["n"], d["k"]
        self.dims_d = tuple(d["dims_d"])

    def execute(self, L, R, D, alpha: float = 1.0, beta: float = 0.0) -> None:
        _check(lib.tt_contract_execute(self._h, _ptr(L), _ptr(R), _ptr(D), float(alpha), float(beta)),
               "tt_contract_execute")

    __call__ = execute

    def timings(self):
        """(transpose L, transpose R, GEMM, transpose D) milliseconds of the last execute."""
        ms = (ctypes.c_float * 4)()
        _check(lib.tt_contract_timings(self._h, ms), "tt_contract_timings")
        return tuple(float(x) for x in ms)

    def describe(self) -> dict:
        return _describe_c(self._h)

    @property
    def flops(self) -> int:
        return 2 * self.m * self.n * self.k

    def destroy(self):
        if self._h is not None:
            _check(lib.tt_contract_destroy(self._h), "tt_contract_destroy")
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def contract_offline(modes_d, dims_l, modes_l, dims_r, modes_r, elem_size: int) -> dict:
    """The contraction's TTGT decomposition without a GPU (JSON description)."""
    h = ctypes.c_void_p()
    _check(lib.tt_contract_plan_offline(ctypes.byref(h), *_marshal(modes_d, dims_l, modes_l, dims_r,
                                                                   modes_r), int(elem_size)),
           "tt_contract_plan_offline")
    try:
        return _describe_c(h)
    finally:
        lib.tt_contract_destroy(h)
