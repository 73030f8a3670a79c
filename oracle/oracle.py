"""CPU oracle for the tensor permutation of arXiv 1705.01598 (cuTT).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this module.  It never imports the product package
(``paper_1705_01598_b200``) and the product never imports it.

Three formulations of the same definition (Section 2):

* ``permute`` / ``permute_range``: the C gather odometer in ``tt_oracle.c``
  (walks the output linearly, P:L52 decode + incremental strides).
* ``permute_threaded``: the same C routine on disjoint output ranges, one
  range per host thread (verification speed only; bit-identical by
  construction, pinned by a test).
* ``permute_scatter_py``: pure-Python *scattered* transpose: read the
  input linearly and write each element to the output position given by
  Eq. (1) with the corrected output stride c(i, O) of DESIGN.md
  reading R2.  Small cases only.

Conventions (readings R1, R5, R6): 0-based dimensions, dims[0] is
the stride-1 dimension, output dimension j is input dimension perm[j].
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tt_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile tt_oracle.c with gcc (plain -O2, no vectorisation tricks)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-shared", "-fPIC", "-Wall", "-Wextra",
             "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i64p = ctypes.POINTER(ctypes.c_int64)
            i32p = ctypes.POINTER(ctypes.c_int)
            lib.oracle_permute.argtypes = [ctypes.c_int, i64p, i32p, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p]
            lib.oracle_permute.restype = ctypes.c_int
            lib.oracle_permute_range.argtypes = [ctypes.c_int, i64p, i32p, ctypes.c_int,
                                                 ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_int64, ctypes.c_int64]
            lib.oracle_permute_range.restype = ctypes.c_int
            lib.oracle_permute_sample.argtypes = [ctypes.c_int, i64p, i32p, ctypes.c_int,
                                                  ctypes.c_void_p, i64p, ctypes.c_int64,
                                                  ctypes.c_void_p]
            lib.oracle_permute_sample.restype = ctypes.c_int
            lib.oracle_permute_scaled.argtypes = [ctypes.c_int, i64p, i32p, ctypes.c_int,
                                                  ctypes.c_void_p, ctypes.c_void_p,
                                                  ctypes.c_double, ctypes.c_double]
            lib.oracle_permute_scaled.restype = ctypes.c_int
            dp = ctypes.POINTER(ctypes.c_double)
            lib.oracle_contract.argtypes = [ctypes.c_int, i32p, ctypes.c_int, i64p, i32p, ctypes.c_int,
                                            i64p, i32p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                            dp, dp, ctypes.c_double, ctypes.c_double]
            lib.oracle_contract.restype = ctypes.c_int
            _lib = lib
    return _lib


_WORD = {4: np.uint32, 8: np.uint64}


def _args(dims, perm, words):
    dims = [int(x) for x in dims]
    perm = [int(x) for x in perm]
    if len(dims) != len(perm):
        raise ValueError("dims and perm differ in length")
    words = np.ascontiguousarray(words)
    esize = words.dtype.itemsize
    if esize not in (4, 8):
        raise ValueError("element size must be 4 or 8 bytes")
    vol = int(np.prod(dims, dtype=np.int64)) if dims else 0
    if words.size != vol:
        raise ValueError(f"input has {words.size} elements, dims give {vol}")
    d = (ctypes.c_int64 * len(dims))(*dims)
    p = (ctypes.c_int * len(perm))(*perm)
    return dims, perm, words.view(_WORD[esize]), esize, vol, d, p


def permute_range(dims, perm, words, out, begin: int, end: int) -> None:
    """Fill out[begin:end] (flat, output order) from the flat input ``words``."""
    dims, perm, words, esize, vol, d, p = _args(dims, perm, words)
    rc = _load().oracle_permute_range(len(dims), d, p, esize, words.ctypes.data,
                                      out.ctypes.data, int(begin), int(end))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")


def permute(dims, perm, words) -> np.ndarray:
    """Output tensor (flat, column-major in output order) of the permutation."""
    dims, perm, words, esize, vol, d, p = _args(dims, perm, words)
    out = np.empty(vol, dtype=words.dtype)
    rc = _load().oracle_permute(len(dims), d, p, esize, words.ctypes.data, out.ctypes.data)
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return out


def permute_threaded(dims, perm, words, threads: int | None = None) -> np.ndarray:
    """``permute`` split over disjoint output ranges on ``threads`` host threads.

    ctypes releases the GIL during the C call, so the ranges run in parallel.
    """
    dims, perm, words, esize, vol, d, p = _args(dims, perm, words)
    out = np.empty(vol, dtype=words.dtype)
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    threads = max(1, min(int(threads), max(1, vol // 4096)))
    lib = _load()
    bounds = [vol * t // threads for t in range(threads + 1)]
    errs = []

    def run(t):
        rc = lib.oracle_permute_range(len(dims), d, p, esize, words.ctypes.data,
                                      out.ctypes.data, bounds[t], bounds[t + 1])
        if rc != 0:
            errs.append(rc)

    ts = [threading.Thread(target=run, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise ValueError("oracle rejected the arguments")
    return out


def permute_sample(dims, perm, words, positions) -> np.ndarray:
    """out[positions] computed one position at a time (P:L52 division decode)."""
    dims, perm, words, esize, vol, d, p = _args(dims, perm, words)
    pos = np.ascontiguousarray(positions, dtype=np.int64)
    vals = np.empty(pos.size, dtype=words.dtype)
    rc = _load().oracle_permute_sample(
        len(dims), d, p, esize, words.ctypes.data,
        pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pos.size, vals.ctypes.data)
    if rc != 0:
        raise ValueError("oracle rejected the arguments or a position")
    return vals


def permute_scaled(dims, perm, words, out_words, alpha: float, beta: float) -> np.ndarray:
    """out = alpha * permute(words) + beta * out_words (float for 4-byte words,
    double for 8-byte; separate RN multiplies and add; beta == 0 ignores
    out_words).  Returns the new output words."""
    dims, perm, words, esize, vol, d, p = _args(dims, perm, words)
    out = np.array(out_words, dtype=words.dtype, copy=True)
    if out.size != vol:
        raise ValueError("output size mismatch")
    rc = _load().oracle_permute_scaled(len(dims), d, p, esize, words.ctypes.data, out.ctypes.data,
                                       float(alpha), float(beta))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return out


def permute_strided(dims, perm, in_buf, in_strides, out_buf, out_strides) -> np.ndarray:
    """Strided form of the permutation (the layouts of tt_plan_strided):
    out[sum_j x[perm[j]] * out_strides[j]] = in[sum_i x[i] * in_strides[i]]
    for every coordinate x (P:L48 scalar positions with caller strides).
    Returns a copy of ``out_buf`` with those positions written; the rest is
    left as given.  The definition written out over all coordinates at once
    (numpy index arithmetic), small and medium sizes."""
    dims = [int(x) for x in dims]
    perm = [int(x) for x in perm]
    n = len(dims)
    x = np.indices(dims, dtype=np.int64).reshape(n, -1)      # x[i] for every element
    src = sum(x[i] * int(in_strides[i]) for i in range(n))
    dst = sum(x[perm[j]] * int(out_strides[j]) for j in range(n))
    if np.unique(dst).size != dst.size:
        raise ValueError("output strides map two elements to one position")
    out = np.array(out_buf, copy=True)
    out[dst] = np.asarray(in_buf)[src]
    return out


# ---------------------------------------------------------------------------
# Pure-Python scattered transpose via Eq. (1), small cases.
# ---------------------------------------------------------------------------

def cumulative_volume(z: int, order, dims) -> int:
    """c(z, {w_j}) of P:L36: 1 if z is first in ``order``, else the product of
    the extents of the dimensions preceding z in ``order``."""
    i = list(order).index(z)
    c = 1
    for w in list(order)[:i]:
        c *= dims[w]
    return c


def scalar_position(x, order, dims) -> int:
    """p({x_j}, {w_j}) = sum_i x_i c(w_i, {w_j}); x listed in ``order``."""
    return sum(xi * cumulative_volume(w, order, dims) for xi, w in zip(x, order))


def transpose_position(p_in: int, dims, perm) -> int:
    """Eq. (1) with the output stride of dimension i read as c(i, O)
    (reading R2): the output position of the element stored at input
    position p_in.  O is the output ordering; dimension i sits at output
    position perm.index(i), so its output stride is the product of the output
    extents before it."""
    n = len(dims)
    ident = list(range(n))
    out_order = list(perm)
    pos = 0
    for i in range(n):
        xi = (p_in // cumulative_volume(i, ident, dims)) % dims[i]   # P:L56 first factor
        pos += xi * cumulative_volume(i, out_order, dims)            # c(i, O)
    return pos


def permute_scatter_py(dims, perm, words) -> np.ndarray:
    """Scattered transpose: read the input linearly, write output
    position transpose_position(p_in)."""
    words = np.asarray(words)
    vol = 1
    for x in dims:
        vol *= int(x)
    out = np.zeros(vol, dtype=words.dtype)
    written = np.zeros(vol, dtype=bool)
    for p_in in range(vol):
        q = transpose_position(p_in, dims, perm)
        if written[q]:
            raise AssertionError("Eq. (1) map is not a bijection")
        written[q] = True
        out[q] = words[p_in]
    return out


def contract(modes_d, dims_l, modes_l, dims_r, modes_r, L, R, D0=None, alpha=1.0, beta=0.0):
    """D = alpha * sum_contracted L * R + beta * D0, in float64, by
    the plain double odometer of tt_oracle.c.  L, R: flat float32/float64
    arrays in column-major order (dim 0 stride-1); D0: flat array or None.
    Returns a flat float64 array in D's column-major order."""
    L = np.ascontiguousarray(L)
    R = np.ascontiguousarray(R)
    if L.dtype != R.dtype or L.dtype not in (np.float32, np.float64):
        raise ValueError("L and R must both be float32 or float64")
    esize = L.dtype.itemsize
    md = [int(x) for x in modes_d]
    ml, mr = [int(x) for x in modes_l], [int(x) for x in modes_r]
    dl, dr = [int(x) for x in dims_l], [int(x) for x in dims_r]
    if L.size != int(np.prod(dl, dtype=np.int64)) or R.size != int(np.prod(dr, dtype=np.int64)):
        raise ValueError("operand sizes do not match their dims")
    ext = {}
    for m, d in list(zip(ml, dl)) + list(zip(mr, dr)):
        ext[m] = d
    vol_d = int(np.prod([ext.get(m, 1) for m in md], dtype=np.int64))
    out = np.empty(vol_d, dtype=np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    d0 = None
    if D0 is not None:
        d0 = np.ascontiguousarray(D0, dtype=np.float64)
        if d0.size != vol_d:
            raise ValueError("D0 size")
    a32 = lambda v: (ctypes.c_int * max(1, len(v)))(*v)  # noqa: E731
    a64 = lambda v: (ctypes.c_int64 * max(1, len(v)))(*v)  # noqa: E731
    rc = _load().oracle_contract(
        len(md), a32(md), len(ml), a64(dl), a32(ml), len(mr), a64(dr), a32(mr), esize,
        L.ctypes.data, R.ctypes.data, d0.ctypes.data_as(dp) if d0 is not None else None,
        out.ctypes.data_as(dp), float(alpha), float(beta))
    if rc != 0:
        raise ValueError("oracle rejected the contraction")
    return out
