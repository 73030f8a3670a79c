"""Seeded synthetic workloads for the tensor-permutation benchmarks.

This module is shared by the oracle side (tests, cpu baseline) and the CUDA
side (bench, parity tests).  It holds NO permutation arithmetic: only seeded
random words, extents and permutations shaped like the paper's benchmark
sets (Section 3, L256-263 Set 1, L289-297 Set 2, L299-309 Set 3,
L283 alignment sweep) and BASELINE.json's configs.  The recipe is restated in
DESIGN.md ("Input recipe").

Conventions: 0-based dims, dims[0] is the stride-1 dimension, output
dimension j is input dimension perm[j] (readings R1, R5, R6).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

SUITE_SEED = 1705
_MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """One step of splitmix64 (a counter-based hash), used to derive case seeds."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def case_seed(index: int, suite_seed: int = SUITE_SEED) -> int:
    return splitmix64(suite_seed ^ int(index))


_CHUNK = 1 << 22  # 64-bit draws per generator stream


def _raw64(count: int, seed: int) -> np.ndarray:
    """``count`` 64-bit draws: stream c of 2^22 draws comes from
    PCG64(seed) jumped c times (stream 0 is PCG64(seed) itself), so the
    streams fill disjoint chunks in parallel host threads (numpy releases
    the GIL while drawing) and the result does not depend on the thread
    count."""
    if count <= _CHUNK:
        return np.random.PCG64(seed).random_raw(count).astype(np.uint64, copy=False)
    import os
    from concurrent.futures import ThreadPoolExecutor
    out = np.empty(count, dtype=np.uint64)
    nch = (count + _CHUNK - 1) // _CHUNK

    def fill(c):
        bg = np.random.PCG64(seed)
        if c:
            bg = bg.jumped(c)
        m = min(_CHUNK, count - c * _CHUNK)
        out[c * _CHUNK:c * _CHUNK + m] = bg.random_raw(m)

    with ThreadPoolExecutor(max(1, min(16, len(os.sched_getaffinity(0))))) as ex:
        list(ex.map(fill, range(nch)))
    return out


def random_words(n: int, esize: int, seed: int) -> np.ndarray:
    """n random 4- or 8-byte words (uint32/uint64) from seeded PCG64 streams.

    Every bit pattern is equally likely, so NaN payloads, infinities,
    subnormals and -0.0 all occur when the words are viewed as floats.
    """
    n = int(n)
    seed = int(seed) & _MASK64
    if esize == 8:
        return _raw64(n, seed)
    if esize == 4:
        return _raw64((n + 1) // 2, seed).view(np.uint32)[:n]
    raise ValueError("esize must be 4 or 8")


def index_words(n: int, esize: int) -> np.ndarray:
    """Debug input A[i] = i (index-encoded)."""
    return np.arange(int(n), dtype=np.uint32 if esize == 4 else np.uint64)


@dataclass(frozen=True)
class Case:
    """One permutation workload: dims (stride-1 first), perm, element size."""

    name: str
    dims: tuple
    perm: tuple
    esize: int
    seed: int = 0
    tags: tuple = field(default_factory=tuple)

    @property
    def rank(self) -> int:
        return len(self.dims)

    @property
    def vol(self) -> int:
        return int(math.prod(self.dims))

    @property
    def nbytes(self) -> int:
        return self.vol * self.esize

    def words(self) -> np.ndarray:
        return random_words(self.vol, self.esize, self.seed)


# ---------------------------------------------------------------------------
# Shape / permutation generators (reading R17, R18).
# ---------------------------------------------------------------------------

def log_uniform_extents(rng: np.random.Generator, rank: int, ratio: float,
                        target_vol: float, tol: float = 0.05) -> tuple:
    """Extents whose largest:smallest ratio is about ``ratio`` and whose
    volume is within ``tol`` of ``target_vol`` where integer rounding allows.

    Draw u_i ~ U[0,1] with one u forced to 0 and one to 1 (the exact ratio),
    extents a * ratio**u_i with a solving prod = target_vol, round, then
    nudge single extents by +-1 until the volume is within tolerance.
    """
    if rank == 1:
        return (int(round(target_vol)),)
    u = rng.random(rank)
    lo, hi = rng.choice(rank, size=2, replace=False)
    u[lo], u[hi] = 0.0, 1.0
    if ratio <= 1:
        u[:] = 0.0
    a = (target_vol / (ratio ** u.sum())) ** (1.0 / rank)
    ext = np.maximum(1, np.rint(a * ratio ** u)).astype(np.int64)
    for _ in range(64 * rank):
        vol = float(np.prod(ext.astype(np.float64)))
        if abs(vol / target_vol - 1.0) <= tol:
            break
        # try every single +-1 nudge, keep the one closest to the target
        best, best_err = None, abs(math.log(vol / target_vol))
        for i in range(rank):
            for dlt in (-1, 1):
                if ext[i] + dlt < 1:
                    continue
                v2 = vol / ext[i] * (ext[i] + dlt)
                err = abs(math.log(v2 / target_vol))
                if err < best_err - 1e-12:
                    best, best_err = (i, dlt), err
        if best is None:
            break
        ext[best[0]] += best[1]
    return tuple(int(x) for x in ext)


def random_nonidentity_perm(rng: np.random.Generator, rank: int,
                            keep_first: bool | None = None) -> tuple:
    """Uniform random non-identity permutation; keep_first=True forces
    perm[0] = 0 (fastest dimension unchanged), False forbids it."""
    if rank < 2:
        raise ValueError("rank >= 2 needed for a non-identity permutation")
    for _ in range(10000):
        p = rng.permutation(rank)
        if (p == np.arange(rank)).all():
            continue
        if keep_first is True and p[0] != 0:
            if rank < 3:
                break
            rest = rng.permutation(np.arange(1, rank))
            if (rest == np.arange(1, rank)).all():
                continue
            p = np.concatenate([[0], rest])
        if keep_first is False and p[0] == 0:
            continue
        return tuple(int(x) for x in p)
    raise ValueError("cannot draw such a permutation")


def nonidentity_perms(rank: int) -> list:
    ident = tuple(range(rank))
    return [p for p in itertools.permutations(range(rank)) if p != ident]


# ---------------------------------------------------------------------------
# Suites (BASELINE.json configs).
# ---------------------------------------------------------------------------

def s0() -> Case:
    """BASELINE.json configs[0]: 7x13x5 fp32, perm (2,0,1)."""
    return Case("S0_7x13x5_p201_f32", (7, 13, 5), (2, 0, 1), 4, case_seed(0), ("S0",))


def s1() -> Case:
    """BASELINE.json configs[1]: 16384x16384 fp32 matrix transpose."""
    return Case("S1_16384x16384_p10_f32", (16384, 16384), (1, 0), 4, case_seed(1), ("S1",))


def s2_ttc() -> list:
    """TTC-style set: 57 fp64 cases, ranks 2-6 = 3/10/12/16/16,
    volumes in [190M, 210M]."""
    rng = np.random.default_rng(case_seed(2))
    cases = []
    idx = 0
    for ratio in (1, 5, 15):
        dims = log_uniform_extents(rng, 2, ratio, 200e6)
        cases.append(Case(f"S2_r2_{idx}", dims, (1, 0), 8, case_seed(1000 + idx), ("S2", "r2")))
        idx += 1
    for p in nonidentity_perms(3):
        for ratio in (1, 15):
            dims = log_uniform_extents(rng, 3, ratio, 200e6)
            cases.append(Case(f"S2_r3_{idx}", dims, p, 8, case_seed(1000 + idx), ("S2", "r3")))
            idx += 1
    for rank, count in ((4, 12), (5, 16), (6, 16)):
        for c in range(count):
            ratio = (1, 5, 15)[c % 3]
            dims = log_uniform_extents(rng, rank, ratio, 200e6)
            keep = True if c % 4 == 0 else None
            p = random_nonidentity_perm(rng, rank, keep_first=keep)
            cases.append(Case(f"S2_r{rank}_{idx}", dims, p, 8, case_seed(1000 + idx),
                              ("S2", f"r{rank}")))
            idx += 1
    assert len(cases) == 57
    return cases


SET2_RANK8 = (5, 3, 2, 4, 35, 33, 37, 40)
SET2_RANK12 = (2, 3, 4, 3, 2, 2, 3, 2, 20, 18, 22, 24)


def s3_random(per_cell: int = 20, ranks=range(2, 13), esizes=(4, 8),
              ratios=(1, 5, 15), set2_random: int = 50) -> list:
    """Random rank 2-12 permutations, fp32 and fp64, volume
    ~ N(200M, 40M) clamped to [120M, 280M]; plus the paper's Set 2 shapes
     with identity, reverse and ``set2_random`` random perms."""
    cases = []
    idx = 0
    for esize in esizes:
        for rank in ranks:
            for ratio in ratios:
                rng = np.random.default_rng(case_seed(3_000_000 + 1000 * rank + 10 * ratio + esize))
                fixed = nonidentity_perms(rank) if rank <= 3 else None
                for c in range(per_cell):
                    vol = float(np.clip(rng.normal(200e6, 40e6), 120e6, 280e6))
                    dims = log_uniform_extents(rng, rank, ratio, vol)
                    if fixed is not None:
                        p = fixed[c % len(fixed)]
                    else:
                        p = random_nonidentity_perm(rng, rank, keep_first=True if c % 5 == 0 else None)
                    cases.append(Case(f"S3_r{rank}_x{ratio}_e{esize}_{c}", dims, p, esize,
                                      case_seed(3_000_000 + idx), ("S3", f"r{rank}", f"e{esize}")))
                    idx += 1
    for dims in (SET2_RANK8, SET2_RANK12):
        rank = len(dims)
        for esize in esizes:
            rng = np.random.default_rng(case_seed(4_000_000 + rank + esize))
            perms = [tuple(range(rank)), tuple(range(rank - 1, -1, -1))]
            perms += [random_nonidentity_perm(rng, rank) for _ in range(set2_random)]
            for c, p in enumerate(perms):
                cases.append(Case(f"SET2_r{rank}_e{esize}_{c}", dims, p, esize,
                                  case_seed(4_000_000 + idx), ("SET2", f"r{rank}", f"e{esize}")))
                idx += 1
    return cases


def s4_alignment() -> list:
    """Square fp32 transposes, side 13952..13968."""
    return [Case(f"S4_{n}", (n, n), (1, 0), 4, case_seed(5_000_000 + n), ("S4",))
            for n in range(13952, 13969)]


S5_DIMS = (112, 112, 112, 104)
S5_LOCAL_PERMS = ((1, 0, 2, 3), (2, 0, 1, 3), (0, 2, 1, 3), (2, 1, 0, 3))
S5_REDIST_PERMS = ((3, 2, 1, 0), (2, 3, 0, 1), (1, 0, 3, 2), (0, 3, 1, 2))


def s5_sharded() -> list:
    """BASELINE.json configs[4]: TAL-SH-shaped fp64 112x112x112x104."""
    cases = []
    for i, p in enumerate(S5_LOCAL_PERMS):
        cases.append(Case(f"S5_local_{i}", S5_DIMS, p, 8, case_seed(6_000_000 + i), ("S5", "local")))
    for i, p in enumerate(S5_REDIST_PERMS):
        cases.append(Case(f"S5_redist_{i}", S5_DIMS, p, 8, case_seed(6_000_100 + i), ("S5", "redist")))
    return cases


def scaled(case: Case, target_vol: int) -> Case:
    """The same permutation on extents scaled down so that the volume is about
    ``target_vol`` (for oracle-sized parity runs).  Extents keep their order
    and shrink by a common factor (never below 1); a ragged tail is kept by
    making scaled extents odd where possible."""
    f = (case.vol / max(1, target_vol)) ** (1.0 / case.rank)
    dims = []
    for d in case.dims:
        s = max(1, int(round(d / f)))
        if s > 2 and s % 2 == 0:
            s += 1
        dims.append(min(s, d))
    return Case(case.name + f"_scaled{target_vol}", tuple(dims), case.perm, case.esize,
                case.seed, case.tags + ("scaled",))
