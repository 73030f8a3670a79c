"""GPU parity: libtt.so's CUDA path vs the CPU oracle, element by element,
bit-exact (tolerance 0, also for float payloads: DESIGN.md reading R12).

Every call goes through the C ABI (the ctypes binding).  Inputs are the
seeded words of tt_workloads (shared generator, no permutation arithmetic).
"""
import itertools
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1705_01598_b200 as tt
from oracle import oracle as orc
import tt_workloads as wl

pytestmark = pytest.mark.gpu

_TD = {4: torch.int32, 8: torch.int64}
_ND = {4: np.int32, 8: np.int64}


def _dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests (no CPU fallback)")
    return torch.device("cuda", 0)


def to_dev(words):
    esize = words.dtype.itemsize
    return torch.from_numpy(words.view(_ND[esize]).copy()).to(_dev())


GUARD = 4096  # sentinel words after every output buffer (no compute-sanitizer on this pool)


def run_gpu(dims, perm, words, offset=0, **opts):
    """Permute on the GPU through tt_plan/tt_execute; returns numpy words.
    The output sits between sentinel words (``offset`` before, GUARD after)
    that must survive: a write outside the output fails the test."""
    esize = words.dtype.itemsize
    n = words.size
    src = torch.empty(n + offset, dtype=_TD[esize], device=_dev())
    src[offset:] = to_dev(words)
    dst = torch.full((n + offset + GUARD,), -0x21524111, dtype=_TD[esize], device=_dev())
    plan = tt.Plan(dims, perm, esize, **opts)
    plan.execute(src[offset:], dst[offset:offset + n])
    torch.cuda.synchronize()
    out = dst[offset:offset + n].cpu().numpy().view(words.dtype)
    if offset:
        assert (dst[:offset].cpu().numpy() == -0x21524111).all(), "wrote before the output"
    assert (dst[offset + n:].cpu().numpy() == -0x21524111).all(), "wrote after the output"
    plan.destroy()
    return out


def check(dims, perm, esize, seed=1, **opts):
    words = wl.random_words(int(np.prod(dims)), esize, seed)
    got = run_gpu(dims, perm, words, **opts)
    want = orc.permute_threaded(dims, perm, words)
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{dims} {perm} e{esize} {opts}: {bad.size} mismatches, first at "
                             f"{bad[:8].tolist()}")


def test_s0_config0():
    c = wl.s0()
    check(c.dims, c.perm, c.esize, seed=c.seed)
    # index-encoded input reproduces the hand-worked golden values
    got = run_gpu(c.dims, c.perm, wl.index_words(455, 4))
    assert got[:12].tolist() == [0, 91, 182, 273, 364, 1, 92, 183, 274, 365, 2, 93]


@pytest.mark.parametrize("esize", [4, 8])
def test_exhaustive_tiny(esize):
    """Every permutation of rank <= 4 with extents in {1, 2, 3, 5}."""
    for rank in (1, 2, 3, 4):
        for dims in itertools.product((1, 2, 3, 5), repeat=rank):
            if rank == 4 and dims.count(1) > 1:
                continue
            words = wl.random_words(int(np.prod(dims)), esize, sum(dims))
            for perm in itertools.permutations(range(rank)):
                got = run_gpu(dims, perm, words)
                np.testing.assert_array_equal(got, orc.permute(dims, perm, words),
                                              err_msg=f"{dims} {perm}")


RANDOM_SHAPES = [
    ((67, 45), (1, 0)),
    ((1000, 999), (1, 0)),
    ((4096, 33), (1, 0)),
    ((33, 4096), (1, 0)),
    ((7, 13, 5), (2, 0, 1)),
    ((129, 65, 7), (2, 1, 0)),
    ((300, 5, 3, 17), (0, 3, 2, 1)),        # fastest dim unchanged
    ((2, 300, 3, 17), (0, 3, 2, 1)),        # fastest unchanged, short rows
    ((5, 3, 2, 4, 35, 33, 37, 40), (7, 4, 0, 5, 2, 6, 3, 1)),  # Set-2 shape
    ((2, 3, 4, 3, 2, 2, 3, 2, 20, 18, 22, 24), tuple(range(11, -1, -1))),
    ((11, 4, 3, 5, 3, 2, 6, 8, 7, 10, 3, 3), (0, 7, 8, 1, 3, 9, 2, 4, 5, 10, 11, 6)),
    ((1, 77, 1, 3, 1), (4, 3, 2, 1, 0)),    # extent-1 dims
    ((1025, 3, 2), (2, 1, 0)),              # large first input, small first output (PackedSplit)
    ((3, 2, 1025), (2, 1, 0)),
]


@pytest.mark.parametrize("esize", [4, 8])
@pytest.mark.parametrize("dims,perm", RANDOM_SHAPES)
def test_shapes(dims, perm, esize):
    vol = int(np.prod(dims))
    if vol > 4_000_000:
        # keep the oracle in seconds: scale down, keep perm and raggedness
        c = wl.scaled(wl.Case("x", dims, perm, esize, 3), 2_000_000)
        dims = c.dims
    check(dims, perm, esize)


@pytest.mark.parametrize("esize", [4, 8])
@pytest.mark.parametrize("run", [(2, 2), (8, 3), (32, 32), (64, 16), (16, 256), (256, 256)])
def test_forced_tiles(run, esize):
    """Force tile geometries so splits, ragged chunks and paddings all occur."""
    for dims, perm in [((37, 29, 11), (2, 0, 1)), ((130, 70), (1, 0)), ((9, 8, 7, 6, 5), (3, 4, 0, 2, 1))]:
        check(dims, perm, esize, run_in=run[0], run_out=run[1])


@pytest.mark.parametrize("esize", [4, 8])
def test_forced_tiled2d(esize):
    """The vectorised 2-D kernel on full, ragged and batched tiles."""
    shapes = [((64, 64), (1, 0)), ((132, 36), (1, 0)), ((6, 10, 7), (1, 2, 0)),
              ((34, 3, 98), (2, 1, 0)), ((8, 5, 12, 3), (2, 3, 0, 1)), ((70, 50), (1, 0)),
              ((1000, 998), (1, 0)), ((36, 7, 44, 3), (2, 0, 3, 1)), ((2, 4, 6), (2, 0, 1)),
              # odd extents: scalar 2-D kernel with padded staging
              ((67, 45), (1, 0)), ((13, 3, 67), (2, 1, 0)), ((1001, 999), (1, 0)),
              ((129, 5, 65), (2, 0, 1))]
    tiles = [(64, 64), (128, 64), (64, 128), (128, 128), (32, 64)] if esize == 4 else \
        [(32, 32), (64, 32), (32, 64), (64, 64)]
    for dims, perm in shapes:
        check(dims, perm, esize, kernel=tt.KERNEL_TILED2D)
        for order in (1, 2):
            for ta, tb in tiles:
                try:
                    tt.Plan(dims, perm, esize, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb)
                except tt.TTError:
                    continue  # tile not instantiated for this vector width
                check(dims, perm, esize, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb,
                      grid_order=order)
        # pointers misaligned for the vector width take the generic fallback
        words = wl.random_words(int(np.prod(dims)), esize, 8)
        got = run_gpu(dims, perm, words, offset=1, kernel=tt.KERNEL_TILED2D)
        np.testing.assert_array_equal(got, orc.permute(dims, perm, words))


@pytest.mark.parametrize("esize", [4, 8])
def test_two_element_vector_2d_kernels(esize):
    """The 2-element-vector 2-D kernels (8-byte vectors of fp32, 16-byte of
    fp64), reachable through the option t2d_vec2 = 1 since the scalar kernel
    is the default for most of their shapes."""
    shapes = [((66, 62), (1, 0)), ((130, 6, 34), (2, 1, 0)), ((1002, 998), (1, 0)),
              ((34, 3, 98), (2, 1, 0)), ((586, 6, 42), (1, 0, 2))]
    tiles = [(32, 64), (64, 64)] if esize == 4 else [(32, 32), (64, 32), (32, 64), (64, 64)]
    for dims, perm in shapes:
        assert tt.Plan(dims, perm, esize, kernel=tt.KERNEL_TILED2D, t2d_vec2=1).describe()["vec"] == 2
        check(dims, perm, esize, kernel=tt.KERNEL_TILED2D, t2d_vec2=1)
        for ta, tb in tiles:
            check(dims, perm, esize, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb, t2d_vec2=1)


@pytest.mark.parametrize("esize", [4, 8])
@pytest.mark.parametrize("stages", [3, 4])
def test_scalar_tiled2d_async_ring(esize, stages):
    """Scalar 2-D kernel with the cp.async ring (tiled2d_sa_kernel): odd
    extents, ragged tiles on both sides, batched dims, every instantiated
    tile, and more CTAs than fit (second partial wave)."""
    shapes = [((67, 45), (1, 0)), ((13, 3, 67), (2, 1, 0)), ((1001, 999), (1, 0)),
              ((129, 5, 65), (2, 0, 1)), ((585, 7, 33), (1, 0, 2)), ((119, 5, 3, 119), (3, 2, 1, 0))]
    tiles = [(64, 64), (128, 64), (64, 128)] if esize == 4 else [(64, 64), (32, 64), (64, 32)]
    for dims, perm in shapes:
        for ta, tb in tiles:
            for cps in (2, 6):
                p = tt.Plan(dims, perm, esize, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb,
                            stages=stages, ctas_per_sm=cps)
                d = p.describe()
                assert d["vec"] == 1 and d["stages"] == stages
                check(dims, perm, esize, kernel=tt.KERNEL_TILED2D, run_in=ta, run_out=tb,
                      stages=stages, ctas_per_sm=cps)


ROW_SHAPES = [((600, 7, 5), (0, 2, 1)), ((256, 3, 5, 2), (0, 3, 1, 2)), ((8, 7, 5), (0, 2, 1)),
              ((6, 5, 7), (0, 2, 1)), ((1001, 3, 4), (0, 2, 1)), ((2, 300, 3, 17), (0, 3, 2, 1)),
              ((128, 2, 2, 2, 2, 2), (0, 5, 3, 1, 4, 2)), ((4, 4), (0, 1)),
              # few long rows: segmented into a new fastest row dim
              ((6144, 5, 3), (0, 2, 1)), ((2048 * 9, 3, 7), (0, 2, 1)), ((4099, 3, 2), (0, 2, 1))]


@pytest.mark.parametrize("esize", [4, 8])
def test_rowcopy_and_widening(esize):
    """Fastest dim unchanged: row copy and widened words (auto), forced row
    copy without widening, and unaligned pointers taking the narrow plan."""
    for dims, perm in ROW_SHAPES:
        check(dims, perm, esize)
        try:
            check(dims, perm, esize, kernel=tt.KERNEL_ROWCOPY)
        except tt.TTError:
            assert dims == (4, 4)  # rank 1 after fusion: copy, not row copy
        words = wl.random_words(int(np.prod(dims)), esize, 12)
        for off in (1, 2):
            got = run_gpu(dims, perm, words, offset=off)
            np.testing.assert_array_equal(got, orc.permute(dims, perm, words))


@pytest.mark.parametrize("esize", [4, 8])
def test_async_stages(esize):
    """The cp.async 3-stage tile pipeline (stages=3) on generic, ragged,
    forced-geometry and widened problems."""
    for dims, perm in RANDOM_SHAPES[:11] + [((37, 29, 11), (2, 0, 1)), ((600, 7, 5), (0, 2, 1))]:
        vol = int(np.prod(dims))
        if vol > 2_000_000:
            dims = wl.scaled(wl.Case("x", dims, perm, esize, 3), 1_000_000).dims
        check(dims, perm, esize, stages=3)
        check(dims, perm, esize, stages=3, kernel=tt.KERNEL_TILE, run_in=8, run_out=5)
        check(dims, perm, esize, kernel=tt.KERNEL_TILE, grid_order=2)  # contiguous tile ranges
    for threads in (64, 256):
        check((97, 89, 3), (1, 2, 0), esize, stages=3, kernel=tt.KERNEL_TILE, threads=threads)


@pytest.mark.parametrize("esize", [4, 8])
def test_slot_dim_map(esize):
    """The slot-dim thread map (tile_sd_kernel) forced on, and the classic
    map forced, on generic, ragged (split slot dims) and small-extent
    problems; the describe output says which map ran."""
    shapes = RANDOM_SHAPES[:11] + [((37, 29, 11), (2, 0, 1)), ((5, 3, 2, 4, 35, 33), (5, 4, 3, 2, 1, 0)),
                                   ((41, 41, 41), (0, 2, 1)), ((46, 46, 46, 7), (3, 1, 0, 2)),
                                   ((3, 5, 7, 11, 13, 2), (4, 2, 0, 5, 3, 1))]
    used = 0
    for dims, perm in shapes:
        vol = int(np.prod(dims))
        if vol > 2_000_000:
            dims = wl.scaled(wl.Case("x", dims, perm, esize, 3), 1_000_000).dims
        j = tt.Plan(dims, perm, esize, slot_dims=1, no_widen=True).describe()
        used += "sd" in j.get("tile", {})
        check(dims, perm, esize, slot_dims=1, no_widen=True)
        check(dims, perm, esize, slot_dims=-1, no_widen=True)
    assert used >= 8


@pytest.mark.parametrize("esize", [4, 8])
@pytest.mark.parametrize("stages", [3, 4])
def test_slot_dim_async_ring(esize, stages):
    """The slot-dim map with a cp.async ring (tile_sd_async_kernel): ragged
    split chunks, small extents, more tiles than CTAs (ring wrap-around) and
    fewer tiles than stages."""
    shapes = RANDOM_SHAPES[:11] + [((37, 29, 11), (2, 0, 1)), ((5, 3, 2, 4, 35, 33), (5, 4, 3, 2, 1, 0)),
                                   ((46, 46, 46, 7), (3, 1, 0, 2)), ((3, 5, 7, 11, 13, 2), (4, 2, 0, 5, 3, 1)),
                                   ((5, 5, 5, 5, 5, 5, 5, 5), (0, 6, 3, 7, 1, 4, 2, 5)), ((6, 7), (1, 0))]
    used = 0
    for dims, perm in shapes:
        vol = int(np.prod(dims))
        if vol > 2_000_000:
            dims = wl.scaled(wl.Case("x", dims, perm, esize, 3), 1_000_000).dims
        j = tt.Plan(dims, perm, esize, slot_dims=1, stages=stages, no_widen=True).describe()
        used += "sd" in j.get("tile", {}) and j["stages"] == stages
        check(dims, perm, esize, slot_dims=1, stages=stages, no_widen=True)
    assert used >= 8


VG_SHAPES = RANDOM_SHAPES[:11] + [
    ((37, 29, 11), (2, 0, 1)), ((5, 3, 2, 4, 35, 33), (5, 4, 3, 2, 1, 0)),
    ((46, 46, 46, 7), (3, 1, 0, 2)), ((3, 5, 7, 11, 13, 2), (4, 2, 0, 5, 3, 1)),
    ((5, 5, 5, 5, 5, 5, 5, 5), (0, 6, 3, 7, 1, 4, 2, 5)), ((9, 7, 5, 3, 5, 7, 9), (6, 4, 2, 0, 1, 3, 5)),
    ((1025, 3, 2), (2, 1, 0)), ((3, 6, 6, 6, 6, 6, 6), (0, 5, 2, 3, 6, 1, 4)), ((6, 7), (1, 0))]


@pytest.mark.parametrize("esize", [4, 8])
@pytest.mark.parametrize("stages", [3, 4])
def test_vector_gather(esize, stages):
    """The vector-gather load phase (tile_vg_kernel): runs copied as 16-byte
    chunks of their aligned superset.  Ragged run tails and ragged non-run
    splits, runs shorter than a chunk, forced tiles, pointers at every
    element offset inside a 16-byte chunk (the shift logic, and the chunks
    that cross the start and the end of the input are clipped)."""
    used = 0
    for dims, perm in VG_SHAPES:
        vol = int(np.prod(dims))
        if vol > 2_000_000:
            dims = wl.scaled(wl.Case("x", dims, perm, esize, 3), 1_000_000).dims
        try:
            j = tt.Plan(dims, perm, esize, vector_gather=1, stages=stages, no_widen=True).describe()
        except tt.TTError:
            continue
        if "vg" not in j.get("tile", {}):
            continue
        used += 1
        check(dims, perm, esize, vector_gather=1, stages=stages, no_widen=True)
        words = wl.random_words(int(np.prod(dims)), esize, 17)
        want = orc.permute(dims, perm, words)
        for off in range(1, 16 // esize):
            got = run_gpu(dims, perm, words, offset=off, vector_gather=1, stages=stages, no_widen=True)
            np.testing.assert_array_equal(got, want, err_msg=f"{dims} {perm} offset {off}")
    assert used >= 10
    for run in [(8, 3), (32, 32), (64, 16), (16, 256)]:
        for dims, perm in [((37, 29, 11), (2, 0, 1)), ((9, 8, 7, 6, 5), (3, 4, 0, 2, 1))]:
            check(dims, perm, esize, run_in=run[0], run_out=run[1], vector_gather=1, stages=stages)


@pytest.mark.parametrize("esize", [4, 8])
def test_tma_2d(esize):
    """The TMA-staged 2-D kernel (tiled2d_tma_kernel, option tma=1): full and
    ragged boxes (the hardware zero-fills loads and clips stores at the
    tensor ends), batch dims up to tensor rank 5, permutations where B is not
    dim 1.  Shapes whose strides are not 16-byte multiples are refused."""
    q = 16 // esize
    shapes = [((64, 64), (1, 0)), ((132, 68), (1, 0)), ((4 * q, 1000 * q), (1, 0)),
              ((96, 5, 40), (2, 1, 0)), ((36, 7, 44, 3), (2, 0, 3, 1)), ((8, 5, 12, 3), (2, 3, 0, 1)),
              ((40, 3, 2, 3, 24), (4, 1, 2, 3, 0)), ((2 * q, 3, 6 * q), (2, 0, 1)),
              ((8, 3, 5, 7, 4), (4, 2, 0, 3, 1))]   # tensor rank 5
    for dims, perm in shapes:
        d = tt.Plan(dims, perm, esize, tma=1).describe()
        assert d["kernel"] == "tiled2d" and d["tma"] == 1
        check(dims, perm, esize, tma=1)
    with pytest.raises(tt.TTError):
        tt.Plan((67, 45), (1, 0), esize, tma=1)


@pytest.mark.parametrize("threads", [64, 96, 256, 512])
def test_forced_threads(threads):
    check((97, 89, 3), (1, 2, 0), 4, threads=threads)
    check((97, 89, 3), (1, 2, 0), 8, threads=threads)


def test_copy_kernel_alignment():
    for esize in (4, 8):
        for n in (1, 3, 17, 1000, 4099):
            words = wl.random_words(n, esize, n)
            for off in (0, 1, 2, 3):
                got = run_gpu((n,), (0,), words, offset=off)
                np.testing.assert_array_equal(got, words)
        check((5, 6, 7), (0, 1, 2), esize)


def test_misaligned_pointers():
    for esize in (4, 8):
        for dims, perm in [((67, 45), (1, 0)), ((7, 13, 5), (2, 0, 1)), ((30, 40, 3), (0, 2, 1))]:
            words = wl.random_words(int(np.prod(dims)), esize, 9)
            for off in (1, 3):
                got = run_gpu(dims, perm, words, offset=off)
                np.testing.assert_array_equal(got, orc.permute(dims, perm, words))


@pytest.mark.parametrize("opts", [{}, {"vector_gather": 1}, {"slot_dims": 1}, {"stages": 3}])
def test_vector_2d_fallback_on_misaligned_pointers(opts):
    """A vector 2-D plan whose pointers are not aligned to its vector width
    runs its generic-tile fallback with the fallback's own kernel choice
    (stages, vector gather, slot-dim map), not the 2-D plan's."""
    for esize, dims in [(4, (256, 132)), (4, (260, 128, 3)), (8, (130, 66))]:
        perm = (1, 0) + tuple(range(2, len(dims)))
        j = tt.Plan(dims, perm, esize, **opts).describe()
        if j["kernel"] != "tiled2d" or j["vec"] == 1:
            continue
        words = wl.random_words(int(np.prod(dims)), esize, 10)
        for off in (1, 3):
            got = run_gpu(dims, perm, words, offset=off, **opts)
            np.testing.assert_array_equal(got, orc.permute(dims, perm, words))


@pytest.mark.parametrize("idx", range(0, 57, 4))
def test_ttc_suite_scaled(idx):
    c = wl.s2_ttc()[idx]
    s = wl.scaled(c, 1_500_000)
    check(s.dims, s.perm, s.esize, seed=c.seed)


@pytest.mark.parametrize("rank", range(2, 13))
def test_random_suite_scaled(rank):
    cases = [c for c in wl.s3_random(per_cell=2, ranks=[rank]) if c.tags[0] == "S3"]
    for c in cases[::3]:
        s = wl.scaled(c, 1_000_000)
        check(s.dims, s.perm, s.esize, seed=c.seed)


def test_set2_shapes_scaled():
    for c in [x for x in wl.s3_random(per_cell=0, set2_random=6) if x.tags[0] == "SET2"]:
        s = wl.scaled(c, 2_000_000)
        check(s.dims, s.perm, s.esize, seed=c.seed)


def _host_ram_ok(nbytes: int) -> bool:
    """Room for the input words, the oracle's output and the copied-back
    GPU output (3 x the tensor) plus a margin."""
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        return True
    return avail > 3 * nbytes + (4 << 30)


def _full_check(case, **opts):
    """Full-size run in bench.py's launch configuration (the planner's plan on
    the seeded words), compared with the oracle's output element by element."""
    if not _host_ram_ok(case.nbytes):
        pytest.skip(f"host RAM below 3 x {case.nbytes} bytes for the full comparison")
    words = case.words()
    src = to_dev(words)
    dst = torch.empty_like(src)
    plan = tt.Plan(case.dims, case.perm, case.esize, **opts)
    plan.execute(src, dst)
    torch.cuda.synchronize()
    del src
    got = dst.cpu().numpy().view(words.dtype)
    del dst
    want = orc.permute_threaded(case.dims, case.perm, words)
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{case.name}: {bad.size} of {case.vol} mismatch, first at {bad[:8].tolist()}")
    plan.destroy()
    del got, want, words
    torch.cuda.empty_cache()


def test_full_size_s1():
    _full_check(wl.s1())


def test_full_size_suite_cases():
    """One full-size case per ~19 of S2, the S5 redistribution shape, and a
    spread of S3 ranks/dtypes: every output element against the oracle."""
    for c in wl.s2_ttc()[::19] + [wl.s5_sharded()[4]]:
        _full_check(c)
    s3 = wl.s3_random(per_cell=1)
    for c in s3[::97]:
        _full_check(c)


def test_index64_path():
    """Volume >= 2^31 elements exercises the 64-bit index kernels (8.6 GB per
    tensor); every element is compared."""
    c = wl.Case("big", (65539, 32771), (1, 0), 4, 123)
    assert c.vol >= (1 << 31)
    assert tt.Plan(c.dims, c.perm, 4).describe()["idx64"] is True
    _full_check(c)


def test_stream_and_errors():
    s = torch.cuda.Stream()
    words = wl.random_words(6000, 4, 1)
    src = to_dev(words)
    dst = torch.empty_like(src)
    plan = tt.Plan((60, 100), (1, 0), 4, stream=s)
    with torch.cuda.stream(s):
        plan.execute(src, dst)
    s.synchronize()
    np.testing.assert_array_equal(dst.cpu().numpy().view(np.uint32), orc.permute((60, 100), (1, 0), words))
    with pytest.raises(tt.TTError):
        plan.execute(src, src)
    plan.destroy()
    with pytest.raises(tt.TTError):
        plan.execute(src, dst)


def test_execute_host_roundtrip():
    dims, perm = (300, 200, 3), (2, 0, 1)
    words = wl.random_words(180000, 8, 4)
    hin = torch.from_numpy(words.view(np.int64).copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    din = torch.empty(hin.shape, dtype=torch.int64, device=_dev())
    dout = torch.empty_like(din)
    plan = tt.Plan(dims, perm, 8)
    plan.execute_host(hin, hout, din, dout)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hout.numpy().view(np.uint64), orc.permute(dims, perm, words))


def test_permute_torch_matches_torch_semantics():
    x = torch.arange(2 * 3 * 4 * 5, dtype=torch.float32, device=_dev()).reshape(2, 3, 4, 5)
    for axes in [(3, 2, 1, 0), (0, 2, 1, 3), (1, 3, 0, 2)]:
        y = tt.permute_torch(x, axes)
        assert torch.equal(y, x.permute(*axes).contiguous())


def test_measured_planning():
    """tt_plan_measure: every candidate it may keep is a valid plan; the kept
    one is bit-exact and reports its measurement."""
    for dims, perm, esize in [((130, 70), (1, 0), 4), ((37, 29, 11, 4), (2, 0, 3, 1), 8),
                              ((600, 7, 5), (0, 2, 1), 4), ((5, 3, 2, 4, 7, 6), (4, 0, 5, 2, 3, 1), 4)]:
        words = wl.random_words(int(np.prod(dims)), esize, 2)
        x = to_dev(words)
        y = torch.empty_like(x)
        plan = tt.Plan(dims, perm, esize, measure=(x, y))
        d = plan.describe()
        assert d["measured"]["candidates"] >= 2 and d["measured"]["best_ms"] > 0
        y.fill_(0)
        plan.execute(x, y)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy().view(words.dtype), orc.permute(dims, perm, words))
        plan.destroy()


@pytest.mark.parametrize("dims,perm,esize", [((2048, 1031, 5), (2, 0, 1), 8), ((4100, 4099), (1, 0), 4),
                                             ((7, 300, 9, 1001), (0, 3, 1, 2), 8)])
def test_execute_host_pipelined(dims, perm, esize):
    """tt_execute_host above 64 MB: chunked H2D (2-D copies) / permute / D2H
    on three streams; bit-exact against the oracle."""
    words = wl.random_words(int(np.prod(dims)), esize, 44)
    nd = _ND[esize]
    hin = torch.from_numpy(words.view(nd).copy()).pin_memory()
    hout = torch.zeros_like(hin).pin_memory()
    din = torch.empty(hin.shape, dtype=_TD[esize], device=_dev())
    dout = torch.empty_like(din)
    plan = tt.Plan(dims, perm, esize)
    assert hin.numel() * esize >= (64 << 20)
    for _ in range(2):   # second call reuses the pipeline
        plan.execute_host(hin, hout, din, dout)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(hout.numpy().view(words.dtype), orc.permute_threaded(dims, perm, words))
        hout.zero_()
    plan.destroy()


@pytest.mark.parametrize("esize", [4, 8])
def test_strided_plans(esize):
    """tt_plan_strided on the GPU vs the strided oracle: padded and reordered
    layouts, positions outside the output layout untouched."""
    from test_planner_cpu import strided_layout
    rng = np.random.default_rng(7 + esize)
    for it in range(12):
        rank = int(rng.integers(2, 7))
        dims = tuple(int(x) for x in rng.integers(1, 14 if rank > 3 else 200, size=rank))
        perm = tuple(int(x) for x in rng.permutation(rank))
        sin, nin, sout, nout = strided_layout(rng, dims, perm)
        inbuf = wl.random_words(nin, esize, it)
        outbuf = wl.random_words(nout, esize, 100 + it)
        want = orc.permute_strided(dims, perm, inbuf, sin, outbuf, sout)
        x = to_dev(inbuf)
        y = to_dev(outbuf)
        plan = tt.Plan(dims, perm, esize, in_strides=sin, out_strides=sout)
        plan.execute(x, y)
        torch.cuda.synchronize()
        got = y.cpu().numpy().view(want.dtype)
        np.testing.assert_array_equal(got, want, err_msg=f"{dims} {perm} {sin} {sout}")
        plan.destroy()
    # a 2-D transpose between padded row pitches (vector 2-D kernel)
    dims, perm, sin, sout = (192, 256), (1, 0), (1, 196), (1, 260)
    inbuf = wl.random_words(196 * 256, esize, 3)
    outbuf = wl.random_words(260 * 192, esize, 4)
    plan = tt.Plan(dims, perm, esize, in_strides=sin, out_strides=sout)
    assert plan.describe()["kernel"] == "tiled2d"
    y = to_dev(outbuf)
    plan.execute(to_dev(inbuf), y)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy().view(outbuf.dtype),
                                  orc.permute_strided(dims, perm, inbuf, sin, outbuf, sout))


@pytest.mark.parametrize("case", range(6))
def test_classification_threshold_shapes(case):
    """The shapes on both sides of the measured classification thresholds
    (test_planner_cpu.RULE_SHAPES), bit-exact on the GPU."""
    from test_planner_cpu import RULE_SHAPES
    dims, perm, esize, kernel = RULE_SHAPES[case]
    plan = tt.Plan(dims, perm, esize)
    assert plan.describe()["kernel"] == kernel
    plan.destroy()
    check(dims, perm, esize, seed=case)


def test_widened_8byte_rows_generic_tile():
    """The rule that sends many widened 8-byte rows to the un-widened generic
    tile: the plan it picks, bit-exact (with and without pointer offsets)."""
    dims, perm = (512, 20000, 2), (0, 2, 1)
    assert tt.Plan(dims, perm, 8).describe()["kernel"] == "tile"
    check(dims, perm, 8, seed=12)
    words = wl.random_words(int(np.prod(dims)), 8, 13)
    np.testing.assert_array_equal(run_gpu(dims, perm, words, offset=1), orc.permute_threaded(dims, perm, words))


@pytest.mark.parametrize("dims,perm,esize", [((597, 41, 85), (2, 1, 0), 8), ((45, 45, 45, 45), (0, 3, 2, 1), 8),
                                             ((5, 29, 7, 31, 81), (4, 0, 3, 1, 2), 8),
                                             ((11, 11, 11, 11, 11, 11), (2, 1, 5, 0, 4, 3), 8),
                                             ((2, 37, 13, 11, 11, 15), (0, 3, 2, 1, 4, 5), 4)])
def test_default_cp_async_slot_dim_plans(dims, perm, esize):
    """Planner-chosen plans of 8-byte words that take the slot-dim map with the
    4-stage cp.async ring at one CTA per SM (api.cu create_plan_w), bit-exact;
    at least the fp64 ones take it on the B200."""
    j = tt.Plan(dims, perm, esize).describe()
    if esize == 8:
        assert j["kernel"] == "tile" and j["stages"] == 4 and "sd" in j["tile"]
    check(dims, perm, esize, seed=5)
