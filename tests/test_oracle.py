"""Pins for the CPU oracle (oracle/) against things other than itself.

Each pin is chosen so that a plausible mistake in the oracle fails it:
* hand-worked golden values (tests/golden/) -- a wrong stride (the printed
  c(w_i,O) of Eq. (1)), the scatter-vs-gather convention, or a swapped
  operand all change B[1] or the output extents;
* closed forms (matrix transpose B[j + i*d1] = A[i + j*d0]);
* a library routine (numpy.transpose) on random shapes;
* an independent pure-Python scatter of Eq. (1);
* invariants: identity, inverse round trip, composition, multiset, sum;
* brute force over every permutation of small ranks with extents in {1,2,3}.
"""
import itertools
import os

import numpy as np
import pytest

from oracle import oracle as orc
import tt_workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def np_ref(dims, perm, words):
    """numpy.transpose of the same column-major data (library routine)."""
    n = len(dims)
    axes = [n - 1 - perm[n - 1 - r] for r in range(n)]
    a = np.asarray(words).reshape(tuple(reversed(dims)))
    return np.ascontiguousarray(a.transpose(axes)).ravel()


def _golden(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split(": ", 1)
            out.setdefault(k.strip(), []).append(v.strip())
    return out


# ---------------------------------------------------------------------------
# hand-worked values
# ---------------------------------------------------------------------------

def test_s0_golden_values():
    g = _golden("s0_7x13x5_p201.txt")
    dims = tuple(int(x) for x in g["dims"][0].split())
    perm = tuple(int(x) for x in g["perm"][0].split())
    assert (dims, perm) == (wl.s0().dims, wl.s0().perm)
    a = wl.index_words(455, 4)
    b = orc.permute(dims, perm, a)
    assert b.tolist()[0:12] == [int(x) for x in g["B[0:12]"][0].split()]
    assert b.tolist()[448:455] == [int(x) for x in g["B[448:455]"][0].split()]
    for pair in g["in_to_out"][0].split():
        i, o = (int(x) for x in pair.split("->"))
        assert int(b[o]) == i
        assert orc.transpose_position(i, dims, perm) == o
    assert int(b.astype(np.int64).sum()) == int(g["sum"][0])
    ext = [int(x) for x in g["out_extents"][0].split()]
    assert ext == [dims[p] for p in perm]


def test_s0_closed_form_all_positions():
    # out = x2 + 5*x0 + 35*x1 for input x0 + 7*x1 + 91*x2 (derived by hand, golden header)
    a = wl.index_words(455, 4)
    b = orc.permute((7, 13, 5), (2, 0, 1), a)
    for x0 in range(7):
        for x1 in range(13):
            for x2 in range(5):
                assert b[x2 + 5 * x0 + 35 * x1] == x0 + 7 * x1 + 91 * x2


def test_spec_examples():
    g = _golden("spec_examples.txt")
    for line in g["cumvol"]:
        d, o, rest = (s.strip() for s in line.split("|"))
        z, want = (int(s) for s in rest.split("->"))
        assert orc.cumulative_volume(z, [int(x) for x in o.split(",")],
                                     [int(x) for x in d.split(",")]) == want
    for line in g["scalarpos"]:
        d, o, rest = (s.strip() for s in line.split("|"))
        x, want = rest.split("->")
        assert orc.scalar_position([int(v) for v in x.split(",")], [int(v) for v in o.split(",")],
                                   [int(v) for v in d.split(",")]) == int(want)
    for line in g["transpos"]:
        d, p, rest = (s.strip() for s in line.split("|"))
        pin, want = (int(s) for s in rest.split("->"))
        assert orc.transpose_position(pin, [int(v) for v in d.split(",")],
                                      [int(v) for v in p.split(",")]) == want
    for line in g["rank2"]:
        d, p, rest = (s.strip() for s in line.split("|"))
        dims = [int(v) for v in d.split(",")]
        perm = [int(v) for v in p.split(",")]
        want = [int(v) for v in rest.split()]
        assert orc.permute(dims, perm, wl.index_words(6, 8)).tolist() == want


def test_matrix_transpose_closed_form():
    d0, d1 = 67, 45
    a = wl.random_words(d0 * d1, 4, 7)
    b = orc.permute((d0, d1), (1, 0), a)
    for i in range(d0):
        for j in range(0, d1, 7):
            assert b[j + i * d1] == a[i + j * d0]


# ---------------------------------------------------------------------------
# library routine, independent formulation, brute force
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("esize", [4, 8])
def test_numpy_random_shapes(esize):
    rng = np.random.default_rng(11)
    for _ in range(120):
        rank = int(rng.integers(1, 8))
        dims = tuple(int(x) for x in rng.integers(1, 9, size=rank))
        perm = tuple(int(x) for x in rng.permutation(rank))
        a = wl.random_words(int(np.prod(dims)), esize, int(rng.integers(1 << 30)))
        np.testing.assert_array_equal(orc.permute(dims, perm, a), np_ref(dims, perm, a))


def test_brute_force_small_ranks():
    """Every permutation of rank <= 4 over extents in {1,2,3} (and a rank-5
    sample): C gather odometer == Python Eq.(1) scatter == numpy."""
    count = 0
    for rank in (1, 2, 3, 4):
        for dims in itertools.product((1, 2, 3), repeat=rank):
            a = wl.index_words(int(np.prod(dims)), 4)
            for perm in itertools.permutations(range(rank)):
                b = orc.permute(dims, perm, a)
                np.testing.assert_array_equal(b, np_ref(dims, perm, a))
                if rank <= 3 or dims.count(1) <= 1:
                    np.testing.assert_array_equal(b, orc.permute_scatter_py(dims, perm, a))
                count += 1
    rng = np.random.default_rng(5)
    for _ in range(60):
        dims = tuple(int(x) for x in rng.integers(1, 4, size=5))
        perm = tuple(int(x) for x in rng.permutation(5))
        a = wl.index_words(int(np.prod(dims)), 8)
        b = orc.permute(dims, perm, a)
        np.testing.assert_array_equal(b, orc.permute_scatter_py(dims, perm, a))
        np.testing.assert_array_equal(b, np_ref(dims, perm, a))
        count += 1
    assert count == 3 + 9 * 2 + 27 * 6 + 81 * 24 + 60


def test_printed_eq1_stride_is_not_a_bijection():
    """DESIGN.md reading R2: Eq.(1) as printed uses c(w_i,O); on the S0 shape
    that map is not a bijection, so the oracle must not use it."""
    dims, perm = (7, 13, 5), (2, 0, 1)

    def printed(p_in):
        pos = 0
        for i in range(3):
            xi = (p_in // orc.cumulative_volume(i, [0, 1, 2], dims)) % dims[i]
            pos += xi * orc.cumulative_volume(perm[i], perm, dims)
        return pos

    assert len({printed(p) for p in range(455)}) < 455
    assert len({orc.transpose_position(p, dims, perm) for p in range(455)}) == 455


# ---------------------------------------------------------------------------
# invariants
# ---------------------------------------------------------------------------

def _inverse(p):
    inv = [0] * len(p)
    for j, pj in enumerate(p):
        inv[pj] = j
    return tuple(inv)


@pytest.mark.parametrize("esize", [4, 8])
def test_invariants(esize):
    rng = np.random.default_rng(3 + esize)
    for _ in range(60):
        rank = int(rng.integers(2, 9))
        dims = tuple(int(x) for x in rng.integers(1, 6, size=rank))
        p = tuple(int(x) for x in rng.permutation(rank))
        q = tuple(int(x) for x in rng.permutation(rank))
        a = wl.random_words(int(np.prod(dims)), esize, int(rng.integers(1 << 30)))
        b = orc.permute(dims, p, a)
        # identity is a bit-identical copy
        np.testing.assert_array_equal(orc.permute(dims, tuple(range(rank)), a), a)
        # inverse round trip: output dims are e[j] = d[p[j]]
        e = tuple(dims[x] for x in p)
        np.testing.assert_array_equal(orc.permute(e, _inverse(p), b), a)
        # composition: T(T(A,p),q) = T(A,r), r[j] = p[q[j]]
        r = tuple(p[q[j]] for j in range(rank))
        np.testing.assert_array_equal(orc.permute(e, q, b), orc.permute(dims, r, a))
        # multiset and wrapping integer sum of bit patterns preserved
        np.testing.assert_array_equal(np.sort(b), np.sort(a))
        assert int(b.sum(dtype=np.uint64)) == int(a.sum(dtype=np.uint64))


def test_fusion_invariance():
    """Adjacent input dims that stay adjacent and in order in the output may be
    merged (BASELINE.json north_star 'fuses contiguous index runs')."""
    dims = (3, 4, 5, 6)
    perm = (2, 3, 0, 1)            # (2,3) and (0,1) are in-order runs
    a = wl.random_words(360, 4, 9)
    np.testing.assert_array_equal(orc.permute(dims, perm, a), orc.permute((12, 30), (1, 0), a))


# ---------------------------------------------------------------------------
# drivers
# ---------------------------------------------------------------------------

def test_threaded_and_sampled_match():
    dims, perm = (33, 17, 9, 5), (3, 1, 0, 2)
    a = wl.random_words(int(np.prod(dims)), 8, 21)
    b = orc.permute(dims, perm, a)
    for t in (1, 2, 3, 8):
        np.testing.assert_array_equal(orc.permute_threaded(dims, perm, a, threads=t), b)
    pos = np.random.default_rng(0).integers(0, b.size, size=500)
    np.testing.assert_array_equal(orc.permute_sample(dims, perm, a, pos), b[pos])
    out = np.zeros_like(b)
    orc.permute_range(dims, perm, a, out, 100, 2000)
    np.testing.assert_array_equal(out[100:2000], b[100:2000])


def test_rejects_bad_arguments():
    a = wl.index_words(6, 4)
    with pytest.raises(ValueError):
        orc.permute((2, 3), (0, 0), a)
    with pytest.raises(ValueError):
        orc.permute((2, 3), (0, 2), a)
    with pytest.raises(ValueError):
        orc.permute((2, 0), (1, 0), np.zeros(0, np.uint32))
    with pytest.raises(ValueError):
        orc.permute((2, 3), (1, 0), np.zeros(6, np.uint16))


def test_float_bits_preserved():
    vals = np.array([np.nan, -0.0, 1e-45, np.inf, -np.inf, 3.0], dtype=np.float32)
    words = vals.view(np.uint32).copy()
    words[0] = 0x7FC12345  # NaN with a payload
    b = orc.permute((2, 3), (1, 0), words)
    assert sorted(b.tolist()) == sorted(words.tolist())
    assert 0x7FC12345 in b.tolist() and 0x80000000 in b.tolist()


def test_workload_generators():
    assert len(wl.s2_ttc()) == 57
    for c in wl.s2_ttc():
        assert 190e6 <= c.vol <= 210e6, c
        assert sorted(c.perm) == list(range(c.rank)) and c.perm != tuple(range(c.rank))
    s3 = wl.s3_random(per_cell=2)
    assert all(120e6 * 0.95 <= c.vol <= 280e6 * 1.05 for c in s3 if c.tags[0] == "S3")
    assert {c.rank for c in s3} == set(range(2, 13))
    np.testing.assert_array_equal(wl.random_words(10, 4, 5), wl.random_words(10, 4, 5))
    assert wl.random_words(10, 8, 5).dtype == np.uint64
    assert wl.s1().vol == 16384 * 16384


def test_permute_strided_pins():
    """Strided oracle form: dense strides reduce to the C gather odometer;
    a brute-force loop over coordinates on a padded, reordered layout."""
    import itertools
    rng = np.random.default_rng(5)
    for _ in range(10):
        rank = int(rng.integers(1, 5))
        dims = [int(x) for x in rng.integers(1, 6, size=rank)]
        perm = [int(x) for x in rng.permutation(rank)]
        vol = int(np.prod(dims))
        words = rng.integers(0, 2**32, size=vol, dtype=np.uint64).astype(np.uint32)
        din = [int(np.prod(dims[:i])) for i in range(rank)]
        dout = [int(np.prod([dims[perm[k]] for k in range(j)])) for j in range(rank)]
        got = orc.permute_strided(dims, perm, words, din, np.zeros(vol, np.uint32), dout)
        np.testing.assert_array_equal(got, orc.permute(dims, perm, words))
        # padded extents, memory order of the output layout reversed
        pin = [d + int(rng.integers(0, 3)) for d in dims]
        sin = [int(np.prod(pin[:i])) for i in range(rank)]
        pout = [dims[perm[j]] + int(rng.integers(0, 3)) for j in range(rank)]
        sout = [0] * rank
        acc = 1
        for j in reversed(range(rank)):
            sout[j] = acc
            acc *= pout[j]
        inbuf = rng.integers(0, 2**32, size=int(np.prod(pin)), dtype=np.uint64).astype(np.uint32)
        outbuf = np.full(acc, 7, np.uint32)
        want = outbuf.copy()
        for x in itertools.product(*[range(d) for d in dims]):
            want[sum(x[perm[j]] * sout[j] for j in range(rank))] = inbuf[sum(x[i] * sin[i] for i in range(rank))]
        np.testing.assert_array_equal(orc.permute_strided(dims, perm, inbuf, sin, outbuf, sout), want)
