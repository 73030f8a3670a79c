"""Accumulate form (SURVEY f-3): out = alpha*perm(in) + beta*out.

CPU pins of the oracle's scaled form against numpy's elementwise float
arithmetic applied to the (separately pinned) permutation -- an independent
formulation -- plus closed forms; GPU parity of tt_execute_scaled against
the oracle.  Floating point here: results are compared bit-exactly where
IEEE 754 fixes them (finite inputs, round-to-nearest, no FMA on either side);
NaN results are compared by position only, since IEEE 754 leaves their
payload open (reading R21).
"""
import numpy as np
import pytest

from oracle import oracle as orc
import tt_workloads as wl

FT = {4: np.float32, 8: np.float64}
WT = {4: np.uint32, 8: np.uint64}


def finite_words(n, esize, seed):
    rng = np.random.default_rng(seed)
    vals = rng.uniform(-4, 4, size=n).astype(FT[esize])
    vals[::7] *= 1e-30          # small and (for float) some subnormal products
    return vals.view(WT[esize])


def np_scaled(dims, perm, words, out_words, alpha, beta):
    esize = words.dtype.itemsize
    f = FT[esize]
    a = orc.permute(dims, perm, words).view(f)
    r = f(alpha) * a                       # numpy: one RN multiply per element
    if beta != 0.0:
        r = r + f(beta) * np.asarray(out_words).view(f)
    return np.asarray(r, dtype=f).view(WT[esize])


@pytest.mark.parametrize("esize", [4, 8])
def test_oracle_scaled_matches_numpy(esize):
    rng = np.random.default_rng(1)
    for _ in range(20):
        rank = int(rng.integers(1, 6))
        dims = tuple(int(x) for x in rng.integers(1, 7, size=rank))
        perm = tuple(int(x) for x in rng.permutation(rank))
        n = int(np.prod(dims))
        a = finite_words(n, esize, int(rng.integers(1 << 30)))
        b = finite_words(n, esize, int(rng.integers(1 << 30)))
        for alpha, beta in [(1.0, 0.0), (1.5, -0.25), (0.1, 0.7), (-3.0, 1.0)]:
            got = orc.permute_scaled(dims, perm, a, b, alpha, beta)
            np.testing.assert_array_equal(got, np_scaled(dims, perm, a, b, alpha, beta))


def test_oracle_scaled_closed_forms():
    dims, perm = (3, 4), (1, 0)
    a = np.arange(12, dtype=np.float64).view(np.uint64)
    b = np.full(12, 10.0).view(np.uint64)
    got = orc.permute_scaled(dims, perm, a, b, 2.0, 0.5).view(np.float64)
    # out[j + 4 i] = 2 * a[i + 3 j] + 5
    for i in range(3):
        for j in range(4):
            assert got[j + 4 * i] == 2.0 * (i + 3 * j) + 5.0
    # alpha = 1, beta = 0 is the plain permutation; beta = 0 ignores NaN in out
    nan_out = np.full(12, np.nan).view(np.uint64)
    np.testing.assert_array_equal(orc.permute_scaled(dims, perm, a, nan_out, 1.0, 0.0),
                                  orc.permute(dims, perm, a))


def _same_floats(got, want, esize):
    g, w = got.view(FT[esize]), want.view(FT[esize])
    nan_g, nan_w = np.isnan(g), np.isnan(w)
    np.testing.assert_array_equal(nan_g, nan_w)
    np.testing.assert_array_equal(got[~nan_g], want[~nan_w])


@pytest.mark.gpu
@pytest.mark.parametrize("esize", [4, 8])
def test_gpu_scaled_parity(esize):
    torch = pytest.importorskip("torch")
    import paper_1705_01598_b200 as tt
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    td = {4: torch.int32, 8: torch.int64}[esize]
    nd = {4: np.int32, 8: np.int64}[esize]
    shapes = [((7, 13, 5), (2, 0, 1)), ((130, 70), (1, 0)), ((600, 7, 5), (0, 2, 1)),
              ((5, 3, 2, 4, 7, 6), (4, 0, 5, 2, 3, 1)), ((1000,), (0,)), ((37, 29, 11), (2, 0, 1))]
    for dims, perm in shapes:
        n = int(np.prod(dims))
        for finite in (True, False):
            a = finite_words(n, esize, 3) if finite else wl.random_words(n, esize, 3)
            b = finite_words(n, esize, 4) if finite else wl.random_words(n, esize, 4)
            x = torch.from_numpy(a.view(nd).copy()).cuda()
            plan = tt.Plan(dims, perm, esize, accumulate=True)
            assert plan.describe()["accumulate"] == 1
            for alpha, beta in [(1.5, -0.25), (1.0, 0.0), (-2.0, 1.0)]:
                y = torch.from_numpy(b.view(nd).copy()).cuda()
                plan.execute_scaled(x, y, alpha, beta)
                torch.cuda.synchronize()
                got = y.cpu().numpy().view(WT[esize])
                want = orc.permute_scaled(dims, perm, a, b, alpha, beta)
                if finite:
                    np.testing.assert_array_equal(got, want)
                else:
                    _same_floats(got, want, esize)
            with pytest.raises(tt.TTError):
                plan.execute(x, y)          # accumulate plans run through execute_scaled
            plan.destroy()
