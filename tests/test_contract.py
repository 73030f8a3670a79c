"""TTGT tensor contraction (SURVEY f-4).

CPU (-m "not gpu"): the contraction oracle (oracle/tt_oracle.c
oracle_contract, the plain double odometer of P:L321's D = D + L.R) pinned
to things other than itself -- numpy matmul and einsum (library routines),
the all-ones closed form, contraction with an identity matrix reducing to
the permutation oracle bit for bit, a full contraction as a dot product,
linearity in alpha/beta -- and the TTGT decomposition the planner derives
(offline plans).
GPU: tt_contract_execute (transposes + cuBLAS GEMM) against the oracle with
a tolerance from the arithmetic: |D_gpu - D| <= c * (k + 2) * u *
(|alpha| * sum_z |L||R| + |beta| * |D0|), u the unit roundoff of the element
type (fp32 GEMMs accumulate in fp32; the oracle in fp64)."""
import string

import numpy as np
import pytest

import paper_1705_01598_b200 as tt
from oracle import oracle as orc
import tt_workloads as wl


def _einsum(modes_d, dims_l, modes_l, dims_r, modes_r, L, R):
    """numpy.einsum on column-major data: reverse shapes and subscripts."""
    labels = sorted(set(modes_l) | set(modes_r))
    ch = {m: string.ascii_letters[i] for i, m in enumerate(labels)}
    sub = lambda ms: "".join(ch[m] for m in reversed(ms))  # noqa: E731
    a = L.reshape(tuple(reversed(dims_l)))
    b = R.reshape(tuple(reversed(dims_r)))
    return np.einsum(f"{sub(modes_l)},{sub(modes_r)}->{sub(modes_d)}", a, b).ravel()


def _rand(n, dtype, seed):
    return np.random.default_rng(seed).standard_normal(n).astype(dtype)


def test_oracle_matmul_pin():
    m, k, n = 7, 11, 5
    L, R = _rand(m * k, np.float64, 1), _rand(k * n, np.float64, 2)
    D = orc.contract((0, 2), (m, k), (0, 1), (k, n), (1, 2), L, R)
    want = L.reshape(k, m).T @ R.reshape(n, k).T        # column-major m x k times k x n
    np.testing.assert_allclose(D.reshape(n, m).T, want, rtol=1e-13, atol=1e-13)


CASES = [  # (modes_d, dims_l, modes_l, dims_r, modes_r)
    ((0, 2), (6, 5), (0, 1), (5, 4), (1, 2)),                     # matmul, direct
    ((2, 0), (6, 5), (0, 1), (5, 4), (1, 2)),                     # D = (LR)^T
    ((0, 2), (5, 6), (1, 0), (4, 5), (2, 1)),                     # both operands op T
    ((2, 3, 0), (3, 2, 4), (0, 5, 1), (2, 4, 5, 3), (5, 1, 2, 3)),
    ((0, 3, 2), (2, 3, 4), (5, 0, 1), (5, 2, 4, 3), (2, 5, 1, 3)),
    ((3, 0, 2, 1), (3, 4, 5, 2), (0, 9, 1, 8), (2, 5, 6, 4), (8, 2, 3, 9)),   # back transpose
    ((0, 7, 1), (4, 3), (0, 1), (2,), (7,)),                      # outer product (no K)
    ((), (3, 4), (0, 1), (4, 3), (1, 0)),                         # full contraction
    ((4, 0), (5, 3, 2, 7), (0, 1, 6, 2), (7, 3, 2, 4), (2, 1, 6, 4)),      # K of 3 labels
]


@pytest.mark.parametrize("case", CASES)
def test_oracle_einsum_pin(case):
    md, dl, ml, dr, mr = case
    L = _rand(int(np.prod(dl)), np.float64, 3)
    R = _rand(int(np.prod(dr)), np.float64, 4)
    D = orc.contract(md, dl, ml, dr, mr, L, R)
    np.testing.assert_allclose(D, _einsum(md, dl, ml, dr, mr, L, R), rtol=1e-12, atol=1e-12)


def test_oracle_closed_forms():
    # all ones: every output is vol(K)
    D = orc.contract((0, 3), (3, 4, 5), (0, 1, 2), (4, 5, 6), (1, 2, 3), np.ones(60), np.ones(120))
    assert D.shape == (18,) and np.all(D == 20.0)
    # full contraction = dot product of the aligned operands
    L, R = _rand(12, np.float64, 5), _rand(12, np.float64, 6)
    d = orc.contract((), (3, 4), (0, 1), (3, 4), (0, 1), L, R)
    assert d.shape == (1,) and abs(d[0] - float(np.dot(L, R))) < 1e-12
    # linearity: alpha X + beta D0
    L, R = _rand(20, np.float64, 7), _rand(15, np.float64, 8)
    X = orc.contract((0, 2), (4, 5), (0, 1), (5, 3), (1, 2), L, R)
    D0 = _rand(12, np.float64, 9)
    Y = orc.contract((0, 2), (4, 5), (0, 1), (5, 3), (1, 2), L, R, D0=D0, alpha=-2.5, beta=0.75)
    np.testing.assert_allclose(Y, -2.5 * X + 0.75 * D0, rtol=1e-14, atol=1e-14)


def test_oracle_identity_contraction_is_the_permutation():
    """L[a,b,c] . I[c,d] with D labelled (d, a, b) is the permutation (2, 0, 1)
    of L: equal to the permutation oracle bit for bit (x*1 and +0 are exact)."""
    dims = (4, 3, 5)
    L = _rand(60, np.float64, 10)
    I = np.eye(5).ravel()
    D = orc.contract((3, 0, 1), dims, (0, 1, 2), (5, 5), (2, 3), L, I)
    P = orc.permute(dims, (2, 0, 1), L.view(np.uint64)).view(np.float64)
    assert np.array_equal(D.view(np.uint64), P.view(np.uint64))


def test_oracle_rejects_non_contractions():
    with pytest.raises(ValueError):   # label of L summed over one operand only
        orc.contract((0,), (3, 4), (0, 1), (3,), (0,), np.ones(12), np.ones(3))
    with pytest.raises(ValueError):   # label of R in neither D nor L
        orc.contract((0, 1), (4, 3), (0, 1), (2,), (7,), np.ones(12), np.ones(2))
    with pytest.raises(ValueError):   # contracted extents differ
        orc.contract((0,), (3, 4), (0, 1), (5,), (1,), np.ones(12), np.ones(5))


def test_ttgt_decomposition_offline():
    d = tt.contract_offline((0, 2), (6, 5), (0, 1), (5, 4), (1, 2), 8)
    assert (d["m"], d["n"], d["k"]) == (6, 4, 5) and d["launches"] == 0 and not d["swap_mn"]
    d = tt.contract_offline((2, 0), (6, 5), (0, 1), (5, 4), (1, 2), 8)
    assert d["swap_mn"] and d["launches"] == 0 and d["dims_d"] == [4, 6]
    d = tt.contract_offline((0, 2), (5, 6), (1, 0), (4, 5), (2, 1), 4)
    assert d["op_l"] == "T" and d["op_r"] == "T" and d["launches"] == 0
    d = tt.contract_offline(*CASES[5], 8)
    assert d["transpose_d"] and d["launches"] >= 1 and d["dims_d"] == [6, 3, 5, 5]
    for bad, st in [(((0, 2), (6, 5), (0, 1), (5, 4), (1, 0)), 2),     # label 0 in L, R and D
                    (((0, 2), (6, 5), (0, 1), (6, 4), (1, 2)), 2),     # contracted extents differ
                    (((0, 1), (6, 5), (0, 1), (5, 4), (1, 2)), 4)]:    # batch label 1
        with pytest.raises(tt.TTError) as e:
            tt.contract_offline(*bad, 8)
        assert e.value.status in (2, 4)


# ---- GPU parity ---------------------------------------------------------------

_U = {4: 2.0 ** -24, 8: 2.0 ** -53}
_DT = {4: np.float32, 8: np.float64}


def _gpu_contract(case, esize, alpha, beta, seed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    md, dl, ml, dr, mr = case
    dt = _DT[esize]
    L = _rand(int(np.prod(dl)), dt, seed)
    R = _rand(int(np.prod(dr)), dt, seed + 1)
    c = tt.Contraction(md, dl, ml, dr, mr, esize)
    vd = int(np.prod(c.dims_d)) if c.dims_d else 1
    D0 = _rand(vd, dt, seed + 2)
    tdt = torch.float32 if esize == 4 else torch.float64
    dev = torch.device("cuda", 0)
    tl, tr = torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev)
    td = torch.from_numpy(D0.copy()).to(dev)
    c.execute(tl, tr, td, alpha, beta)
    torch.cuda.synchronize()
    got = td.cpu().numpy().astype(np.float64)
    want = orc.contract(md, dl, ml, dr, mr, L, R, D0=D0.astype(np.float64), alpha=alpha, beta=beta)
    mag = abs(alpha) * orc.contract(md, dl, ml, dr, mr, np.abs(L), np.abs(R)) + abs(beta) * np.abs(D0)
    tol = 4.0 * (c.k + 2) * _U[esize] * mag + 1e-300
    bad = np.abs(got - want) > tol
    assert not bad.any(), f"{case} e{esize}: {int(bad.sum())} outside the bound, max err " \
                          f"{float(np.max(np.abs(got - want)))}"
    ms = c.timings()
    assert len(ms) == 4 and ms[2] >= 0
    c.destroy()


GPU_CASES = CASES + [
    ((0, 4, 2), (33, 7, 29), (0, 1, 2), (7, 31), (1, 4)),                               # ragged sizes
    ((5, 0, 3, 1), (40, 6, 8, 50), (0, 6, 7, 1), (8, 30, 6, 20), (7, 3, 6, 5)),         # TAL-SH-like
    ((2, 0), (64, 96, 40), (0, 9, 1), (40, 96, 72), (1, 9, 2)),                         # R: K then N, reordered
]


@pytest.mark.gpu
@pytest.mark.parametrize("esize", [4, 8])
@pytest.mark.parametrize("case", GPU_CASES)
def test_gpu_contraction_matches_oracle(case, esize):
    _gpu_contract(case, esize, 1.0, 0.0, 20)
    _gpu_contract(case, esize, -0.5, 1.25, 30)     # accumulate form D = a L.R + b D


@pytest.mark.gpu
def test_gpu_contraction_large_tal_sh_shape():
    """A TAL-SH-shaped fp64 contraction with transposes on every operand at
    a size that spans many tiles (vol(D) = 1.1 M, k = 512), all outputs."""
    case = ((3, 0, 2, 1), (48, 32, 24, 16), (0, 9, 1, 8), (16, 40, 24, 32), (8, 2, 3, 9))
    _gpu_contract(case, 8, 1.0, 0.0, 40)
