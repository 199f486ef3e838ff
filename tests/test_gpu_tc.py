"""tcgen05 int8 tensor-core GEMM (csrc/igemm.cu), the building block of the
fp64 emulation: integer results must be exact (bit-exact int32) for every
shape, including ragged M / N / K tails (TMA zero fill)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (256, 512, 256), (300, 700, 384), (128, 256, 4096),
                                   (1, 1, 16), (129, 257, 144)])
def test_igemm_s8_exact(M, N, K):
    import torch
    from paper_2604_25138_b200 import laker as L
    r = np.random.default_rng(M * 7 + N + K)
    A = r.integers(-128, 128, (M, K), dtype=np.int8)
    B = r.integers(-128, 128, (N, K), dtype=np.int8)
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    Cd = torch.zeros((M, N), dtype=torch.int32, device="cuda")
    L.laker_debug_igemm_s8(Ad, Bd, Cd)
    C = Cd.cpu().numpy()
    bad = np.flatnonzero(C.ravel() != ref.ravel())
    assert bad.size == 0, (bad.size, bad[:5], C.ravel()[bad[:3]], ref.ravel()[bad[:3]])


def _exact_rowcol(A, B, i, j):
    from fractions import Fraction
    return sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(A[i], B[j]))


@pytest.mark.parametrize("M,N,K,S", [(256, 256, 512, 8), (300, 520, 1000, 8), (128, 256, 4096, 7),
                                     (257, 129, 96, 8)])
def test_ozaki_gemm_accuracy(M, N, K, S):
    """fp64 GEMM emulated with S int8 digit slices per input: every input is kept to
    2^-(7S-1) of its row (column) maximum and every level sum is exact, so each
    entry is within (S+2) K 2^-(7S-1) max_k|a_ik| max_k|b_jk| (+ the final fp64
    roundings) of the exact product -- the max-norm form of the fp64 GEMM bound
    K u |a||b|.  Checked against longdouble everywhere and exact rationals on
    sampled entries; rows/columns span 2^+-20 in scale, entries 2^-8 within a row."""
    import torch
    from paper_2604_25138_b200 import laker as L
    r = np.random.default_rng(M + N + K + S)
    A = r.standard_normal((M, K)) * np.exp2(r.integers(-20, 20, (M, 1))) * np.exp2(r.uniform(-8, 0, (M, K)))
    B = r.standard_normal((N, K)) * np.exp2(r.integers(-20, 20, (N, 1)))
    Cd = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    L.laker_debug_ozaki_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), Cd, S)
    C = Cd.cpu().numpy()
    ref = (A.astype(np.longdouble) @ B.astype(np.longdouble).T).astype(np.float64)
    mx = np.outer(np.abs(A).max(axis=1), np.abs(B).max(axis=1))
    bound = (S + 2) * K * 2.0 ** -(7 * S - 1) * mx + 8 * np.finfo(float).eps * np.abs(ref)
    err = np.abs(C - ref)
    assert (err <= bound).all(), (err / mx).max()
    # and in the usual relative sense: comparable to an fp64 GEMM
    absdot = np.abs(A) @ np.abs(B).T
    assert (err / absdot).max() <= (2e-13 if S >= 8 else 2e-11)
    for (i, j) in [(0, 0), (M - 1, N - 1), (M // 2, N // 3)]:
        ex = _exact_rowcol(A, B, i, j)
        assert abs(float(ex - __import__("fractions").Fraction(float(C[i, j])))) <= bound[i, j]


@pytest.mark.parametrize("M,N,K,S", [(256, 384, 512, 8), (300, 130, 1000, 8), (128, 256, 4096, 7),
                                     (257, 129, 96, 5), (129, 200, 640, 3)])
def test_ozaki_level_group_kernel_equals_fused(M, N, K, S):
    """The level-group kernel (each K chunk's slices loaded once, all pairs of <= 4
    levels into resident TMEM buffers) issues the same exact int32 level sums and
    accumulates them in the same fp64 order as the level-streaming kernel: bitwise
    equal results, including ragged M / N / K and S not a multiple of 4."""
    import torch
    from paper_2604_25138_b200 import laker as L
    r = np.random.default_rng(M * 7 + N + K + S)
    A = torch.from_numpy(r.standard_normal((M, K)) * np.exp2(r.integers(-20, 20, (M, 1)))).cuda()
    B = torch.from_numpy(r.standard_normal((N, K))).cuda()
    C1 = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    C2 = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    L.laker_debug_ozaki_gemm(A, B, C1, S, kernel=1)
    L.laker_debug_ozaki_gemm(A, B, C2, S, kernel=0)
    assert torch.equal(C1, C2)
