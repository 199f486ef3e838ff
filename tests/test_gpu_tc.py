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
