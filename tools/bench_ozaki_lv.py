"""Time the Ozaki GEMM kernels on the fit's shapes (4096^3 as in Newton-Schulz, and the
directions product 4096 x 16384 x 16384) through laker_debug_ozaki_gemm, each kernel
(0 level-streaming fused, 2 level groups on chunk-interleaved slices)
checked bitwise against kernel 0 (the level sums are exact integers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402

shapes = [(4096, 4096, 4096), (4096, 4096, 16384), (4096, 16384, 16384), (3584, 16384, 512), (7680, 3584, 512),
          (1000, 777, 1300), (130, 4000, 600)]
kernels = [int(k) for k in os.environ.get("KERNELS", "0,2").split(",")]
reps = int(os.environ.get("REPS", "5"))
for M, N, K in shapes:
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(N, K, dtype=torch.float64, device="cuda", generator=g) * torch.exp(
        torch.randn(N, 1, dtype=torch.float64, device="cuda", generator=g))
    ref = None
    for kern in kernels:
        C = torch.zeros(M, N, dtype=torch.float64, device="cuda")
        L.laker_debug_ozaki_gemm(A, B, C, 8, kern)
        torch.cuda.synchronize()
        if ref is None:
            ref = C.clone()
            err = (C - A @ B.T).abs().max().item() / (A.abs() @ B.abs().T).max().item()
        same = bool(torch.equal(C, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            L.laker_debug_ozaki_gemm(A, B, C, 8, kern)
        e1.record()
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / reps * 1e-3
        print(f"kernel={kern} {M}x{N}x{K}: {dt * 1e3:.3f} ms ({2 * M * N * K / dt / 1e12:.1f} TF/s fp64-equivalent)"
              f" bitwise_vs_k{kernels[0]}={same} relerr_vs_torch={err:.2e}", flush=True)
