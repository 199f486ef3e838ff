"""Time the Ozaki GEMM kernels on the fit's shapes (4096^3 as in Newton-Schulz, and the
directions product 4096 x 16384 x 16384) through laker_debug_ozaki_gemm;
LAKER_OZAKI_LV=0 selects the level-streaming kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402

shapes = [(4096, 4096, 4096), (4096, 16384, 16384)]
for M, N, K in shapes:
    A = torch.randn(M, K, dtype=torch.float64, device="cuda")
    B = torch.randn(N, K, dtype=torch.float64, device="cuda")
    C = torch.zeros(M, N, dtype=torch.float64, device="cuda")
    L.laker_debug_ozaki_gemm(A, B, C, 8)
    torch.cuda.synchronize()
    reps = int(os.environ.get("REPS", "5"))
    t0 = time.perf_counter()
    for _ in range(reps):
        L.laker_debug_ozaki_gemm(A, B, C, 8)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"lv={os.environ.get('LAKER_OZAKI_LV', '1')} {M}x{N}x{K}: {dt * 1e3:.2f} ms "
          f"({2 * M * N * K / dt / 1e12:.1f} TF/s fp64-equivalent)", flush=True)
