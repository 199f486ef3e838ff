"""Throughput of the tcgen05 int8 GEMM (laker_debug_igemm_s8) on square-ish shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_25138_b200 import laker as L

for (M, N, K) in [(4096, 4096, 4096), (8192, 8192, 8192), (4096, 16384, 16384)]:
    A = torch.randint(-64, 64, (M, K), dtype=torch.int8, device="cuda")
    B = torch.randint(-64, 64, (N, K), dtype=torch.int8, device="cuda")
    C = torch.empty((M, N), dtype=torch.int32, device="cuda")
    L.laker_debug_igemm_s8(A, B, C)
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        L.laker_debug_igemm_s8(A, B, C)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"M={M} N={N} K={K}: {dt*1e3:.2f} ms, {2*M*N*K/dt/1e12:.0f} TOPS", flush=True)
