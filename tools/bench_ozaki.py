"""Ozaki (int8 tcgen05) fp64 GEMM vs the DMMA fp64 GEMM on fit-sized shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_25138_b200 import laker as L

for (M, N, K) in [(4096, 4096, 4096), (4096, 16384, 16384)]:
    A = torch.randn((M, K), dtype=torch.float64, device="cuda")
    B = torch.randn((N, K), dtype=torch.float64, device="cuda")
    C = torch.empty((M, N), dtype=torch.float64, device="cuda")
    for S in (7, 8):
        L.laker_debug_ozaki_gemm(A, B, C, S)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            L.laker_debug_ozaki_gemm(A, B, C, S)
        e1.record()
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / 3 * 1e-3
        ref = A @ B.T
        err = ((C - ref).abs().max() / (A.abs() @ B.abs().T).max()).item()
        print(f"M={M} N={N} K={K} S={S}: {dt*1e3:.2f} ms = {2*M*N*K/dt/1e12:.1f} fp64-equiv TF/s, err {err:.2e}", flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        ref = A @ B.T
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"   torch fp64 (cuBLAS DGEMM) {dt*1e3:.2f} ms = {2*M*N*K/dt/1e12:.1f} TF/s", flush=True)
