"""One 4096^3 Ozaki GEMM per kernel variant (0 fused, 2 level groups v2) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402

n = int(os.environ.get("N", "4096"))
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
B = torch.randn(n, n, dtype=torch.float64, device="cuda")
C = torch.zeros(n, n, dtype=torch.float64, device="cuda")
for k in (0, 2):
    L.laker_debug_ozaki_gemm(A, B, C, 8, k)
torch.cuda.synchronize()
print("ok")
