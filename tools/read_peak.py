"""Read-only HBM stream peak on this B200 ("also record the box's
read-only stream peak"): a torch sum over a 4 GiB fp64 buffer (reads only, one
scalar written), best of 10 with CUDA events; beside MEASURED_PEAKS.json's copy
figure (read + write)."""
import json

import torch

x = torch.ones(1 << 29, dtype=torch.float64, device="cuda")  # 4 GiB
for _ in range(3):
    x.sum()
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x.sum()
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) * 1e-3)
print(json.dumps({"read_only_gbs": x.numel() * 8 / best / 1e9, "bytes": x.numel() * 8, "best_s": best,
                  "how": "torch.sum over 4 GiB fp64, best of 10, CUDA events"}))
