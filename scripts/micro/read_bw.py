"""Pure-read HBM bandwidth on this GPU (context for the apply's roofline: MEASURED_PEAKS.json
hbm_gbs is a read+write copy).  torch's sum over 16 GiB of FP64, best of 10, CUDA events."""
import json

import torch

a = torch.rand(2 ** 31, dtype=torch.float64, device="cuda")
best = 1e9
for _ in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s = a.sum()
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
b = a.numel() * 8
c = torch.empty_like(a)
bestc = 1e9
for _ in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c.copy_(a)
    e1.record()
    e1.synchronize()
    bestc = min(bestc, e0.elapsed_time(e1))
print(json.dumps({"read_gbs": b / best / 1e6, "copy_gbs": 2 * b / bestc / 1e6, "bytes": b}))
