"""Write-only HBM bandwidth on this GPU (secondary roofline reference):
torch fill_ of a 16 GiB fp32 tensor, CUDA events, best of 10."""
import json
import torch

x = torch.empty(1 << 32, dtype=torch.float32, device="cuda")
for _ in range(3):
    x.fill_(1.0)
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x.fill_(2.0)
    b.record()
    b.synchronize()
    best = max(best, x.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9)
c = torch.empty_like(x)
bestc = 0.0
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    c.copy_(x)
    b.record()
    b.synchronize()
    bestc = max(bestc, 2 * x.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9)
print(json.dumps({"write_only_gbs": best, "copy_gbs": bestc, "bytes": x.numel() * 4}))
