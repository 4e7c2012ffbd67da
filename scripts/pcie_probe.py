"""D2H bandwidth of this box's host link: 1-D pinned copies of 256 MiB and
a 2-D copy shaped like the staged bank fill (1184 rows of L values)."""
import ctypes
import json
import time

import torch

n = 64 << 20  # 256 MiB fp32
d = torch.empty(n, dtype=torch.float32, device="cuda")
h = torch.empty(4 * n, dtype=torch.float32, pin_memory=True)
s = torch.cuda.Stream()
r = {}
for _ in range(2):
    h[:n].copy_(d, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(8):
    h[(i % 4) * n:(i % 4 + 1) * n].copy_(d, non_blocking=True)
torch.cuda.synchronize()
r["d2h_1d_gbs"] = 8 * n * 4 / (time.perf_counter() - t) / 1e9
cud = ctypes.CDLL("libcudart.so.12") if False else None
# 2-D: 1184 rows of L = n // 1184 values, host pitch 4 * L (bank window)
L = n // 1184
hv = h.view(-1)
t = time.perf_counter()
for i in range(8):
    hv[: 1184 * 4 * L].view(1184, 4 * L)[:, :L].copy_(d[: 1184 * L].view(1184, L), non_blocking=True)
torch.cuda.synchronize()
r["d2h_2d_gbs"] = 8 * 1184 * L * 4 / (time.perf_counter() - t) / 1e9
print(json.dumps(r))
