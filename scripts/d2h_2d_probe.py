"""cudaMemcpy2DAsync (the host-fill staging shape: 1184 rows of L fp32
values, host pitch = one pool segment) vs a 1-D copy of the same bytes."""
import ctypes
import json
import time

import torch

rt = ctypes.CDLL("libcudart.so.12")
P, total = 1184, 1 << 30
seg = total // P
L = (256 << 20) // 4 // P
d = torch.empty(P * L, dtype=torch.float32, device="cuda")
h = torch.empty(total, dtype=torch.float32, pin_memory=True)
s = torch.cuda.Stream()
D2H = 2


def run2d(reps):
    for r in range(reps):
        t0 = (r * L) % (seg - L)
        rt.cudaMemcpy2DAsync(ctypes.c_void_p(h.data_ptr() + 4 * t0), ctypes.c_size_t(seg * 4),
                             ctypes.c_void_p(d.data_ptr()), ctypes.c_size_t(L * 4),
                             ctypes.c_size_t(L * 4), ctypes.c_size_t(P), D2H,
                             ctypes.c_void_p(s.cuda_stream))
    s.synchronize()


def run1d(reps):
    n = P * L
    for r in range(reps):
        off = (r * n) % (total - n)
        rt.cudaMemcpyAsync(ctypes.c_void_p(h.data_ptr() + 4 * off), ctypes.c_void_p(d.data_ptr()),
                           ctypes.c_size_t(n * 4), D2H, ctypes.c_void_p(s.cuda_stream))
    s.synchronize()


out = {}
for name, fn in (("1d", run1d), ("2d", run2d), ("1d_again", run1d), ("2d_again", run2d)):
    fn(2)
    t = time.perf_counter()
    fn(16)
    out[name + "_gbs"] = 16 * P * L * 4 / (time.perf_counter() - t) / 1e9
print(json.dumps(out))
