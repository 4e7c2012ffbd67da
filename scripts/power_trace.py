#!/usr/bin/env python
"""Per-step times of N back-to-back C3/C4-shard fills with nvidia-smi clock and power
samples every 20 ms: shows what the 20-step default bench run sees (sw_power_cap)."""
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1004_3114_b200 as W

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 25
g = W.WallaceState(W.WallaceConfig(pool_exponent=10, throwaway_f=1, seed=99, n_arrays=4,
                                   dtype="f32", pools=1184))
t = torch.empty(1 << 34, dtype=torch.float32, device="cuda")
for _ in range(5):
    g.fill(t)
torch.cuda.synchronize()
samples = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active",
                      "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=lambda: [samples.append((time.time(), l.strip())) for l in p.stdout], daemon=True)
th.start()
time.sleep(0.3)
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
t0 = time.time()
ev[0].record(s)
for k in range(steps):
    g.fill(t)
    ev[k + 1].record(s)
torch.cuda.synchronize()
t1 = time.time()
time.sleep(0.2)
p.terminate()
ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
print("step ms:", " ".join(f"{x:.2f}" for x in ms))
print(f"mean of all {sum(ms) / len(ms):.3f} ms; of steps 10.. {sum(ms[10:]) / max(1, len(ms[10:])):.3f} ms")
if "-q" not in sys.argv:
    for ts, l in samples:
        if t0 - 0.1 <= ts <= t1 + 0.1:
            print(f"{ts - t0:+.3f}s {l}")
