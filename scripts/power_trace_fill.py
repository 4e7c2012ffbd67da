import os, subprocess, sys, threading, time
import torch
t = torch.empty(1 << 34, dtype=torch.float32, device="cuda")
for _ in range(5): t.fill_(1.0)
torch.cuda.synchronize()
samples = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active", "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=lambda: [samples.append((time.time(), l.strip())) for l in p.stdout], daemon=True); th.start()
time.sleep(0.3)
s = torch.cuda.current_stream(); steps = 30
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
t0 = time.time(); ev[0].record(s)
for k in range(steps):
    t.fill_(float(k)); ev[k + 1].record(s)
torch.cuda.synchronize(); t1 = time.time(); time.sleep(0.1); p.terminate()
print("fill_ step ms:", " ".join(f"{ev[k].elapsed_time(ev[k + 1]):.2f}" for k in range(steps)))
for ts, l in samples:
    if t0 - 0.05 <= ts <= t1 + 0.05: print(f"{ts - t0:+.3f}s {l}")
