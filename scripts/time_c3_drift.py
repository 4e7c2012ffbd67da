"""C3 fill time with the drift audit every 64 passes (default) vs never,
to bound the audit's share of the step (exact_sumsq_cta in k_smem)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1004_3114_b200 import WallaceConfig, WallaceState  # noqa: E402

out = torch.empty(1 << 34, dtype=torch.float32, device="cuda")
for drift in (64, 0, 64, 0):
    g = WallaceState(WallaceConfig(pool_exponent=10, throwaway_f=1, seed=2024, n_arrays=4,
                                   dtype="f32", pools=1184, drift_check_period=drift))
    g.fill(out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(4):
        a.record()
        g.fill(out)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    print(f"drift_check_period={drift}: {min(ms):.3f} ms per 2^34 normals")
    del g
