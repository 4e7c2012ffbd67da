"""C1 fill time with and without the periodic drift audit (smem and
cluster engines select by WRNG_GPU_NO_CLUSTER): the audit's share."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1004_3114_b200 import WallaceConfig, WallaceState  # noqa: E402

out = torch.empty(1 << 24, dtype=torch.float64, device="cuda")
for drift in (64, 0):
    g = WallaceState(WallaceConfig(pool_exponent=12, throwaway_f=1, seed=12345, n_arrays=4,
                                   dtype="f64", drift_check_period=drift))
    g.fill(out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.fill(out)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"drift_period={drift}: {best:.3f} ms per 2^24 values")
