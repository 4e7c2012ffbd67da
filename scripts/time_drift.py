"""Times drift_check (exact parallel sum) on a C2-shaped HBM pool."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1004_3114_b200 import WallaceConfig, WallaceState
for tree in (False, True):
    g = WallaceState(WallaceConfig(pool_exponent=20, throwaway_f=2, seed=7, n_arrays=4, dtype="f64", drift_tree=tree))
    g.fill(3 * (4 << 20))
    g.drift_check()
    t0 = time.perf_counter()
    for _ in range(10):
        g.drift_check()
    t1 = time.perf_counter()
    print(f"tree={tree}: drift_check {1e3 * (t1 - t0) / 10:.3f} ms (incl. sync)")
    t0 = time.perf_counter()
    for _ in range(10):
        g.advance_pass()
    t1 = time.perf_counter()
    print(f"advance_pass {1e3 * (t1 - t0) / 10:.3f} ms (incl. sync)")
