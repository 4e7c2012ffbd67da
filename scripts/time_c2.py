#!/usr/bin/env python
"""One C2 step (one 4 x 2^20 fp64 HBM pool, f = 2, 2^30 normals), device-timed; --drift P sets
the audit period (0: none), --tree the parallel (non-reference-order) audit sum: what the
exact audits cost."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--drift", type=int, default=64)
ap.add_argument("--tree", action="store_true")
args = ap.parse_args()
import torch

import paper_1004_3114_b200 as W

g = W.WallaceState(W.WallaceConfig(pool_exponent=20, throwaway_f=2, seed=7, n_arrays=4, dtype="f64",
                                   drift_check_period=args.drift, drift_tree=args.tree))
t = torch.empty(1 << 30, dtype=torch.float64, device="cuda")
g.fill(t)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
best = 1e9
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.fill(t)
    e1.record(s)
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"C2 step (drift {args.drift}{' tree' if args.tree else ''}) {best:.3f} ms, {g.kernel_launches()} launches")
