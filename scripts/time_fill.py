#!/usr/bin/env python
"""Device-timed bank fills of one shape: python scripts/time_fill.py --pool-exponent 9
--dtype f32 --f 1 [--pools N] [--total 2^32]; prints normals/s and the fraction of the
HBM-store roofline (MEASURED_PEAKS.json).  WRNG_GPU_NO_GROUP=1 keeps small pools on
one CTA per pool (A/B against the group engine)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--total", type=int, default=1 << 32)
ap.add_argument("--pool-exponent", type=int, default=8)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--pools", type=int, default=0, help="0: one resident wave")
ap.add_argument("--f", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

import torch

import paper_1004_3114_b200 as W

with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
    peak = float(json.load(fh)["hbm_gbs"])
cfg = W.WallaceConfig(pool_exponent=args.pool_exponent, throwaway_f=args.f, seed=2024,
                      n_arrays=4, dtype=args.dtype)
cfg.pools = args.pools or W.resident_pools(cfg)
g = W.WallaceState(cfg)
esz = 4 if args.dtype == "f32" else 8
t = torch.empty(args.total, dtype=torch.float32 if esz == 4 else torch.float64, device="cuda")
g.fill(t[: cfg.pools * 4096])
torch.cuda.synchronize()
s = torch.cuda.current_stream()
best = None
for _ in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.fill(t)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    best = ms if best is None else min(best, ms)
rate = args.total / (best / 1e3)
print(f"{args.dtype} 4x{1 << args.pool_exponent} f={args.f} pools={cfg.pools} "
      f"{best:.3f} ms {rate:.3e}/s {100 * rate * esz / 1e9 / peak:.1f}%")
