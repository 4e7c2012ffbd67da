#!/usr/bin/env python
"""One warm-up C3 fill then one captured fill (for ncu -k regex:k_smem -s 1 -c 1):
1184 pools, n = 4 fp32 4x1024, seed 2024, f = 1, `--total` normals (default 2^30)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--total", type=int, default=1 << 30)
ap.add_argument("--pool-exponent", type=int, default=10)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--pools", type=int, default=0, help="0: one resident wave")
ap.add_argument("--f", type=int, default=1)
args = ap.parse_args()

import torch

import paper_1004_3114_b200 as W

cfg = W.WallaceConfig(pool_exponent=args.pool_exponent, throwaway_f=args.f, seed=2024,
                      n_arrays=4, dtype=args.dtype)
cfg.pools = args.pools or W.resident_pools(cfg)
g = W.WallaceState(cfg)
t = torch.empty(args.total, dtype=torch.float32 if args.dtype == "f32" else torch.float64,
                device="cuda")
g.fill(t)
g.fill(t)
torch.cuda.synchronize()
g.synchronize()
print(f"pools={cfg.pools} launches={g.kernel_launches()}")
