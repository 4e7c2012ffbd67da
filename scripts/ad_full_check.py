#!/usr/bin/env python
"""Full-size A^2 check: the device Anderson-Darling of a
whole 2^32-value C5 stream against the CPU oracle's A^2 of the same values
(host sort + oracle d_j sum on all host threads).

Usage: python scripts/ad_full_check.py [--total 2^32] [--settings f32:1024:1,f64:1024:1]
Writes profiles/round2/ad_full_check.json.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import torch

    import oracle as O
    import paper_1004_3114_b200 as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--total", type=int, default=1 << 32)
    ap.add_argument("--settings", default="f32:1024:1,f64:1024:1")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round2", "ad_full_check.json"))
    args = ap.parse_args()
    rows = []
    for st in args.settings.split(","):
        dt, N, R = st.split(":")
        N, R = int(N), int(R)
        cfg = W.WallaceConfig(pool_exponent=N.bit_length() - 1, throwaway_f=R, seed=2024,
                              n_arrays=4, dtype=dt)
        cfg.pools = W.resident_pools(cfg)
        t = torch.empty(args.total, dtype=torch.float32 if dt == "f32" else torch.float64,
                        device="cuda")
        W.WallaceState(cfg).fill(t)
        torch.cuda.synchronize()
        t0 = time.time()
        a_dev = W.device_anderson_darling(t)
        t_dev = time.time() - t0
        v = t.cpu().numpy()
        del t
        torch.cuda.empty_cache()
        t0 = time.time()
        v.sort()
        t_sort = time.time() - t0
        t0 = time.time()
        a_or = O.anderson_darling_sorted(v)
        t_or = time.time() - t0
        row = {"setting": st, "pools": cfg.pools, "n": args.total, "ad_device": a_dev,
               "ad_oracle": a_or, "rel_diff": abs(a_dev - a_or) / max(1.0, abs(a_or)),
               "device_s": t_dev, "host_sort_s": t_sort, "oracle_sum_s": t_or,
               "host_threads": os.cpu_count()}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del v
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
