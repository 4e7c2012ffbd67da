#!/usr/bin/env python
"""BASELINE.json config 5: quality/cost sweep on one GPU.

R (passes per output) in {1,2,3,4} x pool 4 x {256, 1024, 4096} per CTA x
{fp32, fp64} x chi rescale {on, off}; 2^32 normals per setting; pools seeded
UniformState(2024, c) (BASELINE names no seed), host (glibc) init.  The
bank holds one wave of pools: wrng_gpu_resident_pools (SMs x CTAs per SM of
the fill kernel).  Reports device-timed throughput (mean of 2 timed fills)
and its fraction of the HBM-store roofline, the first four moments and the
Anderson-Darling A^2 of the FULL 2^32 stream (device reductions, device radix
sort), and moments + A^2 of a bounded sample (the first 2^20 values of pools
0..3) next to the CPU oracle's values for the same sample.

Usage: python scripts/sweep_c5.py [--total 2^32] [--out profiles/round2/c5_sweep.json]
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
    from paper_1004_3114_b200 import (WallaceConfig, WallaceState, device_anderson_darling,
                                      device_moments, resident_pools)

    ap = argparse.ArgumentParser()
    ap.add_argument("--total", type=int, default=1 << 32)
    ap.add_argument("--sample", type=int, default=1 << 20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round2", "c5_sweep.json"))
    ap.add_argument("--only", default=None, help="dtype:N[:R] subset, e.g. f32:256:1")
    ap.add_argument("--pools-per-sm", type=int, default=0, help="override: pools = 148 x this")
    ap.add_argument("--quick", action="store_true", help="subset for smoke runs")
    args = ap.parse_args()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        peak = float(json.load(fh)["hbm_gbs"])
    dev = torch.device("cuda", 0)
    out64 = torch.empty(args.total, dtype=torch.float64, device=dev)
    rows = []
    dtypes = ["f32", "f64"]
    Ns = [256, 1024, 4096]
    Rs = [1, 2, 3, 4]
    modes = [0, 1]
    if args.quick:
        Ns, Rs = [1024], [1, 4]
    for dt in dtypes:
        for N in Ns:
            for R in Rs:
                for mode in modes:
                    if args.only:
                        want = args.only.split(":")
                        if want[0] != dt or int(want[1]) != N or (len(want) > 2 and
                                                                  int(want[2]) != R):
                            continue
                    cfg = WallaceConfig(pool_exponent=N.bit_length() - 1, throwaway_f=R,
                                        scale_mode=mode, seed=2024, n_arrays=4, dtype=dt)
                    P = 148 * args.pools_per_sm if args.pools_per_sm else resident_pools(cfg)
                    cfg.pools = P
                    buf = out64 if dt == "f64" else out64.view(torch.float32)[: args.total]
                    # the timed fills continue a warmed generator; the
                    # statistics use a fresh one so they cover the stream's start
                    g = WallaceState(cfg)
                    g.fill(buf[: P * 4096])  # warm-up
                    torch.cuda.synchronize()
                    s = torch.cuda.current_stream()
                    times = []
                    for _ in range(2):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        g.fill(buf[: args.total])
                        e1.record(s)
                        e1.synchronize()
                        times.append(e0.elapsed_time(e1))
                    g.synchronize()
                    ms = sum(times) / len(times)
                    rate = args.total / (ms / 1e3)
                    esz = 4 if dt == "f32" else 8
                    WallaceState(cfg).fill(buf[: args.total])
                    torch.cuda.synchronize()
                    mom = device_moments(buf[: args.total])
                    ad_full = device_anderson_darling(buf[: args.total])
                    # bounded sample: first `sample` values of pools 0..3 (fresh
                    # generator so the sample is the stream's beginning)
                    g2 = WallaceState(cfg)
                    per = args.sample
                    gs = g2.fill(np.empty(per * P, dtype=np.float32 if dt == "f32" else np.float64))
                    gsamp = np.concatenate([gs[p * per:(p + 1) * per] for p in range(4)])
                    osamp = np.concatenate([
                        O.OracleState(pool_exponent=N.bit_length() - 1, throwaway_f=R,
                                      scale_mode=mode, seed=2024, stream=p, n_arrays=4,
                                      dtype=O.F32 if dt == "f32" else O.F64).fill(per)
                        for p in range(4)])
                    mg, mo = O.moments(gsamp), O.moments(osamp)
                    row = {
                        "dtype": dt, "N": N, "R": R, "chisq": mode == 0, "pools": P,
                        "normals": args.total, "ms": ms, "normals_per_s": rate,
                        "hbm_store_frac": rate * esz / 1e9 / peak,
                        "moments_full": {k: mom[k] for k in ("m1", "m2", "m3", "m4")},
                        "ad_full": ad_full,
                        "sample": f"pools 0..3, first {per} values each",
                        "gpu_sample": {"m1": mg["m1"], "m2": mg["m2"], "m3": mg["m3"],
                                       "m4": mg["m4"], "ad": O.anderson_darling(gsamp)},
                        "oracle_sample": {"m1": mo["m1"], "m2": mo["m2"], "m3": mo["m3"],
                                          "m4": mo["m4"], "ad": O.anderson_darling(osamp)},
                        "max_rel_diff_sample": float(np.max(
                            np.abs(gsamp.astype(np.float64) - osamp.astype(np.float64)) /
                            np.maximum(1.0, np.abs(osamp.astype(np.float64))))),
                    }
                    rows.append(row)
                    print(f"{dt} N={N:5d} R={R} chisq={mode == 0!s:5s} pools={P:5d} "
                          f"{rate:.3e}/s {100 * row['hbm_store_frac']:5.1f}% "
                          f"m2={mom['m2']:.6f} m4={mom['m4']:.5f} A2(2^32)={ad_full:.3f} "
                          f"AD gpu={row['gpu_sample']['ad']:.4f} oracle={row['oracle_sample']['ad']:.4f}",
                          flush=True)
                    del g, g2
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump({"config": "BASELINE.json configs[4] (C5)", "peak_gbs": peak, "rows": rows},
                  fh, indent=1)
    md = [f"| dtype | N | R | chisq | pools | normals/s | frac | m1 | m2 | m3 | m4 | A^2 (2^32) | "
          f"A^2 sample gpu | A^2 sample oracle |", "|" + "---|" * 14]
    for r in rows:
        m = r["moments_full"]
        md.append(f"| {r['dtype']} | {r['N']} | {r['R']} | {'on' if r['chisq'] else 'off'} | "
                  f"{r['pools']} | {r['normals_per_s']:.3e} | {100 * r['hbm_store_frac']:.1f}% | "
                  f"{m['m1']:+.2e} | {m['m2']:.6f} | {m['m3']:+.2e} | {m['m4']:.5f} | "
                  f"{r['ad_full']:.3f} | {r['gpu_sample']['ad']:.4f} | "
                  f"{r['oracle_sample']['ad']:.4f} |")
    with open(os.path.splitext(args.out)[0] + "_table.md", "w") as fh:
        fh.write("\n".join(md) + "\n")


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(f"sweep done in {time.time() - t0:.1f}s")
