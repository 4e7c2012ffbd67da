#!/usr/bin/env python
"""Restates the paper's speed-up claim on B200 (
SURVEY.md §6, §8(f)4): Wallace vs Box-Muller vs polar, on the GPU and with
the unmodified reference on the host cores.

GPU: 2^32 normals per method into one fp32 device array (16 GiB, far larger
than L2), 1184 streams (8 per SM), device-timed with CUDA events, best of 3
after a warm-up.  Wallace at f = 1..4 (n = 4, N = 1024: the C3 shape) also
gives the cost model t(f) = a f + b the paper states as (6.8 f + 3.2) ns on
the VP2200 and the reference's acceptance gate
t(3)/t(1) in [1.5, 4.5] (acceptance.cpp:222-230).

CPU: the reference library (oracle/_ref), all host threads, thread t =
stream t, 64Ki-value fill calls (tools/main.cpp:287-312), a bounded sample.

Usage: python scripts/methods_bench.py [--out profiles/round1/methods.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import torch

    import oracle as O
    from paper_1004_3114_b200 import WallaceConfig, WallaceState, method_fill

    ap = argparse.ArgumentParser()
    ap.add_argument("--total", type=int, default=1 << 32)
    ap.add_argument("--cpu-per-thread", type=int, default=1 << 24)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round1", "methods.json"))
    args = ap.parse_args()
    n = args.total
    pools = 8 * 148
    buf = torch.empty(n, dtype=torch.float32, device="cuda")

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    rows = []
    for f in (1, 2, 3, 4):
        g = WallaceState(WallaceConfig(pool_exponent=10, throwaway_f=f, seed=2024, n_arrays=4,
                                       dtype="f32", pools=pools))
        ms = timed(lambda: g.fill(buf))
        rows.append({"where": "gpu", "method": "wallace", "f": f, "math": "f32 (n=4 pools)",
                     "ms": ms, "normals_per_s": n / (ms / 1e3), "ns_per_normal_per_stream":
                     ms * 1e6 / (n / pools)})
        del g
    for method in ("boxmuller", "polar"):
        for f64 in (True, False):
            ms = timed(lambda: method_fill(method, buf, 2024, 0, pools, f64_math=f64))
            rows.append({"where": "gpu", "method": method, "math": "f64" if f64 else "f32",
                         "ms": ms, "normals_per_s": n / (ms / 1e3),
                         "ns_per_normal_per_stream": ms * 1e6 / (n / pools)})
    torch.cuda.synchronize()
    del buf

    threads = os.cpu_count() or 1
    if O.ref_available():
        per = args.cpu_per_thread
        for f in (1, 3):
            O.ref_bench_threads(10, f, 0, 1, 0, threads, per // 8)
            s = O.ref_bench_threads(10, f, 0, 1, 0, threads, per)
            rows.append({"where": "cpu", "method": "wallace", "f": f, "math": "f64 (n=2)",
                         "threads": threads, "s": s, "normals_per_s": threads * per / s})
        for method in ("boxmuller", "polar"):
            O.ref_bench_methods(method, threads, per // 8)
            s = O.ref_bench_methods(method, threads, per)
            rows.append({"where": "cpu", "method": method, "math": "f64", "threads": threads,
                         "s": s, "normals_per_s": threads * per / s})

    def rate(where, method, **kw):
        for r in rows:
            if r["where"] == where and r["method"] == method and all(
                    r.get(k) == v for k, v in kw.items()):
                return r["normals_per_s"]
        return None

    # cost model t(f) = a f + b per stream (least squares over f = 1..4)
    fs = [r["f"] for r in rows if r["where"] == "gpu" and r["method"] == "wallace"]
    ts = [r["ns_per_normal_per_stream"] for r in rows
          if r["where"] == "gpu" and r["method"] == "wallace"]
    mf, mt = sum(fs) / len(fs), sum(ts) / len(ts)
    a = sum((x - mf) * (y - mt) for x, y in zip(fs, ts)) / sum((x - mf) ** 2 for x in fs)
    b = mt - a * mf
    summary = {
        "gpu_speedup_wallace_f3_over_polar_f64": rate("gpu", "wallace", f=3) / rate(
            "gpu", "polar", math="f64"),
        "gpu_speedup_wallace_f3_over_polar_f32": rate("gpu", "wallace", f=3) / rate(
            "gpu", "polar", math="f32"),
        "gpu_speedup_wallace_f1_over_boxmuller_f32": rate("gpu", "wallace", f=1) / rate(
            "gpu", "boxmuller", math="f32"),
        "gpu_cost_model_ns_per_normal_per_stream": {"a": a, "b": b},
        "gpu_t3_over_t1": ts[2] / ts[0],
        "paper": "VP2200/10: (6.8 f + 3.2) ns; f = 3 is 3.2x faster than polar (PAPER.md:482-489)",
    }
    if rate("cpu", "polar"):
        summary["cpu_speedup_wallace_f3_over_polar"] = rate("cpu", "wallace", f=3) / rate(
            "cpu", "polar")
        summary["gpu_over_cpu_wallace_f3"] = rate("gpu", "wallace", f=3) / rate(
            "cpu", "wallace", f=3)
    out = {"normals_gpu": n, "streams_gpu": pools, "rows": rows, "summary": summary}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    for r in rows:
        print(json.dumps(r))
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
