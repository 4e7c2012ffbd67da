#!/usr/bin/env python
"""Benchmark of the Wallace pool-regeneration hot path (BASELINE.json).

Workload at every N (one curve): the C4 shard ("c4w")
— n = 4, fp32, 4 x 1024 floats per pool in shared memory, 8 pools per SM x
148 SMs = 1184 pools per GPU, GPU g's pool c seeded UniformState(99 + g, c),
1 pass per output, 2^34 normals per GPU per step (weak scaling: N GPUs
generate N x 2^34; at N = 4 that is exactly C4's 2^36 split evenly), no
inter-GPU communication on the generation path.  At N = 1 that is C3's
shape with C4's seed; the N = 1 line also carries the exact C3 config (seed
2024), C4 at N = 1 (2^36 per step, strong-scaling form), C1, C2, C5's
smallest pools (fp32 / fp64 4x256, R = 1, one resident wave) and the GPU
at the reference's only mode (n = 2 fp64, "matched_reference"), all
measured in the same run.  `--config c1 | c2 | c3 | c4` makes one of them
the line's workload instead (c4: 2^36 split evenly, strong scaling).
Steps of 2^34 (≈11 ms) keep the timed region short enough that the board's
power cap does not engage (20 steps of C4's 2^36 ran at a median 1886 MHz
under sw_power_cap, 3 % slower).

One "step" = the step's normals through the C ABI (wrng_gpu_fill_f32/_f64,
device output).  `value` is device-timed whole-job normals/s (CUDA events on
the launch stream, max over ranks).  `e2e` is the same metric through the
same public call with a pinned HOST output buffer (generation overlapped
with D2H inside the library), on a bounded sample.

`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU) and fails when the node has fewer GPUs.

`--impl reference` times the reference's own CPU implementation (the
unmodified library built from /root/reference into oracle/_ref) on all host
cores instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "N(0,1) normals/sec per GPU and whole box; % of HBM-store roofline"
UNIT = "normals/s"
SMS = 148

CONFIGS = {
    # name: (n_arrays, dtype, pool_exponent, throwaway_f, pools, seed, total normals)
    "c1": dict(n_arrays=4, dtype="f64", pool_exponent=12, throwaway_f=1, pools=1,
               seed=12345, total=1 << 24, desc="C1 fp64 n=4 4x4096 pool, seed 12345, f=1"),
    "c2": dict(n_arrays=4, dtype="f64", pool_exponent=20, throwaway_f=2, pools=1, seed=7,
               total=1 << 30, desc="C2 fp64 n=4 one HBM-resident 4x2^20 pool, seed 7, f=2"),
    "c3": dict(n_arrays=4, dtype="f32", pool_exponent=10, throwaway_f=1, pools=8 * SMS,
               seed=2024, total=1 << 34,
               desc="C3 fp32 n=4 4x1024 smem pool per CTA, 8 CTAs/SM x 148, seed 2024, f=1"),
    "c4w": dict(n_arrays=4, dtype="f32", pool_exponent=10, throwaway_f=1, pools=8 * SMS,
                seed=99, total=1 << 34,
                desc="C4 shard: fp32 n=4 per-CTA 4x1024 pools, 1184 per GPU, GPU g seeded 99+g, "
                     "2^34 per GPU per step (weak scaling; N=4 is C4's 2^36)"),
    "c4": dict(n_arrays=4, dtype="f32", pool_exponent=10, throwaway_f=1, pools=8 * SMS,
               seed=99, total=1 << 36,
               desc="C4 fp32 n=4 per-CTA pools, GPU g seeded 99+g, 2^36 total split evenly"),
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def free_port() -> int:
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    return port


def self_launch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: one rank per GPU, launched the
    way the driver does it."""
    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} needs {n} CUDA devices; this node has {have}",
              file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation on all host cores
# ---------------------------------------------------------------------------
def run_reference(args, cfgname: str, world: int, rank: int):
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O

    c = CONFIGS[cfgname]
    threads = cpu_threads()
    if not O.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libwrng_ref.so not built"}))
        return 0
    # The reference implements n = 2 fp64 only: time it at
    # the workload's pool size and pass count, thread t = stream t.  The
    # workload stores every normal (bench.py's line: into HBM; its e2e leg:
    # into a host array), so the reference's threads fill their segments of
    # one host array much larger than the caches (value).  Its CLI bench loop
    # (refilling one 64Ki buffer that stays in cache, proj/tools/main.cpp:
    # 287-312) is timed too and reported as `bench_loop`.
    per_thread = int(args.ref_sample_per_thread)
    seg = min(per_thread, 1 << 24)  # 128 MiB of fp64 per thread
    reps = max(1, per_thread // seg)
    per_thread = seg * reps
    p, f = c["pool_exponent"], c["throwaway_f"]
    seed = c["seed"]
    arr = np.zeros(threads * seg, dtype=np.float64)  # touched before timing
    for _ in range(args.warmup):
        O.ref_bench_array(p, f, 0, seed, 0, threads, seg, arr)
    times = []
    for _ in range(args.steps):
        times.append(sum(O.ref_bench_array(p, f, 0, seed, 0, threads, seg, arr)
                         for _ in range(reps)))
    loop_times = [O.ref_bench_threads(p, f, 0, seed, 0, threads, per_thread)
                  for _ in range(max(1, min(args.steps, 3)))]
    total = per_thread * threads
    ms = 1e3 * statistics.mean(times)
    value = total / (ms / 1e3)
    loop_value = total / statistics.mean(loop_times)
    sample = (f"reference WallaceState n=2 fp64 (the only mode it implements), "
              f"N=2^{p}, f={f}, chisq, seed {seed}, {threads} threads, thread t = stream t "
              f"filling its {seg}-value segment of one {threads * seg * 8 >> 20} MiB host "
              f"array {reps}x per step with fill(span) in 64Ki chunks")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if cfgname == "c4" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator state)",
        "config": {"workload": c["desc"], "reference_mode": "n=2 fp64", "pool_exponent": p,
                   "throwaway_f": f, "host_threads": threads},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "bench_loop": {"value": loop_value, "unit": UNIT,
                       "sample": (f"the reference CLI's bench loop: {threads} threads x "
                                  f"{per_thread} values, each refilling one 64Ki buffer "
                                  f"(cache-resident; proj/tools/main.cpp:287-312)")},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def cpu_baseline_port(c, seconds_target: float):
    """The oracle restatement (n = 4 / fp32, same workload semantics) on all
    host cores, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes as C

    import oracle as O

    threads = cpu_threads()
    cfg = O.OrConfig(c["n_arrays"], O.F64 if c["dtype"] == "f64" else O.F32, c["pool_exponent"],
                     c["throwaway_f"], O.CHISQ, 0, 64, c["seed"], 0)
    lib = O.oracle_lib()
    # calibrate: 2^20 values per thread
    probe = 1 << 20
    t = lib.or_bench_threads(C.byref(cfg), threads, probe, 1 << 16)
    per_thread = int(min(1 << 30, max(probe, probe * seconds_target / max(t, 1e-6))))
    t = lib.or_bench_threads(C.byref(cfg), threads, per_thread, 1 << 16)
    value = per_thread * threads / t
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"oracle/wallace_oracle.c (n={c['n_arrays']} {c['dtype']} restatement, "
                       f"not reference code), N=2^{c['pool_exponent']}, f={c['throwaway_f']}, "
                       f"{threads} threads x {per_thread} values, pools = streams 0..{threads - 1}, "
                       f"{t:.2f} s wall")}


def roofline_of(gen, per_gpu: int, esize: int, nslabs: int, step_ms: list, cfgname: str):
    """Roofline of the dominant kernel: one fill kernel per output slab
    (smem engine), or the whole step (HBM engine: persistent runs + audits);
    algorithmic bytes = stored output bytes."""
    peak, peak_src = peaks()
    if gen.engine() == "smem":
        kernel_ms = statistics.mean(step_ms) / nslabs
        algo_bytes = per_gpu * esize / nslabs
    else:
        kernel_ms = statistics.mean(step_ms)
        algo_bytes = per_gpu * esize
    achieved = algo_bytes / (kernel_ms / 1e3) / 1e9
    # DRAM traffic per launch: dram__bytes_read + dram__bytes_write of the
    # committed `ncu --set full` capture (profiles/traffic.json), expressed
    # per output byte and scaled to this launch.
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                tj = json.load(fh).get("c3" if cfgname in ("c4", "c4w") else cfgname)
            if tj:
                traffic = tj["dram_bytes_per_output_byte"] * algo_bytes
                traffic_src = tj["source"]
        except Exception:
            traffic = None
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peak_src, "algorithmic_bytes_per_launch": algo_bytes,
            "kernel_ms": kernel_ms}


def make_gen(c: dict, seed: int, local: int, **over):
    from paper_1004_3114_b200 import WallaceConfig, WallaceState

    kw = dict(pool_exponent=c["pool_exponent"], throwaway_f=c["throwaway_f"], seed=seed,
              stream_id=0, n_arrays=c["n_arrays"], dtype=c["dtype"], pools=c["pools"],
              device=local)
    kw.update(over)
    return WallaceState(WallaceConfig(**kw))


MAX_SLAB_GIB = float(os.environ.get("WRNG_BENCH_MAX_SLAB_GIB", "160"))


def timed_device_fills(gen, per_gpu: int, dtype: str, steps: int, warmup: int, dev,
                       barrier=None, on_start=None):
    """`steps` timed steps of per_gpu normals into a device buffer (when the
    step does not fit HBM: the largest halving of it that fits, at most
    MAX_SLAB_GIB, re-used within the step — every value is still stored; C4
    at N = 1 is 2 slabs of 128 GiB, measured 1.7 % faster than 4 of 64).
    Returns (step_ms list, elapsed_ms, launches, nslabs)."""
    import torch

    out_dtype = torch.float32 if dtype == "f32" else torch.float64
    esize = 4 if dtype == "f32" else 8
    free, _ = torch.cuda.mem_get_info(dev)
    slab = per_gpu
    while slab * esize > min(free - (8 << 30), int(MAX_SLAB_GIB * (1 << 30))):
        slab = (slab + 1) // 2
    nslabs = math.ceil(per_gpu / slab)
    out = torch.empty(slab, dtype=out_dtype, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        left = per_gpu
        while left > 0:
            n = min(slab, left)
            gen.fill(out[:n], stream=stream)
            left -= n

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    gen.synchronize()
    if on_start:
        on_start()
    if barrier:
        barrier()
    torch.cuda.synchronize(dev)
    launches0 = gen.kernel_launches()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for k in range(steps):
        step()
        ev[k + 1].record(stream)
    torch.cuda.synchronize(dev)
    launches = gen.kernel_launches() - launches0
    if barrier:
        barrier()
    gen.synchronize()  # surfaces any device-raised error
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    elapsed_ms = ev[0].elapsed_time(ev[-1])
    del out
    return step_ms, elapsed_ms, launches, nslabs


def host_e2e(gen, n: int, dtype: str, steps: int):
    """The public call with pinned HOST output: n normals per step."""
    import torch

    host = torch.empty(n, dtype=torch.float32 if dtype == "f32" else torch.float64,
                       pin_memory=True)
    hv = host.numpy()
    gen.fill(hv)  # warm (allocates staging)
    t0 = time.perf_counter()
    for _ in range(steps):
        gen.fill(hv)
    dt = time.perf_counter() - t0
    del hv, host
    return dt


def sub_bench(name: str, c: dict, seed: int, per_gpu: int, steps: int, warmup: int, local: int,
              dev, e2e_n: int = 0, e2e_steps: int = 2, **over):
    """A secondary config measured in the same run (N = 1 line)."""
    import torch

    gen = make_gen(c, seed, local, **over)
    esize = 4 if c["dtype"] == "f32" else 8
    step_ms, elapsed, launches, nslabs = timed_device_fills(gen, per_gpu, c["dtype"], steps,
                                                            warmup, dev)
    ms = elapsed / steps
    r = roofline_of(gen, per_gpu, esize, nslabs, step_ms, name)
    d = {"workload": c["desc"], "value": per_gpu / (ms / 1e3), "unit": UNIT,
         "ms_per_step": ms, "steps": steps, "warmup": warmup, "normals_per_step": per_gpu,
         "dtype": c["dtype"], "engine": gen.engine(), "gpu_launches": launches,
         "roofline_frac": r["frac"], "achieved_gbs": r["achieved"]}
    if e2e_n:
        n = min(e2e_n, per_gpu)
        dt = host_e2e(gen, n, c["dtype"], e2e_steps)
        d["e2e"] = {"value": n * e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": n * esize,
                    "sample": f"{n} normals per step into pinned host memory"}
    del gen
    torch.cuda.empty_cache()
    return d


MATCHED = dict(n_arrays=2, dtype="f64", pool_exponent=10, throwaway_f=1, pools=8 * SMS,
               seed=2024, total=1 << 32,
               desc="the reference's only mode: n=2 fp64 N=2^10 f=1, 1184 pools (seed 2024), "
                    "2^32 normals per step")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--total", type=int, default=None, help="override normals per step")
    ap.add_argument("--e2e-sample", type=int, default=1 << 30)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=2.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the C1/C2/C3/matched-reference sub-results of the N = 1 line")
    ap.add_argument("--ref-sample-per-thread", type=float, default=float(1 << 26))
    args = ap.parse_args()

    world, rank, local = dist_setup()
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1 and args.impl == "ours":
        return self_launch(args.gpus)
    if args.impl == "ours" and args.gpus is not None and args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    cfgname = args.config or "c4w"
    if args.impl == "reference":
        return run_reference(args, cfgname, max(world, args.gpus or 1), rank)

    import torch

    if torch.cuda.device_count() <= local:
        print(f"bench.py: rank {rank} needs cuda:{local}; {torch.cuda.device_count()} visible",
              file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    from paper_1004_3114_b200.sharding import shard

    c = dict(CONFIGS[cfgname])
    total = args.total or c["total"]
    if cfgname == "c4":
        # 2^36 normals in total split evenly; GPU g seeded 99 + g (strong scaling)
        sh = shard(total, world, rank, c["seed"])
        seed, per_gpu = sh.seed, sh.count
        scaling = "strong"
    elif cfgname == "c4w":
        # C4's seeding, a fixed 2^34 per GPU (weak scaling)
        seed, per_gpu = c["seed"] + rank, total
        scaling = "weak"
    else:
        # c1..c3 at N > 1: every GPU runs the whole config on its own seed
        seed = c["seed"] + (rank if world > 1 else 0)
        per_gpu = total
        scaling = "weak"
    esize = 4 if c["dtype"] == "f32" else 8
    gen = make_gen(c, seed, local)

    # ---- timed region -----------------------------------------------------
    clocks = ClockSampler(local)
    barrier = (lambda: torch.distributed.barrier()) if world > 1 else None
    step_ms, elapsed_ms, launches, nslabs = timed_device_fills(
        gen, per_gpu, c["dtype"], args.steps, args.warmup, dev, barrier=barrier,
        on_start=lambda: (clocks.start(), time.sleep(0.3)))
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    total_normals = total if cfgname == "c4" else per_gpu * world
    value = total_normals / (ms_per_step / 1e3)
    roofline = roofline_of(gen, per_gpu, esize, nslabs, step_ms, cfgname)

    # ---- e2e: same public call, HOST output (pinned), bounded sample -------
    # every rank runs it; at N > 1 the slowest rank's time counts
    n_e2e = min(args.e2e_sample if world == 1 else min(args.e2e_sample, 1 << 28), per_gpu)
    dt = host_e2e(gen, n_e2e, c["dtype"], args.e2e_steps)
    e2e_value = n_e2e * args.e2e_steps / dt
    if world > 1:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_value = n_e2e * args.e2e_steps * world / float(t.item())
    e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 0,
           "d2h_bytes_per_step": n_e2e * esize,
           "sample": f"{n_e2e} normals per rank per step into pinned host memory via "
                     f"wrng_gpu_fill_{c['dtype']}(out_is_device=0); generator state is "
                     f"device-resident, so no host->device input bytes; PCIe-bound"}
    engine = gen.engine()
    del gen
    torch.cuda.empty_cache()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": c["dtype"],
        "data": "synthetic (seeded generator pools; no dataset)",
        "config": {"workload": c["desc"], "normals_per_step": total_normals,
                   "normals_per_gpu": per_gpu, "pools_per_gpu": c["pools"],
                   "n_arrays": c["n_arrays"], "pool_exponent": c["pool_exponent"],
                   "throwaway_f": c["throwaway_f"], "seed_base": c["seed"],
                   "engine": engine, "output_slabs_per_step": nslabs,
                   "l2": "output per step >> 126 MB L2 (no flush needed)",
                   "parallelism": f"independent pools, {world} GPU(s), no collective"},
        "per_gpu_value": value / world,
        "roofline": roofline,
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_extras:
        # secondary configs, measured in the same run on the same box
        line["c3"] = sub_bench("c3", CONFIGS["c3"], 2024, 1 << 34, 3, 2, local, dev)
        line["c4_strong"] = sub_bench("c4", CONFIGS["c4"], 99, 1 << 36, 3, 1, local, dev)
        line["c2"] = sub_bench("c2", CONFIGS["c2"], 7, 1 << 30, 3, 1, local, dev,
                               e2e_n=1 << 27)
        line["c1"] = sub_bench("c1", CONFIGS["c1"], 12345, 1 << 24, 3, 1, local, dev)
        # C5's smallest pools (configs[4], R = 1): the group engine, several
        # pools per warp, one resident wave
        from paper_1004_3114_b200 import WallaceConfig, resident_pools
        for nm, dt in (("c5_f32_4x256", "f32"), ("c5_f64_4x256", "f64")):
            c5 = dict(n_arrays=4, dtype=dt, pool_exponent=8, throwaway_f=1, seed=2024,
                      total=1 << 32, pools=1)
            c5["pools"] = resident_pools(WallaceConfig(
                pool_exponent=8, throwaway_f=1, n_arrays=4, dtype=dt, device=local))
            c5["desc"] = (f"C5 {dt} n=4 4x256 pools, R=1, chi rescale on, {c5['pools']} pools "
                          f"(one resident wave), seed 2024, 2^32 normals per step")
            line[nm] = sub_bench(nm, c5, 2024, 1 << 32, 3, 2, local, dev)
        line["matched_reference"] = sub_bench(
            "matched", MATCHED, 2024, MATCHED["total"], 3, 2, local, dev, e2e_n=1 << 28)
        line["matched_reference"]["note"] = (
            "GPU through the same C ABI at the reference arm's mode (n=2 fp64); its e2e "
            "(fp64 into pinned host memory) is PCIe-bound, compare it with the --impl "
            "reference line")
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_port(c, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
