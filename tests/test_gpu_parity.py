"""GPU parity tests: the sm_100a path through the C ABI vs the CPU oracle
and the reference library.

Bars (BASELINE.json north_star):
  * uniform words, index/offset/stride selection: bit-exact;
  * fp64 pool values: bit-exact when the initial pool comes from the host
    (glibc) Box-Muller (init_on_host=True, or an imported reference state);
    with the device Box-Muller init (CUDA libm, a few ulp from glibc):
    |gpu - ref| <= 1e-12 * max(1, |ref|)   (TOL64 below);
  * fp32 outputs: bit-exact with host init; otherwise relative 1e-6 (TOL32);
  * moments m1..m4 and Anderson-Darling A^2 of the GPU stream equal the
    oracle's on the same parameters (they are computed from identical
    values when the streams are bit-exact).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-6
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def W():
    import paper_1004_3114_b200 as W

    return W


def gpu_state(W, **kw):
    return W.WallaceState(W.WallaceConfig(**kw))


def oracle_state(**kw):
    m = dict(kw)
    m.pop("init_on_host", None)
    force = m.pop("force_hbm", None)  # noqa: F841  (engine choice is GPU-only)
    dt = O.F64 if m.pop("dtype", "f64") == "f64" else O.F32
    return O.OracleState(pool_exponent=m.pop("pool_exponent", 10), throwaway_f=m.pop("throwaway_f", 3),
                         scale_mode=m.pop("scale_mode", 0), restart_interval=m.pop("restart_interval_passes", 0),
                         drift_period=m.pop("drift_check_period", 64), seed=m.pop("seed", 0),
                         stream=m.pop("stream_id", 0), n_arrays=m.pop("n_arrays", 2), dtype=dt)


def assert_bits(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype
    if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
        i = int(np.argmax(a != b))
        raise AssertionError(f"first difference at {i}: {a[i]!r} != {b[i]!r}")


def assert_close(a, b, tol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert float(err.max()) <= tol, f"max normwise error {err.max():.3e} > {tol}"


# ---------------------------------------------------------------------------
# uniform generator (uniform.cpp:13-51; test_uniform.cpp)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", load("golden_ref.json")["uniform"],
                         ids=lambda c: f"{c['seed']}-{c['stream']}")
def test_device_lfg_words_match_reference_golden(W, case):
    words = W.lfg_words(int(case["seed"]), int(case["stream"]), 1, len(case["words"]))[0]
    assert [f"{int(w):016x}" for w in words] == case["words"]


def test_device_lfg_streams_many_pools(W):
    pools, count = 37, 3000
    words = W.lfg_words(2024, 5, pools, count)
    for p in (0, 1, 17, 36):
        u = O.OracleUniform(2024, 5 + p)
        assert_bits(words[p], np.array([u.next_word() for _ in range(count)], dtype=np.uint64))
    assert len({int(words[p, 0]) for p in range(pools)}) == pools


@pytest.mark.parametrize("n_arrays,dtype", [(2, "f64"), (4, "f32")])
def test_uniform_state_after_create_and_fill(W, n_arrays, dtype):
    kw = dict(pool_exponent=10, throwaway_f=2, seed=77, n_arrays=n_arrays, dtype=dtype)
    g = gpu_state(W, **kw)
    o = oracle_state(**kw)
    for cnt in (0, 5, 5000):
        g.fill(cnt)
        o.fill(cnt)
        us = g.uniform_state()
        t, r, s, d = o.uniform()
        assert_bits(us.lag_table, t)
        assert (us.cursor_r, us.cursor_s, us.draws) == (r, s, d)


# ---------------------------------------------------------------------------
# initial pool (wallace.cpp:158-167)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n_arrays,dtype,p", [(2, "f64", 12), (4, "f64", 10), (4, "f32", 10),
                                              (2, "f32", 8), (4, "f64", 20)])
def test_initial_pool(W, n_arrays, dtype, p):
    kw = dict(pool_exponent=p, seed=12345, n_arrays=n_arrays, dtype=dtype)
    o = oracle_state(**kw)
    vo, to, wo = o.pool()
    host = gpu_state(W, init_on_host=True, **kw).active_pool()
    assert_bits(host.arrays.reshape(-1), vo)
    assert host.tracked_sumsq == to and host.withheld == wo
    dev = gpu_state(W, init_on_host=False, **kw).active_pool()
    tol = TOL64 if dtype == "f64" else TOL32
    # element-wise RELATIVE bar: the init values are single libm evaluations
    # (log, sqrt, cos, sin), a few ulp apart between CUDA and glibc
    a = dev.arrays.reshape(-1)
    rel = np.abs(a - vo) / np.abs(vo)
    assert float(rel.max()) <= tol, f"max relative error {rel.max():.3e}"
    assert_close(a, vo, tol)
    assert abs(dev.tracked_sumsq / to - 1) < 1e-12
    assert abs(dev.withheld - wo) < 1e-12


# ---------------------------------------------------------------------------
# the reference's own n = 2 fp64 generator, pinned by golden_ref.json
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("engine", ["smem", "hbm"])
@pytest.mark.parametrize("case", load("golden_ref.json")["cases"], ids=lambda c: c["name"])
def test_n2_stream_matches_reference_golden(W, case, engine):
    g = gpu_state(W, pool_exponent=case["pool_exponent"], throwaway_f=case["throwaway_f"],
                  scale_mode=case["scale_mode"], seed=case["seed"], stream_id=case["stream"],
                  init_on_host=True, force_hbm=engine == "hbm")
    v = g.fill(case["count"])
    assert [float(x).hex() for x in v[:16]] == case["fill_head_hex"]
    assert sha(v) == case["fill_sha256"]
    c = case["counters"]
    assert (g.pass_count(), g.numbers_emitted(), g.avail()) == (
        c["pass_count"], c["numbers_emitted"], c["avail"])
    pool = g.active_pool()
    assert sha(pool.arrays.reshape(-1)) == case["final_pool_sha256"]
    assert pool.tracked_sumsq.hex() == case["final_tracked_hex"]
    assert pool.withheld.hex() == case["final_withheld_hex"]
    assert hashlib.sha256(g.save_state()).hexdigest() == case["state_sha256"]


@pytest.mark.parametrize("case", load("golden_ref.json")["cases"][:4], ids=lambda c: c["name"])
def test_n2_params_match_reference_golden(W, case):
    g = gpu_state(W, pool_exponent=case["pool_exponent"], throwaway_f=case["throwaway_f"],
                  scale_mode=case["scale_mode"], seed=case["seed"], stream_id=case["stream"],
                  init_on_host=True)
    for want in case["params"]:
        p = g.advance_pass()
        assert [p.alpha, p.beta] == want["stride"] and [p.gamma, p.delta] == want["offset"]
        assert p.rot.c.hex() == want["c_hex"] and p.rot.s.hex() == want["s_hex"]
        assert p.scale.hex() == want["scale_hex"] and p.target_sumsq.hex() == want["target_hex"]


@pytest.mark.parametrize("case", load("golden_n4.json")["cases"], ids=lambda c: c["name"])
@pytest.mark.parametrize("engine", ["smem", "hbm"])
def test_n4_stream_matches_oracle_golden(W, case, engine):
    g = gpu_state(W, pool_exponent=case["pool_exponent"], throwaway_f=case["throwaway_f"],
                  scale_mode=case["scale_mode"], seed=case["seed"], stream_id=case["stream"],
                  n_arrays=case["n_arrays"], dtype=case["dtype"], init_on_host=True,
                  force_hbm=engine == "hbm")
    v = g.fill(case["count"])
    assert [float(x).hex() for x in v[:16]] == case["fill_head_hex"]
    assert sha(v) == case["fill_sha256"]
    pool = g.active_pool()
    assert sha(pool.arrays.reshape(-1)) == case["final_pool_sha256"]
    assert pool.tracked_sumsq.hex() == case["final_tracked_hex"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("p,f,mode,seed,restart", [
    (8, 1, 0, 1, 0), (9, 3, 1, 2, 0), (10, 2, 0, 3, 0), (12, 1, 0, 12345, 0),
    (10, 3, 0, 1, 100), (9, 1, 0, 4, 7), (11, 2, 1, 5, 5)])
@pytest.mark.parametrize("engine", ["smem", "hbm"])
def test_n2_against_live_reference_library(W, p, f, mode, seed, restart, engine):
    r = O.RefState(pool_exponent=p, throwaway_f=f, scale_mode=mode, seed=seed,
                   restart_interval=restart)
    g = gpu_state(W, pool_exponent=p, throwaway_f=f, scale_mode=mode, seed=seed,
                  restart_interval_passes=restart, init_on_host=True, force_hbm=engine == "hbm")
    for cnt in (0, 1, 2 << p, 3 * (2 << p) + 5, 70 * (2 << p) + 3):
        assert_bits(g.fill(cnt), r.fill(cnt))
        rc = r.counters()
        assert (g.pass_count(), g.numbers_emitted(), g.avail()) == (
            rc["pass_count"], rc["numbers_emitted"], rc["avail"])
    for _ in range(5):
        a, b = g.advance_pass(), r.advance_pass()
        assert (a.alpha, a.beta, a.gamma, a.delta) == tuple(b.stride[:2]) + tuple(b.offset[:2])
        assert a.scale == b.scale and a.target_sumsq == b.target and a.rot.c == b.c


# ---------------------------------------------------------------------------
# device-initialised pools: tolerance bars
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n_arrays,dtype,p,f", [(2, "f64", 12, 1), (4, "f64", 12, 1),
                                                (4, "f32", 10, 1), (4, "f64", 8, 3)])
def test_device_init_stream_within_tolerance(W, n_arrays, dtype, p, f):
    """Device (CUDA libm) init: pool values start a few ulp off glibc's, and
    passes mix them linearly, so a value near zero can carry an absolute
    error of ~ulp(max |pool|): the bar is normwise, |d| <= tol * max(1, |ref|),
    the 1e-12 (fp64) / 1e-6 (fp32) of BASELINE's north star."""
    kw = dict(pool_exponent=p, throwaway_f=f, seed=12345, n_arrays=n_arrays, dtype=dtype)
    g, o = gpu_state(W, init_on_host=False, **kw), oracle_state(**kw)
    cnt = 70 * (n_arrays << p)  # crosses the drift audit at pass 64
    tol = TOL64 if dtype == "f64" else TOL32
    assert_close(g.fill(cnt), o.fill(cnt), tol)
    # parameters never depend on pool values: index streams stay bit-exact
    a, b = g.advance_pass(), o.advance_pass()
    assert a.strides == list(b.stride)[:n_arrays] and a.offsets == list(b.offset)[:n_arrays]
    assert a.variant == b.variant


# ---------------------------------------------------------------------------
# banks of independent pools (C3 / C4 layout)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("pools,count", [(16, 16 * 3 * 4095 + 5), (37, 1000), (5, 3)])
def test_bank_fill_matches_oracle_bank(W, pools, count):
    g = gpu_state(W, pool_exponent=10, throwaway_f=1, seed=2024, n_arrays=4, dtype="f32",
                  pools=pools, init_on_host=True)
    out = g.fill(count)
    ref = O.bank_fill(count, pools, seed=2024, pool_exponent=10, throwaway_f=1, n_arrays=4,
                      dtype=O.F32)
    assert_bits(out, ref)


def test_bank_fill_c3_shape_subset(W):
    """All 1184 pools of C3, a short segment each; pools spot-checked."""
    pools = 8 * 148
    g = gpu_state(W, pool_exponent=10, throwaway_f=1, seed=2024, n_arrays=4, dtype="f32",
                  pools=pools, init_on_host=True)
    per = 2 * 4095 + 3
    out = g.fill(pools * per + 768)  # first 768 pools get one more value, like 2^34
    base = 0
    for p in range(pools):
        ln = per + (1 if p < 768 else 0)
        if p in (0, 1, 767, 768, 1183):
            o = O.OracleState(pool_exponent=10, throwaway_f=1, seed=2024, stream=p, n_arrays=4,
                              dtype=O.F32)
            assert_bits(out[base:base + ln], o.fill(ln))
        base += ln
    assert base == out.size


def test_c3_full_size_segment_ends_bit_exact(W):
    """The whole C3 step (2^34 fp32 normals, 1184 pools, ~3544 refills and
    55 drift audits per pool, bulk-copy emission) into one device array:
    the first and last 4096 values of several pool segments equal the
    oracle's stream for that pool, bit for bit; the device moments of the
    full array are within the reference's CLT-style bounds."""
    import torch

    pools = 8 * 148
    total = 1 << 34
    free, _ = torch.cuda.mem_get_info()
    if free < total * 4 + (12 << 30):
        pytest.skip("needs 76 GiB of free device memory")
    g = gpu_state(W, pool_exponent=10, throwaway_f=1, seed=2024, n_arrays=4, dtype="f32",
                  pools=pools, init_on_host=True)
    out = torch.empty(total, dtype=torch.float32, device="cuda")
    g.fill(out)
    torch.cuda.synchronize()
    per, extra = divmod(total, pools)
    for p in (0, 767, 768, 1183):
        start = p * per + min(p, extra)
        ln = per + (1 if p < extra else 0)
        ref = O.OracleState(pool_exponent=10, throwaway_f=1, seed=2024, stream=p, n_arrays=4,
                            dtype=O.F32).fill(ln)
        assert_bits(out[start:start + 4096].cpu().numpy(), ref[:4096])
        assert_bits(out[start + ln - 4096:start + ln].cpu().numpy(), ref[-4096:])
    # moments of all 2^34 values (fp64 sums on the device, in slabs)
    s1 = s2 = s4 = 0.0
    for k in range(0, total, 1 << 28):  # 2 GiB fp64 temporaries per slab
        x = out[k:k + (1 << 28)].double()
        x2 = x * x
        s1 += float(x.sum())
        s2 += float(x2.sum())
        s4 += float((x2 * x2).sum())
        del x, x2
    n = float(total)
    m1, m2, m4 = s1 / n, s2 / n, s4 / n
    # z-scores with variances 1, 2, 96 (stats.cpp:89-108); a generous bound
    assert abs(m1) * n ** 0.5 < 6 and abs(m2 - 1) * (n / 2) ** 0.5 < 6 * 10
    assert abs(m4 - 3) < 5e-3


def test_bank_calls_continue_streams(W):
    pools = 7
    g = gpu_state(W, pool_exponent=8, throwaway_f=2, seed=9, n_arrays=4, dtype="f32", pools=pools,
                  init_on_host=True)
    a = g.fill(pools * 1500)
    b = g.fill(pools * 3001)
    for p in (0, 3, 6):
        o = O.OracleState(pool_exponent=8, throwaway_f=2, seed=9, stream=p, n_arrays=4,
                          dtype=O.F32)
        assert_bits(a[p * 1500:(p + 1) * 1500], o.fill(1500))
        assert_bits(b[p * 3001:(p + 1) * 3001], o.fill(3001))


def test_device_tensor_fill_equals_host_fill(W):
    import torch

    kw = dict(pool_exponent=10, throwaway_f=1, seed=4, n_arrays=4, dtype="f32", pools=11)
    g1, g2 = gpu_state(W, **kw), gpu_state(W, **kw)
    t = torch.empty(11 * 9000 + 4, dtype=torch.float32, device="cuda")
    g1.fill(t)
    torch.cuda.synchronize()
    h = g2.fill(t.numel())
    assert_bits(t.cpu().numpy(), h)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g1.fill(t, stream=s)
    s.synchronize()
    assert_bits(t.cpu().numpy(), g2.fill(t.numel()))


# Bulk-copy emission (smem engine, unit output): the pool is kept rotated in
# shared memory to match the output's 16-byte phase; every phase, ragged
# ends, leftovers across calls, drift audits and restarts on a rotated pool.
@pytest.mark.parametrize("dt,n,p", [("f32", 4, 10), ("f32", 2, 8), ("f64", 2, 10),
                                    ("f64", 4, 12), ("f32", 4, 13), ("f64", 4, 8)])
def test_bulk_emission_every_output_phase(W, dt, n, p):
    import torch

    pools = 3
    tdt = torch.float32 if dt == "f32" else torch.float64
    odt = O.F32 if dt == "f32" else O.F64
    cap = n * (1 << p) - 1
    counts = (pools * (3 * cap + 7), pools * (cap + 1) + 2)  # full refills, tails, leftovers
    vec = 4 if dt == "f32" else 2
    for off in range(vec):
        # (restarts re-initialise with the device Box-Muller, which is only
        # tolerance-equal to glibc: covered bulk-vs-warp-store below)
        kw = dict(pool_exponent=p, throwaway_f=1, seed=5 + off, n_arrays=n, dtype=dt, pools=pools,
                  init_on_host=True, drift_check_period=2)
        g = gpu_state(W, **kw)
        orc = [O.OracleState(pool_exponent=p, throwaway_f=1, seed=5 + off, stream=q, n_arrays=n,
                             dtype=odt, drift_period=2) for q in range(pools)]
        for c in counts:
            buf = torch.full((c + vec,), 7.0, dtype=tdt, device="cuda")
            g.fill(buf[off:off + c])
            torch.cuda.synchronize()
            got = buf.cpu().numpy()
            assert np.all(got[:off] == 7.0) and np.all(got[off + c:] == 7.0), "wrote outside"
            got = got[off:off + c]
            per, extra = divmod(c, pools)
            base = 0
            for q in range(pools):
                ln = per + (1 if q < extra else 0)
                assert_bits(got[base:base + ln], orc[q].fill(ln))
                base += ln
        # the pool written back after rotated emission is in natural order
        for q in range(pools):
            gp = g.active_pool(q)
            ov, ot, ow = orc[q].pool()
            assert_bits(gp.arrays.reshape(-1), ov)
            assert (gp.tracked_sumsq, gp.withheld) == (ot, ow)


@pytest.mark.parametrize("dt,n", [("f32", 4), ("f64", 2)])
def test_bulk_and_warp_store_emission_agree(W, dt, n):
    """WRNG_GPU_NO_BULK switches full-refill emission to warp stores; both
    paths must produce the same bits, through drift audits and restarts on a
    rotated pool (subprocess: the switch is read when the library loads)."""
    import subprocess
    import sys

    tdt = "torch.float32" if dt == "f32" else "torch.float64"
    code = (
        "import numpy as np, torch, hashlib\n"
        "import paper_1004_3114_b200 as W\n"
        f"g = W.WallaceState(W.WallaceConfig(pool_exponent=10, throwaway_f=1, seed=3, n_arrays={n},"
        f" dtype='{dt}', pools=37, drift_check_period=2, restart_interval_passes=3))\n"
        f"t = torch.empty(37 * 20000 + 11, dtype={tdt}, device='cuda')\n"
        "h = hashlib.sha256()\n"
        "for a, b in ((1, 37 * 9000 + 2), (37 * 9000 + 2, 37 * 20000 + 11)):\n"
        "    g.fill(t[a:b]); torch.cuda.synchronize(); h.update(t[a:b].cpu().numpy().tobytes())\n"
        "p = g.active_pool(5)\n"
        "h.update(p.arrays.tobytes()); h.update(np.array([p.tracked_sumsq, p.withheld]).tobytes())\n"
        "print(h.hexdigest())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"WRNG_GPU_NO_BULK": "1"}):
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=e, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]


@pytest.mark.parametrize("n,dt,p", [(4, "f64", 12), (2, "f64", 11), (4, "f32", 13)])
def test_cluster_engine_matches_oracle(W, n, dt, p):
    """The opt-in cluster engine (WRNG_GPU_CLUSTER=1, one pool over 8 CTAs,
    DSMEM gathers) is bit-identical to the oracle through drift audits,
    leftovers and fp32/fp64 outputs (subprocess: the switch is read at load)."""
    import subprocess
    import sys

    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, 'oracle')\n"
        "import oracle as O, torch\n"
        "import paper_1004_3114_b200 as W\n"
        f"kw = dict(pool_exponent={p}, throwaway_f=2, seed=31, n_arrays={n}, dtype='{dt}',"
        " drift_check_period=3)\n"
        "g = W.WallaceState(W.WallaceConfig(init_on_host=True, **kw))\n"
        f"o = O.OracleState(pool_exponent={p}, throwaway_f=2, seed=31, n_arrays={n},"
        f" dtype=O.{'F64' if dt == 'f64' else 'F32'}, drift_period=3)\n"
        f"tdt = torch.{'float64' if dt == 'f64' else 'float32'}\n"
        "ok = True\n"
        f"for c in (5 * {n} * 2**{p} + 17, 3 * {n} * 2**{p} - 5, 1000):\n"
        "    t = torch.empty(c, dtype=tdt, device='cuda'); g.fill(t); torch.cuda.synchronize()\n"
        "    ok &= bool(np.array_equal(t.cpu().numpy(), o.fill(c)))\n"
        "pv, pt, pw = o.pool(); gp = g.active_pool()\n"
        "ok &= bool(np.array_equal(gp.arrays.reshape(-1), pv)) and gp.tracked_sumsq == pt\n"
        "print('OK' if ok else 'MISMATCH')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=300, env=dict(os.environ, WRNG_GPU_CLUSTER="1"))
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().splitlines()[-1] == "OK"


@pytest.mark.parametrize("n,dt,p,f,drift,restart", [
    (4, "f64", 15, 2, 0, 0),   # no audits: runs split only at 64 passes
    (2, "f32", 16, 3, 5, 0),   # audits split the runs
    (4, "f32", 14, 1, 3, 7),   # restarts inside the fill
])
def test_hbm_persistent_runs_match_oracle(W, n, dt, p, f, drift, restart):
    """HBM pools with many storage rows (C = N / 512 up to 128): the
    persistent run kernel (grid barrier between passes, TMA row pipeline,
    emission tiles) is bit-identical to the oracle for long fills, leftover
    windows, partial refills and generic (mu, sigma / other width) output."""
    kw = dict(pool_exponent=p, throwaway_f=f, seed=77, n_arrays=n, dtype=dt,
              drift_check_period=drift, restart_interval_passes=restart)
    g = gpu_state(W, init_on_host=True, force_hbm=True, **kw)
    assert g.engine() == "hbm"
    o = oracle_state(**kw)
    cap = n * (1 << p) - 1
    for cnt in (70 * cap + 3, 5, 2 * cap - 7):
        assert_bits(g.fill(cnt), o.fill(cnt))
    other = "f32" if dt == "f64" else "f64"
    onp = np.float32 if other == "f32" else np.float64
    assert_bits(g.fill(3 * cap + 1, 0.5, 2.0), o.fill(3 * cap + 1, 0.5, 2.0))
    assert_bits(g.fill(2 * cap, dtype=other), o.fill(2 * cap, out_dtype=onp))
    pv, pt, pw = o.pool()
    gp = g.active_pool()
    assert np.array_equal(gp.arrays.reshape(-1).astype(np.float64), pv)
    assert (gp.tracked_sumsq, gp.withheld) == (pt, pw)


def test_hbm_run_and_stepwise_paths_agree(W):
    """WRNG_GPU_HBM_STEPWISE=1 (one launch per pass and per emission),
    WRNG_GPU_HBM_FLOW=1 (row-level dataflow, no grid barrier) and the
    default persistent runs give the same bits (subprocess: the switch is
    read when the library loads)."""
    import subprocess
    import sys

    code = (
        "import numpy as np, hashlib\n"
        "import paper_1004_3114_b200 as W\n"
        "g = W.WallaceState(W.WallaceConfig(pool_exponent=17, throwaway_f=2, seed=9, n_arrays=4,"
        " dtype='f64', drift_check_period=6, force_hbm=True))\n"
        "h = hashlib.sha256()\n"
        "for c in (40 * 4 * 2**17 + 9, 17, 4 * 2**17):\n"
        "    h.update(g.fill(c).tobytes())\n"
        "p = g.active_pool()\n"
        "h.update(p.arrays.tobytes()); h.update(np.array([p.tracked_sumsq, p.withheld]).tobytes())\n"
        "print(h.hexdigest())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"WRNG_GPU_HBM_STEPWISE": "1"}, {"WRNG_GPU_HBM_FLOW": "1"}):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1] == outs[2]


def test_hbm_run_small_then_large_pool_in_one_process(W):
    """The run kernel's cached grid must suit every pool size: a small forced
    HBM pool first (short rows), then a large one, in a fresh process."""
    import subprocess
    import sys

    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, 'oracle')\n"
        "import oracle as O\n"
        "import paper_1004_3114_b200 as W\n"
        "ok = True\n"
        "for p in (8, 16):\n"
        "    kw = dict(pool_exponent=p, throwaway_f=2, seed=5, n_arrays=4, dtype='f64')\n"
        "    g = W.WallaceState(W.WallaceConfig(init_on_host=True, force_hbm=True, **kw))\n"
        "    o = O.OracleState(pool_exponent=p, throwaway_f=2, seed=5, n_arrays=4, dtype=O.F64)\n"
        "    c = 3 * 4 * 2**p + 11\n"
        "    ok &= bool(np.array_equal(g.fill(c), o.fill(c)))\n"
        "print('OK' if ok else 'MISMATCH')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().splitlines()[-1] == "OK"


def test_host_fill_larger_than_staging(W):
    """Host output larger than the 2 x 256 MiB staging slabs (f32 bank)."""
    g = gpu_state(W, pool_exponent=10, throwaway_f=1, seed=31, n_arrays=4, dtype="f32", pools=148,
                  init_on_host=True)
    n = (1 << 27) + 12345  # 512 MiB + tail -> 3 slabs
    out = g.fill(n)
    per, extra = divmod(n, 148)
    for p in (0, 147):
        start = p * per + min(p, extra)
        ln = per + (1 if p < extra else 0)
        o = O.OracleState(pool_exponent=10, throwaway_f=1, seed=31, stream=p, n_arrays=4,
                          dtype=O.F32)
        head = o.fill(4096)
        assert_bits(out[start:start + 4096], head)
        if p == 147:
            o.fill(ln - 4096 - 10)
            assert_bits(out[start + ln - 10:start + ln], o.fill(10))


# ---------------------------------------------------------------------------
# emission: mu, sigma, output dtypes (wallace.cpp:198-216; test_wallace_state.cpp:69-109)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype,out_dtype", [("f64", "f64"), ("f64", "f32"), ("f32", "f64"),
                                             ("f32", "f32")])
def test_mu_sigma_and_output_dtypes(W, dtype, out_dtype):
    kw = dict(pool_exponent=9, throwaway_f=2, seed=21, n_arrays=4, dtype=dtype)
    g, o = gpu_state(W, init_on_host=True, **kw), oracle_state(**kw)
    odt = np.float64 if out_dtype == "f64" else np.float32
    for mu, sigma, cnt in ((5.0, 2.0, 3000), (0.0, 1.0, 100), (-1.5, 0.25, 5000), (7.0, 0.0, 5)):
        a = g.fill(cnt, mu, sigma, dtype=out_dtype)
        b = o.fill(cnt, mu, sigma, out_dtype=odt)
        assert_bits(a, b)
    assert np.all(g.fill(5, 7.0, 0.0) == 7.0)


def test_fill_edge_cases(W):
    g = gpu_state(W, pool_exponent=10, throwaway_f=3, seed=1)
    assert g.fill(0).size == 0
    assert g.numbers_emitted() == 0 and g.pass_count() == 0
    with pytest.raises(ValueError):
        g.fill(np.empty(1), 0.0, -1.0)
    with pytest.raises(ValueError):
        W.WallaceState(W.WallaceConfig(pool_exponent=7))
    with pytest.raises(ValueError):
        W.WallaceState(W.WallaceConfig(pool_exponent=21))
    with pytest.raises(ValueError):
        W.WallaceState(W.WallaceConfig(throwaway_f=0))
    with pytest.raises(ValueError):
        W.WallaceState(W.WallaceConfig(throwaway_f=3, restart_interval_passes=3))
    with pytest.raises(ValueError):
        W.WallaceState(W.WallaceConfig(n_arrays=3))


def test_emission_accounting(W):
    # test_wallace_state.cpp:97-109: refills = ceil(c / (2N - 1)) over split calls
    cap = 2047
    for total in (1, cap, cap + 1, 3 * cap + 5):
        g = gpu_state(W, pool_exponent=10, throwaway_f=3, seed=1)
        first = total // 2
        g.fill(first)
        g.fill(total - first)
        assert g.numbers_emitted() == total
        assert g.pass_count() // 3 == (total + cap - 1) // cap


def test_refill_and_advance_pass_counters(W):
    for f in (1, 3):
        g = gpu_state(W, pool_exponent=10, throwaway_f=f, seed=1)
        g.refill()
        assert g.avail() == 2047 and g.pass_count() == f
        g.refill()
        assert g.pass_count() == 2 * f
        g.advance_pass()
        assert g.avail() == 0 and g.pass_count() == 2 * f + 1


# ---------------------------------------------------------------------------
# sum of squares, drift audit, restart (wallace.cpp:188-236)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n_arrays", [2, 4])
def test_chisq_post_refill_sum_equals_target(W, n_arrays):
    g = gpu_state(W, pool_exponent=10, throwaway_f=3, seed=1, n_arrays=n_arrays)
    for _ in range(20):
        g.refill()
        p = g.active_pool()
        assert abs(p.direct_sumsq() / p.tracked_sumsq - 1) < 1e-9


def test_fixed_mode_conserves_sum(W):
    g = gpu_state(W, pool_exponent=10, throwaway_f=1, seed=1, scale_mode=W.ScaleMode.fixed,
                  n_arrays=4)
    q0 = g.active_pool().direct_sumsq()
    for _ in range(50):
        g.advance_pass()
    assert abs(g.active_pool().direct_sumsq() / q0 - 1) <= 1e-12


@pytest.mark.parametrize("n,bound", [(2, 2 ** 0.5), (4, 2.0)])
def test_outlier_band_fixed_mode(W, n, bound):
    """acceptance.cpp:207-220 on the GPU: with the sum of squares fixed, one
    pass moves the largest |value| by at most the transform's norm bound
    (sqrt 2 for the n = 2 rotation; 2 for the n = 4 matrices, whose rows
    have four entries of size 1/2 or 1/2 and 1/2-1), over 1000 passes."""
    g = gpu_state(W, pool_exponent=10, throwaway_f=1, seed=7, scale_mode=W.ScaleMode.fixed,
                  n_arrays=n)
    before = g.active_pool().max_abs()
    for _ in range(1000):
        g.advance_pass()
        after = g.active_pool().max_abs()
        eps = 1e-12 * before
        assert before / bound - eps <= after <= bound * before + eps
        before = after


def test_threaded_independent_streams(W):
    """test_wallace_state.cpp:175-191 on the GPU: three host threads, each
    with its own generator (stream 0, 1, 2) and CUDA stream, fill at the
    same time; each stream equals its sequential run, and they differ."""
    import threading

    def run(sid):
        g = gpu_state(W, pool_exponent=10, throwaway_f=3, seed=0, stream_id=sid, n_arrays=4)
        return g.fill(100000)

    par = [None] * 3

    def worker(i):
        par[i] = run(i)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(3):
        assert_bits(par[i], run(i))
    assert not np.array_equal(par[0], par[1])


def test_cost_model_ratio_on_gpu(W):
    """acceptance.cpp:222-230: t(f=3) / t(f=1) in [1.5, 4.5], here for the
    C3-shaped bank (1184 fp32 n = 4 pools) on the device."""
    import torch

    out = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    t = {}
    for f in (1, 3):
        g = gpu_state(W, pool_exponent=10, throwaway_f=f, seed=2024, n_arrays=4, dtype="f32",
                      pools=1184)
        g.fill(out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(3):
            a.record()
            g.fill(out)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        t[f] = best
    assert 1.5 <= t[3] / t[1] <= 4.5, t


def test_drift_check_raises_and_corrects(W):
    g = gpu_state(W, pool_exponent=10, throwaway_f=3, seed=1)
    g.refill()
    p = g.active_pool()
    p.arrays[0, 17] += 1000.0
    g.set_active_pool(p)
    with pytest.raises(W.CorruptedStateError):
        g.drift_check()
    g2 = gpu_state(W, pool_exponent=10, throwaway_f=3, seed=1, init_on_host=True)
    g2.refill()
    p2 = g2.active_pool()
    actual = p2.direct_sumsq()
    p2.tracked_sumsq = actual * (1 + 1e-5)
    g2.set_active_pool(p2)
    g2.drift_check()
    assert g2.active_pool().tracked_sumsq == actual


@pytest.mark.parametrize("force_hbm", [False, True])
def test_drift_guard_at_periodic_checkpoint(W, force_hbm):
    # acceptance.cpp:263-286
    g = gpu_state(W, pool_exponent=10, throwaway_f=3, seed=13, drift_check_period=6,
                  force_hbm=force_hbm)
    g.refill()  # pass_count 3
    p = g.active_pool()
    p.arrays[0, 0] += 1000.0
    g.set_active_pool(p)
    with pytest.raises(W.CorruptedStateError):
        g.refill()  # crosses 6 -> audit


@pytest.mark.parametrize("force_hbm,n,f", [(False, 2, 3), (True, 2, 3), (False, 4, 1),
                                         (True, 4, 2)])
def test_state_after_mid_fill_audit_failure_matches_oracle(W, force_hbm, n, f):
    """A fill whose audit raises corrupted_state_error leaves the generator
    exactly where the reference's exception leaves it (wallace.cpp:188-196,
    225-234): the audited refill's passes done, no later pass drawn — lag
    table, cursor, draws, counters and pool all equal the oracle's."""
    kw = dict(pool_exponent=10, throwaway_f=f, seed=13, drift_check_period=4 * f, n_arrays=n)
    g = gpu_state(W, force_hbm=force_hbm, **kw)
    o = oracle_state(**kw)
    cap = n * 1024 - 1
    assert_bits(g.fill(2 * cap + 7), o.fill(2 * cap + 7))
    p = g.active_pool()
    p.arrays[0, 17] += 1000.0
    g.set_active_pool(p)
    ov, ot, ow = o.pool()
    ov[17] += 1000.0
    o.set_pool(ov, ot, ow)
    with pytest.raises(W.CorruptedStateError):
        g.fill(10 * cap)
    with pytest.raises(O.OracleError):
        o.fill(10 * cap)
    oc = o.counters()
    assert (g.pass_count(), g.avail()) == (oc["pass_count"], oc["avail"])
    t, r, s_, d = o.uniform()
    us = g.uniform_state()
    assert_bits(us.lag_table, t)
    assert (us.cursor_r, us.draws) == (r, d)
    pv, pt, pw = o.pool()
    gp = g.active_pool()
    assert_bits(gp.arrays.reshape(-1), pv)
    assert (gp.tracked_sumsq, gp.withheld) == (pt, pw)


@pytest.mark.parametrize("force_hbm", [False, True])
def test_uniform_state_write_back(W, force_hbm):
    """The mutable uniform_state() (wallace.hpp:158): a generator whose
    uniform state is overwritten with another stream's draws that stream's
    pass parameters next; malformed cursors are rejected."""
    a = gpu_state(W, pool_exponent=10, seed=5, force_hbm=force_hbm)
    b = gpu_state(W, pool_exponent=10, seed=9, force_hbm=force_hbm)
    a.fill(3000)
    b.fill(5000)
    a.set_uniform_state(b.uniform_state())
    ua, ub = a.uniform_state(), b.uniform_state()
    assert_bits(ua.lag_table, ub.lag_table)
    assert (ua.cursor_r, ua.cursor_s, ua.draws) == (ub.cursor_r, ub.cursor_s, ub.draws)
    pa, pb = a.advance_pass(), b.advance_pass()
    assert (pa.alpha, pa.beta, pa.gamma, pa.delta, pa.rot.c, pa.rot.s) == (
        pb.alpha, pb.beta, pb.gamma, pb.delta, pb.rot.c, pb.rot.s)
    bad = b.uniform_state()
    bad.cursor_s = (bad.cursor_r + 1) % 607
    with pytest.raises(ValueError):
        a.set_uniform_state(bad)


@pytest.mark.parametrize("n,dt,p", [(2, "f64", 10), (4, "f32", 8), (4, "f64", 11)])
def test_small_host_fills_bit_exact(W, n, dt, p):
    """Host fills of at most one refill's worth are served from the host
    window (capi.cu fill_window): random sizes, mu/sigma and output widths,
    interleaved with device-path fills, advance_pass, refill and a save/load
    round trip — every value and counter as the oracle's."""
    kw = dict(pool_exponent=p, throwaway_f=2, seed=41, n_arrays=n, dtype=dt, drift_check_period=5,
              restart_interval_passes=9)
    g = gpu_state(W, **kw)
    o = oracle_state(**kw)
    cap = n * (1 << p) - 1
    rng = np.random.default_rng(p)
    for it in range(60):
        cnt = int(rng.integers(0, cap + 1)) if it % 7 else int(rng.integers(cap, 3 * cap))
        mu, sigma = (0.0, 1.0) if it % 3 else (float(rng.normal()), float(rng.uniform(0, 3)))
        od = ("f64", np.float64) if it % 2 else ("f32", np.float32)
        assert_bits(g.fill(cnt, mu, sigma, dtype=od[0]), o.fill(cnt, mu, sigma, out_dtype=od[1]))
        if it % 11 == 5:
            g.advance_pass()
            o.advance_pass()
        if it % 13 == 7:
            g.refill()
            o.refill()
        if it == 30:
            g = W.WallaceState.load_state(g.save_state())
        oc = o.counters()
        assert (g.pass_count(), g.numbers_emitted(), g.avail()) == (
            oc["pass_count"], oc["numbers_emitted"], oc["avail"])


def test_zero_tracked_sum_raises(W):
    g = gpu_state(W, pool_exponent=10, seed=3)
    p = g.active_pool()
    p.tracked_sumsq = 0.0
    g.set_active_pool(p)
    with pytest.raises(W.CorruptedStateError):
        g.advance_pass()


def test_drift_stays_tiny_over_1000_passes(W):
    g = gpu_state(W, pool_exponent=10, throwaway_f=1, seed=1)
    for _ in range(10):
        g.fill(100 * 2047)
    p = g.active_pool()
    assert abs(p.direct_sumsq() / p.tracked_sumsq - 1) <= 1e-9


def test_restart_deterministic_and_close_to_oracle(W):
    kw = dict(pool_exponent=10, throwaway_f=3, seed=1, restart_interval_passes=100)
    a, b = gpu_state(W, init_on_host=False, **kw), gpu_state(W, init_on_host=False, **kw)
    va, vb = a.fill(300000), b.fill(300000)
    assert_bits(va, vb)
    assert a.pass_count() > 300
    assert_close(va, oracle_state(**kw).fill(300000), TOL64)


@pytest.mark.parametrize("n,dt,p,f,restart,hbm,pools", [
    (2, "f64", 10, 3, 100, False, 1),   # test_wallace_state.cpp:152-173's config
    (4, "f64", 12, 1, 9, False, 3),     # bank: pools restart at different calls
    (4, "f32", 10, 2, 5, False, 5),
    (2, "f64", 14, 2, 7, True, 1),      # HBM engine
    (4, "f64", 15, 1, 4, True, 2),
])
def test_host_init_restarts_bit_exact(W, n, dt, p, f, restart, hbm, pools):
    """Restarts of a host-initialised handle run glibc's Box-Muller on the
    host from the device's uniform state (wallace.cpp:236), so the stream
    stays bit-identical to the oracle across every restart — fills, refill(),
    restart() and a save/load round trip."""
    kw = dict(pool_exponent=p, throwaway_f=f, seed=21, n_arrays=n, dtype=dt,
              restart_interval_passes=restart)
    g = gpu_state(W, init_on_host=True, force_hbm=hbm, pools=pools, **kw)
    cap = n * (1 << p) - 1
    if pools == 1:
        o = oracle_state(**kw)
        for cnt in (7 * cap + 5, 1, 25 * cap, 3):
            assert_bits(g.fill(cnt), o.fill(cnt))
        g.refill()
        o.refill()
        g.restart()
        o.restart()
        assert_bits(g.fill(4 * cap + 2), o.fill(4 * cap + 2))
        pv, pt, pw = o.pool()
        gp = g.active_pool()
        assert np.array_equal(gp.arrays.reshape(-1), pv) and (gp.tracked_sumsq, gp.withheld) == (pt, pw)
        t, r, s, d = o.uniform()
        us = g.uniform_state()
        assert_bits(us.lag_table, t)
        assert (us.cursor_r, us.draws) == (r, d)
        h = W.WallaceState.load_state(g.save_state(), force_hbm=hbm)
        assert_bits(h.fill(12 * cap), o.fill(12 * cap))
    else:
        # per-pool streams: pool q of the bank equals a single-pool oracle
        # state run through the same per-call segment lengths
        orc = [oracle_state(**dict(kw, stream_id=q)) for q in range(pools)]
        for cnt in (pools * 9 * cap + 2, 5, pools * 13 * cap + pools - 1):
            got = g.fill(cnt)
            base, extra = divmod(cnt, pools)
            off = 0
            for q in range(pools):
                ln = base + (1 if q < extra else 0)
                assert_bits(got[off:off + ln], orc[q].fill(ln))
                off += ln


# ---------------------------------------------------------------------------
# persistence (serialize.cpp; test_serialize.cpp)
# ---------------------------------------------------------------------------
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_state_roundtrip_with_reference_library(W):
    r = O.RefState(pool_exponent=10, throwaway_f=3, seed=11)
    r.fill(3500)
    g = W.WallaceState.load_state(r.save_state())
    assert g.save_state() == r.save_state()
    assert_bits(g.fill(100000), r.fill(100000))
    assert g.save_state() == r.save_state()
    # and the other direction
    r2 = O.RefState.load_state(g.save_state())
    assert_bits(g.fill(7777), r2.fill(7777))


@pytest.mark.parametrize("n_arrays,dtype,pools", [(4, "f32", 3), (4, "f64", 1), (2, "f32", 2)])
def test_state_v2_roundtrip(W, n_arrays, dtype, pools):
    g = gpu_state(W, pool_exponent=9, throwaway_f=2, seed=5, n_arrays=n_arrays, dtype=dtype,
                  pools=pools)
    g.fill(pools * 1234)
    data = g.save_state()
    h = W.WallaceState.load_state(data)
    assert h.save_state() == data
    assert_bits(g.fill(pools * 5000), h.fill(pools * 5000))


def test_state_rejects_malformed(W):
    g = gpu_state(W, seed=1)
    data = bytearray(g.save_state())
    bad = bytearray(data)
    bad[0] ^= 0xFF
    with pytest.raises(W.MalformedStateError) as e:
        W.WallaceState.load_state(bytes(bad))
    assert e.value.kind == W.StateErrorKind.bad_magic
    bad = bytearray(data)
    bad[4:8] = b"\xff\xff\xff\xff"
    with pytest.raises(W.MalformedStateError) as e:
        W.WallaceState.load_state(bytes(bad))
    assert e.value.kind == W.StateErrorKind.unsupported_version
    for keep in (0, 3, 8, 73, 500, len(data) - 1):
        with pytest.raises(W.MalformedStateError) as e:
            W.WallaceState.load_state(bytes(data[:keep]))
        assert e.value.kind == W.StateErrorKind.truncated
    bad = bytearray(data)
    bad[8] = 42
    with pytest.raises(W.MalformedStateError) as e:
        W.WallaceState.load_state(bytes(bad))
    assert e.value.kind == W.StateErrorKind.field_range
    with pytest.raises(W.MalformedStateError) as e:
        W.WallaceState.load_state(bytes(data) + b"\0")
    assert e.value.kind == W.StateErrorKind.field_range


def test_import_reference_state_then_gpu_continues_bit_exact(W):
    """No host init involved: the state bytes come from the oracle's n = 2
    fp64 run of the reference's own algorithm, so every value downstream is
    the GPU kernels' arithmetic."""
    o = O.OracleState(pool_exponent=12, throwaway_f=1, seed=12345)
    o.fill(10000)
    if O.ref_available():
        r = O.RefState(pool_exponent=12, throwaway_f=1, seed=12345)
        r.fill(10000)
        g = W.WallaceState.load_state(r.save_state())
    else:
        pytest.skip("needs the reference library to serialise a state")
    for engine_force in (False, True):
        gg = W.WallaceState.load_state(g.save_state(), force_hbm=engine_force)
        oo = O.OracleState(pool_exponent=12, throwaway_f=1, seed=12345)
        oo.fill(10000)
        assert_bits(gg.fill(200000), oo.fill(200000))


# ---------------------------------------------------------------------------
# statistics (stats.cpp:89-108, acceptance.cpp:168-177) + Anderson-Darling
# ---------------------------------------------------------------------------
def test_moments_and_ad_match_oracle_c1(W):
    """C1 (n=4 fp64 4x4096, seed 12345, f=1): 2^24 normals."""
    import torch

    kw = dict(pool_exponent=12, throwaway_f=1, seed=12345, n_arrays=4, dtype="f64")
    g = gpu_state(W, init_on_host=True, **kw)
    t = torch.empty(1 << 24, dtype=torch.float64, device="cuda")
    g.fill(t)
    v = t.cpu().numpy()
    ref = oracle_state(**kw).fill(1 << 24)
    assert_bits(v, ref)
    mg = W.device_moments(t)
    mo = O.moments(ref)
    for k in ("m1", "m2", "m3", "m4"):
        assert abs(mg[k] - mo[k]) <= 1e-12 * max(1.0, abs(mo[k]))
    assert O.anderson_darling(v) == O.anderson_darling(ref)
    # CLT bands of acceptance.cpp:168-177 (4 sigma at n = 2^24)
    n = float(1 << 24)
    assert abs(mo["m1"]) <= 4 / n ** 0.5
    assert abs(mo["m2"] - 1) <= 4 * (2 / n) ** 0.5
    assert abs(mo["m3"]) <= 4 * (15 / n) ** 0.5
    assert abs(mo["m4"] - 3) <= 4 * (96 / n) ** 0.5
    assert O.anderson_darling(ref) < 4.0


@pytest.mark.parametrize("n_arrays,dtype", [(2, "f64"), (4, "f32")])
def test_moments_1e7_at_f3(W, n_arrays, dtype):
    # acceptance.cpp:168-177, on the GPU stream
    g = gpu_state(W, seed=1, throwaway_f=3, n_arrays=n_arrays, dtype=dtype)
    v = g.fill(10_000_000).astype(np.float64)
    m = O.moments(v)
    assert abs(m["m1"]) <= 0.00127 and abs(m["m2"] - 1) <= 0.00179 and abs(m["m4"] - 3) <= 0.0124


# ---------------------------------------------------------------------------
# C2 (HBM-resident 4 x 2^20 fp64 pool, f = 2)
# ---------------------------------------------------------------------------
def test_c2_head_bit_exact_and_full_properties(W):
    kw = dict(pool_exponent=20, throwaway_f=2, seed=7, n_arrays=4, dtype="f64")
    g = gpu_state(W, init_on_host=True, **kw)
    assert g.engine() == "hbm"
    o = oracle_state(**kw)
    n = 3 * (4 << 20)
    assert_bits(g.fill(n), o.fill(n))
    p = g.active_pool()
    assert abs(p.direct_sumsq() / p.tracked_sumsq - 1) < 1e-9
    us = g.uniform_state()
    assert_bits(us.lag_table, o.uniform()[0])
