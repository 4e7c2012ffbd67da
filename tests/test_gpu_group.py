"""Group engine (csrc/group_engine.cu: 2 or 4 small n = 4 pools per warp) vs
the CPU oracle, bit for bit: streams, counters, generator state, pools, drift
audits and a failing audit — the same bars as the one-CTA-per-pool engine
(test_gpu_parity.py), on the shapes the group engine takes over (4x256 fp32 /
fp64, 4x512 fp32; unit device/host fills without restarts)."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    import paper_1004_3114_b200 as W

    return W


def assert_bits(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype
    if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
        i = int(np.argmax(a != b))
        raise AssertionError(f"first difference at {i} of {a.size}: {a[i]!r} != {b[i]!r}")


def odt(dt):
    return O.F32 if dt == "f32" else O.F64


def test_group_engine_is_selected(W):
    """resident_pools() reports the group kernel's residency for the shapes it
    takes: whole warps of 2 pools, 16 (fp32) / 8 (fp64) warps per SM — for
    f = 1 fills the 3/4 of that which measured fastest; restarts stay on one
    CTA per pool."""
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    per_sm = lambda **kw: W.resident_pools(W.WallaceConfig(pool_exponent=8, n_arrays=4, **kw)) / sms
    assert per_sm(dtype="f32", throwaway_f=1) == 24
    assert per_sm(dtype="f32", throwaway_f=2) == 32
    assert per_sm(dtype="f64", throwaway_f=1) == 12
    assert per_sm(dtype="f64", throwaway_f=2) == 16
    assert per_sm(dtype="f32", throwaway_f=2, restart_interval_passes=100) <= 18


@pytest.mark.parametrize("dt,p,f,drift,mode,pools,per", [
    ("f32", 8, 1, 64, 0, 16, 5 * 1023 + 11),
    ("f32", 8, 1, 64, 0, 8, 200 * 1023 + 1),    # three audits per pool
    ("f32", 8, 2, 3, 0, 7, 9 * 1023 + 5),       # an audit every other refill, ragged warp
    ("f32", 8, 4, 64, 1, 4, 40 * 1023),         # fixed-sum mode
    ("f32", 8, 3, 0, 0, 5, 33 * 1023 + 1000),   # no audits; 99 passes = several word batches
    ("f64", 8, 1, 64, 0, 6, 70 * 1023 + 1),
    ("f64", 8, 3, 4, 0, 5, 11 * 1023 + 77),
    ("f64", 8, 2, 64, 1, 3, 40 * 1023 + 2),
    ("f32", 9, 1, 64, 0, 5, 70 * 2047 + 3),
    ("f32", 9, 2, 5, 0, 2, 12 * 2047),
])
def test_group_bank_fill_matches_oracle(W, dt, p, f, drift, mode, pools, per):
    count = pools * per + (pools // 2)  # the first pools hold one value more
    g = W.WallaceState(W.WallaceConfig(pool_exponent=p, throwaway_f=f, seed=77, n_arrays=4, dtype=dt,
                                       pools=pools, drift_check_period=drift, scale_mode=mode,
                                       init_on_host=True))
    out = g.fill(count)
    ref = O.bank_fill(count, pools, seed=77, pool_exponent=p, throwaway_f=f, n_arrays=4,
                      dtype=odt(dt), drift_period=drift, scale_mode=mode)
    assert_bits(out, ref)


@pytest.mark.parametrize("dt,p", [("f32", 8), ("f64", 8), ("f32", 9)])
def test_group_device_fills_continue_stream_every_phase(W, dt, p):
    """Successive device fills of one pool at every output phase and ragged
    length (leftover windows, partial last refills, bulk spans of any
    alignment), then the whole state against the oracle's."""
    import torch

    tdt = torch.float32 if dt == "f32" else torch.float64
    kw = dict(pool_exponent=p, throwaway_f=2, seed=31, n_arrays=4, drift_check_period=6)
    g = W.WallaceState(W.WallaceConfig(dtype=dt, init_on_host=True, **kw))
    o = O.OracleState(dtype=odt(dt), drift_period=6,
                      **{k: v for k, v in kw.items() if k != "drift_check_period"})
    cap = 4 * (1 << p) - 1
    buf = torch.zeros(8 * cap + 64, dtype=tdt, device="cuda:0")
    sizes = [1, 2, cap - 3, cap, cap + 1, 3 * cap + 5, 7, 2 * cap, 13, cap - 1, 5 * cap + 2]
    for i, n in enumerate(sizes):
        off = (i * 5 + 1) % 9
        buf.fill_(-7.0)
        g.fill(buf[off:off + n])
        torch.cuda.synchronize()
        h = buf.cpu().numpy()
        assert_bits(h[off:off + n], o.fill(n))
        assert np.all(h[:off] == -7.0) and np.all(h[off + n:] == -7.0)
    oc = o.counters()
    assert (g.pass_count(), g.avail(), g.numbers_emitted()) == (oc["pass_count"], oc["avail"],
                                                                 oc["numbers_emitted"])
    t, r, s_, d = o.uniform()
    us = g.uniform_state()
    assert_bits(us.lag_table, t)
    assert (us.cursor_r, us.draws) == (r, d)
    pv, pt, pw = o.pool()
    gp = g.active_pool()
    assert_bits(gp.arrays.reshape(-1), pv)
    assert (gp.tracked_sumsq, gp.withheld) == (pt, pw)


def test_group_fills_interleave_with_single_pool_operations(W):
    """advance_pass / refill / drift_check run on the one-CTA-per-pool kernel
    over the same device state; the stream continues bit-exact across them."""
    import torch

    kw = dict(pool_exponent=8, throwaway_f=1, seed=5, n_arrays=4)
    g = W.WallaceState(W.WallaceConfig(dtype="f32", init_on_host=True, **kw))
    o = O.OracleState(dtype=O.F32, **kw)
    t = torch.empty(5000, dtype=torch.float32, device="cuda:0")
    g.fill(t)
    assert_bits(t.cpu().numpy(), o.fill(5000))
    g.advance_pass()
    o.advance_pass()
    g.refill()
    o.refill()
    g.drift_check()
    o.drift_check()
    g.fill(t[:3001])
    assert_bits(t[:3001].cpu().numpy(), o.fill(3001))
    assert g.pass_count() == o.counters()["pass_count"]


@pytest.mark.parametrize("dt,f", [("f32", 1), ("f64", 2)])
def test_group_state_after_mid_fill_audit_failure(W, dt, f):
    """A failing audit inside a group-engine fill leaves lag table, cursor,
    draws, counters and pool where the reference's exception leaves them
    (words drawn ahead are un-drawn)."""
    import torch

    tdt = torch.float32 if dt == "f32" else torch.float64
    kw = dict(pool_exponent=8, throwaway_f=f, seed=13, n_arrays=4)
    g = W.WallaceState(W.WallaceConfig(dtype=dt, drift_check_period=4 * f, init_on_host=True, **kw))
    o = O.OracleState(dtype=odt(dt), drift_period=4 * f, **kw)
    cap = 4 * 256 - 1
    t = torch.empty(10 * cap, dtype=tdt, device="cuda:0")
    g.fill(t[:2 * cap + 7])
    assert_bits(t[:2 * cap + 7].cpu().numpy(), o.fill(2 * cap + 7))
    p = g.active_pool()
    p.arrays[0, 17] += 1000.0
    g.set_active_pool(p)
    ov, ot, ow = o.pool()
    ov[17] += 1000.0
    o.set_pool(ov, ot, ow)
    with pytest.raises(W.CorruptedStateError):
        g.fill(t)
        g.synchronize()
    with pytest.raises(O.OracleError):
        o.fill(10 * cap)
    oc = o.counters()
    assert (g.pass_count(), g.avail()) == (oc["pass_count"], oc["avail"])
    tb, r, s_, d = o.uniform()
    us = g.uniform_state()
    assert_bits(us.lag_table, tb)
    assert (us.cursor_r, us.draws) == (r, d)
    pv, pt, pw = o.pool()
    gp = g.active_pool()
    assert_bits(gp.arrays.reshape(-1), pv)
    assert (gp.tracked_sumsq, gp.withheld) == (pt, pw)


def test_group_zero_tracked_sum_raises_after_draws(W):
    """select_pass_params draws the pass's words, then rejects a pool whose
    tracked sum is not positive (wallace.cpp:54-61): same generator state as
    the oracle after the error."""
    import torch

    kw = dict(pool_exponent=8, throwaway_f=1, seed=3, n_arrays=4)
    g = W.WallaceState(W.WallaceConfig(dtype="f32", init_on_host=True, **kw))
    o = O.OracleState(dtype=O.F32, **kw)
    t = torch.empty(4000, dtype=torch.float32, device="cuda:0")
    g.fill(t[:1023])
    o.fill(1023)
    p = g.active_pool()
    p.tracked_sumsq = 0.0
    g.set_active_pool(p)
    ov, ot, ow = o.pool()
    o.set_pool(ov, 0.0, ow)
    with pytest.raises(W.CorruptedStateError):
        g.fill(t)
        g.synchronize()
    with pytest.raises(O.OracleError):
        o.fill(4000)
    tb, r, s_, d = o.uniform()
    us = g.uniform_state()
    assert_bits(us.lag_table, tb)
    assert (us.cursor_r, us.draws) == (r, d)
    assert g.pass_count() == o.counters()["pass_count"]


def test_group_large_bank_one_wave(W):
    """One resident wave of 4x256 fp32 pools, a few hundred refills each:
    first/last pools and a middle one bit-exact, segment layout intact."""
    cfg = W.WallaceConfig(pool_exponent=8, throwaway_f=1, seed=2024, n_arrays=4, dtype="f32",
                          init_on_host=True)
    pools = W.resident_pools(cfg)
    cfg.pools = pools
    g = W.WallaceState(cfg)
    per = 300 * 1023 + 17
    import torch

    t = torch.empty(pools * per + 5, dtype=torch.float32, device="cuda:0")
    g.fill(t)
    torch.cuda.synchronize()
    base = 0
    for p in range(pools):
        ln = per + (1 if p < 5 else 0)
        if p in (0, 1, 4, 5, pools // 2 + 1, pools - 1):
            o = O.OracleState(pool_exponent=8, throwaway_f=1, seed=2024, stream=p, n_arrays=4,
                              dtype=O.F32)
            assert_bits(t[base:base + ln].cpu().numpy(), o.fill(ln))
        base += ln
    assert base == t.numel()


def test_group_full_size_c5_stream(W):
    """BASELINE configs[4] at full size on the group engine: 2^32 fp32 normals from one
    resident wave of 4x256 pools (~1180 refills and 18 drift audits per pool) into one
    device array: the first and last 4096 values of several pool segments equal the
    oracle's bit for bit, and the whole array's moments are N(0, 1)'s."""
    import torch

    total = 1 << 32
    free, _ = torch.cuda.mem_get_info(0)
    if free < total * 4 + (4 << 30):
        pytest.skip("needs 20 GiB of free device memory")
    cfg = W.WallaceConfig(pool_exponent=8, throwaway_f=1, seed=2024, n_arrays=4, dtype="f32",
                          init_on_host=True)
    pools = W.resident_pools(cfg)
    cfg.pools = pools
    g = W.WallaceState(cfg)
    t = torch.empty(total, dtype=torch.float32, device="cuda:0")
    g.fill(t)
    torch.cuda.synchronize()
    base_len, extra = divmod(total, pools)
    for p in (0, 1, extra - 1, extra, pools // 2, pools - 1):
        ln = base_len + (1 if p < extra else 0)
        off = p * base_len + min(p, extra)
        o = O.OracleState(pool_exponent=8, throwaway_f=1, seed=2024, stream=p, n_arrays=4,
                          dtype=O.F32)
        ref = o.fill(ln)
        assert_bits(t[off:off + 4096].cpu().numpy(), ref[:4096])
        assert_bits(t[off + ln - 4096:off + ln].cpu().numpy(), ref[-4096:])
    assert g.pass_count(pools - 1) == -(-base_len // 1023)
    m = W.device_moments(t)
    assert abs(m["m1"]) < 1e-4 and abs(m["m2"] - 1.0) < 1e-4 and abs(m["m4"] - 3.0) < 2e-3
    del t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dt,p,f", [("f32", 8, 1), ("f64", 8, 2), ("f32", 9, 3)])
def test_group_and_one_cta_per_pool_engines_agree(W, dt, p, f):
    """WRNG_GPU_NO_GROUP keeps small pools on one CTA per pool; both engines
    must produce the same bits and leave the same state, through drift audits
    and ragged device fills (subprocess: the switch is read when the library
    loads)."""
    import subprocess
    import sys

    tdt = "torch.float32" if dt == "f32" else "torch.float64"
    cap = 4 * (1 << p) - 1
    code = (
        "import numpy as np, torch, hashlib\n"
        "import paper_1004_3114_b200 as W\n"
        f"g = W.WallaceState(W.WallaceConfig(pool_exponent={p}, throwaway_f={f}, seed=3, n_arrays=4,"
        f" dtype='{dt}', pools=11, drift_check_period=5))\n"
        f"t = torch.empty(11 * 40 * {cap} + 13, dtype={tdt}, device='cuda')\n"
        "h = hashlib.sha256()\n"
        f"for a, b in ((1, 11 * 9 * {cap} + 2), (11 * 9 * {cap} + 2, t.numel())):\n"
        "    g.fill(t[a:b]); torch.cuda.synchronize(); h.update(t[a:b].cpu().numpy().tobytes())\n"
        "for q in (0, 5, 10):\n"
        "    pl = g.active_pool(q); us = g.uniform_state(q)\n"
        "    h.update(pl.arrays.tobytes()); h.update(np.array([pl.tracked_sumsq, pl.withheld]).tobytes())\n"
        "    h.update(us.lag_table.tobytes()); h.update(np.array([us.cursor_r, us.draws, g.pass_count(q), g.avail(q)]).tobytes())\n"
        "print(h.hexdigest())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"WRNG_GPU_NO_GROUP": "1"}):
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=e, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]


def test_group_one_pool_of_a_warp_fails_the_other_completes(W):
    """The two groups of a warp never wait for one another: when pool 1's audit
    fails mid-fill, pool 0 (same warp) still completes its whole segment, and
    both pools end in the states the oracle reaches for them separately."""
    import torch

    kw = dict(pool_exponent=8, throwaway_f=1, seed=21, n_arrays=4)
    g = W.WallaceState(W.WallaceConfig(dtype="f32", drift_check_period=4, pools=2,
                                       init_on_host=True, **kw))
    o = [O.OracleState(dtype=O.F32, drift_period=4, stream=q, **kw) for q in (0, 1)]
    cap = 4 * 256 - 1
    t = torch.full((2 * 9 * cap,), -5.0, dtype=torch.float32, device="cuda:0")
    g.fill(t[:2 * (cap + 3)])
    for q in (0, 1):
        assert_bits(t[q * (cap + 3):(q + 1) * (cap + 3)].cpu().numpy(), o[q].fill(cap + 3))
    p1 = g.active_pool(1)
    p1.arrays[2, 5] += 1000.0
    g.set_active_pool(p1, 1)
    ov, ot, ow = o[1].pool()
    ov[2 * 256 + 5] += 1000.0
    o[1].set_pool(ov, ot, ow)
    per = 9 * cap
    with pytest.raises(W.CorruptedStateError):
        g.fill(t)
        g.synchronize()
    assert_bits(t[:per].cpu().numpy(), o[0].fill(per))      # pool 0: the whole segment
    with pytest.raises(O.OracleError):
        o[1].fill(per)
    for q in (0, 1):
        oc = o[q].counters()
        assert (g.pass_count(q), g.avail(q)) == (oc["pass_count"], oc["avail"]), q
        tb, r, s_, d = o[q].uniform()
        us = g.uniform_state(q)
        assert_bits(us.lag_table, tb)
        assert (us.cursor_r, us.draws) == (r, d)
        pv, pt, pw = o[q].pool()
        gp = g.active_pool(q)
        assert_bits(gp.arrays.reshape(-1), pv)
        assert (gp.tracked_sumsq, gp.withheld) == (pt, pw)
