"""C2 (one HBM-resident 4 x 2^20 fp64 pool, f = 2, seed 7) parity at full
size, and the exact parallel drift sum against the sequential one.

The HBM engine's drift audit (hbm_engine.cu k_sum_chunks -> k_sum_segs ->
k_sum_walk) must reproduce Pool::direct_sumsq's left-to-right fp64 sum
(/root/reference/proj/src/wallace.cpp:13-18) bit for bit, because
drift_check adopts the recomputed value (wallace.cpp:225-234) and every later
chi-squared scale depends on it.  These tests compare it with the oracle's
sequential loop (oracle/wallace_oracle.c or_direct_sumsq, via
OracleState.drift_check) at 4 * 2^20 terms, on term sets chosen to stress
the algorithm: many binades, exact rounding ties, absorbed tiny terms,
zeros, and the C2 generator's own pools after hundreds of passes.
"""
import hashlib

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

C2 = dict(pool_exponent=20, throwaway_f=2, seed=7, n_arrays=4, dtype="f64")


@pytest.fixture(scope="module")
def W():
    import paper_1004_3114_b200 as W

    return W


def assert_bits(a, b, where=""):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype
    if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
        i = int(np.argmax(a.view(np.uint8) != b.view(np.uint8))) // a.itemsize
        raise AssertionError(f"{where}first difference at {i}: {a[i]!r} != {b[i]!r}")


def c2_oracle(**over):
    kw = dict(C2, **over)
    return O.OracleState(pool_exponent=kw["pool_exponent"], throwaway_f=kw["throwaway_f"],
                         seed=kw["seed"], n_arrays=kw["n_arrays"],
                         dtype=O.F64 if kw["dtype"] == "f64" else O.F32,
                         drift_period=kw.get("drift_check_period", 64))


def test_c2_through_three_drift_audits_bit_exact(W):
    """C2 with host (glibc) init, filled until pass 200: the audits at
    passes 64, 128 and 192 adopt the exact sequential sum, so every value
    after them is bit-identical to the oracle (host-output fills of 2^25)."""
    g = W.WallaceState(W.WallaceConfig(init_on_host=True, **C2))
    assert g.engine() == "hbm"
    o = c2_oracle()
    chunk = 1 << 25
    k = 0
    while g.pass_count() < 200:
        assert_bits(g.fill(chunk), o.fill(chunk), f"chunk {k}: ")
        k += 1
    oc = o.counters()
    assert (g.pass_count(), g.numbers_emitted(), g.avail()) == (
        oc["pass_count"], oc["numbers_emitted"], oc["avail"])
    pv, pt, pw = o.pool()
    gp = g.active_pool()
    assert_bits(gp.arrays.reshape(-1), pv)
    assert (gp.tracked_sumsq, gp.withheld) == (pt, pw)
    t, r, s, d = o.uniform()
    us = g.uniform_state()
    assert_bits(us.lag_table, t)
    assert (us.cursor_r, us.cursor_s, us.draws) == (r, s, d)


def test_c2_full_step_bit_exact(W):
    """One whole C2 bench step — 2^30 normals into a DEVICE array (the
    bench's path: one fill call, persistent runs, 8 audits) — equals the
    oracle's 2^30 values; compared slice by slice, plus a sha256 of both."""
    import torch

    g = W.WallaceState(W.WallaceConfig(init_on_host=True, **C2))
    o = c2_oracle()
    n = 1 << 30
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    g.fill(t)
    torch.cuda.synchronize()
    hg, ho = hashlib.sha256(), hashlib.sha256()
    step = 1 << 26
    for i in range(0, n, step):
        a = t[i:i + step].cpu().numpy()
        b = o.fill(step)
        hg.update(a.tobytes())
        ho.update(b.tobytes())
        assert_bits(a, b, f"offset {i}: ")
    assert hg.hexdigest() == ho.hexdigest()
    assert g.pass_count() == o.counters()["pass_count"] == 514


def test_c2_drift_every_refill_bit_exact(W):
    """Forced drift period 1 on the C2 pool: an exact audit after every
    refill (f = 1), each adopted value feeding the next pass's scale."""
    over = dict(throwaway_f=1, drift_check_period=1)
    g = W.WallaceState(W.WallaceConfig(init_on_host=True, **dict(C2, **over)))
    o = c2_oracle(**over)
    cap = 4 * (1 << 20) - 1
    for cnt in (10 * cap + 11, 3 * cap - 4):
        assert_bits(g.fill(cnt), o.fill(cnt))
    assert g.active_pool().tracked_sumsq == o.pool()[1]


def _term_sets(n, rng):
    """Pools whose sequential sum of squares is hard to reproduce."""
    z = rng.standard_normal(n)
    sets = {"normal": z}
    # many binades: |v| from 2^-30 to 2^30, so large terms absorb small ones
    sets["binades"] = z * np.exp2(rng.integers(-30, 31, n).astype(np.float64))
    # ascending magnitudes: the running sum crosses a power of two every few terms
    sets["ascending"] = np.sort(np.abs(z)) * np.exp2(np.linspace(-20, 20, n))
    # exact rounding ties: one big head puts the sum in [2^55, 2^56) (ulp 8)
    # and every 2.0 adds 4 = half an ulp, so round-half-even decides each add;
    # scattered 1.0 / 3.0 terms flip the parity of the running sum
    ties = np.full(n, 2.0)
    ties[0] = 189812531.0  # 189812531^2 ~ 2^55.0
    flip = rng.integers(1, n, n // 64)
    ties[flip] = rng.choice([1.0, 3.0, -2.0, 0.5], flip.size)
    sets["ties"] = ties
    # zeros, underflowing squares and sign mix
    zz = z.copy()
    zz[rng.integers(0, n, n // 8)] = 0.0
    zz[rng.integers(0, n, n // 16)] = 1e-170
    sets["zeros_tiny"] = zz
    # a small head then a long run of equal values (long tie-free plateaus)
    eq = np.full(n, 0.75)
    eq[: n // 3] = rng.standard_normal(n // 3) * 1e-3
    sets["plateau"] = eq
    return sets


@pytest.mark.parametrize("engine,n_arrays,p,dtype", [
    ("hbm", 4, 20, "f64"),   # C2 size: 4 * 2^20 terms (k_sum_* pipeline)
    ("hbm", 4, 20, "f32"),   # fp32 pool, terms squared in fp64
    ("hbm", 2, 17, "f64"),
    ("smem", 4, 12, "f64"),  # exact_sumsq_cta (one CTA)
    ("smem", 2, 10, "f64"),
])
def test_exact_drift_sum_equals_sequential_sum(W, engine, n_arrays, p, dtype):
    """drift_check on a written pool adopts exactly the oracle's sequential
    sum (the tracked value is set 1e-6 off so the audit must replace it)."""
    rng = np.random.default_rng(1234 + p)
    n = n_arrays << p
    g = W.WallaceState(W.WallaceConfig(pool_exponent=p, n_arrays=n_arrays, dtype=dtype,
                                       seed=5, init_on_host=True,
                                       force_hbm=engine == "hbm"))
    assert g.engine() == engine
    o = O.OracleState(pool_exponent=p, n_arrays=n_arrays, seed=5,
                      dtype=O.F64 if dtype == "f64" else O.F32)
    for name, v in _term_sets(n, rng).items():
        if dtype == "f32":
            v = v.astype(np.float32).astype(np.float64)
            v[np.abs(v) > 1e30] = 1.0
        exact = _oracle_direct_sumsq(o, v)
        pool = g.active_pool()
        pool.arrays[:] = v.reshape(n_arrays, -1)
        pool.tracked_sumsq = exact * (1.0 + 1e-6)
        pool.withheld = 0.25
        g.set_active_pool(pool)
        g.drift_check()
        got = g.active_pool().tracked_sumsq
        assert got == exact, f"{name}: {got!r} != {exact!r} ({(got - exact) / exact:.3e})"


def _oracle_direct_sumsq(o, v):
    """or_direct_sumsq through the oracle's drift_check: set the tracked sum
    within 1e-3 of the truth, audit, read the adopted (sequential) value."""
    approx = float(np.dot(v, v))
    o.set_pool(v, approx * (1.0 + 1e-7) if approx > 0 else 1.0, 0.25)
    o.drift_check()
    return o.pool()[1]
