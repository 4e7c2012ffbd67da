"""The reference's free functions through the drop-in (wallace.hpp:77-111,
uniform.hpp:16-40): host parts against the oracle / reference golden
vectors on CPU, the GPU regenerate against the naive modular oracle of
test_wallace_core.cpp:15-27 bit for bit."""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def W():
    import paper_1004_3114_b200 as W

    return W


def test_uniform_state_matches_reference_golden(W):
    with open(os.path.join(GOLDEN, "golden_ref.json")) as fh:
        cases = json.load(fh)["uniform"]
    for case in cases:
        us = W.UniformState(int(case["seed"]), int(case["stream"]))
        assert [f"{us.next_word():016x}" for _ in case["words"]] == case["words"]
    u = W.UniformState(12345, 0)
    o = O.OracleUniform(12345, 0)
    for m in (2, 3, 1024, 1 << 20):
        assert u.next_int_below(m) == o.next_int_below(m)
    assert u.next_uniform() == o.next_uniform()
    assert u.draws == 5
    with pytest.raises(ValueError):
        u.next_int_below(0)
    with pytest.raises(ValueError):
        u.next_int_below((1 << 20) + 1)


def test_known_answers(W):
    # test_wallace_core.cpp:42-45, 58-62
    t = 0.0 + (2.0 * 2048 - 1.0) ** 0.5
    assert W.chi2_target(0.0, 2048) == 0.5 * t * t  # 2047.5 to 1e-12, as the reference
    assert abs(W.chi2_target(1.0, 2048) - 2111.9921870231046) < 0.01
    r = W.rotation_from_t(2.0 - 3.0 ** 0.5, 0)
    assert abs(r.c - 3.0 ** 0.5 / 2) < 1e-15 and abs(r.s - 0.5) < 1e-15
    r1, r2 = W.rotation_from_t(0.4, 1), W.rotation_from_t(0.4, 2)
    r0 = W.rotation_from_t(0.4, 0)
    assert (r1.c, r1.s) == (r0.c, -r0.s) and (r2.c, r2.s) == (-r0.c, r0.s)


@pytest.mark.parametrize("n_arrays", [2, 4])
def test_select_pass_params_matches_oracle_draws(W, n_arrays):
    """Same draws and scalars as the device engines' first pass (golden):
    a fresh GPU state's advance_pass equals select_pass_params on a host
    UniformState over the same initial pool."""
    p = 10
    o = O.OracleState(pool_exponent=p, throwaway_f=1, seed=31, n_arrays=n_arrays)
    vals, tracked, withheld = o.pool()
    us = W.UniformState(31, 0)
    for _ in range(n_arrays * (1 << p) + 2):  # init_pool's Box-Muller uniforms
        us.next_uniform()
    pool = W.Pool(vals.reshape(n_arrays, -1), tracked, withheld)
    got = W.select_pass_params(us, pool)
    ref = o.advance_pass()
    assert got.strides == list(ref.stride)[:n_arrays]
    assert got.offsets == list(ref.offset)[:n_arrays]
    assert got.scale == ref.scale and got.target_sumsq == ref.target
    if n_arrays == 2:
        assert (got.rot.c, got.rot.s) == (ref.c, ref.s)
    else:
        assert got.variant == ref.variant
    t, r, s, d = o.uniform()
    assert np.array_equal(us.lag_table, t) and (us.cursor_r, us.draws) == (r, d)


def test_select_pass_params_raises_after_draws(W):
    us = W.UniformState(3, 0)
    pool = W.Pool(np.zeros((2, 256)), 0.0, 0.1)
    with pytest.raises(W.CorruptedStateError):
        W.select_pass_params(us, pool)
    assert us.draws == 6  # wallace.cpp:54-61: the draws happen first


def test_plan_segments_cover_and_reject(W):
    # test_wallace_core.cpp:105-157: segments tile [0, N) and keep both
    # strided indices affine; bad strides/offsets -> invalid_argument
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = 1 << int(rng.integers(8, 14))
        a, b = int(rng.choice([3, 5])), int(rng.choice([7, 11]))
        g, d = int(rng.integers(0, n)), int(rng.integers(0, n))
        pp = W.PassParams(a, b, g, d, W.Rotation2(1.0, 0.0), 1.0, 1.0)
        segs = W.plan_segments(pp, n)
        assert segs[0][0] == 0 and segs[-1][1] == n - 1
        assert len(segs) <= a + b + 1
        for (lo, hi, jx, jy), nxt in zip(segs, segs[1:] + [None]):
            if nxt:
                assert nxt[0] == hi + 1
            for j in (lo, hi):
                assert a * j + jx == (a * j + g) % n and b * j + jy == (b * j + d) % n
    with pytest.raises(ValueError):
        W.plan_segments(W.PassParams(4, 7, 0, 0, W.Rotation2(1, 0), 1, 1), 256)
    with pytest.raises(ValueError):
        W.plan_segments(W.PassParams(3, 7, 256, 0, W.Rotation2(1, 0), 1, 1), 256)


def _naive(src, p, n_arrays):
    """regenerate_naive (test_wallace_core.cpp:15-27) / docs/n4_spec.md §3."""
    n = src.shape[1]
    j = np.arange(n, dtype=np.uint64)
    if n_arrays == 2:
        kc, ks = p.rot.c * p.scale, p.rot.s * p.scale
        xs = src[0][(np.uint64(p.alpha) * j + np.uint64(p.gamma)) % np.uint64(n)]
        ys = src[1][(np.uint64(p.beta) * j + np.uint64(p.delta)) % np.uint64(n)]
        return np.stack([kc * xs + ks * ys, kc * ys - ks * xs])
    x = [src[m][(np.uint64(p.strides[m]) * j + np.uint64(p.offsets[m])) % np.uint64(n)]
         for m in range(4)]
    if p.variant == 0:
        k = 0.5 * p.scale
        ps, qs, rs, ss = x[0] + x[1], x[0] - x[1], x[2] + x[3], x[2] - x[3]
        return np.stack([k * (ps + rs), k * (qs + ss), k * (ps - rs), k * (qs - ss)])
    t = 0.5 * ((x[0] + x[1]) + (x[2] + x[3]))
    return np.stack([p.scale * (t - x[m]) for m in range(4)])


@pytest.mark.gpu
@pytest.mark.parametrize("n_arrays", [2, 4])
def test_gpu_regenerate_equals_naive_oracle(W, n_arrays):
    """acceptance.cpp:94-114 / test_wallace_core.cpp:203-217: 100 random
    pools and draws, the GPU pass bit-identical to the modular oracle."""
    us = W.UniformState(77, 0)
    for _ in range(100):
        n = 256 << us.next_int_below(3)
        src = np.random.default_rng(us.next_word() & 0xFFFF).standard_normal((n_arrays, n))
        q = 0.0
        for v in src.reshape(-1).tolist():
            q += v * v
        pool = W.Pool(src, q, float(src[-1, -1]))
        p = W.select_pass_params(us, pool)
        out = W.regenerate(pool, p)
        ref = _naive(src, p, n_arrays)
        assert np.array_equal(out.arrays.view(np.uint64), ref.view(np.uint64))
        assert out.withheld == ref[-1, -1] and out.tracked_sumsq == p.target_sumsq
