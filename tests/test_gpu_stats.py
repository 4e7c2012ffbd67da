"""GPU tests of the on-device validation statistics:
u/v chi-squared (stats.cpp:10-38 with the CLI's pairing, tools/main.cpp:
160-193), autocorrelation (stats.cpp:110-127), chi2_sf (stats.cpp:40-87) and
the generate-and-check path (wrng_gpu_validate), against the reference's
golden statistics and the CPU oracle.

Bars: bin counts exact (device exp/atan may differ from glibc by an ulp, so
a value sitting on a bin edge could move one bin: allowed for at most 2
pairs per test); chi-squared statistics exact when the counts are; r within
1e-12 absolute (the device sums in tree order, the reference left to right);
moments within 1e-12 relative.
"""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
STATS = json.load(open(os.path.join(GOLDEN, "golden_ref.json")))["stats"]


@pytest.fixture(scope="module")
def W():
    import paper_1004_3114_b200 as W

    return W


def cuda(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def counts_close(a, b, max_moves=2):
    d = np.abs(a.astype(np.int64) - b.astype(np.int64))
    assert int(d.sum()) <= 2 * max_moves, f"{int(d.sum())} count differences"


def golden_stream():
    g = STATS["stream"]
    return O.OracleState(pool_exponent=g["pool_exponent"], throwaway_f=g["throwaway_f"],
                         seed=g["seed"]).fill(g["count"])


def test_device_uv_chi2_matches_reference_golden(W):
    v = golden_stream()
    r = W.device_uv_chi2(cuda(v), 1000)
    gold = STATS["uv_k1000"]
    cu, cv, sk = O.uv_counts(v, 1000)
    counts_close(r["counts_u"], cu)
    counts_close(r["counts_v"], cv)
    assert r["skipped"] == sk == 0
    if np.array_equal(r["counts_u"], cu):
        assert r["u"]["statistic"] == gold["u_statistic"]
        assert r["u"]["p_value"] == gold["u_p"]
    if np.array_equal(r["counts_v"], cv):
        assert r["v"]["statistic"] == gold["v_statistic"]
        assert r["v"]["p_value"] == gold["v_p"]
    assert r["u"]["sample_count"] == gold["samples"]


def test_device_autocorr_matches_reference_golden(W):
    v = cuda(golden_stream())
    for lag, want in STATS["autocorr"].items():
        assert abs(W.device_autocorr(v, int(lag)) - want) <= 1e-12


@pytest.mark.parametrize("row", STATS["chi2_sf"], ids=lambda r: f"{r[0]}-{r[1]}")
def test_chi2_sf_matches_reference_golden(W, row):
    x, dof, p = row
    assert W.chi2_sf(x, dof) == p


def test_device_stats_f32_stream_and_edges(W):
    v = O.OracleState(pool_exponent=10, throwaway_f=1, seed=7, n_arrays=4,
                      dtype=O.F32).fill(300001)
    v[10] = v[11] = 0.0  # a (0, 0) pair is skipped (stats.cpp:11)
    v[21] = 0.0          # y == 0: v = copysign(pi/2, x) (stats.cpp:13)
    r = W.device_uv_chi2(cuda(v), 777)
    cu, cv, sk = O.uv_counts(v, 777)
    assert r["skipped"] == sk == 1
    counts_close(r["counts_u"], cu)
    counts_close(r["counts_v"], cv)
    assert abs(W.device_autocorr(cuda(v), 3) - O.autocorr(v, 3)) <= 1e-12
    with pytest.raises(ValueError):
        W.device_autocorr(cuda(v[:4]), 3)  # needs n >= lag + 2 (stats.cpp:112-113)


def test_validate_single_pool_equals_reference_statistics(W):
    g = STATS["stream"]
    st = W.WallaceState(W.WallaceConfig(pool_exponent=g["pool_exponent"],
                                        throwaway_f=g["throwaway_f"], seed=g["seed"],
                                        init_on_host=True))
    r = W.validate(st, g["count"], k=1000, lag=1)
    v = golden_stream()
    m = O.moments(v)
    for key in ("m1", "m2", "m3", "m4"):
        assert abs(r[key] - m[key]) <= 1e-12 * max(1.0, abs(m[key]))
    cu, cv, _ = O.uv_counts(v, 1000)
    counts_close(r["counts_u"], cu)
    counts_close(r["counts_v"], cv)
    if np.array_equal(r["counts_u"], cu):
        assert r["u_statistic"] == STATS["uv_k1000"]["u_statistic"]
    assert abs(r["autocorr"] - STATS["autocorr"]["1"]) <= 1e-12
    assert r["n"] == g["count"] and r["uv_samples"] == 100000
    # the generator advanced exactly as fill(count) would
    o = O.OracleState(pool_exponent=g["pool_exponent"], throwaway_f=g["throwaway_f"],
                      seed=g["seed"])
    o.fill(g["count"])
    assert np.array_equal(st.fill(5000), o.fill(5000))


@pytest.mark.parametrize("pools,count,lag", [(5, 5 * 40000 + 3, 7), (1, 20_000_001, 100)])
def test_validate_bank_multi_window_matches_oracle(W, pools, count, lag):
    kw = dict(pool_exponent=10, throwaway_f=1, seed=21, n_arrays=4, dtype="f32", pools=pools,
              init_on_host=True)
    st = W.WallaceState(W.WallaceConfig(**kw))
    r = W.validate(st, count, k=500, lag=lag)
    per, extra = divmod(count, pools)
    streams = [O.OracleState(pool_exponent=10, throwaway_f=1, seed=21, stream=p, n_arrays=4,
                             dtype=O.F32).fill(per + (1 if p < extra else 0))
               for p in range(pools)]
    allv = np.concatenate(streams).astype(np.float64)
    n = allv.size
    for j, key in enumerate(("m1", "m2", "m3", "m4"), start=1):
        want = float(np.sum(allv ** j)) / n
        assert abs(r[key] - want) <= 1e-11 * max(1.0, abs(want)), key
    cu = np.zeros(500, dtype=np.uint64)
    cv = np.zeros(500, dtype=np.uint64)
    for s in streams:  # pairs within each pool's stream
        a, b, _ = O.uv_counts(s, 500)
        cu += a
        cv += b
    counts_close(r["counts_u"], cu)
    counts_close(r["counts_v"], cv)
    m = allv.mean()
    num = sum(float(np.dot(s[:-lag].astype(np.float64) - m, s[lag:].astype(np.float64) - m))
              for s in streams)
    den = sum(float(np.sum((s[:-lag].astype(np.float64) - m) ** 2)) for s in streams)
    assert abs(r["autocorr"] - num / den) <= 1e-10
    # every pool advanced as a fill of `count` would
    nxt = st.fill(pools * 10)
    for p in range(pools):
        o = O.OracleState(pool_exponent=10, throwaway_f=1, seed=21, stream=p, n_arrays=4,
                          dtype=O.F32)
        o.fill(per + (1 if p < extra else 0))
        assert np.array_equal(nxt[p * 10:(p + 1) * 10], o.fill(10))
