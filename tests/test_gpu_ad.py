"""Anderson-Darling A^2 on the device (csrc/stats_ad.cu) against the CPU
oracle (oracle/wallace_oracle.c ad_sorted), BASELINE north_star: "the first
four moments and an Anderson-Darling statistic match".  The reference has no
AD: the oracle's A^2 is pinned below to the textbook
formula summed exactly (math.fsum) on small samples (CPU tests), and the
device value must equal the oracle's to 1e-9 relative on the same values."""
import math

import numpy as np
import pytest

import oracle as O

REL = 1e-9


def textbook_ad(v):
    z = np.sort(np.asarray(v, dtype=np.float64))
    n = z.size
    r = 1 / math.sqrt(2)
    terms = [(2 * i + 1) * (math.log(0.5 * math.erfc(-z[i] * r))
                            + math.log(0.5 * math.erfc(z[n - 1 - i] * r))) for i in range(n)]
    return -n - math.fsum(terms) / n


@pytest.mark.parametrize("n,kind", [(7, "normal"), (1000, "normal"), (20000, "normal"),
                                    (5000, "ties"), (3000, "shifted")])
def test_oracle_ad_matches_textbook_formula(n, kind):
    rng = np.random.default_rng(n)
    v = rng.standard_normal(n)
    if kind == "ties":
        v = np.round(v * 4) / 4  # few distinct values
    if kind == "shifted":
        v = v * 1.3 + 0.2  # not N(0,1): large A^2
    a, b = O.anderson_darling(v), textbook_ad(v)
    assert abs(a - b) <= 1e-10 * max(1.0, abs(b)), (a, b)
    assert O.anderson_darling_sorted(np.sort(v), 3) == pytest.approx(a, rel=1e-13)


@pytest.fixture(scope="module")
def W():
    import paper_1004_3114_b200 as W

    return W


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,n,kind", [
    ("f64", 1 << 20, "normal"), ("f32", 1 << 20, "normal"), ("f64", 12345, "normal"),
    ("f32", (1 << 16) + 7, "ties"), ("f64", 1 << 18, "ties"), ("f32", 3 << 20, "shifted"),
    ("f64", 1000, "tiny_tail"),
])
def test_device_ad_equals_oracle(W, dtype, n, kind):
    """Device radix sort + compensated sum vs the oracle on the same values:
    many ties (sort stability is irrelevant, equal values give equal terms),
    negative zero, ragged tile sizes, and far-tail values."""
    import torch

    rng = np.random.default_rng(n)
    v = rng.standard_normal(n)
    if kind == "ties":
        v = np.round(v * 8) / 8
        v[:5] = -0.0
    if kind == "shifted":
        v = v * 0.9 - 0.05
    if kind == "tiny_tail":
        v[:10] = [-8.5, 8.4, -7.9, 7.7, -6.0, 6.1, 1e-300, -1e-300, 0.0, 3.0]
    v = v.astype(np.float64 if dtype == "f64" else np.float32)
    t = torch.from_numpy(v).cuda()
    got = W.device_anderson_darling(t)
    ref = O.anderson_darling(v)
    assert abs(got - ref) <= REL * max(1.0, abs(ref)), (got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_validate_reports_ad_of_the_generated_stream(W, dtype):
    """wrng_gpu_validate_ex(WRNG_GPU_VALIDATE_AD): A^2 of every generated
    value (a C5-shaped bank) equals the oracle's A^2 of the same stream, and
    the moments match; the stream is regenerated here through fill()."""
    kw = dict(pool_exponent=10, throwaway_f=1, seed=2024, n_arrays=4, dtype=dtype, pools=148 * 8)
    n = (1 << 24) + 333
    res = W.validate(W.WallaceState(W.WallaceConfig(**kw)), n, ad=True)
    vals = W.WallaceState(W.WallaceConfig(**kw)).fill(n)
    ref = O.anderson_darling(vals)
    assert res["ad_n"] == n
    assert abs(res["ad_a2"] - ref) <= REL * max(1.0, abs(ref)), (res["ad_a2"], ref)
    m = O.moments(vals.astype(np.float64))
    for k in ("m1", "m2", "m3", "m4"):
        assert abs(res[k] - m[k]) <= 1e-12 * max(1.0, abs(m[k]))
