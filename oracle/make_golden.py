"""TEST INFRASTRUCTURE ONLY — writes tests/golden/*.json.

* golden_ref.json: outputs of the UNMODIFIED reference library
  (oracle/_ref/libwrng_ref.so built from /root/reference/proj/src by
  oracle/Makefile): uniform words, pass parameters, fill prefixes, counters
  and sums for the reference's n = 2 fp64 generator.  These pin the oracle
  (and through it the GPU path) to the reference itself.
* golden_n4.json: outputs of the oracle restatement in its n = 4 and fp32
  modes (no reference code exists for them — "parity unpinned" by reference
  tests; these files freeze the restatement so regressions show up).

Run from the repo root: python oracle/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle as O  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def h(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def params_dict(p, n_arrays):
    d = p.as_dict(n_arrays)
    d["scale_hex"] = float(p.scale).hex()
    d["target_hex"] = float(p.target).hex()
    d["c_hex"] = float(p.c).hex()
    d["s_hex"] = float(p.s).hex()
    return d


# Configs named by BASELINE.json / SURVEY.md §8(d), in the reference's n=2
# fp64 mode (the only mode the reference implements).
REF_CASES = [
    # name, p, f, mode, seed, stream, count
    ("C1_n2_analogue", 12, 1, O.CHISQ, 12345, 0, 3 * 8191 + 5),
    ("C2_n2_analogue", 20, 2, O.CHISQ, 7, 0, 5000),
    ("C3_n2_cta0", 10, 1, O.CHISQ, 2024, 0, 3 * 2047 + 11),
    ("C3_n2_cta1", 10, 1, O.CHISQ, 2024, 1, 2047),
    ("C4_n2_rank0", 10, 1, O.CHISQ, 99, 0, 2047),
    ("defaults_seed1", 10, 3, O.CHISQ, 1, 0, 3 * 2047 + 1),
    ("fixed_p8", 8, 2, O.FIXED, 5, 3, 2000),
    ("drift_crossing", 8, 3, O.CHISQ, 11, 0, 70 * 511),
]


def ref_golden():
    out = {"source": "oracle/_ref/libwrng_ref.so (reference proj/src, -O3 -ffp-contract=off)",
           "uniform": [], "cases": []}
    for seed, stream in [(12345, 0), (7, 0), (2024, 0), (2024, 1), (99, 0), (1, 0), (0, 0),
                         (2**64 - 1, 5)]:
        u = O.RefUniform(seed, stream)
        words = [u.next_word() for _ in range(40)]
        out["uniform"].append({"seed": str(seed), "stream": str(stream),
                               "words": [f"{w:016x}" for w in words]})
    for name, p, f, mode, seed, stream, count in REF_CASES:
        st = O.RefState(pool_exponent=p, throwaway_f=f, scale_mode=mode, seed=seed,
                        stream=stream)
        pool0, tracked0, withheld0 = st.pool()
        # parameters of the first two passes on a twin state
        twin = O.RefState(pool_exponent=p, throwaway_f=f, scale_mode=mode, seed=seed,
                          stream=stream)
        params = [params_dict(twin.advance_pass(), 2) for _ in range(2)]
        v = st.fill(count)
        c = st.counters()
        pool1, tracked1, withheld1 = st.pool()
        out["cases"].append({
            "name": name, "pool_exponent": p, "throwaway_f": f, "scale_mode": mode,
            "seed": seed, "stream": stream, "count": count,
            "init_tracked_hex": tracked0.hex(), "init_withheld_hex": withheld0.hex(),
            "init_pool_sha256": h(pool0),
            "params": params,
            "fill_head_hex": [float(x).hex() for x in v[:16]],
            "fill_tail_hex": [float(x).hex() for x in v[-8:]],
            "fill_sha256": h(v),
            "counters": c,
            "final_tracked_hex": tracked1.hex(), "final_withheld_hex": withheld1.hex(),
            "final_pool_sha256": h(pool1),
            "state_sha256": hashlib.sha256(st.save_state()).hexdigest(),
        })
    # known answers quoted by the reference tests
    L = O.ref_lib()
    out["chi2_target_0_2048"] = L.ref_chi2_target(0.0, 2048)
    out["chi2_target_1_2048"] = L.ref_chi2_target(1.0, 2048)
    # validation statistics of a reference stream (stats.cpp:10-127, the
    # CLI's u/v pairing tools/main.cpp:160-193)
    st = O.RefState(pool_exponent=10, throwaway_f=3, seed=1)
    v = st.fill(200000)
    uv = O.ref_uv_chi2(v, 1000)
    out["stats"] = {
        "stream": {"pool_exponent": 10, "throwaway_f": 3, "seed": 1, "count": 200000,
                   "sha256": h(v)},
        "uv_k1000": uv,
        "autocorr": {str(lag): O.ref_autocorr(v, lag) for lag in (1, 2, 5, 100)},
        "chi2_sf": [[x, d, O.ref_chi2_sf(x, d)] for x, d in
                    ((1000.0, 999), (50.0, 10), (0.5, 3), (842.0, 999), (1156.0, 999))],
    }
    return out


N4_CASES = [
    # name, n, dtype, p, f, mode, seed, stream, count
    ("C1", 4, O.F64, 12, 1, O.CHISQ, 12345, 0, 2 * 16383 + 9),
    ("C2_head", 4, O.F64, 20, 2, O.CHISQ, 7, 0, 6000),
    ("C3_cta0", 4, O.F32, 10, 1, O.CHISQ, 2024, 0, 3 * 4095 + 3),
    ("C3_cta1183", 4, O.F32, 10, 1, O.CHISQ, 2024, 1183, 4095),
    ("C4_rank7_cta5", 4, O.F32, 10, 1, O.CHISQ, 106, 5, 4095),
    ("C5_f64_fixed_p8_R3", 4, O.F64, 8, 3, O.FIXED, 2024, 0, 2 * 1023 + 1),
    ("C5_f32_p12_R4", 4, O.F32, 12, 4, O.CHISQ, 2024, 2, 16383),
    ("n2_f32", 2, O.F32, 10, 2, O.CHISQ, 3, 0, 3000),
    ("drift_crossing_n4", 4, O.F64, 8, 1, O.CHISQ, 11, 0, 70 * 1023),
]


def n4_golden():
    out = {"source": "oracle/liboracle.so (restatement; parity unpinned by reference tests)",
           "cases": []}
    for name, n, dt, p, f, mode, seed, stream, count in N4_CASES:
        st = O.OracleState(pool_exponent=p, throwaway_f=f, scale_mode=mode, seed=seed,
                           stream=stream, n_arrays=n, dtype=dt)
        pool0, tracked0, withheld0 = st.pool()
        twin = O.OracleState(pool_exponent=p, throwaway_f=f, scale_mode=mode, seed=seed,
                             stream=stream, n_arrays=n, dtype=dt)
        params = [params_dict(twin.advance_pass(), n) for _ in range(2)]
        v = st.fill(count)
        pool1, tracked1, withheld1 = st.pool()
        m = O.moments(v)
        out["cases"].append({
            "name": name, "n_arrays": n, "dtype": "f64" if dt == O.F64 else "f32",
            "pool_exponent": p, "throwaway_f": f, "scale_mode": mode, "seed": seed,
            "stream": stream, "count": count,
            "init_tracked_hex": tracked0.hex(), "init_withheld_hex": withheld0.hex(),
            "init_pool_sha256": h(pool0),
            "params": params,
            "fill_head_hex": [float(x).hex() for x in v[:16]],
            "fill_sha256": h(v),
            "counters": st.counters(),
            "final_tracked_hex": tracked1.hex(), "final_withheld_hex": withheld1.hex(),
            "final_pool_sha256": h(pool1),
            "moments": {k: (float(x).hex() if k != "n" else x) for k, x in m.items()},
            "anderson_darling_hex": O.anderson_darling(v).hex(),
        })
    return out


def main():
    os.makedirs(GOLDEN, exist_ok=True)
    O.build()
    if O.ref_available():
        with open(os.path.join(GOLDEN, "golden_ref.json"), "w") as fh:
            json.dump(ref_golden(), fh, indent=1)
    else:
        print("reference library not built; golden_ref.json left unchanged")
    with open(os.path.join(GOLDEN, "golden_n4.json"), "w") as fh:
        json.dump(n4_golden(), fh, indent=1)
    print("wrote", os.listdir(GOLDEN))


if __name__ == "__main__":
    main()
