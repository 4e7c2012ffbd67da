"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU checkers.

* ``Oracle``  — oracle/liboracle.so, the C restatement (wallace_oracle.c).
* ``Ref``     — oracle/_ref/libwrng_ref.so, the UNMODIFIED reference library
  (/root/reference/proj/src) behind our extern "C" shim (ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
``--impl reference`` arm) may import this module.  The product package never
does: it fails loudly when its CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwrng_ref.so")

OK, EINVAL, ECORRUPT = 0, 1, 2
F64, F32 = 0, 1
CHISQ, FIXED = 0, 1


class Params(C.Structure):
    """Flat PassParams (wallace.hpp:22-30); shared by oracle, ref shim and product."""

    _fields_ = [
        ("stride", C.c_uint32 * 4),
        ("offset", C.c_uint32 * 4),
        ("variant", C.c_uint32),
        ("pad_", C.c_uint32),
        ("c", C.c_double),
        ("s", C.c_double),
        ("scale", C.c_double),
        ("target", C.c_double),
    ]

    def as_dict(self, n_arrays: int = 4) -> dict:
        return {
            "stride": list(self.stride)[:n_arrays],
            "offset": list(self.offset)[:n_arrays],
            "variant": int(self.variant),
            "c": float(self.c),
            "s": float(self.s),
            "scale": float(self.scale),
            "target": float(self.target),
        }


class OrConfig(C.Structure):
    _fields_ = [
        ("n_arrays", C.c_uint32),
        ("dtype", C.c_uint32),
        ("pool_exponent", C.c_uint32),
        ("throwaway_f", C.c_uint32),
        ("scale_mode", C.c_uint32),
        ("restart_interval", C.c_uint64),
        ("drift_period", C.c_uint64),
        ("seed", C.c_uint64),
        ("stream", C.c_uint64),
    ]


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def build(quiet: bool = True) -> None:
    """Build liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_oracle_lib = None
_ref_lib = None


def oracle_lib():
    global _oracle_lib
    if _oracle_lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        u64, u32, dbl, vp = C.c_uint64, C.c_uint32, C.c_double, C.c_void_p
        lib.or_next_word.restype = u64
        lib.or_next_word.argtypes = [vp]
        lib.or_next_uniform.restype = dbl
        lib.or_next_uniform.argtypes = [vp]
        lib.or_next_int_below.argtypes = [vp, u32, C.POINTER(u32)]
        lib.or_uniform_init.argtypes = [vp, u64, u64]
        lib.or_chi2_target.restype = dbl
        lib.or_chi2_target.argtypes = [dbl, u32]
        lib.or_rotation_from_t.argtypes = [dbl, u32, C.POINTER(dbl), C.POINTER(dbl)]
        lib.or_box_muller_pair.argtypes = [dbl, dbl, C.POINTER(dbl), C.POINTER(dbl)]
        lib.or_select_params.argtypes = [vp, u32, u32, dbl, dbl, u32, C.POINTER(Params)]
        lib.or_regenerate.argtypes = [u32, u32, u32, vp, vp, C.POINTER(Params)]
        lib.or_direct_sumsq.restype = dbl
        lib.or_direct_sumsq.argtypes = [u32, u32, u32, vp]
        lib.or_state_create.argtypes = [C.POINTER(OrConfig), C.POINTER(vp)]
        lib.or_state_destroy.argtypes = [vp]
        lib.or_state_advance_pass.argtypes = [vp, C.POINTER(Params)]
        lib.or_state_refill.argtypes = [vp]
        lib.or_state_fill_f64.argtypes = [vp, vp, C.c_size_t, dbl, dbl]
        lib.or_state_fill_f32.argtypes = [vp, vp, C.c_size_t, dbl, dbl]
        lib.or_state_drift_check.argtypes = [vp]
        lib.or_state_restart.argtypes = [vp]
        lib.or_state_counters.argtypes = [vp, vp]
        lib.or_state_get_pool.argtypes = [vp, vp, vp]
        lib.or_state_set_pool.argtypes = [vp, vp, vp]
        lib.or_state_get_uniform.argtypes = [vp, vp, C.POINTER(u32), C.POINTER(u32),
                                             C.POINTER(u64)]
        lib.or_bank_fill_f32.argtypes = [C.POINTER(OrConfig), u32, u64, vp, dbl, dbl]
        lib.or_bank_fill_f64.argtypes = [C.POINTER(OrConfig), u32, u64, vp, dbl, dbl]
        lib.or_bench_threads.restype = dbl
        lib.or_bench_threads.argtypes = [C.POINTER(OrConfig), u32, u64, u32]
        lib.or_moments_f64.argtypes = [vp, C.c_size_t, vp]
        lib.or_moments_f32.argtypes = [vp, C.c_size_t, vp]
        lib.or_anderson_darling_f64.restype = dbl
        lib.or_anderson_darling_f64.argtypes = [vp, C.c_size_t]
        lib.or_ad_sorted_threads.restype = dbl
        lib.or_ad_sorted_threads.argtypes = [vp, C.c_size_t, C.c_int]
        lib.or_ad_sorted_f32_threads.restype = dbl
        lib.or_ad_sorted_f32_threads.argtypes = [vp, C.c_size_t, C.c_int]
        lib.or_anderson_darling_f32.restype = dbl
        lib.or_anderson_darling_f32.argtypes = [vp, C.c_size_t]
        lib.or_method_bank_fill.argtypes = [C.c_int, u64, u64, u32, u64, vp]
        lib.or_to_uv.argtypes = [dbl, dbl, C.POINTER(dbl), C.POINTER(dbl)]
        lib.or_chi2_bin.restype = C.c_int64
        lib.or_chi2_bin.argtypes = [dbl, u32, dbl, dbl]
        for nm in ("or_uv_counts_f64", "or_uv_counts_f32"):
            getattr(lib, nm).restype = u64
            getattr(lib, nm).argtypes = [vp, C.c_size_t, u32, vp, vp]
        lib.or_chi2_statistic.restype = dbl
        lib.or_chi2_statistic.argtypes = [vp, u32]
        lib.or_chi2_sf.restype = dbl
        lib.or_chi2_sf.argtypes = [dbl, u32]
        for nm in ("or_autocorr_f64", "or_autocorr_f32"):
            getattr(lib, nm).restype = dbl
            getattr(lib, nm).argtypes = [vp, C.c_size_t, C.c_size_t]
        _oracle_lib = lib
    return _oracle_lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref_lib
    if _ref_lib is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference)")
        lib = C.CDLL(REF_SO)
        u64, u32, u8, dbl, vp = C.c_uint64, C.c_uint32, C.c_uint8, C.c_double, C.c_void_p
        lib.ref_uniform_create.restype = vp
        lib.ref_uniform_create.argtypes = [u64, u64]
        lib.ref_uniform_destroy.argtypes = [vp]
        lib.ref_uniform_next_word.restype = u64
        lib.ref_uniform_next_word.argtypes = [vp]
        lib.ref_uniform_next_uniform.restype = dbl
        lib.ref_uniform_next_uniform.argtypes = [vp]
        lib.ref_uniform_next_int_below.argtypes = [vp, u32, C.POINTER(u32)]
        lib.ref_uniform_get.argtypes = [vp, vp, C.POINTER(u32), C.POINTER(u32),
                                        C.POINTER(u64)]
        lib.ref_uniform_set.argtypes = [vp, vp, u32, u32, u64]
        lib.ref_chi2_target.restype = dbl
        lib.ref_chi2_target.argtypes = [dbl, u32]
        lib.ref_rotation_from_t.argtypes = [dbl, u32, C.POINTER(dbl), C.POINTER(dbl)]
        lib.ref_box_muller_pair.argtypes = [dbl, dbl, C.POINTER(dbl), C.POINTER(dbl)]
        lib.ref_box_muller_fill.argtypes = [vp, vp, C.c_size_t, dbl, dbl]
        lib.ref_select_pass_params.argtypes = [vp, u32, dbl, dbl, u8, C.POINTER(Params)]
        lib.ref_regenerate.argtypes = [u32, vp, vp, vp, vp, C.POINTER(Params),
                                       C.POINTER(dbl), C.POINTER(dbl)]
        lib.ref_moments.argtypes = [vp, C.c_size_t, vp]
        lib.ref_polar_fill.argtypes = [vp, vp, C.c_size_t, dbl, dbl]
        lib.ref_bench_methods.restype = dbl
        lib.ref_bench_methods.argtypes = [C.c_int, u32, u64, u64]
        lib.ref_uv_chi2.argtypes = [vp, C.c_size_t, u32, vp]
        lib.ref_chi2_sf.argtypes = [dbl, u32, C.POINTER(dbl)]
        lib.ref_autocorr.argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(dbl)]
        lib.ref_state_create.argtypes = [u32, u32, u8, u64, u64, u64, u64, C.POINTER(vp)]
        lib.ref_state_destroy.argtypes = [vp]
        lib.ref_state_fill.argtypes = [vp, vp, C.c_size_t, dbl, dbl]
        lib.ref_state_advance_pass.argtypes = [vp, C.POINTER(Params)]
        lib.ref_state_refill.argtypes = [vp]
        lib.ref_state_drift_check.argtypes = [vp]
        lib.ref_state_restart.argtypes = [vp]
        lib.ref_state_counters.argtypes = [vp, vp]
        lib.ref_state_get_pool.argtypes = [vp, vp, vp, vp]
        lib.ref_state_set_pool.argtypes = [vp, vp, vp, vp]
        lib.ref_state_uniform.argtypes = [vp, vp, C.POINTER(u32), C.POINTER(u32),
                                          C.POINTER(u64)]
        lib.ref_state_save.restype = C.c_size_t
        lib.ref_state_save.argtypes = [vp, vp, C.c_size_t]
        lib.ref_state_load.argtypes = [vp, C.c_size_t, C.POINTER(vp)]
        lib.ref_bench_threads.restype = dbl
        lib.ref_bench_threads.argtypes = [u32, u32, u8, u64, u64, u32, u64, u32]
        lib.ref_bench_array.restype = dbl
        lib.ref_bench_array.argtypes = [u32, u32, u8, u64, u64, u32, u64, u64,
                                        C.c_void_p]
        _ref_lib = lib
    return _ref_lib


# ---------------------------------------------------------------------------
# Object wrappers
# ---------------------------------------------------------------------------
class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(rc, what)


class OracleUniform:
    """or_uniform — UniformState restated (uniform.cpp:23-51)."""

    class _S(C.Structure):
        _fields_ = [("table", C.c_uint64 * 607), ("r", C.c_uint32), ("s", C.c_uint32),
                    ("seed", C.c_uint64), ("stream", C.c_uint64), ("draws", C.c_uint64)]

    def __init__(self, seed: int, stream: int = 0):
        self.lib = oracle_lib()
        self.s = self._S()
        self.lib.or_uniform_init(C.byref(self.s), seed, stream)

    def next_word(self) -> int:
        return self.lib.or_next_word(C.byref(self.s))

    def next_uniform(self) -> float:
        return self.lib.or_next_uniform(C.byref(self.s))

    def next_int_below(self, m: int) -> int:
        out = C.c_uint32()
        _check(self.lib.or_next_int_below(C.byref(self.s), m, C.byref(out)), "next_int_below")
        return out.value

    @property
    def table(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.s.table).copy()


class OracleState:
    """or_state — WallaceState restated, n in {2, 4}, dtype in {f64, f32}."""

    def __init__(self, pool_exponent=10, throwaway_f=3, scale_mode=CHISQ,
                 restart_interval=0, drift_period=64, seed=0, stream=0,
                 n_arrays=2, dtype=F64):
        self.lib = oracle_lib()
        self.cfg = OrConfig(n_arrays, dtype, pool_exponent, throwaway_f, scale_mode,
                            restart_interval, drift_period, seed, stream)
        self.h = C.c_void_p()
        _check(self.lib.or_state_create(C.byref(self.cfg), C.byref(self.h)), "create")
        self.n_arrays, self.dtype, self.N = n_arrays, dtype, 1 << pool_exponent

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.or_state_destroy(self.h)
            self.h = None

    def fill(self, count: int, mu=0.0, sigma=1.0, out_dtype=None) -> np.ndarray:
        out_dtype = out_dtype or (np.float64 if self.dtype == F64 else np.float32)
        out = np.empty(count, dtype=out_dtype)
        fn = self.lib.or_state_fill_f64 if out_dtype == np.float64 else self.lib.or_state_fill_f32
        _check(fn(self.h, out.ctypes.data, count, mu, sigma), "fill")
        return out

    def advance_pass(self) -> Params:
        p = Params()
        _check(self.lib.or_state_advance_pass(self.h, C.byref(p)), "advance_pass")
        return p

    def refill(self):
        _check(self.lib.or_state_refill(self.h), "refill")

    def drift_check(self):
        _check(self.lib.or_state_drift_check(self.h), "drift_check")

    def restart(self):
        self.lib.or_state_restart(self.h)

    def counters(self):
        c = np.zeros(4, dtype=np.uint64)
        self.lib.or_state_counters(self.h, c.ctypes.data)
        return {"pass_count": int(c[0]), "numbers_emitted": int(c[1]),
                "avail": int(c[2]), "pool_size": int(c[3])}

    def pool(self):
        v = np.empty(self.n_arrays * self.N, dtype=np.float64)
        tw = np.empty(2, dtype=np.float64)
        self.lib.or_state_get_pool(self.h, v.ctypes.data, tw.ctypes.data)
        return v, float(tw[0]), float(tw[1])

    def set_pool(self, vals: np.ndarray, tracked: float, withheld: float):
        v = np.ascontiguousarray(vals, dtype=np.float64)
        tw = np.array([tracked, withheld], dtype=np.float64)
        self.lib.or_state_set_pool(self.h, v.ctypes.data, tw.ctypes.data)

    def uniform(self):
        t = np.empty(607, dtype=np.uint64)
        r, s, d = C.c_uint32(), C.c_uint32(), C.c_uint64()
        self.lib.or_state_get_uniform(self.h, t.ctypes.data, C.byref(r), C.byref(s), C.byref(d))
        return t, r.value, s.value, d.value


def bank_fill(count: int, pools: int, *, seed: int, stream: int = 0, pool_exponent=10,
              throwaway_f=1, scale_mode=CHISQ, drift_period=64, restart_interval=0,
              n_arrays=4, dtype=F32, mu=0.0, sigma=1.0) -> np.ndarray:
    lib = oracle_lib()
    cfg = OrConfig(n_arrays, dtype, pool_exponent, throwaway_f, scale_mode,
                   restart_interval, drift_period, seed, stream)
    out = np.empty(count, dtype=np.float32 if dtype == F32 else np.float64)
    fn = lib.or_bank_fill_f32 if dtype == F32 else lib.or_bank_fill_f64
    _check(fn(C.byref(cfg), pools, count, out.ctypes.data, mu, sigma), "bank_fill")
    return out


def moments(v: np.ndarray) -> dict:
    lib = oracle_lib()
    out = np.zeros(5, dtype=np.float64)
    v = np.ascontiguousarray(v)
    fn = lib.or_moments_f64 if v.dtype == np.float64 else lib.or_moments_f32
    fn(v.ctypes.data, v.size, out.ctypes.data)
    return {"n": int(out[0]), "m1": out[1], "m2": out[2], "m3": out[3], "m4": out[4]}


def anderson_darling(v: np.ndarray) -> float:
    lib = oracle_lib()
    v = np.ascontiguousarray(v)
    fn = lib.or_anderson_darling_f64 if v.dtype == np.float64 else lib.or_anderson_darling_f32
    return float(fn(v.ctypes.data, v.size))


def anderson_darling_sorted(z: np.ndarray, threads: int = 0) -> float:
    """A^2 of an already sorted float32/float64 sample on `threads` host threads
    (same d_j sum as anderson_darling; for 2^32-value samples)."""
    lib = oracle_lib()
    th = threads or (os.cpu_count() or 1)
    if z.dtype == np.float32:
        z = np.ascontiguousarray(z)
        return float(lib.or_ad_sorted_f32_threads(z.ctypes.data, z.size, th))
    z = np.ascontiguousarray(z, dtype=np.float64)
    return float(lib.or_ad_sorted_threads(z.ctypes.data, z.size, th))


def method_bank_fill(method: str, seed: int, stream0: int, pools: int, count: int) -> np.ndarray:
    """Box-Muller ("boxmuller") or polar ("polar") fills of `pools` fresh
    UniformState(seed, stream0 + p) streams, pool-major (reference.cpp:41-63)."""
    out = np.empty(count, dtype=np.float64)
    oracle_lib().or_method_bank_fill(0 if method == "boxmuller" else 1, seed, stream0, pools,
                                     count, out.ctypes.data)
    return out


def uv_counts(v: np.ndarray, k: int):
    """Pairs (v[2i], v[2i+1]) -> to_uv -> k-bin counts of u and v
    (stats.cpp:10-38 as tools/main.cpp:160-193 uses them)."""
    lib = oracle_lib()
    v = np.ascontiguousarray(v)
    cu = np.zeros(k, dtype=np.uint64)
    cv = np.zeros(k, dtype=np.uint64)
    fn = lib.or_uv_counts_f64 if v.dtype == np.float64 else lib.or_uv_counts_f32
    skipped = int(fn(v.ctypes.data, v.size, k, cu.ctypes.data, cv.ctypes.data))
    return cu, cv, skipped


def chi2_statistic(counts: np.ndarray) -> float:
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    return float(oracle_lib().or_chi2_statistic(c.ctypes.data, c.size))


def chi2_sf(statistic: float, dof: int) -> float:
    return float(oracle_lib().or_chi2_sf(statistic, dof))


def autocorr(v: np.ndarray, lag: int) -> float:
    lib = oracle_lib()
    v = np.ascontiguousarray(v)
    fn = lib.or_autocorr_f64 if v.dtype == np.float64 else lib.or_autocorr_f32
    return float(fn(v.ctypes.data, v.size, lag))


def ref_uv_chi2(v: np.ndarray, k: int) -> dict:
    """The reference's own to_uv + chi2_bins on float64 values."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros(6, dtype=np.float64)
    _check(ref_lib().ref_uv_chi2(v.ctypes.data, v.size, k, out.ctypes.data), "ref_uv_chi2")
    return {"u_statistic": out[0], "u_p": out[1], "v_statistic": out[2], "v_p": out[3],
            "samples": int(out[4]), "dof": int(out[5])}


def ref_chi2_sf(statistic: float, dof: int) -> float:
    r = C.c_double()
    _check(ref_lib().ref_chi2_sf(statistic, dof, C.byref(r)), "ref_chi2_sf")
    return r.value


def ref_autocorr(v: np.ndarray, lag: int) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    r = C.c_double()
    _check(ref_lib().ref_autocorr(v.ctypes.data, v.size, lag, C.byref(r)), "ref_autocorr")
    return r.value


class RefUniform:
    def __init__(self, seed: int, stream: int = 0):
        self.lib = ref_lib()
        self.h = self.lib.ref_uniform_create(seed, stream)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_uniform_destroy(self.h)
            self.h = None

    def next_word(self) -> int:
        return self.lib.ref_uniform_next_word(self.h)

    def next_uniform(self) -> float:
        return self.lib.ref_uniform_next_uniform(self.h)

    def next_int_below(self, m: int) -> int:
        out = C.c_uint32()
        _check(self.lib.ref_uniform_next_int_below(self.h, m, C.byref(out)), "next_int_below")
        return out.value

    def get(self):
        t = np.empty(607, dtype=np.uint64)
        r, s, d = C.c_uint32(), C.c_uint32(), C.c_uint64()
        self.lib.ref_uniform_get(self.h, t.ctypes.data, C.byref(r), C.byref(s), C.byref(d))
        return t, r.value, s.value, d.value

    def box_muller_fill(self, n: int, mu=0.0, sigma=1.0) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.lib.ref_box_muller_fill(self.h, out.ctypes.data, n, mu, sigma)
        return out

    def polar_fill(self, n: int, mu=0.0, sigma=1.0) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.lib.ref_polar_fill(self.h, out.ctypes.data, n, mu, sigma)
        return out


def ref_bench_methods(method: str, threads: int, per_thread: int, seed: int = 1) -> float:
    """Wall seconds for `threads` reference Box-Muller / polar streams of
    per_thread values each (64Ki-value fill calls)."""
    return float(ref_lib().ref_bench_methods(0 if method == "boxmuller" else 1, threads,
                                             per_thread, seed))


class RefState:
    """The reference's WallaceState (n = 2, fp64) through the shim."""

    def __init__(self, pool_exponent=10, throwaway_f=3, scale_mode=CHISQ,
                 restart_interval=0, drift_period=64, seed=0, stream=0, _handle=None):
        self.lib = ref_lib()
        self.h = C.c_void_p()
        if _handle is not None:
            self.h = _handle
        else:
            _check(self.lib.ref_state_create(pool_exponent, throwaway_f, scale_mode,
                                             restart_interval, drift_period, seed, stream,
                                             C.byref(self.h)), "ref create")
        self.N = self.counters()["pool_size"]

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_state_destroy(self.h)
            self.h = None

    def fill(self, count: int, mu=0.0, sigma=1.0) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        _check(self.lib.ref_state_fill(self.h, out.ctypes.data, count, mu, sigma), "fill")
        return out

    def advance_pass(self) -> Params:
        p = Params()
        _check(self.lib.ref_state_advance_pass(self.h, C.byref(p)), "advance_pass")
        return p

    def refill(self):
        _check(self.lib.ref_state_refill(self.h), "refill")

    def drift_check(self):
        _check(self.lib.ref_state_drift_check(self.h), "drift_check")

    def restart(self):
        self.lib.ref_state_restart(self.h)

    def counters(self):
        c = np.zeros(4, dtype=np.uint64)
        self.lib.ref_state_counters(self.h, c.ctypes.data)
        return {"pass_count": int(c[0]), "numbers_emitted": int(c[1]),
                "avail": int(c[2]), "pool_size": int(c[3])}

    def pool(self):
        x = np.empty(self.N)
        y = np.empty(self.N)
        tw = np.empty(2)
        self.lib.ref_state_get_pool(self.h, x.ctypes.data, y.ctypes.data, tw.ctypes.data)
        return np.concatenate([x, y]), float(tw[0]), float(tw[1])

    def set_pool(self, vals, tracked, withheld):
        v = np.ascontiguousarray(vals, dtype=np.float64)
        tw = np.array([tracked, withheld])
        x = np.ascontiguousarray(v[: self.N])
        y = np.ascontiguousarray(v[self.N:])
        self.lib.ref_state_set_pool(self.h, x.ctypes.data, y.ctypes.data, tw.ctypes.data)

    def uniform(self):
        t = np.empty(607, dtype=np.uint64)
        r, s, d = C.c_uint32(), C.c_uint32(), C.c_uint64()
        self.lib.ref_state_uniform(self.h, t.ctypes.data, C.byref(r), C.byref(s), C.byref(d))
        return t, r.value, s.value, d.value

    def save_state(self) -> bytes:
        n = self.lib.ref_state_save(self.h, None, 0)
        buf = (C.c_uint8 * n)()
        self.lib.ref_state_save(self.h, buf, n)
        return bytes(buf)

    @classmethod
    def load_state(cls, data: bytes) -> "RefState":
        lib = ref_lib()
        h = C.c_void_p()
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        _check(lib.ref_state_load(buf, len(data), C.byref(h)), "load_state")
        return cls(_handle=h)


def ref_bench_array(pool_exponent, f, mode, seed, stream0, threads, per_thread, out,
                    chunk=1 << 16) -> float:
    """Reference threads filling their segments of one host array `out`
    (float64, >= threads * per_thread values); returns wall seconds."""
    assert out.dtype == np.float64 and out.size >= threads * per_thread
    return ref_lib().ref_bench_array(pool_exponent, f, mode, seed, stream0, threads,
                                     per_thread, chunk, out.ctypes.data)


def ref_bench_threads(pool_exponent, f, mode, seed, stream0, threads, per_thread,
                      chunk=1 << 16) -> float:
    return ref_lib().ref_bench_threads(pool_exponent, f, mode, seed, stream0, threads,
                                       per_thread, chunk)
