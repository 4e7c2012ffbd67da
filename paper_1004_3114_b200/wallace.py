"""Python mirror of the reference generator interface over the GPU C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/wrng/wallace.hpp (WallaceConfig, ScaleMode,
PassParams, Pool, WallaceState) and errors.hpp (corrupted_state_error,
malformed_state_error{kind}); std::invalid_argument maps to ValueError.  The
C++ mirror for C++ callers is include/wrng_gpu/wallace.hpp.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Union

import numpy as np

from . import _lib as L

lib = L.lib


class ScaleMode(enum.IntEnum):  # wallace.hpp:52-55
    chisq = 0
    fixed = 1


class StateErrorKind(enum.IntEnum):  # errors.hpp:15-20
    bad_magic = 0
    unsupported_version = 1
    truncated = 2
    field_range = 3


class CorruptedStateError(RuntimeError):
    """wrng::corrupted_state_error (errors.hpp:10-13)."""


class MalformedStateError(RuntimeError):
    """wrng::malformed_state_error (errors.hpp:22-32)."""

    def __init__(self, kind: StateErrorKind, what: str):
        super().__init__(what)
        self.kind = kind


class CudaError(RuntimeError):
    """Device-side failure (no reference analogue)."""


_MALFORMED = {
    L.EMALFORMED_BAD_MAGIC: StateErrorKind.bad_magic,
    L.EMALFORMED_VERSION: StateErrorKind.unsupported_version,
    L.EMALFORMED_TRUNCATED: StateErrorKind.truncated,
    L.EMALFORMED_FIELD_RANGE: StateErrorKind.field_range,
}


def _raise(rc: int, what: str, h=None):
    if rc == L.OK:
        return
    msg = what
    if h is not None:
        detail = lib.wrng_gpu_last_error(h)
        if detail:
            msg = f"{what}: {detail.decode()}"
    if rc == L.EINVAL:
        raise ValueError(msg)
    if rc == L.ECORRUPT:
        raise CorruptedStateError(msg)
    if rc in _MALFORMED:
        raise MalformedStateError(_MALFORMED[rc], msg)
    raise CudaError(f"{msg} (status {rc})")


@dataclass
class WallaceConfig:
    """wallace.hpp:57-65, plus the B200 extensions (n_arrays, dtype, pools, ...)."""

    pool_exponent: int = 10
    throwaway_f: int = 3
    scale_mode: ScaleMode = ScaleMode.chisq
    restart_interval_passes: int = 0
    drift_check_period: int = 64
    seed: int = 0
    stream_id: int = 0
    # extensions
    n_arrays: int = 2          # 2 (reference) or 4 (docs/n4_spec.md)
    dtype: str = "f64"         # "f64" | "f32"
    pools: int = 1             # independent pools, pool p = stream_id + p
    device: int = 0
    # glibc Box-Muller for the initial pool and every restart: bit-exact with
    # the reference (default, as in the C++ drop-in); False runs it on the
    # device (CUDA libm, within a few ulp of glibc)
    init_on_host: bool = True
    force_hbm: bool = False     # HBM-resident engine even when smem would fit
    drift_tree: bool = False    # parallel (non-reference-order) drift sum

    def to_c(self) -> L.Config:
        c = L.Config()
        lib.wrng_gpu_config_default(C.byref(c))
        c.pool_exponent = self.pool_exponent
        c.throwaway_f = self.throwaway_f
        c.scale_mode = int(self.scale_mode)
        c.restart_interval_passes = self.restart_interval_passes
        c.drift_check_period = self.drift_check_period
        c.seed = self.seed & (2**64 - 1)
        c.stream_id = self.stream_id & (2**64 - 1)
        c.n_arrays = self.n_arrays
        c.dtype = L.F64 if self.dtype == "f64" else L.F32
        c.pools = self.pools
        c.device = self.device
        c.flags = ((L.FLAG_INIT_HOST if self.init_on_host else 0)
                   | (L.FLAG_FORCE_HBM if self.force_hbm else 0)
                   | (L.FLAG_DRIFT_TREE if self.drift_tree else 0))
        return c

    @classmethod
    def from_c(cls, c: L.Config) -> "WallaceConfig":
        return cls(pool_exponent=c.pool_exponent, throwaway_f=c.throwaway_f,
                   scale_mode=ScaleMode(c.scale_mode),
                   restart_interval_passes=c.restart_interval_passes,
                   drift_check_period=c.drift_check_period, seed=c.seed,
                   stream_id=c.stream_id, n_arrays=c.n_arrays,
                   dtype="f64" if c.dtype == L.F64 else "f32", pools=c.pools,
                   device=c.device, init_on_host=bool(c.flags & L.FLAG_INIT_HOST),
                   force_hbm=bool(c.flags & L.FLAG_FORCE_HBM),
                   drift_tree=bool(c.flags & L.FLAG_DRIFT_TREE))


@dataclass
class Rotation2:  # wallace.hpp:14-17
    c: float
    s: float


@dataclass
class PassParams:
    """wallace.hpp:22-30; n = 4 adds strides[2:], offsets[2:] and `variant`."""

    alpha: int
    beta: int
    gamma: int
    delta: int
    rot: Rotation2
    scale: float
    target_sumsq: float
    strides: List[int] = field(default_factory=list)
    offsets: List[int] = field(default_factory=list)
    variant: int = 0

    @classmethod
    def from_c(cls, p: L.Params, n_arrays: int) -> "PassParams":
        return cls(alpha=p.stride[0], beta=p.stride[1], gamma=p.offset[0], delta=p.offset[1],
                   rot=Rotation2(p.c, p.s), scale=p.scale, target_sumsq=p.target_sumsq,
                   strides=list(p.stride)[:n_arrays], offsets=list(p.offset)[:n_arrays],
                   variant=p.variant)


@dataclass
class Pool:
    """wallace.hpp:36-50: the live pool as host arrays (arrays[m] is x_m)."""

    arrays: np.ndarray  # (n_arrays, N) float64
    tracked_sumsq: float
    withheld: float

    @property
    def x(self) -> np.ndarray:
        return self.arrays[0]

    @property
    def y(self) -> np.ndarray:
        return self.arrays[1]

    def n(self) -> int:
        return self.arrays.shape[1]

    def direct_sumsq(self) -> float:
        """Sequential sum, arrays in order (wallace.hpp:44-46)."""
        q = 0.0
        for v in self.arrays.reshape(-1).tolist():
            q += v * v
        return q

    def max_abs(self) -> float:
        return float(np.max(np.abs(self.arrays)))


@dataclass
class UniformStateView:
    """uniform.hpp:16-29 snapshot."""

    lag_table: np.ndarray
    cursor_r: int
    cursor_s: int
    draws: int


# ---- the reference's free functions (wallace.hpp:77-111, uniform.hpp) -------
class UniformState:
    """uniform.hpp:16-40 on the host (seeded by wrng_gpu_uniform_seed; the
    per-word recurrence mirrors uniform.cpp:34-51)."""

    def __init__(self, seed: int = 0, stream_id: int = 0):
        self._s = L.Uniform()
        lib.wrng_gpu_uniform_seed(C.byref(self._s), seed & (2**64 - 1), stream_id & (2**64 - 1))

    @property
    def lag_table(self) -> np.ndarray:
        return np.ctypeslib.as_array(self._s.lag_table).copy()

    cursor_r = property(lambda self: self._s.cursor_r)
    cursor_s = property(lambda self: self._s.cursor_s)
    draws = property(lambda self: self._s.draws)
    seed = property(lambda self: self._s.seed)
    stream_id = property(lambda self: self._s.stream_id)

    def next_word(self) -> int:
        s = self._s
        w = (s.lag_table[s.cursor_r] + s.lag_table[s.cursor_s]) & (2**64 - 1)
        s.lag_table[s.cursor_r] = w
        s.cursor_r = 0 if s.cursor_r + 1 == 607 else s.cursor_r + 1
        s.cursor_s = 0 if s.cursor_s + 1 == 607 else s.cursor_s + 1
        return w

    def next_uniform(self) -> float:
        self._s.draws += 1
        return float(self.next_word() >> 11) * 2.0 ** -53

    def next_int_below(self, m: int) -> int:
        if m < 1 or m > (1 << 20):
            raise ValueError("next_int_below: m must be in [1, 2^20]")
        return int(self.next_uniform() * m)


def chi2_target(r: float, nu: int) -> float:
    """wallace.cpp:27-31."""
    return float(lib.wrng_gpu_chi2_target(r, nu))


def rotation_from_t(t: float, region: int) -> Rotation2:
    """wallace.cpp:33-42."""
    c, s = C.c_double(), C.c_double()
    lib.wrng_gpu_rotation_from_t(t, region, C.byref(c), C.byref(s))
    return Rotation2(c.value, s.value)


def rotation_from_uniform(us: UniformState) -> Rotation2:
    """wallace.cpp:44-49."""
    c, s = C.c_double(), C.c_double()
    lib.wrng_gpu_rotation_from_uniform(C.byref(us._s), C.byref(c), C.byref(s))
    return Rotation2(c.value, s.value)


def select_pass_params(us: UniformState, pool: "Pool", mode: ScaleMode = ScaleMode.chisq):
    """wallace.cpp:51-70 (n = 4 pools: docs/n4_spec.md §2)."""
    p = L.Params()
    na, n = pool.arrays.shape
    _raise(lib.wrng_gpu_select_pass_params(C.byref(us._s), na, n, int(mode), pool.tracked_sumsq,
                                           pool.withheld, C.byref(p)), "select_pass_params")
    return PassParams.from_c(p, na)


def _params_c(p: "PassParams", n_arrays: int) -> L.Params:
    c = L.Params()
    if n_arrays == 2:
        c.stride[0], c.stride[1], c.offset[0], c.offset[1] = p.alpha, p.beta, p.gamma, p.delta
    else:
        for m in range(4):
            c.stride[m], c.offset[m] = p.strides[m], p.offsets[m]
        c.variant = p.variant
    c.c, c.s, c.scale, c.target_sumsq = p.rot.c, p.rot.s, p.scale, p.target_sumsq
    return c


def plan_segments(params: "PassParams", n: int) -> list:
    """wallace.cpp:72-111: [(low, high, jx, jy), ...]."""
    c = _params_c(params, 2)
    cnt = C.c_uint32()
    _raise(lib.wrng_gpu_plan_segments(C.byref(c), n, None, 0, C.byref(cnt)), "plan_segments")
    segs = (L.Segment * cnt.value)()
    _raise(lib.wrng_gpu_plan_segments(C.byref(c), n, segs, cnt.value, C.byref(cnt)),
           "plan_segments")
    return [(s.low, s.high, s.jx, s.jy) for s in segs]


def regenerate(src: "Pool", params: "PassParams", device: int = 0) -> "Pool":
    """One pass (wallace.cpp:113-137) of a host pool, computed on the GPU."""
    na, n = src.arrays.shape
    a = np.ascontiguousarray(src.arrays, dtype=np.float64)
    out = np.empty_like(a)
    c = _params_c(params, na)
    w = C.c_double()
    _raise(lib.wrng_gpu_regenerate(a.ctypes.data, out.ctypes.data, na, n, C.byref(c), C.byref(w),
                                   device), "regenerate")
    return Pool(out, params.target_sumsq, w.value)


def _is_device_tensor(t) -> bool:
    return hasattr(t, "data_ptr") and getattr(t, "is_cuda", False)


class WallaceState:
    """wallace.hpp:113-174 on the B200.  One handle may hold `pools`
    independent generators; every call applies to all of them, and fill
    writes pool p's stream into the p-th contiguous segment."""

    def __init__(self, config: Optional[WallaceConfig] = None, *, _handle=None):
        if _handle is not None:
            self._h = _handle
            c = L.Config()
            _raise(lib.wrng_gpu_get_config(self._h, C.byref(c)), "get_config")
            self._cfg = WallaceConfig.from_c(c)
            return
        self._cfg = config or WallaceConfig()
        c = self._cfg.to_c()
        h = C.c_void_p()
        _raise(lib.wrng_gpu_create(C.byref(c), C.byref(h)), "WallaceState")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.wrng_gpu_destroy(h)
            self._h = None

    # ---- generation -------------------------------------------------------
    def fill(self, out: Union[int, np.ndarray, "object"], mu: float = 0.0,
             sigma: float = 1.0, *, dtype: Optional[str] = None, stream=None):
        """fill(count) -> numpy array (host output, synchronous);
        fill(ndarray) fills a host array in place;
        fill(torch CUDA tensor) fills device memory in place, enqueued on
        `stream` (default: torch's current stream) without a host sync."""
        if isinstance(out, (int, np.integer)):
            dt = dtype or self._cfg.dtype
            arr = np.empty(int(out), dtype=np.float64 if dt == "f64" else np.float32)
            self.fill(arr, mu, sigma)
            return arr
        if isinstance(out, np.ndarray):
            if not out.flags.c_contiguous or out.dtype not in (np.float32, np.float64):
                raise ValueError("fill: contiguous float32/float64 array required")
            fn = lib.wrng_gpu_fill_f64 if out.dtype == np.float64 else lib.wrng_gpu_fill_f32
            _raise(fn(self._h, out.ctypes.data if out.size else None, out.size, mu, sigma, 0,
                      None), "fill", self._h)
            return out
        if _is_device_tensor(out):
            import torch

            if not out.is_contiguous() or out.dtype not in (torch.float32, torch.float64):
                raise ValueError("fill: contiguous float32/float64 CUDA tensor required")
            if stream is None:
                stream = torch.cuda.current_stream(out.device)
            sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
            fn = lib.wrng_gpu_fill_f64 if out.dtype == torch.float64 else lib.wrng_gpu_fill_f32
            _raise(fn(self._h, out.data_ptr() if out.numel() else None, out.numel(), mu, sigma,
                      1, sptr), "fill", self._h)
            return out
        raise TypeError("fill: expected a count, a numpy array or a CUDA tensor")

    def advance_pass(self):
        P = self._cfg.pools
        arr = (L.Params * P)()
        _raise(lib.wrng_gpu_advance_pass(self._h, arr), "advance_pass", self._h)
        out = [PassParams.from_c(arr[p], self._cfg.n_arrays) for p in range(P)]
        return out[0] if P == 1 else out

    def refill(self):
        _raise(lib.wrng_gpu_refill(self._h), "refill", self._h)

    def drift_check(self):
        _raise(lib.wrng_gpu_drift_check(self._h), "drift_check", self._h)

    def restart(self):
        _raise(lib.wrng_gpu_restart(self._h), "restart", self._h)

    def synchronize(self):
        _raise(lib.wrng_gpu_synchronize(self._h), "synchronize", self._h)

    # ---- persistence (serialize.cpp:82-169) -----------------------------------
    def save_state(self) -> bytes:
        n = C.c_size_t()
        _raise(lib.wrng_gpu_export_state(self._h, None, 0, C.byref(n)), "save_state", self._h)
        buf = (C.c_uint8 * n.value)()
        _raise(lib.wrng_gpu_export_state(self._h, buf, n.value, C.byref(n)), "save_state",
               self._h)
        return bytes(buf)

    @classmethod
    def load_state(cls, data: bytes, device: int = 0, *, force_hbm: bool = False,
                   drift_tree: bool = False, init_on_host: bool = True) -> "WallaceState":
        h = C.c_void_p()
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
        flags = ((L.FLAG_FORCE_HBM if force_hbm else 0) | (L.FLAG_DRIFT_TREE if drift_tree else 0)
                 | (L.FLAG_INIT_HOST if init_on_host else 0))
        _raise(lib.wrng_gpu_import_state(buf, len(data), device, flags, C.byref(h)),
               "load_state")
        return cls(_handle=h)

    # ---- accessors (wallace.hpp:148-160) -----------------------------------
    @property
    def config(self) -> WallaceConfig:
        return self._cfg

    def _counters(self, pool: int = 0) -> L.Counters:
        c = L.Counters()
        _raise(lib.wrng_gpu_get_counters(self._h, pool, C.byref(c)), "counters")
        return c

    def pool_size(self) -> int:
        return 1 << self._cfg.pool_exponent

    def pass_count(self, pool: int = 0) -> int:
        return self._counters(pool).pass_count

    def numbers_emitted(self, pool: int = 0) -> int:
        return self._counters(pool).numbers_emitted

    def avail(self, pool: int = 0) -> int:
        return self._counters(pool).avail

    def active_pool(self, pool: int = 0) -> Pool:
        n = self._cfg.n_arrays * self.pool_size()
        v = np.empty(n, dtype=np.float64)
        t, w = C.c_double(), C.c_double()
        _raise(lib.wrng_gpu_read_pool(self._h, pool, v.ctypes.data, C.byref(t), C.byref(w)),
               "active_pool", self._h)
        return Pool(v.reshape(self._cfg.n_arrays, -1), t.value, w.value)

    def set_active_pool(self, p: Pool, pool: int = 0):
        v = np.ascontiguousarray(p.arrays, dtype=np.float64).reshape(-1)
        _raise(lib.wrng_gpu_write_pool(self._h, pool, v.ctypes.data, p.tracked_sumsq,
                                       p.withheld), "set_active_pool", self._h)

    def uniform_state(self, pool: int = 0) -> UniformStateView:
        t = np.empty(607, dtype=np.uint64)
        r, s, d = C.c_uint32(), C.c_uint32(), C.c_uint64()
        _raise(lib.wrng_gpu_read_uniform(self._h, pool, t.ctypes.data, C.byref(r), C.byref(s),
                                         C.byref(d)), "uniform_state", self._h)
        return UniformStateView(t, r.value, s.value, d.value)

    def set_uniform_state(self, u: UniformStateView, pool: int = 0):
        """Overwrites the device uniform generator (the reference's mutable
        uniform_state(), wallace.hpp:158)."""
        t = np.ascontiguousarray(u.lag_table, dtype=np.uint64)
        _raise(lib.wrng_gpu_write_uniform(self._h, pool, t.ctypes.data, u.cursor_r, u.cursor_s,
                                          u.draws), "set_uniform_state", self._h)

    def kernel_launches(self) -> int:
        return int(lib.wrng_gpu_kernel_launches(self._h))

    def engine(self) -> str:
        return lib.wrng_gpu_engine(self._h).decode()

    @property
    def handle(self):
        return self._h


def device_moments(t, device: int = 0, stream=None) -> dict:
    """n, m1..m4 of a CUDA tensor by the device reduction (validation only)."""
    import torch

    out = np.zeros(5, dtype=np.float64)
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    fn = lib.wrng_gpu_moments_f32 if t.dtype == torch.float32 else lib.wrng_gpu_moments_f64
    _raise(fn(t.data_ptr(), t.numel(), out.ctypes.data, device, stream.cuda_stream),
           "moments")
    return {"n": int(out[0]), "m1": out[1], "m2": out[2], "m3": out[3], "m4": out[4]}


def resident_pools(config: WallaceConfig) -> int:
    """Pools the shared-memory engine keeps resident at once for fills of
    `config` on its device (SMs x CTAs per SM); 0 for HBM-engine configs.
    Banks of this size (or a multiple) run in whole waves."""
    c = config.to_c()
    r = int(lib.wrng_gpu_resident_pools(C.byref(c)))
    if r < 0:
        _raise(-r, "resident_pools")
    return r


def lfg_words(seed: int, stream_id: int, pools: int, count: int, device: int = 0) -> np.ndarray:
    """First `count` next_word() outputs of UniformState(seed, stream_id + p)."""
    out = np.empty((pools, count), dtype=np.uint64)
    _raise(lib.wrng_gpu_lfg_words(seed, stream_id, pools, count, out.ctypes.data, device),
           "lfg_words")
    return out


# ---- validation statistics on the device ---------------
def _dev_args(t, stream):
    import torch

    if not (t.is_cuda and t.is_contiguous()) or t.dtype not in (torch.float32, torch.float64):
        raise ValueError("expected a contiguous float32/float64 CUDA tensor")
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    return t.data_ptr(), 1 if t.dtype == torch.float32 else 0, t.device.index or 0, \
        stream.cuda_stream


def device_anderson_darling(t, stream=None) -> float:
    """A^2 of a CUDA tensor's values against N(0, 1), on the device."""
    ptr, f32, dev, st = _dev_args(t, stream)
    a = C.c_double()
    _raise(lib.wrng_gpu_anderson_darling(ptr, f32, t.numel(), C.byref(a), dev, st),
           "anderson_darling")
    return a.value


def chi2_sf(statistic: float, dof: int) -> float:
    """Survival function of chi-squared(dof) (stats.cpp:40-87)."""
    return float(lib.wrng_gpu_chi2_sf(statistic, dof))


def _chi2_report(counts: np.ndarray) -> dict:
    total = int(counts.sum())
    k = counts.size
    expected = total / k
    stat = 0.0
    for c in counts.tolist():  # bin order, as chi2_bins sums (stats.cpp:30-35)
        d = float(c) - expected
        stat += d * d / expected
    return {"statistic": stat, "dof": k - 1, "p_value": chi2_sf(stat, k - 1), "bin_count": k,
            "sample_count": total}


def device_uv_chi2(t, k: int = 1000, stream=None) -> dict:
    """u/v uniformity of a CUDA tensor of normals, paired (2i, 2i+1) as the
    reference CLI's uniformity test (tools/main.cpp:160-193; stats.cpp:10-38):
    {"u": Chi2Report, "v": Chi2Report, "skipped": pairs (0, 0), "counts_u",
    "counts_v"}."""
    ptr, f32, dev, st = _dev_args(t, stream)
    cu = np.zeros(k, dtype=np.uint64)
    cv = np.zeros(k, dtype=np.uint64)
    sk = C.c_uint64()
    _raise(lib.wrng_gpu_uv_counts(ptr, f32, t.numel(), k, cu.ctypes.data, cv.ctypes.data,
                                  C.byref(sk), dev, st), "uv_counts")
    return {"u": _chi2_report(cu), "v": _chi2_report(cv), "skipped": int(sk.value),
            "counts_u": cu, "counts_v": cv}


def device_autocorr(t, lag: int, stream=None) -> float:
    """autocorr_at_lag(t, lag).r (stats.cpp:110-127) on the device."""
    ptr, f32, dev, st = _dev_args(t, stream)
    r = C.c_double()
    _raise(lib.wrng_gpu_autocorr(ptr, f32, t.numel(), lag, C.byref(r), dev, st), "autocorr")
    return r.value


def validate(state: "WallaceState", count: int, k: int = 1000, lag: int = 1,
             ad: bool = False) -> dict:
    """Generate `count` values of `state` (advancing it exactly like
    state.fill(count)) and check them on the device: moments with z-scores,
    u/v chi-squared, autocorrelation at `lag`, and with ad=True the
    Anderson-Darling A^2 of all `count` values (device radix sort).  No
    values reach the host."""
    v = L.Validation()
    cu = np.zeros(k, dtype=np.uint64)
    cv = np.zeros(k, dtype=np.uint64)
    _raise(lib.wrng_gpu_validate_ex(state._h, count, k, lag, L.VALIDATE_AD if ad else 0,
                                    cu.ctypes.data, cv.ctypes.data, C.byref(v)),
           "validate", state._h)
    out = {f: getattr(v, f) for f, _ in L.Validation._fields_}
    out["counts_u"], out["counts_v"] = cu, cv
    return out


# ---- Box-Muller / polar baselines (reference.cpp:9-63) ----------------------
def method_fill(method: str, t, seed: int, stream_id: int = 0, pools: int = 1, mu: float = 0.0,
                sigma: float = 1.0, f64_math: bool = True, stream=None):
    """Fill the CUDA tensor `t` with `pools` fresh Box-Muller ("boxmuller") or
    polar ("polar") streams UniformState(seed, stream_id + p), pool-major
    (asynchronous on `stream`)."""
    ptr, f32, dev, st = _dev_args(t, stream)
    m = {"boxmuller": 0, "polar": 1}[method]
    _raise(lib.wrng_gpu_method_fill(m, seed, stream_id, pools, ptr, f32, t.numel(), mu, sigma,
                                    1 if f64_math else 0, dev, st), "method_fill")
    return t
