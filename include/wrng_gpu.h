/*
 * wrng_gpu.h — C ABI of the B200 (sm_100a) Wallace normal generator.
 *
 * This is the drop-in boundary for the reference's generator interface
 * (/root/reference/proj/include/wrng/wallace.hpp).  Every entry point below
 * replaces one reference member / free function, cited as file:line.  No C++
 * types, exceptions or torch types cross it: plain pointers, sizes and status
 * codes.  include/wrng_gpu/wallace.hpp wraps it back into the reference's C++
 * API (WallaceConfig / WallaceState, same exception types).
 *
 * Generalisations over the reference (all default to the reference's
 * behaviour: n_arrays = 2, dtype = f64, pools = 1):
 *   - n_arrays = 4: Wallace's 4x4 orthogonal variant (docs/n4_spec.md);
 *   - dtype = f32 pools (all per-pass scalars still computed in f64);
 *   - pools = P independent generators in one handle ("bank"); pool p is
 *     the reference state (seed, stream_id + p) (uniform.cpp:23-26).  A fill
 *     of `count` values writes pool p's stream into the contiguous segment of
 *     count/P (+1 for p < count % P) values starting at sum of the previous
 *     segments ("pool-major").
 *
 * Threading: a handle is single-owner (wallace.hpp:113-114); distinct handles
 * may be used concurrently from different host threads.
 */
#ifndef WRNG_GPU_H
#define WRNG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WRNG_GPU_ABI_VERSION 2

/* Status codes.  Map 1:1 onto the reference's exceptions:
 *   EINVAL     std::invalid_argument      (wallace.cpp:141-149, 199;
 *                                           uniform.cpp:48-49)
 *   ECORRUPT   wrng::corrupted_state_error (errors.hpp:10-13;
 *                                           wallace.cpp:59-61, 229-232)
 *   EMALFORMED_* wrng::malformed_state_error{kind} (errors.hpp:15-32;
 *                                           serialize.cpp:63-66, 76-78, 117-169)
 *   ECUDA / ENOMEM / ENODEV: device-side failures (no reference analogue). */
typedef enum wrng_gpu_status {
    WRNG_GPU_OK = 0,
    WRNG_GPU_EINVAL = 1,
    WRNG_GPU_ECORRUPT = 2,
    WRNG_GPU_EMALFORMED_BAD_MAGIC = 3,
    WRNG_GPU_EMALFORMED_VERSION = 4,
    WRNG_GPU_EMALFORMED_TRUNCATED = 5,
    WRNG_GPU_EMALFORMED_FIELD_RANGE = 6,
    WRNG_GPU_ECUDA = 7,
    WRNG_GPU_ENOMEM = 8,
    WRNG_GPU_ENODEV = 9
} wrng_gpu_status;

enum { WRNG_GPU_F64 = 0, WRNG_GPU_F32 = 1 };
enum { WRNG_GPU_CHISQ = 0, WRNG_GPU_FIXED = 1 }; /* ScaleMode, wallace.hpp:52-55 */

/* Config flags. */
enum {
    /* Initial pool from the host (glibc libm) instead of the device
     * Box-Muller kernel: bit-identical to the reference's init_pool
     * (wallace.cpp:158-167).  The device path agrees to a few ulp. */
    WRNG_GPU_INIT_HOST = 1u << 0,
    /* Engine selection (default: shared-memory pools when a pool fits in
     * one CTA's shared memory, else HBM-resident double-buffered pools). */
    WRNG_GPU_FORCE_HBM = 1u << 1,
    /* drift_check by a fast parallel reduction instead of the reference's
     * left-to-right order (Pool::direct_sumsq, wallace.hpp:44-46).  Off by
     * default: the default path reproduces the sequential sum bit-exactly. */
    WRNG_GPU_DRIFT_TREE = 1u << 2
};

/* WallaceConfig (wallace.hpp:57-65) + the B200 extensions. */
typedef struct wrng_gpu_config {
    uint32_t pool_exponent;           /* N = 2^p per array, p in [8, 20] */
    uint32_t throwaway_f;             /* >= 1: passes per exposed pool */
    uint32_t scale_mode;              /* WRNG_GPU_CHISQ | WRNG_GPU_FIXED */
    uint32_t n_arrays;                /* 2 (reference) or 4 */
    uint64_t restart_interval_passes; /* 0 = never, else > throwaway_f */
    uint64_t drift_check_period;      /* passes between audits, 0 = never */
    uint64_t seed;
    uint64_t stream_id;               /* pool p uses stream_id + p */
    uint32_t dtype;                   /* WRNG_GPU_F64 | WRNG_GPU_F32 */
    uint32_t pools;                   /* >= 1 independent pools */
    int32_t device;                   /* CUDA device ordinal */
    uint32_t flags;                   /* WRNG_GPU_* flags */
} wrng_gpu_config;

/* PassParams (wallace.hpp:22-30), flattened for n in {2, 4}.
 * n = 2: stride = {alpha, beta}, offset = {gamma, delta}, (c, s) = rot.
 * n = 4: stride[0..3], offset[0..3], variant in {0, 1} (docs/n4_spec.md). */
typedef struct wrng_gpu_params {
    uint32_t stride[4];
    uint32_t offset[4];
    uint32_t variant;
    uint32_t pad_;
    double c;
    double s;
    double scale;
    double target_sumsq;
} wrng_gpu_params;

typedef struct wrng_gpu_counters {
    uint64_t pass_count;      /* WallaceState::pass_count (wallace.hpp:150) */
    uint64_t numbers_emitted; /* WallaceState::numbers_emitted (:151) */
    uint64_t avail;           /* WallaceState::avail (:152) */
    uint32_t active;          /* double-buffer flag (wallace.hpp:168) */
    uint32_t pool_size;       /* N (wallace.hpp:149) */
} wrng_gpu_counters;

typedef struct wrng_gpu wrng_gpu_t;

/* Reference defaults: p = 10, f = 3, chisq, no restart, drift 64, seed 0,
 * stream 0 (wallace.hpp:57-65); n = 2, f64, 1 pool, device 0, no flags. */
void wrng_gpu_config_default(wrng_gpu_config* cfg);

/* WallaceState::WallaceState (wallace.cpp:139-156): validates, seeds each
 * pool's uniform generator (uniform.cpp:23-32) and fills the initial pools
 * (wallace.cpp:158-167).  EINVAL on a bad config. */
wrng_gpu_status wrng_gpu_create(const wrng_gpu_config* cfg, wrng_gpu_t** out);
void wrng_gpu_destroy(wrng_gpu_t* g);

/* WallaceState::fill (wallace.cpp:198-216), every pool, pool-major output.
 * out_is_device != 0: `out` is device memory and the work is enqueued on
 * `stream` (a cudaStream_t, NULL = legacy default) without a host sync; a
 * device-detected ECORRUPT is returned by the next synchronising call.
 * out_is_device == 0: `out` is host memory (pinned or pageable); generation
 * is overlapped with the device-to-host copies and the call returns when all
 * values are in `out`.  sigma < 0 -> EINVAL (wallace.cpp:199). */
wrng_gpu_status wrng_gpu_fill_f64(wrng_gpu_t* g, double* out, uint64_t count,
                                  double mu, double sigma, int out_is_device,
                                  void* stream);
wrng_gpu_status wrng_gpu_fill_f32(wrng_gpu_t* g, float* out, uint64_t count,
                                  double mu, double sigma, int out_is_device,
                                  void* stream);

/* WallaceState::advance_pass (wallace.cpp:169-178) on every pool; the
 * parameters used are written to params[p] when params != NULL. */
wrng_gpu_status wrng_gpu_advance_pass(wrng_gpu_t* g, wrng_gpu_params* params);
/* WallaceState::refill (wallace.cpp:188-196) on every pool. */
wrng_gpu_status wrng_gpu_refill(wrng_gpu_t* g);
/* WallaceState::drift_check (wallace.cpp:225-234) on every pool. */
wrng_gpu_status wrng_gpu_drift_check(wrng_gpu_t* g);
/* WallaceState::restart (wallace.cpp:236) on every pool. */
wrng_gpu_status wrng_gpu_restart(wrng_gpu_t* g);

/* Accessors (wallace.hpp:148-160). */
wrng_gpu_status wrng_gpu_get_config(const wrng_gpu_t* g, wrng_gpu_config* out);
wrng_gpu_status wrng_gpu_get_counters(const wrng_gpu_t* g, uint32_t pool,
                                      wrng_gpu_counters* out);
/* active_pool() (wallace.hpp:156-157): values (n_arrays * N, array-major,
 * widened to double), tracked_sumsq, withheld. */
wrng_gpu_status wrng_gpu_read_pool(wrng_gpu_t* g, uint32_t pool, double* values,
                                   double* tracked_sumsq, double* withheld);
/* Mutable active_pool(): overwrite the live pool (tests model callers that
 * scribble over the work area, test_wallace_state.cpp:128-150). */
wrng_gpu_status wrng_gpu_write_pool(wrng_gpu_t* g, uint32_t pool, const double* values,
                                    double tracked_sumsq, double withheld);
/* uniform_state() (wallace.hpp:158): lag table, cursors, draws. */
wrng_gpu_status wrng_gpu_read_uniform(wrng_gpu_t* g, uint32_t pool, uint64_t* table607,
                                      uint32_t* cursor_r, uint32_t* cursor_s,
                                      uint64_t* draws);

/* Overwrites pool `pool`'s uniform generator (the mutable uniform_state(),
 * wallace.hpp:158).  EINVAL unless cursor_r < 607 and
 * cursor_s = (cursor_r + 334) mod 607 (serialize.cpp:145-148). */
wrng_gpu_status wrng_gpu_write_uniform(wrng_gpu_t* g, uint32_t pool, const uint64_t* table607,
                                       uint32_t cursor_r, uint32_t cursor_s, uint64_t draws);

/* save_state / load_state (serialize.cpp:82-169).  A handle with n = 2,
 * f64, 1 pool exports the reference's "WRNG" v1 bytes exactly; anything else
 * exports v2 (docs/n4_spec.md §6).  export: *size receives the byte count;
 * bytes are copied only when cap >= *size (buf may be NULL to query). */
wrng_gpu_status wrng_gpu_export_state(wrng_gpu_t* g, uint8_t* buf, size_t cap,
                                      size_t* size);
wrng_gpu_status wrng_gpu_import_state(const uint8_t* bytes, size_t size, int32_t device,
                                      uint32_t flags, wrng_gpu_t** out);

/* Blocks until the handle's queued work is done; reports device errors. */
wrng_gpu_status wrng_gpu_synchronize(wrng_gpu_t* g);
/* Message of the handle's last failing call ("" when none). */
const char* wrng_gpu_last_error(const wrng_gpu_t* g);
/* Pools the shared-memory engine keeps resident at once on cfg->device for
 * fills of this configuration (SMs x CTAs per SM of the fill kernel x pools
 * per CTA): a bank of this many pools, or a multiple, runs in whole waves.
 * For small n = 4 pools (4x256, fp32 4x512: several pools per warp) at
 * throwaway_f = 1 it is the count that measured fastest, below the occupancy
 * limit (fills of f = 1 are bound by the number of concurrent output
 * streams).  0 when the configuration runs on the HBM engine; < 0 (a negated
 * wrng_gpu_status) on error. */
int64_t wrng_gpu_resident_pools(const wrng_gpu_config* cfg);
/* Number of this library's kernels launched by the handle so far. */
uint64_t wrng_gpu_kernel_launches(const wrng_gpu_t* g);
/* Name of the engine the handle runs: "smem" or "hbm". */
const char* wrng_gpu_engine(const wrng_gpu_t* g);

/* Validation reductions on device data: n, m1..m4
 * from per-block fp64 partial sums (tree order).  Synchronous. */
wrng_gpu_status wrng_gpu_moments_f32(const float* dev, uint64_t n, double* out5,
                                     int32_t device, void* stream);
wrng_gpu_status wrng_gpu_moments_f64(const double* dev, uint64_t n, double* out5,
                                     int32_t device, void* stream);

/* ---- validation statistics on the device ------------
 * u/v uniformity counts of a DEVICE array of n normals: pairs
 * (v[2i], v[2i+1]) -> to_uv (stats.cpp:10-16) -> k bins of u on [0, 1] and
 * of v on [-pi/2, pi/2] (chi2_bins, stats.cpp:18-38), paired as the CLI's
 * uniformity test does (tools/main.cpp:160-193); (0, 0) pairs are skipped.
 * counts_u / counts_v: host arrays of k, overwritten.  1 < k <= 8192.
 * Synchronous. */
wrng_gpu_status wrng_gpu_uv_counts(const void* dev, int32_t is_f32, uint64_t n, uint32_t k,
                                   uint64_t* counts_u, uint64_t* counts_v, uint64_t* skipped,
                                   int32_t device, void* stream);
/* autocorr_at_lag (stats.cpp:110-127) of a DEVICE array, from one-pass raw
 * sums (sum z_t z_{t+lag}, sum z_t, sum z_{t+lag}, sum z_t^2) and the mean.
 * EINVAL unless n >= lag + 2.  Synchronous. */
wrng_gpu_status wrng_gpu_autocorr(const void* dev, int32_t is_f32, uint64_t n, uint64_t lag,
                                  double* r, int32_t device, void* stream);
/* chi2_sf (stats.cpp:40-87): survival function of chi-squared(dof). */
double wrng_gpu_chi2_sf(double statistic, uint32_t dof);

/* Generate-and-check with no host copy of the values: advances every pool
 * exactly as wrng_gpu_fill_*(g, count) would (pool p: count / pools values,
 * one more for p < count % pools), generating into an L2-sized device slab
 * and reducing each slab on the device.  Pairs (u/v) and lags (autocorr)
 * are taken within each pool's stream; statistics are pooled over pools
 * (for one pool they are the reference's, stats.cpp / tools/main.cpp).
 * counts_u / counts_v: optional host arrays of k. */
typedef struct wrng_gpu_validation {
    uint64_t n;                       /* values generated and checked */
    double m1, m2, m3, m4;            /* moments (stats.cpp:89-108 + m3) */
    double z1, z2, z4;                /* standardized deviations (stats.cpp:103-105) */
    uint64_t uv_samples, uv_skipped;  /* pairs binned / (0, 0) pairs skipped */
    uint32_t k, dof;                  /* bins, k - 1 */
    double u_statistic, u_p, v_statistic, v_p;  /* chi2_bins of u and v */
    uint64_t lag;
    double autocorr;                  /* r at lag */
    /* WRNG_GPU_VALIDATE_AD: Anderson-Darling A^2 of all `n` values against
     * N(0, 1) (simple hypothesis; device radix sort, stats_ad.cu), else NAN */
    double ad_a2;
    uint64_t ad_n;
} wrng_gpu_validation;
wrng_gpu_status wrng_gpu_validate(wrng_gpu_t* g, uint64_t count, uint32_t k, uint64_t lag,
                                  uint64_t* counts_u, uint64_t* counts_v,
                                  wrng_gpu_validation* out);
enum { WRNG_GPU_VALIDATE_AD = 1u << 0 };
/* wrng_gpu_validate plus the statistics selected by `what` (needs device
 * scratch of 2 keys per value for WRNG_GPU_VALIDATE_AD: 32 GiB at 2^32
 * fp32 values; ENOMEM when it does not fit). */
wrng_gpu_status wrng_gpu_validate_ex(wrng_gpu_t* g, uint64_t count, uint32_t k, uint64_t lag,
                                     uint32_t what, uint64_t* counts_u, uint64_t* counts_v,
                                     wrng_gpu_validation* out);
/* Anderson-Darling A^2 against N(0, 1) of a DEVICE array of n values
 * (f32 or f64), computed on the device: radix sort of order-preserving keys,
 * then sum_j d_j with d_j = -1 - [(2j+1) ln Phi(z_j) + (2n-2j-1) ln(1-Phi(z_j))]/n
 * in compensated arithmetic.  Synchronous; allocates 2 keys per value. */
wrng_gpu_status wrng_gpu_anderson_darling(const void* dev, int32_t is_f32, uint64_t n, double* a2,
                                          int32_t device, void* stream);

/* ---- Box-Muller / polar baselines (reference.cpp:9-63) --
 * The methods the paper compares Wallace against, on the
 * GPU: stream p = UniformState(seed, stream_id + p) fills count / pools
 * values (+1 for p < count % pools) as a FRESH box_muller_fill (method 0)
 * or polar_fill (method 1) would, pool-major into DEVICE memory, on
 * `stream` (asynchronous).  f64_math = 1 evaluates the reference's fp64
 * expressions (CUDA libm: within a few ulp of glibc); 0 uses fp32 math
 * (logf, sqrtf, sincospif) as a throughput baseline. */
wrng_gpu_status wrng_gpu_method_fill(int32_t method, uint64_t seed, uint64_t stream_id,
                                     uint32_t pools, void* dev_out, int32_t out_f32,
                                     uint64_t count, double mu, double sigma, int32_t f64_math,
                                     int32_t device, void* stream);

/* Device uniform generator, for bit-exact stream checks: the first `count`
 * next_word() outputs of UniformState(seed, stream_id + p) for p < pools,
 * pool-major (uniform.cpp:23-40). */
wrng_gpu_status wrng_gpu_lfg_words(uint64_t seed, uint64_t stream_id, uint32_t pools,
                                   uint64_t count, uint64_t* host_out, int32_t device);

/* ---- the reference's free functions on host data ------------------------
 * (proj/include/wrng/{uniform,wallace,reference,stats}.hpp).  These serve
 * callers that drive passes on their own value-type pools and uniform
 * states, as the reference's tests do; include/wrng_gpu/wallace.hpp wraps
 * them under the reference's names.  Floating-point helpers live here (built
 * with FMA contraction off) so their bits never depend on how the caller is
 * compiled.  wrng_gpu_regenerate runs the pass on the GPU. */

/* UniformState (uniform.hpp:16-40) as plain data; the drop-in's
 * wrng::UniformState has exactly this layout. */
typedef struct wrng_gpu_uniform {
    uint64_t lag_table[607];
    uint32_t cursor_r;
    uint32_t cursor_s;
    uint64_t seed;
    uint64_t stream_id;
    uint64_t draws;
} wrng_gpu_uniform;

/* Segment (wallace.hpp:70-75) */
typedef struct wrng_gpu_segment {
    uint32_t low;
    uint32_t high;
    int64_t jx;
    int64_t jy;
} wrng_gpu_segment;

/* UniformState::UniformState(seed, stream_id) (uniform.cpp:23-32). */
void wrng_gpu_uniform_seed(wrng_gpu_uniform* us, uint64_t seed, uint64_t stream_id);
/* Pool::direct_sumsq's loop (wallace.cpp:13-18) continued from q: returns
 * q + v[0]^2 + ... + v[n-1]^2 added left to right, each product rounded. */
double wrng_gpu_sumsq_continue(double q, const double* v, uint64_t n);
/* chi2_target (wallace.cpp:27-31). */
double wrng_gpu_chi2_target(double r, uint32_t nu);
/* rotation_from_t / rotation_from_uniform (wallace.cpp:33-49). */
void wrng_gpu_rotation_from_t(double t, uint32_t region, double* c, double* s);
void wrng_gpu_rotation_from_uniform(wrng_gpu_uniform* us, double* c, double* s);
/* select_pass_params (wallace.cpp:51-70; n = 4: docs/n4_spec.md §2) on a
 * host uniform state.  ECORRUPT (after the draws, with *out holding the
 * drawn indices) when tracked_sumsq is not > 0; EINVAL for bad arguments. */
wrng_gpu_status wrng_gpu_select_pass_params(wrng_gpu_uniform* us, uint32_t n_arrays, uint32_t N,
                                            uint32_t scale_mode, double tracked_sumsq,
                                            double withheld, wrng_gpu_params* out);
/* plan_segments (wallace.cpp:72-111): *count receives the number of
 * segments; they are written when out != NULL and cap >= *count.  EINVAL as
 * the reference's invalid_argument (strides not coprime to N, offsets out of
 * range). */
wrng_gpu_status wrng_gpu_plan_segments(const wrng_gpu_params* p, uint32_t N,
                                       wrng_gpu_segment* out, uint32_t cap, uint32_t* count);
/* regenerate (wallace.cpp:113-137; n = 4: docs/n4_spec.md §3): one pass
 * from host arrays src (n_arrays * N fp64, array-major) to dst, computed on
 * GPU `device`; *withheld_out = dst's last value.  Synchronous. */
wrng_gpu_status wrng_gpu_regenerate(const double* src, double* dst, uint32_t n_arrays, uint32_t N,
                                    const wrng_gpu_params* p, double* withheld_out,
                                    int32_t device);
/* box_muller_pair / _next, polar_transform / _next (reference.cpp:9-37);
 * wrng_gpu_normal_fill = box_muller_fill (method 0) / polar_fill (1)
 * (reference.cpp:41-63). */
wrng_gpu_status wrng_gpu_box_muller_pair(double u1, double u2, double* x, double* y);
void wrng_gpu_box_muller_next(wrng_gpu_uniform* us, double* x, double* y);
void wrng_gpu_polar_transform(double v1, double v2, double* x, double* y);
void wrng_gpu_polar_next(wrng_gpu_uniform* us, double* x, double* y);
void wrng_gpu_normal_fill(int32_t method, wrng_gpu_uniform* us, double* out, uint64_t n,
                          double mu, double sigma);
/* to_uv, chi2_bins' statistic, moments (+ m3), autocorr_at_lag on host
 * arrays (stats.cpp:10-127), in the reference's sequential order.
 * moments: out7 = {m1, m2, m3, m4, z1, z2, z4}. */
void wrng_gpu_to_uv(double x, double y, double* u, double* v, int32_t* skip);
wrng_gpu_status wrng_gpu_chi2_bins(const double* values, uint64_t n, uint32_t k, double lo,
                                   double hi, double* statistic);
wrng_gpu_status wrng_gpu_moments_host(const double* values, uint64_t n, double* out7);
wrng_gpu_status wrng_gpu_autocorr_host(const double* values, uint64_t n, uint64_t lag,
                                       double* r);
/* sumsq_distribution_check's reduction (stats.cpp:136-145) of n recorded
 * targets: mean_var = {sample mean, population variance (>= 0)}. */
void wrng_gpu_target_stats(const double* s, uint64_t n, double* mean_var);

#ifdef __cplusplus
}
#endif
#endif /* WRNG_GPU_H */
