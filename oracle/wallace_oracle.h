/* TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into the product.
 *
 * Plain-C restatement of the reference's Wallace generator
 * (/root/reference/proj/src/{uniform,reference,wallace}.cpp) generalised to
 * the n = 4 / fp32 modes frozen in docs/n4_spec.md.  Its n = 2 fp64 mode is
 * pinned bit-for-bit against the reference library itself (oracle/_ref, built
 * from the reference sources) and against the committed golden vectors in
 * tests/golden/.  The n = 4 and fp32 modes reuse the same uniform generator,
 * Box-Muller initialisation, chi-squared target, draw order and emission
 * order; their values are pinned only by this restatement's own golden files
 * ("parity unpinned" by reference tests — SURVEY.md §8(c)).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction: the reference's
 * Release build emits none).
 */
#ifndef WALLACE_ORACLE_H
#define WALLACE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_EINVAL = 1, OR_ECORRUPT = 2 };
enum { OR_F64 = 0, OR_F32 = 1 };
enum { OR_CHISQ = 0, OR_FIXED = 1 };

#define OR_TABLE 607u
#define OR_SHORT_LAG 273u
#define OR_MAX_INT_BOUND (1u << 20)

/* UniformState (uniform.hpp:16-40). */
typedef struct {
    uint64_t table[OR_TABLE];
    uint32_t r, s;
    uint64_t seed, stream, draws;
} or_uniform;

/* PassParams flattened (wallace.hpp:22-30).  n = 2: stride = {alpha, beta},
 * offset = {gamma, delta}, (c, s) the rotation.  n = 4: stride[0..3],
 * offset[0..3], variant selects the 4x4 matrix. */
typedef struct {
    uint32_t stride[4];
    uint32_t offset[4];
    uint32_t variant;
    uint32_t pad_;
    double c, s;
    double scale;
    double target;
} or_params;

typedef struct {
    uint32_t n_arrays;      /* 2 (reference) or 4 */
    uint32_t dtype;         /* OR_F64 / OR_F32 */
    uint32_t pool_exponent; /* N = 2^p, [8, 20] */
    uint32_t throwaway_f;   /* >= 1 */
    uint32_t scale_mode;    /* OR_CHISQ / OR_FIXED */
    uint64_t restart_interval;
    uint64_t drift_period;
    uint64_t seed, stream;
} or_config;

typedef struct {
    void* v;        /* n_arrays * N values, array-major (x0 | x1 | ...) */
    double tracked; /* tracked sum of squares */
    double withheld;
} or_pool;

typedef struct {
    or_config cfg;
    uint32_t n;         /* N */
    or_uniform us;
    or_pool pools[2];
    uint32_t active;
    uint64_t pass_count, avail, emitted;
} or_state;

/* ---- uniform.cpp ---- */
void or_uniform_init(or_uniform* u, uint64_t seed, uint64_t stream);
uint64_t or_next_word(or_uniform* u);
double or_next_uniform(or_uniform* u);
int or_next_int_below(or_uniform* u, uint32_t m, uint32_t* out);

/* ---- reference.cpp / wallace.cpp free functions ---- */
int or_box_muller_pair(double u1, double u2, double* x, double* y);
void or_box_muller_next(or_uniform* u, double* x, double* y);
void or_box_muller_fill(or_uniform* u, double* out, size_t n);
void or_polar_next(or_uniform* u, double* x, double* y);
void or_polar_fill(or_uniform* u, double* out, size_t n);
void or_method_bank_fill(int method, uint64_t seed, uint64_t stream0, uint32_t pools,
                         uint64_t count, double* out);
double or_chi2_target(double r, uint32_t nu);
void or_rotation_from_t(double t, uint32_t region, double* c, double* s);
int or_select_params(or_uniform* u, uint32_t n_arrays, uint32_t n, double tracked,
                     double withheld, uint32_t mode, or_params* p);
void or_regenerate(uint32_t n_arrays, uint32_t dtype, uint32_t n, const void* src,
                   void* dst, const or_params* p);
double or_direct_sumsq(uint32_t n_arrays, uint32_t dtype, uint32_t n, const void* v);

/* ---- WallaceState ---- */
int or_state_create(const or_config* cfg, or_state** out);
void or_state_destroy(or_state* st);
int or_state_advance_pass(or_state* st, or_params* p);
int or_state_refill(or_state* st);
int or_state_fill_f64(or_state* st, double* out, size_t count, double mu, double sigma);
int or_state_fill_f32(or_state* st, float* out, size_t count, double mu, double sigma);
int or_state_drift_check(or_state* st);
void or_state_restart(or_state* st);
void or_state_counters(const or_state* st, uint64_t* out4); /* pass, emitted, avail, N */
/* Active pool values widened to double, plus {tracked, withheld}. */
void or_state_get_pool(const or_state* st, double* vals, double* tw);
void or_state_set_pool(or_state* st, const double* vals, const double* tw);
void or_state_get_uniform(const or_state* st, uint64_t* table, uint32_t* r,
                          uint32_t* s, uint64_t* draws);

/* ---- bank of independent pools (pool p = stream + p), CTA-major output ---- */
int or_bank_fill_f32(const or_config* cfg, uint32_t pools, uint64_t count,
                     float* out, double mu, double sigma);
int or_bank_fill_f64(const or_config* cfg, uint32_t pools, uint64_t count,
                     double* out, double mu, double sigma);
/* CPU baseline timing: `threads` pthreads, thread t owns state stream0 + t and
 * fills per_thread values in `chunk`-sized calls.  Returns wall seconds. */
double or_bench_threads(const or_config* cfg, uint32_t threads, uint64_t per_thread,
                        uint32_t chunk);

/* ---- statistics (stats.cpp:89-108 + m3 + Anderson-Darling) ---- */
/* out: n, m1, m2, m3, m4 (sequential sums, left to right). */
void or_moments_f64(const double* v, size_t n, double* out5);
void or_moments_f32(const float* v, size_t n, double* out5);
/* A^2 of the simple hypothesis N(0,1); sorts a private copy. */
double or_anderson_darling_f64(const double* v, size_t n);
double or_anderson_darling_f32(const float* v, size_t n);
/* A^2 of an already sorted sample, summed on `threads` host threads. */
double or_ad_sorted_threads(const double* z, size_t n, int threads);
double or_ad_sorted_f32_threads(const float* z, size_t n, int threads);

/* ---- uniformity and serial-correlation checks (stats.cpp:10-38, 110-127;
 * the CLI's pairing, tools/main.cpp:160-193) ---- */
/* to_uv: u = exp(-(x^2 + y^2)/2), v = atan(x / y) (y == 0: copysign(pi/2, x));
 * returns 1 (skip) for the (0, 0) pair. */
int or_to_uv(double x, double y, double* u, double* v);
/* chi2_bins' bin index of v in [lo, hi] with k bins (values == hi -> k - 1);
 * -1 when v is outside [lo, hi]. */
int64_t or_chi2_bin(double v, uint32_t k, double lo, double hi);
/* Pairs (v[2i], v[2i+1]), i < n/2, mapped by to_uv; u binned on [0, 1] and
 * v on [-pi/2, pi/2] into k bins each.  Returns the skipped-pair count. */
uint64_t or_uv_counts_f64(const double* v, size_t n, uint32_t k, uint64_t* cu, uint64_t* cv);
uint64_t or_uv_counts_f32(const float* v, size_t n, uint32_t k, uint64_t* cu, uint64_t* cv);
/* chi2_bins' statistic from counts (expected = total / k, summed in bin order). */
double or_chi2_statistic(const uint64_t* counts, uint32_t k);
/* chi2_sf (stats.cpp:40-87): regularized upper incomplete gamma. */
double or_chi2_sf(double statistic, uint32_t dof);
/* autocorr_at_lag (stats.cpp:110-127): r, two-pass, sequential sums. */
double or_autocorr_f64(const double* v, size_t n, size_t lag);
double or_autocorr_f32(const float* v, size_t n, size_t lag);

#ifdef __cplusplus
}
#endif
#endif
