/* TEST INFRASTRUCTURE ONLY — CPU oracle (see wallace_oracle.h).
 *
 * Every function cites the reference line range it restates.  Paths are
 * relative to /root/reference/proj.  Compile with -ffp-contract=off: every
 * floating-point expression below is evaluated exactly as written, one
 * rounding per operation, like the reference's FMA-free Release build.
 */
#define _GNU_SOURCE
#include "wallace_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------
 * Uniform generator: additive lagged Fibonacci (607, 273) mod 2^64.
 * ---------------------------------------------------------------------- */

/* splitmix64 finalizer over a counter (uniform.cpp:13-19). */
static uint64_t splitmix64(uint64_t* s) {
    *s += 0x9E3779B97F4A7C15ull;
    uint64_t z = *s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t v, unsigned k) { return (v << k) | (v >> (64 - k)); }

/* UniformState::UniformState (uniform.cpp:23-32). */
void or_uniform_init(or_uniform* u, uint64_t seed, uint64_t stream) {
    uint64_t s = seed ^ rotl64(stream, 32);
    for (uint32_t i = 0; i < OR_TABLE; ++i) u->table[i] = splitmix64(&s);
    u->r = 0;
    u->s = OR_TABLE - OR_SHORT_LAG;
    u->seed = seed;
    u->stream = stream;
    for (uint32_t i = 0; i < 10 * OR_TABLE; ++i) or_next_word(u);
    u->draws = 0;
}

/* UniformState::next_word (uniform.cpp:34-40). */
uint64_t or_next_word(or_uniform* u) {
    uint64_t w = u->table[u->r] + u->table[u->s];
    u->table[u->r] = w;
    if (++u->r == OR_TABLE) u->r = 0;
    if (++u->s == OR_TABLE) u->s = 0;
    return w;
}

/* UniformState::next_uniform (uniform.cpp:42-45): top 53 bits * 2^-53. */
double or_next_uniform(or_uniform* u) {
    ++u->draws;
    return (double)(or_next_word(u) >> 11) * 0x1.0p-53;
}

/* UniformState::next_int_below (uniform.cpp:47-51). */
int or_next_int_below(or_uniform* u, uint32_t m, uint32_t* out) {
    if (m < 1 || m > OR_MAX_INT_BOUND) return OR_EINVAL;
    *out = (uint32_t)(or_next_uniform(u) * m);
    return OR_OK;
}

static uint32_t nib(or_uniform* u, uint32_t m) {
    uint32_t v = 0;
    or_next_int_below(u, m, &v); /* callers pass m in [1, 2^20] */
    return v;
}

/* ------------------------------------------------------------------------
 * Box-Muller (reference.cpp:9-22, 41-51)
 * ---------------------------------------------------------------------- */

/* box_muller_pair (reference.cpp:9-15). */
int or_box_muller_pair(double u1, double u2, double* x, double* y) {
    if (!(u1 > 0.0 && u1 < 1.0)) return OR_EINVAL;
    const double pi = 3.141592653589793; /* std::numbers::pi */
    double radius = sqrt(-2.0 * log(u1));
    double angle = 2.0 * pi * u2;
    *x = radius * cos(angle);
    *y = radius * sin(angle);
    return OR_OK;
}

/* box_muller_next (reference.cpp:17-22): u1 == 0 maps to 2^-53. */
void or_box_muller_next(or_uniform* u, double* x, double* y) {
    double u1 = or_next_uniform(u);
    if (u1 == 0.0) u1 = 0x1.0p-53;
    double u2 = or_next_uniform(u);
    or_box_muller_pair(u1, u2, x, y);
}

/* box_muller_fill with mu = 0, sigma = 1 (reference.cpp:41-58): pairs in
 * order, `mu + sigma * z` evaluated literally (so -0.0 becomes +0.0), an odd
 * count drops the final partner. */
void or_box_muller_fill(or_uniform* u, double* out, size_t n) {
    volatile double mu = 0.0, sigma = 1.0;
    size_t i = 0;
    double x, y;
    while (i + 1 < n) {
        or_box_muller_next(u, &x, &y);
        out[i++] = mu + sigma * x;
        out[i++] = mu + sigma * y;
    }
    if (i < n) {
        or_box_muller_next(u, &x, &y);
        out[i] = mu + sigma * x;
    }
}

/* polar_transform / polar_next (reference.cpp:24-39): Marsaglia's polar
 * method, (v1, v2) = 2u - 1 accepted when 0 < v1^2 + v2^2 < 1. */
void or_polar_next(or_uniform* u, double* x, double* y) {
    for (;;) {
        double v1 = 2.0 * or_next_uniform(u) - 1.0;
        double v2 = 2.0 * or_next_uniform(u) - 1.0;
        double s = v1 * v1 + v2 * v2;
        if (s > 0.0 && s < 1.0) {
            double f = sqrt(-2.0 * log(s) / s);
            *x = v1 * f;
            *y = v2 * f;
            return;
        }
    }
}

/* polar_fill with mu = 0, sigma = 1 (reference.cpp:46-63). */
void or_polar_fill(or_uniform* u, double* out, size_t n) {
    volatile double mu = 0.0, sigma = 1.0;
    size_t i = 0;
    double x, y;
    while (i + 1 < n) {
        or_polar_next(u, &x, &y);
        out[i++] = mu + sigma * x;
        out[i++] = mu + sigma * y;
    }
    if (i < n) {
        or_polar_next(u, &x, &y);
        out[i] = mu + sigma * x;
    }
}

/* Bank of method fills: stream p = UniformState(seed, stream0 + p) fills
 * count / pools values (+1 for p < count % pools), pool-major; method 0
 * Box-Muller, 1 polar. */
void or_method_bank_fill(int method, uint64_t seed, uint64_t stream0, uint32_t pools,
                         uint64_t count, double* out) {
    const uint64_t base = count / pools, extra = count % pools;
    uint64_t off = 0;
    for (uint32_t p = 0; p < pools; ++p) {
        const uint64_t len = base + (p < extra ? 1 : 0);
        or_uniform u;
        or_uniform_init(&u, seed, stream0 + p);
        if (method == 0)
            or_box_muller_fill(&u, out + off, len);
        else
            or_polar_fill(&u, out + off, len);
        off += len;
    }
}

/* ------------------------------------------------------------------------
 * Pass parameters (wallace.cpp:27-70) and the n = 4 extension
 * (docs/n4_spec.md §2).
 * ---------------------------------------------------------------------- */

/* chi2_target (wallace.cpp:27-31): S = (r + sqrt(2 nu - 1))^2 / 2. */
double or_chi2_target(double r, uint32_t nu) {
    double t = r + sqrt(2.0 * nu - 1.0);
    return 0.5 * t * t;
}

/* rotation_from_t (wallace.cpp:33-42). */
void or_rotation_from_t(double t, uint32_t region, double* c, double* s) {
    double t2 = t * t;
    double cc = (1.0 - t2) / (1.0 + t2);
    double ss = 2.0 * t / (1.0 + t2);
    switch (region) {
        case 0: *c = cc; *s = ss; break;
        case 1: *c = cc; *s = -ss; break;
        default: *c = -cc; *s = ss; break;
    }
}

static const uint32_t kStrideSets4[4][2] = {{3, 5}, {7, 11}, {13, 17}, {19, 23}};

/* select_pass_params (wallace.cpp:51-70).  The tracked > 0 check runs AFTER
 * every draw, so a failing call still advances the uniform state. */
int or_select_params(or_uniform* u, uint32_t n_arrays, uint32_t n, double tracked,
                     double withheld, uint32_t mode, or_params* p) {
    memset(p, 0, sizeof(*p));
    if (n_arrays == 2) {
        p->stride[0] = nib(u, 2) == 0 ? 3 : 5;
        p->stride[1] = nib(u, 2) == 0 ? 7 : 11;
        p->offset[0] = nib(u, n);
        p->offset[1] = nib(u, n);
        /* rotation_from_uniform (wallace.cpp:44-49) */
        const double kTanLo = 0.26794919243112270;
        const double kTanHi = 0.57735026918962576;
        double t = kTanLo + (kTanHi - kTanLo) * or_next_uniform(u);
        or_rotation_from_t(t, nib(u, 3), &p->c, &p->s);
    } else {
        for (int m = 0; m < 4; ++m) p->stride[m] = kStrideSets4[m][nib(u, 2)];
        for (int m = 0; m < 4; ++m) p->offset[m] = nib(u, n);
        p->variant = nib(u, 2);
    }
    if (!(tracked > 0.0)) return OR_ECORRUPT;
    if (mode == OR_CHISQ) {
        p->target = or_chi2_target(withheld, n_arrays * n);
        p->scale = sqrt(p->target / tracked);
    } else {
        p->scale = 1.0;
        p->target = tracked;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * Regeneration pass: wallace.cpp:113-137 with naive modular indexing, which
 * the reference pins bit-identical to its segmented loop
 * (tests/test_wallace_core.cpp:15-27, 203-217).
 * ---------------------------------------------------------------------- */
void or_regenerate(uint32_t n_arrays, uint32_t dtype, uint32_t n, const void* src,
                   void* dst, const or_params* p) {
    const uint32_t mask = n - 1;
    if (dtype == OR_F64) {
        const double* s = (const double*)src;
        double* d = (double*)dst;
        if (n_arrays == 2) {
            const double kc = p->c * p->scale;
            const double ks = p->s * p->scale;
            for (uint32_t j = 0; j < n; ++j) {
                double xs = s[(p->stride[0] * (uint64_t)j + p->offset[0]) & mask];
                double ys = s[n + ((p->stride[1] * (uint64_t)j + p->offset[1]) & mask)];
                d[j] = kc * xs + ks * ys;
                d[n + j] = kc * ys - ks * xs;
            }
        } else {
            const double k = 0.5 * p->scale;
            const double sc = p->scale;
            for (uint32_t j = 0; j < n; ++j) {
                double a = s[0 * n + ((p->stride[0] * (uint64_t)j + p->offset[0]) & mask)];
                double b = s[1 * n + ((p->stride[1] * (uint64_t)j + p->offset[1]) & mask)];
                double c = s[2 * n + ((p->stride[2] * (uint64_t)j + p->offset[2]) & mask)];
                double e = s[3 * n + ((p->stride[3] * (uint64_t)j + p->offset[3]) & mask)];
                if (p->variant == 0) { /* (1/2) H4, Sylvester order */
                    double pp = a + b, q = a - b, r = c + e, ss = c - e;
                    d[0 * n + j] = k * (pp + r);
                    d[1 * n + j] = k * (q + ss);
                    d[2 * n + j] = k * (pp - r);
                    d[3 * n + j] = k * (q - ss);
                } else { /* (1/2) J - I */
                    double t = 0.5 * ((a + b) + (c + e));
                    d[0 * n + j] = sc * (t - a);
                    d[1 * n + j] = sc * (t - b);
                    d[2 * n + j] = sc * (t - c);
                    d[3 * n + j] = sc * (t - e);
                }
            }
        }
    } else {
        const float* s = (const float*)src;
        float* d = (float*)dst;
        if (n_arrays == 2) {
            const float kc = (float)(p->c * p->scale);
            const float ks = (float)(p->s * p->scale);
            for (uint32_t j = 0; j < n; ++j) {
                float xs = s[(p->stride[0] * (uint64_t)j + p->offset[0]) & mask];
                float ys = s[n + ((p->stride[1] * (uint64_t)j + p->offset[1]) & mask)];
                d[j] = kc * xs + ks * ys;
                d[n + j] = kc * ys - ks * xs;
            }
        } else {
            const float k = (float)(0.5 * p->scale);
            const float sc = (float)p->scale;
            for (uint32_t j = 0; j < n; ++j) {
                float a = s[0 * n + ((p->stride[0] * (uint64_t)j + p->offset[0]) & mask)];
                float b = s[1 * n + ((p->stride[1] * (uint64_t)j + p->offset[1]) & mask)];
                float c = s[2 * n + ((p->stride[2] * (uint64_t)j + p->offset[2]) & mask)];
                float e = s[3 * n + ((p->stride[3] * (uint64_t)j + p->offset[3]) & mask)];
                if (p->variant == 0) {
                    float pp = a + b, q = a - b, r = c + e, ss = c - e;
                    d[0 * n + j] = k * (pp + r);
                    d[1 * n + j] = k * (q + ss);
                    d[2 * n + j] = k * (pp - r);
                    d[3 * n + j] = k * (q - ss);
                } else {
                    float t = 0.5f * ((a + b) + (c + e));
                    d[0 * n + j] = sc * (t - a);
                    d[1 * n + j] = sc * (t - b);
                    d[2 * n + j] = sc * (t - c);
                    d[3 * n + j] = sc * (t - e);
                }
            }
        }
    }
}

/* Pool::direct_sumsq (wallace.cpp:13-18): arrays in order, left to right;
 * fp32 values are widened (the product of two floats is exact in double). */
double or_direct_sumsq(uint32_t n_arrays, uint32_t dtype, uint32_t n, const void* v) {
    double q = 0.0;
    size_t total = (size_t)n_arrays * n;
    if (dtype == OR_F64) {
        const double* d = (const double*)v;
        for (size_t i = 0; i < total; ++i) q += d[i] * d[i];
    } else {
        const float* f = (const float*)v;
        for (size_t i = 0; i < total; ++i) q += (double)f[i] * (double)f[i];
    }
    return q;
}

/* ------------------------------------------------------------------------
 * WallaceState (wallace.cpp:139-236)
 * ---------------------------------------------------------------------- */

static size_t esize(uint32_t dtype) { return dtype == OR_F64 ? 8 : 4; }

/* init_pool (wallace.cpp:158-167): Box-Muller fill of each array in order,
 * then withheld = the .x of one more pair (its .y is dropped). */
static void init_pool(or_state* st) {
    or_pool* pool = &st->pools[st->active];
    const uint32_t n = st->n;
    double* tmp = (double*)malloc(sizeof(double) * n);
    for (uint32_t m = 0; m < st->cfg.n_arrays; ++m) {
        or_box_muller_fill(&st->us, tmp, n);
        if (st->cfg.dtype == OR_F64) {
            memcpy((double*)pool->v + (size_t)m * n, tmp, sizeof(double) * n);
        } else {
            float* f = (float*)pool->v + (size_t)m * n;
            for (uint32_t j = 0; j < n; ++j) f[j] = (float)tmp[j];
        }
    }
    free(tmp);
    double x, y;
    or_box_muller_next(&st->us, &x, &y);
    pool->withheld = x;
    pool->tracked = or_direct_sumsq(st->cfg.n_arrays, st->cfg.dtype, n, pool->v);
    st->avail = 0;
}

/* Constructor + validation (wallace.cpp:139-156). */
int or_state_create(const or_config* cfg, or_state** out) {
    *out = NULL;
    if (cfg->pool_exponent < 8 || cfg->pool_exponent > 20) return OR_EINVAL;
    if (cfg->throwaway_f < 1) return OR_EINVAL;
    if (cfg->restart_interval > 0 && cfg->restart_interval <= cfg->throwaway_f)
        return OR_EINVAL;
    if (cfg->n_arrays != 2 && cfg->n_arrays != 4) return OR_EINVAL;
    if (cfg->dtype > 1 || cfg->scale_mode > 1) return OR_EINVAL;
    or_state* st = (or_state*)calloc(1, sizeof(or_state));
    st->cfg = *cfg;
    st->n = 1u << cfg->pool_exponent;
    or_uniform_init(&st->us, cfg->seed, cfg->stream);
    for (int b = 0; b < 2; ++b)
        st->pools[b].v = calloc((size_t)cfg->n_arrays * st->n, esize(cfg->dtype));
    init_pool(st);
    *out = st;
    return OR_OK;
}

void or_state_destroy(or_state* st) {
    if (!st) return;
    free(st->pools[0].v);
    free(st->pools[1].v);
    free(st);
}

/* advance_pass (wallace.cpp:169-178). */
int or_state_advance_pass(or_state* st, or_params* p) {
    or_pool* src = &st->pools[st->active];
    or_pool* dst = &st->pools[1 - st->active];
    or_params local;
    if (!p) p = &local;
    int rc = or_select_params(&st->us, st->cfg.n_arrays, st->n, src->tracked,
                              src->withheld, st->cfg.scale_mode, p);
    if (rc) return rc;
    or_regenerate(st->cfg.n_arrays, st->cfg.dtype, st->n, src->v, dst->v, p);
    dst->tracked = p->target;
    /* withheld = last slot of the last array (wallace.cpp:136) */
    size_t last = (size_t)st->cfg.n_arrays * st->n - 1;
    dst->withheld = st->cfg.dtype == OR_F64 ? ((double*)dst->v)[last]
                                            : (double)((float*)dst->v)[last];
    st->active = 1 - st->active;
    ++st->pass_count;
    st->avail = 0;
    return OR_OK;
}

static int crossed(uint64_t before, uint64_t after, uint64_t period) {
    return period > 0 && after / period > before / period;
}

/* drift_check (wallace.cpp:225-234). */
int or_state_drift_check(or_state* st) {
    or_pool* pool = &st->pools[st->active];
    double rec = or_direct_sumsq(st->cfg.n_arrays, st->cfg.dtype, st->n, pool->v);
    double rel = fabs(rec / pool->tracked - 1.0);
    if (!(rel <= 1e-3)) return OR_ECORRUPT;
    pool->tracked = rec;
    return OR_OK;
}

void or_state_restart(or_state* st) { init_pool(st); } /* wallace.cpp:236 */

/* refill (wallace.cpp:188-196). */
int or_state_refill(or_state* st) {
    const uint64_t before = st->pass_count;
    for (uint32_t i = 0; i < st->cfg.throwaway_f; ++i) {
        int rc = or_state_advance_pass(st, NULL);
        if (rc) return rc;
    }
    st->avail = (uint64_t)st->cfg.n_arrays * st->n - 1;
    if (crossed(before, st->pass_count, st->cfg.drift_period)) {
        int rc = or_state_drift_check(st);
        if (rc) return rc;
    }
    if (st->cfg.restart_interval > 0 &&
        crossed(before, st->pass_count, st->cfg.restart_interval))
        or_state_restart(st);
    return OR_OK;
}

/* fill (wallace.cpp:198-216): emission order array 0..n-1, each left to
 * right, the final slot withheld; out = mu + sigma * v. */
static int fill_any(or_state* st, void* out, int out_f32, size_t count, double mu,
                    double sigma) {
    if (sigma < 0.0) return OR_EINVAL;
    const uint64_t cap = (uint64_t)st->cfg.n_arrays * st->n - 1;
    size_t done = 0;
    while (done < count) {
        if (st->avail == 0) {
            int rc = or_state_refill(st);
            if (rc) return rc;
        }
        const or_pool* pool = &st->pools[st->active];
        uint64_t pos = cap - st->avail;
        uint64_t take = count - done < st->avail ? count - done : st->avail;
        for (uint64_t i = pos; i < pos + take; ++i) {
            double v = st->cfg.dtype == OR_F64 ? ((const double*)pool->v)[i]
                                               : (double)((const float*)pool->v)[i];
            double o = mu + sigma * v;
            if (out_f32)
                ((float*)out)[done++] = (float)o;
            else
                ((double*)out)[done++] = o;
        }
        st->avail -= take;
    }
    st->emitted += count;
    return OR_OK;
}

int or_state_fill_f64(or_state* st, double* out, size_t count, double mu, double sigma) {
    return fill_any(st, out, 0, count, mu, sigma);
}
int or_state_fill_f32(or_state* st, float* out, size_t count, double mu, double sigma) {
    return fill_any(st, out, 1, count, mu, sigma);
}

void or_state_counters(const or_state* st, uint64_t* out4) {
    out4[0] = st->pass_count;
    out4[1] = st->emitted;
    out4[2] = st->avail;
    out4[3] = st->n;
}

void or_state_get_pool(const or_state* st, double* vals, double* tw) {
    const or_pool* p = &st->pools[st->active];
    size_t total = (size_t)st->cfg.n_arrays * st->n;
    for (size_t i = 0; i < total; ++i)
        vals[i] = st->cfg.dtype == OR_F64 ? ((const double*)p->v)[i]
                                          : (double)((const float*)p->v)[i];
    tw[0] = p->tracked;
    tw[1] = p->withheld;
}

void or_state_set_pool(or_state* st, const double* vals, const double* tw) {
    or_pool* p = &st->pools[st->active];
    size_t total = (size_t)st->cfg.n_arrays * st->n;
    for (size_t i = 0; i < total; ++i) {
        if (st->cfg.dtype == OR_F64)
            ((double*)p->v)[i] = vals[i];
        else
            ((float*)p->v)[i] = (float)vals[i];
    }
    p->tracked = tw[0];
    p->withheld = tw[1];
}

void or_state_get_uniform(const or_state* st, uint64_t* table, uint32_t* r,
                          uint32_t* s, uint64_t* draws) {
    memcpy(table, st->us.table, sizeof(st->us.table));
    *r = st->us.r;
    *s = st->us.s;
    *draws = st->us.draws;
}

/* ------------------------------------------------------------------------
 * Banks of independent pools: pool p is the state
 * (seed, stream + p); the output is CTA-major, pool p owning a contiguous
 * segment of count/P (+1 for p < count % P) values.
 * ---------------------------------------------------------------------- */
static int bank_fill(const or_config* cfg, uint32_t pools, uint64_t count, void* out,
                     int f32, double mu, double sigma) {
    uint64_t base = count / pools, extra = count % pools, off = 0;
    for (uint32_t p = 0; p < pools; ++p) {
        or_config c = *cfg;
        c.stream = cfg->stream + p;
        or_state* st;
        int rc = or_state_create(&c, &st);
        if (rc) return rc;
        uint64_t len = base + (p < extra ? 1 : 0);
        rc = f32 ? or_state_fill_f32(st, (float*)out + off, len, mu, sigma)
                 : or_state_fill_f64(st, (double*)out + off, len, mu, sigma);
        or_state_destroy(st);
        if (rc) return rc;
        off += len;
    }
    return OR_OK;
}
int or_bank_fill_f32(const or_config* cfg, uint32_t pools, uint64_t count, float* out,
                     double mu, double sigma) {
    return bank_fill(cfg, pools, count, out, 1, mu, sigma);
}
int or_bank_fill_f64(const or_config* cfg, uint32_t pools, uint64_t count, double* out,
                     double mu, double sigma) {
    return bank_fill(cfg, pools, count, out, 0, mu, sigma);
}

typedef struct {
    or_state* st;
    uint64_t per_thread;
    uint32_t chunk;
    double sink;
} bench_arg;

static void* bench_worker(void* a) {
    bench_arg* b = (bench_arg*)a;
    int f32 = b->st->cfg.dtype == OR_F32;
    void* buf = malloc((size_t)b->chunk * 8);
    uint64_t done = 0;
    double sink = 0.0;
    while (done < b->per_thread) {
        uint64_t take = b->per_thread - done < b->chunk ? b->per_thread - done : b->chunk;
        if (f32) {
            or_state_fill_f32(b->st, (float*)buf, take, 0.0, 1.0);
            sink += ((float*)buf)[take / 2];
        } else {
            or_state_fill_f64(b->st, (double*)buf, take, 0.0, 1.0);
            sink += ((double*)buf)[take / 2];
        }
        done += take;
    }
    b->sink = sink;
    free(buf);
    return NULL;
}

double or_bench_threads(const or_config* cfg, uint32_t threads, uint64_t per_thread,
                        uint32_t chunk) {
    bench_arg* args = (bench_arg*)calloc(threads, sizeof(bench_arg));
    pthread_t* tids = (pthread_t*)calloc(threads, sizeof(pthread_t));
    for (uint32_t t = 0; t < threads; ++t) {
        or_config c = *cfg;
        c.stream = cfg->stream + t;
        or_state_create(&c, &args[t].st);
        args[t].per_thread = per_thread;
        args[t].chunk = chunk;
    }
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (uint32_t t = 0; t < threads; ++t)
        pthread_create(&tids[t], NULL, bench_worker, &args[t]);
    for (uint32_t t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    for (uint32_t t = 0; t < threads; ++t) or_state_destroy(args[t].st);
    free(args);
    free(tids);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* ------------------------------------------------------------------------
 * Statistics: moments (stats.cpp:89-108, plus the third moment) and the
 * Anderson-Darling A^2 of the simple hypothesis N(0, 1) (new).
 * ---------------------------------------------------------------------- */
void or_moments_f64(const double* v, size_t n, double* out5) {
    double s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    for (size_t i = 0; i < n; ++i) {
        double x = v[i], x2 = x * x;
        s1 += x;
        s2 += x2;
        s3 += x2 * x;
        s4 += x2 * x2;
    }
    double dn = (double)n;
    out5[0] = dn;
    out5[1] = s1 / dn;
    out5[2] = s2 / dn;
    out5[3] = s3 / dn;
    out5[4] = s4 / dn;
}

void or_moments_f32(const float* v, size_t n, double* out5) {
    double s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    for (size_t i = 0; i < n; ++i) {
        double x = v[i], x2 = x * x;
        s1 += x;
        s2 += x2;
        s3 += x2 * x;
        s4 += x2 * x2;
    }
    double dn = (double)n;
    out5[0] = dn;
    out5[1] = s1 / dn;
    out5[2] = s2 / dn;
    out5[3] = s3 / dn;
    out5[4] = s4 / dn;
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* A^2 = -n - (1/n) sum_{i=1..n} (2i-1) [ln Phi(z_(i)) + ln(1 - Phi(z_(n+1-i)))],
 * Phi(z) = erfc(-z/sqrt2)/2 and 1 - Phi(z) = erfc(z/sqrt2)/2 (no cancellation
 * in either tail). */
/* A^2 of the simple N(0,1) hypothesis on a sorted sample (new: the reference
 * has no AD; SURVEY.md §8(c) "parity unpinned").  The textbook form
 *   A^2 = -n - (1/n) sum_i (2i+1) [ln Phi(z_i) + ln(1 - Phi(z_{n-1-i}))]
 * subtracts two O(n) quantities; regrouped per sorted value j,
 *   A^2 = sum_j d_j,  d_j = -1 - [(2j+1) ln Phi(z_j) + (2n-2j-1) ln(1-Phi(z_j))] / n,
 * every d_j is O(1) and the sum stays accurate at n = 2^32.  Summed with
 * Neumaier compensation over [j0, j1) (the GPU kernel, stats_ad.cu, uses the
 * same d_j). */
static void ad_terms(const double* z, const float* zf, size_t n, size_t j0, size_t j1,
                     double* sum, double* comp) {
    const double rs2 = 0.70710678118654752440;
    const double dn = (double)n;
    double s = 0.0, c = 0.0;
    for (size_t j = j0; j < j1; ++j) {
        const double x = z ? z[j] : (double)zf[j];
        const double lo = log(0.5 * erfc(-x * rs2));
        const double hi = log(0.5 * erfc(x * rs2));
        const double wj = 2.0 * (double)j + 1.0;
        const double d = -1.0 - (wj * lo + (2.0 * dn - wj) * hi) / dn;
        const double t = s + d;
        c += fabs(s) >= fabs(d) ? (s - t) + d : (d - t) + s;
        s = t;
    }
    *sum = s;
    *comp = c;
}

static double ad_sorted(const double* z, size_t n) {
    double s, c;
    ad_terms(z, NULL, n, 0, n, &s, &c);
    return s + c;
}

typedef struct {
    const double* z;
    const float* zf;
    size_t n, j0, j1;
    double s, c;
} ad_job;

static void* ad_worker(void* arg) {
    ad_job* j = (ad_job*)arg;
    ad_terms(j->z, j->zf, j->n, j->j0, j->j1, &j->s, &j->c);
    return NULL;
}

static double ad_sorted_threads(const double* z, const float* zf, size_t n, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    ad_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t].z = z;
        jobs[t].zf = zf;
        jobs[t].n = n;
        jobs[t].j0 = n * (size_t)t / (size_t)threads;
        jobs[t].j1 = n * (size_t)(t + 1) / (size_t)threads;
        pthread_create(&th[t], NULL, ad_worker, &jobs[t]);
    }
    double s = 0.0, c = 0.0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        const double d = jobs[t].s, t2 = s + d;
        c += (fabs(s) >= fabs(d) ? (s - t2) + d : (d - t2) + s) + jobs[t].c;
        s = t2;
    }
    return s + c;
}

/* A^2 of an already sorted sample on `threads` host threads (large n). */
double or_ad_sorted_threads(const double* z, size_t n, int threads) {
    return ad_sorted_threads(z, NULL, n, threads);
}
double or_ad_sorted_f32_threads(const float* z, size_t n, int threads) {
    return ad_sorted_threads(NULL, z, n, threads);
}

double or_anderson_darling_f64(const double* v, size_t n) {
    double* z = (double*)malloc(sizeof(double) * n);
    memcpy(z, v, sizeof(double) * n);
    qsort(z, n, sizeof(double), cmp_double);
    double a = ad_sorted(z, n);
    free(z);
    return a;
}

double or_anderson_darling_f32(const float* v, size_t n) {
    double* z = (double*)malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; ++i) z[i] = v[i];
    qsort(z, n, sizeof(double), cmp_double);
    double a = ad_sorted(z, n);
    free(z);
    return a;
}

/* ------------------------------------------------------------------------
 * Uniformity / serial-correlation checks (restated from stats.cpp:10-38,
 * 40-87 and 110-127; pairing as tools/main.cpp:160-193).
 * ---------------------------------------------------------------------- */
int or_to_uv(double x, double y, double* u, double* v) {
    /* stats.cpp:10-16 */
    if (x == 0.0 && y == 0.0) {
        *u = 0.0;
        *v = 0.0;
        return 1;
    }
    *u = exp(-0.5 * (x * x + y * y));
    *v = y == 0.0 ? copysign(1.5707963267948966, x) : atan(x / y);
    return 0;
}

int64_t or_chi2_bin(double v, uint32_t k, double lo, double hi) {
    /* stats.cpp:24-29 */
    if (!(v >= lo && v <= hi)) return -1;
    const double width = hi - lo;
    uint32_t bin = (uint32_t)((v - lo) / width * k);
    if (bin >= k) bin = k - 1;
    return (int64_t)bin;
}

static uint64_t uv_counts(const double* vd, const float* vf, size_t n, uint32_t k, uint64_t* cu,
                          uint64_t* cv) {
    const double kPi2 = 1.5707963267948966; /* tools/main.cpp:162 */
    uint64_t skipped = 0;
    memset(cu, 0, k * sizeof(uint64_t));
    memset(cv, 0, k * sizeof(uint64_t));
    for (size_t i = 0; i + 1 < n; i += 2) {
        const double x = vd ? vd[i] : (double)vf[i];
        const double y = vd ? vd[i + 1] : (double)vf[i + 1];
        double u, v;
        if (or_to_uv(x, y, &u, &v)) {
            ++skipped;
            continue;
        }
        ++cu[or_chi2_bin(u, k, 0.0, 1.0)];
        ++cv[or_chi2_bin(v, k, -kPi2, kPi2)];
    }
    return skipped;
}

uint64_t or_uv_counts_f64(const double* v, size_t n, uint32_t k, uint64_t* cu, uint64_t* cv) {
    return uv_counts(v, NULL, n, k, cu, cv);
}

uint64_t or_uv_counts_f32(const float* v, size_t n, uint32_t k, uint64_t* cu, uint64_t* cv) {
    return uv_counts(NULL, v, n, k, cu, cv);
}

double or_chi2_statistic(const uint64_t* counts, uint32_t k) {
    /* stats.cpp:30-35 */
    uint64_t total = 0;
    for (uint32_t i = 0; i < k; ++i) total += counts[i];
    const double expected = (double)total / k;
    double statistic = 0.0;
    for (uint32_t i = 0; i < k; ++i) {
        const double d = (double)counts[i] - expected;
        statistic += d * d / expected;
    }
    return statistic;
}

static double gamma_p_series(double a, double x) {
    /* stats.cpp:44-55 */
    double ap = a, term = 1.0 / a, sum = term;
    for (int i = 0; i < 100000; ++i) {
        ap += 1.0;
        term *= x / ap;
        sum += term;
        if (fabs(term) < fabs(sum) * 1e-16) break;
    }
    return sum * exp(-x + a * log(x) - lgamma(a));
}

static double gamma_q_contfrac(double a, double x) {
    /* stats.cpp:57-75 (modified Lentz) */
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 100000; ++i) {
        const double an = -i * (i - a);
        b += 2.0;
        d = an * d + b;
        if (fabs(d) < tiny) d = tiny;
        c = b + an / c;
        if (fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (fabs(del - 1.0) < 1e-16) break;
    }
    return h * exp(-x + a * log(x) - lgamma(a));
}

double or_chi2_sf(double statistic, uint32_t dof) {
    /* stats.cpp:79-87 */
    if (statistic < 0.0 || dof < 1) return NAN;
    if (statistic == 0.0) return 1.0;
    const double a = 0.5 * dof, x = 0.5 * statistic;
    return x < a + 1.0 ? 1.0 - gamma_p_series(a, x) : gamma_q_contfrac(a, x);
}

static double autocorr(const double* vd, const float* vf, size_t n, size_t lag) {
    /* stats.cpp:110-127 */
    if (n < lag + 2) return NAN;
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) mean += vd ? vd[i] : (double)vf[i];
    mean /= (double)n;
    const size_t pairs = n - lag;
    double num = 0.0, den = 0.0;
    for (size_t t = 0; t < pairs; ++t) {
        const double a = (vd ? vd[t] : (double)vf[t]) - mean;
        num += a * ((vd ? vd[t + lag] : (double)vf[t + lag]) - mean);
        den += a * a;
    }
    return den == 0.0 ? NAN : num / den;
}

double or_autocorr_f64(const double* v, size_t n, size_t lag) { return autocorr(v, NULL, n, lag); }
double or_autocorr_f32(const float* v, size_t n, size_t lag) { return autocorr(NULL, v, n, lag); }
