// B200 (sm_100a) kernels for the Wallace pool-regeneration hot path.
//
// Reference path (paths relative to /root/reference/proj):
//   uniform generator      src/uniform.cpp:13-51
//   Box-Muller init        src/reference.cpp:9-22, 41-58; src/wallace.cpp:158-167
//   pass parameters        src/wallace.cpp:27-70
//   regeneration pass      src/wallace.cpp:113-137 (segmented; we use the
//                          modular form pinned identical by
//                          tests/test_wallace_core.cpp:203-217)
//   refill / fill / drift  src/wallace.cpp:169-236
//
// Compiled with -fmad=false: every floating-point expression is evaluated
// exactly as written (one rounding per operation), matching the reference's
// FMA-free Release build.  Only sqrt/div (IEEE on device),
// +, -, * and conversions appear on the parity path; log/cos/sin appear only
// in the device Box-Muller initialisation (a few ulp from glibc).
//
// Two engines:
//   * smem  — one CTA per pool, the pool resident in shared memory for the
//             whole fill call; each pass is an in-place permutation+transform
//             staged through registers (gather -> barrier -> transform ->
//             scatter), the last pass of every refill stores the exposed
//             values straight from registers to HBM (coalesced, lane-
//             consecutive columns).
//   * hbm   — pools too large for shared memory: double-buffered in HBM/L2,
//             one grid-wide launch per pass, host-driven control.
#include <cstdio>

#include "internal.h"

namespace wg {

// ---------------------------------------------------------------------------
// Scalar helpers (bit-exact restatements)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double u53(uint64_t w) {
    // next_uniform (uniform.cpp:42-45): top 53 bits * 2^-53
    return (double)(w >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ uint32_t nib(uint64_t w, uint32_t m) {
    // next_int_below (uniform.cpp:47-51)
    return (uint32_t)(u53(w) * (double)m);
}
__device__ __forceinline__ double chi2_target(double r, uint32_t nu) {
    // wallace.cpp:27-31
    double t = r + sqrt(2.0 * (double)nu - 1.0);
    return 0.5 * t * t;
}
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    // uniform.cpp:13-19, counter form: output i = mix(s0 + (i + 1) * golden)
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__constant__ uint32_t c_stride4[4][2] = {{3, 5}, {7, 11}, {13, 17}, {19, 23}};

// Pass parameters from the K = 6 (n=2) / 9 (n=4) uniform words of one pass,
// in the reference's draw order (wallace.cpp:54-58; docs/n4_spec.md §2).
// Returns 0, or WRNG_GPU_ECORRUPT when tracked is not positive (checked
// after the draws, wallace.cpp:59-61).
template <int NA>
__device__ int make_params(const uint64_t* w, uint32_t N, double tracked, double withheld,
                           uint32_t mode, wrng_gpu_params& p) {
    if (NA == 2) {
        p.stride[0] = nib(w[0], 2) == 0 ? 3 : 5;
        p.stride[1] = nib(w[1], 2) == 0 ? 7 : 11;
        p.stride[2] = p.stride[3] = 0;
        p.offset[0] = nib(w[2], N);
        p.offset[1] = nib(w[3], N);
        p.offset[2] = p.offset[3] = 0;
        p.variant = 0;
        // rotation_from_uniform / rotation_from_t (wallace.cpp:33-49)
        const double kTanLo = 0x1.126145e9ecd56p-2;    // 0.26794919243112270
        const double kTanSpan = 0x1.3cd3a2c8198e2p-2;  // kTanHi - kTanLo
        double t = kTanLo + kTanSpan * u53(w[4]);
        uint32_t region = nib(w[5], 3);
        double t2 = t * t;
        double c = (1.0 - t2) / (1.0 + t2);
        double s = 2.0 * t / (1.0 + t2);
        if (region == 0) {
            p.c = c; p.s = s;
        } else if (region == 1) {
            p.c = c; p.s = -s;
        } else {
            p.c = -c; p.s = s;
        }
    } else {
        for (int m = 0; m < 4; ++m) p.stride[m] = c_stride4[m][nib(w[m], 2)];
        for (int m = 0; m < 4; ++m) p.offset[m] = nib(w[4 + m], N);
        p.variant = nib(w[8], 2);
        p.c = 0.0;
        p.s = 0.0;
    }
    p.pad_ = 0;
    if (!(tracked > 0.0)) return WRNG_GPU_ECORRUPT;
    if (mode == WRNG_GPU_CHISQ) {
        p.target_sumsq = chi2_target(withheld, NA * N);
        p.scale = sqrt(p.target_sumsq / tracked);
    } else {
        p.scale = 1.0;
        p.target_sumsq = tracked;
    }
    return 0;
}

// Box-Muller pair (reference.cpp:9-22), u1 == 0 mapped to 2^-53.
__device__ __forceinline__ void box_muller(uint64_t w1, uint64_t w2, double& x, double& y) {
    double u1 = u53(w1);
    if (u1 == 0.0) u1 = 0x1.0p-53;
    double u2 = u53(w2);
    const double pi = 0x1.921fb54442d18p+1;
    double radius = sqrt(-2.0 * log(u1));
    double angle = 2.0 * pi * u2;
    x = radius * cos(angle);
    y = radius * sin(angle);
}

// Output element: mu + sigma * v (wallace.cpp:209-212), in double, then
// narrowed for f32 outputs.  unit (mu = 0, sigma = 1) keeps the reference's
// -0.0 -> +0.0 of `0 + 1 * v` without the double multiply.
template <typename T>
__device__ __forceinline__ void put_out(void* out, uint64_t i, T v, uint32_t out_f32,
                                        uint32_t unit, double mu, double sigma) {
    if (unit) {
        if (out_f32)
            static_cast<float*>(out)[i] = (float)v + 0.0f;
        else
            static_cast<double*>(out)[i] = (double)v + 0.0;
    } else {
        double o = mu + sigma * (double)v;
        if (out_f32)
            static_cast<float*>(out)[i] = (float)o;
        else
            static_cast<double*>(out)[i] = o;
    }
}

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ bool crossed(uint64_t before, uint64_t after, uint64_t period) {
    // wallace.cpp:182-184
    return period > 0 && after / period > before / period;
}

// ---------------------------------------------------------------------------
// CTA-cooperative uniform generator.
//
// x_n = x_{n-607} + x_{n-273} (mod 2^64).  With the table as a 607-word ring
// and cursor r, word k of a step (k < 273) reads slots r+k and r+k+334 and
// writes slot r+k: no slot written in a step is read by another thread of
// the same step, so up to 256 consecutive words are produced in parallel.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t lfg_word_at(uint64_t* tab, uint32_t r, uint32_t k) {
    uint32_t i = r + k;
    i = i >= kTable ? i - kTable : i;
    uint32_t s = i + kGap;
    s = s >= kTable ? s - kTable : s;
    uint64_t w = tab[i] + tab[s];
    tab[i] = w;
    return w;
}

struct Ctl {
    // current pass parameters
    uint32_t stride[4];
    uint32_t offset[4];
    uint32_t variant;
    int32_t error;
    double c0d, c1d;   // n=2: (kc, ks); n=4: (k = scale/2, scale)
    float c0f, c1f;
    double target;
    // pool scalars of the active buffer
    double tracked;
    double withheld;
    double prev_tracked, prev_withheld;
    uint32_t r;
    uint32_t active;
    uint64_t draws;
    uint32_t have_prev;
    uint32_t pad_;
};

// Generates `total` words in steps of `step` (<= 256, <= blockDim) into
// wbuf; fn(base, cnt) runs on all threads after each step.
template <typename F>
__device__ void lfg_bulk(uint64_t* tab, Ctl* ctl, uint64_t* wbuf, uint64_t total,
                         uint32_t step, F fn) {
    uint32_t r = ctl->r;
    for (uint64_t base = 0; base < total; base += step) {
        uint32_t cnt = (uint32_t)umin64(step, total - base);
        if (threadIdx.x < cnt) wbuf[threadIdx.x] = lfg_word_at(tab, r, threadIdx.x);
        r += cnt;
        r = r >= kTable ? r - kTable : r;
        __syncthreads();
        fn(base, cnt);
        __syncthreads();
    }
    if (threadIdx.x == 0) ctl->r = r;
    __syncthreads();
}

// Seeds the generator (uniform.cpp:23-32): table[i] = splitmix64 output i of
// seed ^ rotl(stream, 32), then 6070 discarded words, draws = 0.
__device__ void lfg_seed(uint64_t* tab, Ctl* ctl, uint64_t* wbuf, uint64_t seed,
                         uint64_t stream, uint32_t step) {
    const uint64_t s0 = seed ^ ((stream << 32) | (stream >> 32));
    for (uint32_t i = threadIdx.x; i < kTable; i += blockDim.x)
        tab[i] = splitmix64(s0 + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull);
    if (threadIdx.x == 0) {
        ctl->r = 0;
        ctl->draws = 0;
    }
    __syncthreads();
    lfg_bulk(tab, ctl, wbuf, kWarmup, step, [](uint64_t, uint32_t) {});
    if (threadIdx.x == 0) ctl->draws = 0;
    __syncthreads();
}

// Sequential sum of squares, Pool::direct_sumsq order (wallace.cpp:13-18).
template <typename T>
__device__ double seq_sumsq(const T* v, uint32_t n) {
    double q = 0.0;
#pragma unroll 8
    for (uint32_t i = 0; i < n; ++i) {
        double d = (double)v[i];
        q = q + d * d;
    }
    return q;
}

// init_pool (wallace.cpp:158-167) into a pool array `pool` (shared or
// global): Box-Muller pairs fill arrays 0..n-1 in order, then withheld = .x
// of one more pair; tracked = sequential sum.  Consumes n*N + 2 uniforms.
template <typename T>
__device__ void init_pool_dev(T* pool, uint64_t nvals, uint64_t* tab, Ctl* ctl,
                              uint64_t* wbuf, uint32_t step) {
    lfg_bulk(tab, ctl, wbuf, nvals + 2, step, [&](uint64_t base, uint32_t cnt) {
        for (uint32_t k = threadIdx.x; k < cnt / 2; k += blockDim.x) {
            double x, y;
            box_muller(wbuf[2 * k], wbuf[2 * k + 1], x, y);
            uint64_t i = base + 2 * k;
            if (i < nvals) {
                // fill_from_pairs: out = mu + sigma * z with mu = 0, sigma = 1
                pool[i] = (T)(x + 0.0);
                pool[i + 1] = (T)(y + 0.0);
            } else {
                ctl->withheld = x;
            }
        }
    });
    if (threadIdx.x == 0) {
        ctl->draws += nvals + 2;
        ctl->tracked = seq_sumsq(pool, (uint32_t)nvals);
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Shared-memory engine
// ---------------------------------------------------------------------------
template <typename T, int NA, int J>
struct SmemPass {
    // One regeneration pass in place on the shared pool.  Returns false on a
    // device-detected error (ctl->error set).
    static __device__ bool run(T* pool, uint64_t* tab, uint64_t* wbuf, Ctl* ctl,
                               const KernelArgs& a, uint32_t N, bool last_in_launch,
                               T* prev_gmem, uint64_t emit_n, void* out_p,
                               wrng_gpu_params* rec) {
        constexpr int K = NA == 2 ? 6 : 9;
        const uint32_t tid = threadIdx.x, nth = blockDim.x, mask = N - 1;
        // (1) warp 0: K uniform words, then lane 0 derives the parameters.
        if (tid < 32) {
            uint32_t r = ctl->r;
            if (tid < K) wbuf[tid] = lfg_word_at(tab, r, tid);
            __syncwarp();
            if (tid == 0) {
                r += K;
                ctl->r = r >= kTable ? r - kTable : r;
                ctl->draws += K;
                wrng_gpu_params p;
                int err = make_params<NA>(wbuf, N, ctl->tracked, ctl->withheld, a.mode, p);
                ctl->error = err;
                if (!err) {
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        ctl->stride[m] = p.stride[m];
                        ctl->offset[m] = p.offset[m];
                    }
                    ctl->variant = p.variant;
                    ctl->target = p.target_sumsq;
                    if (NA == 2) {
                        // regenerate folds the scale into the matrix (wallace.cpp:116-117)
                        ctl->c0d = p.c * p.scale;
                        ctl->c1d = p.s * p.scale;
                    } else {
                        ctl->c0d = 0.5 * p.scale;
                        ctl->c1d = p.scale;
                    }
                    ctl->c0f = (float)ctl->c0d;
                    ctl->c1f = (float)ctl->c1d;
                    if (rec) *rec = p;
                }
            }
        }
        __syncthreads();
        if (ctl->error) return false;

        uint32_t st[NA], of[NA];
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            st[m] = ctl->stride[m];
            of[m] = ctl->offset[m];
        }
        // (2) gather: column j = tid + k * nth, lane-consecutive -> odd strides
        //     hit 32 distinct banks (fp32) / 2 wavefronts (fp64).
        T v[NA][J];
#pragma unroll
        for (int k = 0; k < J; ++k) {
            const uint32_t j = tid + k * nth;
#pragma unroll
            for (int m = 0; m < NA; ++m) v[m][k] = pool[m * N + ((st[m] * j + of[m]) & mask)];
        }
        if (last_in_launch) {
            // Keep the pre-pass pool as the inactive buffer (wallace.hpp:167).
#pragma unroll
            for (int k = 0; k < J; ++k) {
                const uint32_t j = tid + k * nth;
#pragma unroll
                for (int m = 0; m < NA; ++m)
                    prev_gmem[m * N + ((st[m] * j + of[m]) & mask)] = v[m][k];
            }
            if (tid == 0) {
                ctl->prev_tracked = ctl->tracked;
                ctl->prev_withheld = ctl->withheld;
                ctl->have_prev = 1;
            }
        }
        __syncthreads();

        // (3) transform, store in place, emit.
        const uint32_t variant = ctl->variant;
        T c0, c1;
        if (sizeof(T) == 4) {
            c0 = (T)ctl->c0f;
            c1 = (T)ctl->c1f;
        } else {
            c0 = (T)ctl->c0d;
            c1 = (T)ctl->c1d;
        }
        const double target = ctl->target;
#pragma unroll
        for (int k = 0; k < J; ++k) {
            const uint32_t j = tid + k * nth;
            T y[NA];
            if (NA == 2) {
                // dst.x = kc*xs + ks*ys ; dst.y = kc*ys - ks*xs (wallace.cpp:130-131)
                T xs = v[0][k], ys = v[1][k];
                y[0] = c0 * xs + c1 * ys;
                y[1] = c0 * ys - c1 * xs;
            } else {
                T a0 = v[0][k], a1 = v[NA > 1 ? 1 : 0][k], a2 = v[NA > 2 ? 2 : 0][k],
                  a3 = v[NA > 3 ? 3 : 0][k];
                if (variant == 0) {
                    // (1/2) H4 (docs/n4_spec.md §3)
                    T pp = a0 + a1, q = a0 - a1, r = a2 + a3, s = a2 - a3;
                    y[0] = c0 * (pp + r);
                    y[NA > 1 ? 1 : 0] = c0 * (q + s);
                    y[NA > 2 ? 2 : 0] = c0 * (pp - r);
                    y[NA > 3 ? 3 : 0] = c0 * (q - s);
                } else {
                    // (1/2) J - I
                    T t = (T)0.5 * ((a0 + a1) + (a2 + a3));
                    y[0] = c1 * (t - a0);
                    y[NA > 1 ? 1 : 0] = c1 * (t - a1);
                    y[NA > 2 ? 2 : 0] = c1 * (t - a2);
                    y[NA > 3 ? 3 : 0] = c1 * (t - a3);
                }
            }
#pragma unroll
            for (int m = 0; m < NA; ++m) {
                pool[m * N + j] = y[m];
                const uint64_t flat = (uint64_t)m * N + j;
                if (flat < emit_n) put_out(out_p, flat, y[m], a.out_f32, a.unit, a.mu, a.sigma);
            }
            if (j == N - 1) ctl->withheld = (double)y[NA - 1];  // wallace.cpp:136
        }
        if (tid == 0) {
            ctl->tracked = target;  // wallace.cpp:135
            ctl->active ^= 1u;
        }
        __syncthreads();
        return true;
    }
};

template <typename T, int NA, int J>
__global__ void __launch_bounds__(1024, 1) k_smem(KernelArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t N = a.N;
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    const uint32_t p = blockIdx.x;
    const uint64_t nvals = (uint64_t)NA * N;
    const uint64_t cap = nvals - 1;
    const uint32_t step = nth < 256 ? nth : 256;

    T* pool = reinterpret_cast<T*>(sm);
    uint64_t* tab = reinterpret_cast<uint64_t*>(sm + nvals * sizeof(T));
    uint64_t* wbuf = tab + 608;
    Ctl* ctl = reinterpret_cast<Ctl*>(wbuf + 256);

    PoolMeta* meta = a.meta + p;
    LfgState* lg = a.lfg + p;
    // A device-raised error is sticky until the host observes it: the pool
    // stays frozen at the failure point (wrng_gpu_synchronize reports it).
    if (a.op != OP_INIT && meta->error) return;

    // ---- load state -------------------------------------------------------
    uint64_t pc, avail, emitted;
    uint32_t active0;
    if (a.op == OP_INIT) {
        pc = avail = emitted = 0;
        active0 = 0;
        if (tid == 0) {
            ctl->active = 0;
            ctl->error = 0;
            ctl->have_prev = 0;
        }
        lfg_seed(tab, ctl, wbuf, a.seed, a.stream0 + p, step);
    } else {
        pc = meta->pass_count;
        avail = meta->avail;
        emitted = meta->emitted;
        active0 = meta->active;
        for (uint32_t i = tid; i < kTable; i += nth) tab[i] = lg->table[i];
        if (tid == 0) {
            ctl->r = lg->r;
            ctl->draws = lg->draws;
            ctl->active = active0;
            ctl->tracked = meta->tracked[active0];
            ctl->withheld = meta->withheld[active0];
            ctl->error = 0;
            ctl->have_prev = 0;
        }
        const uint4* src = reinterpret_cast<const uint4*>(
            static_cast<const T*>(a.buf[active0]) + (uint64_t)p * nvals);
        uint4* dst = reinterpret_cast<uint4*>(pool);
        const uint32_t nvec = (uint32_t)(nvals * sizeof(T) / 16);
        for (uint32_t i = tid; i < nvec; i += nth) dst[i] = src[i];
    }
    __syncthreads();

    // After the last pass of this launch the inactive buffer must hold that
    // pass's source pool (advance_pass swaps, wallace.cpp:170-174): the
    // buffer index active *before* the pass.
    auto prev_of = [&](uint32_t act_before) -> T* {
        return static_cast<T*>(a.buf[act_before]) + (uint64_t)p * nvals;
    };

    const uint64_t len = a.lay.len_base + (p < a.lay.len_extra ? 1 : 0);
    const uint64_t out_base =
        (uint64_t)p * a.lay.off_stride + (p < a.lay.off_extra ? p : a.lay.off_extra);
    const uint32_t f = a.f;

    // ---- total passes of this launch (to know the last one) ---------------
    uint64_t total_passes = 0;
    if (a.op == OP_FILL) {
        uint64_t rem = len;
        uint64_t av = avail;
        if (av > 0 && rem > 0) rem -= umin64(rem, av);
        if (a.restart == 0) {
            total_passes = (rem + cap - 1) / cap * f;
        } else {
            uint64_t c = pc;
            while (rem > 0) {
                uint64_t before = c;
                c += f;
                total_passes += f;
                if (crossed(before, c, a.restart)) continue;
                rem -= umin64(rem, cap);
            }
        }
    } else if (a.op == OP_PASSES) {
        total_passes = a.npasses;
    } else if (a.op == OP_REFILL) {
        total_passes = f;
    }

    uint64_t pass_i = 0;
    int err = 0;
    auto do_pass = [&](uint64_t emit_n, void* out_p, wrng_gpu_params* rec) -> bool {
        ++pass_i;
        const bool last = pass_i == total_passes;
        bool ok = SmemPass<T, NA, J>::run(pool, tab, wbuf, ctl, a, N, last,
                                          last ? prev_of(ctl->active) : nullptr, emit_n,
                                          out_p, rec);
        if (!ok) return false;
        ++pc;
        return true;
    };
    auto drift_check = [&]() -> bool {
        // wallace.cpp:225-234
        if (tid == 0) {
            double rec = seq_sumsq(pool, (uint32_t)nvals);
            double rel = fabs(rec / ctl->tracked - 1.0);
            if (!(rel <= 1e-3))
                ctl->error = WRNG_GPU_ECORRUPT;
            else
                ctl->tracked = rec;
        }
        __syncthreads();
        return ctl->error == 0;
    };
    auto restart = [&]() {
        init_pool_dev(pool, nvals, tab, ctl, wbuf, step);
        avail = 0;
    };
    // refill (wallace.cpp:188-196) with the exposed window fused into the
    // last pass.  Returns false on error.
    auto refill = [&](uint64_t emit_want, void* out_p, uint64_t& emitted_now) -> bool {
        const uint64_t before = pc;
        const bool will_restart = a.restart > 0 && crossed(before, before + f, a.restart);
        const uint64_t emit_n = will_restart ? 0 : emit_want;
        for (uint32_t i = 0; i < f; ++i) {
            if (!do_pass(i + 1 == f ? emit_n : 0, out_p, nullptr)) return false;
        }
        avail = cap;
        if (crossed(before, pc, a.drift) && !drift_check()) return false;
        if (will_restart) {
            restart();
            emitted_now = 0;
            return true;
        }
        emitted_now = emit_n;
        return true;
    };

    if (a.op == OP_FILL) {
        uint64_t done = 0;
        char* outc = static_cast<char*>(a.out);
        const uint32_t esz = a.out_f32 ? 4 : 8;
        if (avail > 0 && len > 0) {
            // leftover of the current pool: flat [pos, pos + take)
            const uint64_t take = umin64(len, avail);
            const uint64_t pos = cap - avail;
            void* o = outc + out_base * esz;
            for (uint64_t i = tid; i < take; i += nth)
                put_out(o, i, pool[pos + i], a.out_f32, a.unit, a.mu, a.sigma);
            done = take;
            avail -= take;
        }
        while (done < len) {
            uint64_t got = 0;
            void* o = outc + (out_base + done) * esz;
            if (!refill(umin64(len - done, cap), o, got)) {
                err = ctl->error;
                break;
            }
            done += got;
            avail -= got;
        }
        if (!err) emitted += len;
    } else if (a.op == OP_PASSES) {
        for (uint32_t i = 0; i < a.npasses; ++i) {
            wrng_gpu_params* rec =
                (a.params_out && i + 1 == a.npasses) ? a.params_out + p : nullptr;
            if (!do_pass(0, nullptr, rec)) {
                err = ctl->error;
                break;
            }
            avail = 0;
        }
    } else if (a.op == OP_REFILL) {
        uint64_t got;
        if (!refill(0, nullptr, got)) err = ctl->error;
    } else if (a.op == OP_DRIFT) {
        if (!drift_check()) err = ctl->error;
    } else if (a.op == OP_RESTART || a.op == OP_INIT) {
        restart();
    }

    // ---- write back -------------------------------------------------------
    __syncthreads();
    const uint32_t act = ctl->active;
    {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<T*>(a.buf[act]) + (uint64_t)p * nvals);
        const uint4* src = reinterpret_cast<const uint4*>(pool);
        const uint32_t nvec = (uint32_t)(nvals * sizeof(T) / 16);
        for (uint32_t i = tid; i < nvec; i += nth) dst[i] = src[i];
    }
    for (uint32_t i = tid; i < kTable; i += nth) lg->table[i] = tab[i];
    if (tid == 0) {
        lg->r = ctl->r;
        lg->draws = ctl->draws;
        meta->tracked[act] = ctl->tracked;
        meta->withheld[act] = ctl->withheld;
        if (ctl->have_prev) {
            meta->tracked[act ^ 1u] = ctl->prev_tracked;
            meta->withheld[act ^ 1u] = ctl->prev_withheld;
        }
        if (a.op == OP_INIT) {
            meta->tracked[1] = 0.0;
            meta->withheld[1] = 0.0;
        }
        meta->active = act;
        meta->pass_count = pc;
        meta->avail = avail;
        meta->emitted = emitted;
        meta->error = (uint32_t)err;  // 0 here unless this launch failed
    }
}

// Largest pool (bytes) one CTA keeps in shared memory.  Leaves room for the
// lag table (4.9 KiB), word staging (2 KiB) and control block.
static constexpr uint32_t kSmemPoolMax = 192 * 1024;

static uint32_t smem_bytes(uint32_t n_arrays, uint32_t dtype, uint32_t N) {
    const uint32_t es = dtype == WRNG_GPU_F64 ? 8 : 4;
    return n_arrays * N * es + 608 * 8 + 256 * 8 + (uint32_t)sizeof(Ctl);
}

bool smem_engine_fits(uint32_t n_arrays, uint32_t dtype, uint32_t N) {
    const uint32_t es = dtype == WRNG_GPU_F64 ? 8 : 4;
    return (uint64_t)n_arrays * N * es <= kSmemPoolMax;
}

// Columns per thread: enough independent gathers per thread for latency
// hiding, within 64 registers at 1024 threads/SM.
EngineShape smem_engine_shape(uint32_t n_arrays, uint32_t dtype, uint32_t N) {
    const uint32_t regs_per_col = n_arrays * (dtype == WRNG_GPU_F64 ? 2 : 1);
    uint32_t j = 32 / regs_per_col;  // 32 data registers
    if (j > 16) j = 16;
    while (N / j < 32 && j > 4) j /= 2;
    while (N / j > 1024) j *= 2;
    EngineShape s;
    s.j = j;
    s.threads = N / j;
    s.smem = smem_bytes(n_arrays, dtype, N);
    return s;
}

template <typename T, int NA>
static cudaError_t launch_smem_t(const KernelArgs& a, cudaStream_t st, const EngineShape& s) {
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)s.smem);
        if (e != cudaSuccess) return e;
        kern<<<a.pools, s.threads, s.smem, st>>>(a);
        return cudaGetLastError();
    };
    switch (s.j) {
        case 4: return go(k_smem<T, NA, 4>);
        case 8: return go(k_smem<T, NA, 8>);
        case 16: return go(k_smem<T, NA, 16>);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_smem(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                        cudaStream_t st) {
    EngineShape s = smem_engine_shape(n_arrays, dtype, a.N);
    if (dtype == WRNG_GPU_F64)
        return n_arrays == 2 ? launch_smem_t<double, 2>(a, st, s)
                             : launch_smem_t<double, 4>(a, st, s);
    return n_arrays == 2 ? launch_smem_t<float, 2>(a, st, s)
                         : launch_smem_t<float, 4>(a, st, s);
}

// ---------------------------------------------------------------------------
// HBM engine (pools larger than shared memory; one pool per launch row)
// ---------------------------------------------------------------------------

// One warp per pool: the LFG-dependent part of `npass` consecutive passes'
// parameters (strides, offsets, variant / rotation).  The scale needs the
// previous pass's withheld value and is derived inside each pass kernel.
template <int NA>
__global__ void k_hbm_params(uint32_t N, LfgState* lfg, wrng_gpu_params* params,
                             uint32_t npass, PoolMeta* meta) {
    constexpr int K = NA == 2 ? 6 : 9;
    __shared__ uint64_t tab[kTable];
    __shared__ uint64_t w[32];
    LfgState* lg = lfg + blockIdx.x;
    if (meta[blockIdx.x].error) return;
    for (uint32_t i = threadIdx.x; i < kTable; i += 32) tab[i] = lg->table[i];
    uint32_t r = lg->r;
    __syncwarp();
    for (uint32_t ps = 0; ps < npass; ++ps) {
        if (threadIdx.x < K) w[threadIdx.x] = lfg_word_at(tab, r, threadIdx.x);
        __syncwarp();
        r += K;
        r = r >= kTable ? r - kTable : r;
        if (threadIdx.x == 0) {
            wrng_gpu_params p;
            // tracked = 1 placeholder: scale/target are recomputed per pass.
            make_params<NA>(w, N, 1.0, 0.0, WRNG_GPU_FIXED, p);
            params[(uint64_t)blockIdx.x * npass + ps] = p;
        }
        __syncwarp();
    }
    for (uint32_t i = threadIdx.x; i < kTable; i += 32) lg->table[i] = tab[i];
    if (threadIdx.x == 0) {
        lg->r = r;
        lg->draws += (uint64_t)K * npass;
    }
}

cudaError_t launch_hbm_params(uint32_t n_arrays, uint32_t N, LfgState* lfg,
                              wrng_gpu_params* params, uint32_t npass, PoolMeta* meta,
                              cudaStream_t st) {
    if (n_arrays == 2)
        k_hbm_params<2><<<1, 32, 0, st>>>(N, lfg, params, npass, meta);
    else
        k_hbm_params<4><<<1, 32, 0, st>>>(N, lfg, params, npass, meta);
    return cudaGetLastError();
}

constexpr uint32_t kHbmThreads = 256;
constexpr uint32_t kHbmJ = 4;

template <typename T, int NA>
__global__ void __launch_bounds__(kHbmThreads) k_hbm_pass(KernelArgs a,
                                                          wrng_gpu_params* params,
                                                          HbmPass ps) {
    __shared__ double s_c0, s_c1, s_target, s_scale;
    __shared__ int s_err;
    const uint32_t N = a.N, mask = N - 1;
    PoolMeta* meta = a.meta;
    const uint32_t src = ps.src, dst = src ^ 1u;
    const wrng_gpu_params prm = params[ps.param_idx];
    if (threadIdx.x == 0) {
        int err = meta->error ? -1 : 0;
        double tracked = meta->tracked[src], withheld = meta->withheld[src];
        if (!err) {
            if (!(tracked > 0.0)) {
                err = WRNG_GPU_ECORRUPT;
            } else {
                double target, scale;
                if (a.mode == WRNG_GPU_CHISQ) {
                    target = chi2_target(withheld, NA * N);
                    scale = sqrt(target / tracked);
                } else {
                    scale = 1.0;
                    target = tracked;
                }
                s_target = target;
                s_scale = scale;
                if (NA == 2) {
                    s_c0 = prm.c * scale;
                    s_c1 = prm.s * scale;
                } else {
                    s_c0 = 0.5 * scale;
                    s_c1 = scale;
                }
            }
        }
        s_err = err;
    }
    __syncthreads();
    if (s_err) {
        if (s_err > 0 && blockIdx.x == 0 && threadIdx.x == 0) meta->error = s_err;
        return;
    }
    const T* sp = static_cast<const T*>(a.buf[src]);
    T* dp = static_cast<T*>(a.buf[dst]);
    T c0, c1;
    if (sizeof(T) == 4) {
        c0 = (T)(float)s_c0;
        c1 = (T)(float)s_c1;
    } else {
        c0 = (T)s_c0;
        c1 = (T)s_c1;
    }
    uint32_t stv[NA], ofv[NA];
#pragma unroll
    for (int m = 0; m < NA; ++m) {
        stv[m] = prm.stride[m];
        ofv[m] = prm.offset[m];
    }
    const uint32_t nth = blockDim.x;
    const uint32_t j0 = blockIdx.x * (nth * kHbmJ) + threadIdx.x;
    T v[NA][kHbmJ];
#pragma unroll
    for (int k = 0; k < (int)kHbmJ; ++k) {
        const uint32_t j = j0 + k * nth;
#pragma unroll
        for (int m = 0; m < NA; ++m)
            v[m][k] = __ldg(sp + (uint64_t)m * N + ((stv[m] * j + ofv[m]) & mask));
    }
    char* outc = static_cast<char*>(a.out) + ps.out_off * (a.out_f32 ? 4 : 8);
#pragma unroll
    for (int k = 0; k < (int)kHbmJ; ++k) {
        const uint32_t j = j0 + k * nth;
        T y[NA];
        if (NA == 2) {
            T xs = v[0][k], ys = v[1][k];
            y[0] = c0 * xs + c1 * ys;
            y[1] = c0 * ys - c1 * xs;
        } else {
            T a0 = v[0][k], a1 = v[NA > 1 ? 1 : 0][k], a2 = v[NA > 2 ? 2 : 0][k],
              a3 = v[NA > 3 ? 3 : 0][k];
            if (prm.variant == 0) {
                T pp = a0 + a1, q = a0 - a1, r = a2 + a3, s = a2 - a3;
                y[0] = c0 * (pp + r);
                y[NA > 1 ? 1 : 0] = c0 * (q + s);
                y[NA > 2 ? 2 : 0] = c0 * (pp - r);
                y[NA > 3 ? 3 : 0] = c0 * (q - s);
            } else {
                T t = (T)0.5 * ((a0 + a1) + (a2 + a3));
                y[0] = c1 * (t - a0);
                y[NA > 1 ? 1 : 0] = c1 * (t - a1);
                y[NA > 2 ? 2 : 0] = c1 * (t - a2);
                y[NA > 3 ? 3 : 0] = c1 * (t - a3);
            }
        }
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            dp[(uint64_t)m * N + j] = y[m];
            const uint64_t flat = (uint64_t)m * N + j;
            if (flat < ps.emit_n) put_out(outc, flat, y[m], a.out_f32, a.unit, a.mu, a.sigma);
        }
        if (j == N - 1) meta->withheld[dst] = (double)y[NA - 1];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        params[ps.param_idx].scale = s_scale;
        params[ps.param_idx].target_sumsq = s_target;
        meta->tracked[dst] = s_target;
        meta->active = dst;
        meta->pass_count += 1;
        meta->avail = ps.end_refill ? (uint64_t)NA * N - 1 - ps.emit_n : 0;
    }
}

cudaError_t launch_hbm_pass(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                            wrng_gpu_params* params, const HbmPass& ps,
                            cudaStream_t st) {
    const uint32_t nth = a.N / kHbmJ < kHbmThreads ? a.N / kHbmJ : kHbmThreads;
    const uint32_t grid = a.N / (nth * kHbmJ);
    if (dtype == WRNG_GPU_F64) {
        if (n_arrays == 2)
            k_hbm_pass<double, 2><<<grid, nth, 0, st>>>(a, params, ps);
        else
            k_hbm_pass<double, 4><<<grid, nth, 0, st>>>(a, params, ps);
    } else {
        if (n_arrays == 2)
            k_hbm_pass<float, 2><<<grid, nth, 0, st>>>(a, params, ps);
        else
            k_hbm_pass<float, 4><<<grid, nth, 0, st>>>(a, params, ps);
    }
    return cudaGetLastError();
}

template <typename T>
__global__ void k_hbm_emit(KernelArgs a, uint32_t buf, uint64_t pos, uint64_t take,
                           uint64_t out_off) {
    if (a.meta->error) return;
    const T* sp = static_cast<const T*>(a.buf[buf]) + pos;
    char* o = static_cast<char*>(a.out) + out_off * (a.out_f32 ? 4 : 8);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < take;
         i += (uint64_t)gridDim.x * blockDim.x)
        put_out(o, i, sp[i], a.out_f32, a.unit, a.mu, a.sigma);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.meta->avail -= take;
}

cudaError_t launch_hbm_emit(uint32_t, uint32_t dtype, const KernelArgs& a, uint32_t buf,
                            uint64_t pos, uint64_t take, uint64_t out_off,
                            cudaStream_t st) {
    uint32_t grid = (uint32_t)umin64((take + 255) / 256, 148 * 8);
    if (grid == 0) grid = 1;
    if (dtype == WRNG_GPU_F64)
        k_hbm_emit<double><<<grid, 256, 0, st>>>(a, buf, pos, take, out_off);
    else
        k_hbm_emit<float><<<grid, 256, 0, st>>>(a, buf, pos, take, out_off);
    return cudaGetLastError();
}

// drift_check on an HBM pool.  Default: one thread, left-to-right, exactly
// Pool::direct_sumsq (wallace.cpp:13-18).  tree != 0: blocked parallel
// reduction (documented deviation, relative error ~1e-16 * log n).
template <typename T>
__global__ void k_hbm_drift_seq(KernelArgs a, uint32_t buf, uint64_t nvals) {
    if (a.meta->error || threadIdx.x != 0) return;
    const T* v = static_cast<const T*>(a.buf[buf]);
    double q = 0.0;
#pragma unroll 16
    for (uint64_t i = 0; i < nvals; ++i) {
        double d = (double)v[i];
        q = q + d * d;
    }
    double rel = fabs(q / a.meta->tracked[buf] - 1.0);
    if (!(rel <= 1e-3))
        a.meta->error = WRNG_GPU_ECORRUPT;
    else
        a.meta->tracked[buf] = q;
}

template <typename T>
__global__ void k_hbm_drift_tree_partial(KernelArgs a, uint32_t buf, uint64_t nvals,
                                         double* partial) {
    __shared__ double red[256];
    const T* v = static_cast<const T*>(a.buf[buf]);
    double q = 0.0;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < nvals; i += gridDim.x * 256ull) {
        double d = (double)v[i];
        q += d * d;
    }
    red[threadIdx.x] = q;
    __syncthreads();
    for (uint32_t s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void k_hbm_drift_tree_final(KernelArgs a, uint32_t buf, const double* partial,
                                       uint32_t nb) {
    if (a.meta->error || threadIdx.x != 0) return;
    double q = 0.0;
    for (uint32_t i = 0; i < nb; ++i) q += partial[i];
    double rel = fabs(q / a.meta->tracked[buf] - 1.0);
    if (!(rel <= 1e-3))
        a.meta->error = WRNG_GPU_ECORRUPT;
    else
        a.meta->tracked[buf] = q;
}

cudaError_t launch_hbm_drift(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                             uint32_t buf, int tree, double* scratch, cudaStream_t st) {
    const uint64_t nvals = (uint64_t)n_arrays * a.N;
    if (!tree) {
        if (dtype == WRNG_GPU_F64)
            k_hbm_drift_seq<double><<<1, 32, 0, st>>>(a, buf, nvals);
        else
            k_hbm_drift_seq<float><<<1, 32, 0, st>>>(a, buf, nvals);
        return cudaGetLastError();
    }
    const uint32_t nb = 296;
    if (dtype == WRNG_GPU_F64)
        k_hbm_drift_tree_partial<double><<<nb, 256, 0, st>>>(a, buf, nvals, scratch);
    else
        k_hbm_drift_tree_partial<float><<<nb, 256, 0, st>>>(a, buf, nvals, scratch);
    k_hbm_drift_tree_final<<<1, 32, 0, st>>>(a, buf, scratch, nb);
    return cudaGetLastError();
}

// init_pool / restart of an HBM pool: one CTA generates the n*N + 2 uniforms
// 256 at a time and writes Box-Muller values straight to the pool buffer.
template <typename T>
__global__ void __launch_bounds__(256) k_hbm_init(KernelArgs a, uint32_t buf, int seed_lfg,
                                                  uint32_t n_arrays) {
    __shared__ uint64_t tab[608];
    __shared__ uint64_t wbuf[256];
    __shared__ Ctl ctl;
    LfgState* lg = a.lfg;
    PoolMeta* meta = a.meta;
    if (!seed_lfg && meta->error) return;
    if (seed_lfg) {
        if (threadIdx.x == 0) ctl.active = 0;
        lfg_seed(tab, &ctl, wbuf, a.seed, a.stream0, 256);
    } else {
        for (uint32_t i = threadIdx.x; i < kTable; i += 256) tab[i] = lg->table[i];
        if (threadIdx.x == 0) {
            ctl.r = lg->r;
            ctl.draws = lg->draws;
        }
        __syncthreads();
    }
    T* pool = static_cast<T*>(a.buf[buf]);
    init_pool_dev(pool, (uint64_t)n_arrays * a.N, tab, &ctl, wbuf, 256);
    for (uint32_t i = threadIdx.x; i < kTable; i += 256) lg->table[i] = tab[i];
    if (threadIdx.x == 0) {
        lg->r = ctl.r;
        lg->draws = ctl.draws;
        meta->tracked[buf] = ctl.tracked;
        meta->withheld[buf] = ctl.withheld;
        meta->avail = 0;
        if (seed_lfg) {
            meta->tracked[buf ^ 1u] = 0.0;
            meta->withheld[buf ^ 1u] = 0.0;
            meta->active = buf;
            meta->pass_count = 0;
            meta->emitted = 0;
            meta->error = 0;
        }
    }
}

cudaError_t launch_hbm_init(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                            uint32_t buf, int seed_lfg, cudaStream_t st) {
    if (dtype == WRNG_GPU_F64)
        k_hbm_init<double><<<1, 256, 0, st>>>(a, buf, seed_lfg, n_arrays);
    else
        k_hbm_init<float><<<1, 256, 0, st>>>(a, buf, seed_lfg, n_arrays);
    return cudaGetLastError();
}

__global__ void k_setmeta(PoolMeta* meta, uint64_t pass_count, uint64_t avail,
                          uint64_t emitted, uint32_t active) {
    if (meta->error) return;
    meta->pass_count = pass_count;
    meta->avail = avail;
    meta->emitted = emitted;
    meta->active = active;
}

cudaError_t launch_hbm_setmeta(PoolMeta* meta, uint64_t pass_count, uint64_t avail,
                               uint64_t emitted, uint32_t active, cudaStream_t st) {
    k_setmeta<<<1, 1, 0, st>>>(meta, pass_count, avail, emitted, active);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Validation moments (stats.cpp:89-108 + m3): per-block fp64 partial sums
// (s1..s4), summed in block order by one thread.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_moments_partial(const T* v, uint64_t n, double* partials) {
    __shared__ double red[4][256];
    double s[4] = {0, 0, 0, 0};
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
        double x = (double)v[i], x2 = x * x;
        s[0] += x;
        s[1] += x2;
        s[2] += x2 * x;
        s[3] += x2 * x2;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) red[k][threadIdx.x] = s[k];
    __syncthreads();
    for (uint32_t st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st)
#pragma unroll
            for (int k = 0; k < 4; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x < 4) partials[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void k_moments_final(const double* partials, uint32_t nb, uint64_t n,
                                double* out5) {
    if (threadIdx.x != 0) return;
    double s[4] = {0, 0, 0, 0};
    for (uint32_t b = 0; b < nb; ++b)
        for (int k = 0; k < 4; ++k) s[k] += partials[b * 4 + k];
    double dn = (double)n;
    out5[0] = dn;
    for (int k = 0; k < 4; ++k) out5[1 + k] = s[k] / dn;
}

cudaError_t launch_moments(const void* v, int is_f32, uint64_t n, double* partials,
                           uint32_t nblocks, double* out5_dev, cudaStream_t st) {
    if (is_f32)
        k_moments_partial<float><<<nblocks, 256, 0, st>>>(static_cast<const float*>(v), n,
                                                          partials);
    else
        k_moments_partial<double><<<nblocks, 256, 0, st>>>(static_cast<const double*>(v), n,
                                                           partials);
    k_moments_final<<<1, 32, 0, st>>>(partials, nblocks, n, out5_dev);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Raw uniform words (tests): pool p = UniformState(seed, stream0 + p).
// ---------------------------------------------------------------------------
__global__ void k_lfg_words(uint64_t seed, uint64_t stream0, uint64_t count, uint64_t* out) {
    __shared__ uint64_t tab[608];
    __shared__ uint64_t wbuf[256];
    __shared__ Ctl ctl;
    lfg_seed(tab, &ctl, wbuf, seed, stream0 + blockIdx.x, 256);
    uint64_t* o = out + (uint64_t)blockIdx.x * count;
    lfg_bulk(tab, &ctl, wbuf, count, 256, [&](uint64_t base, uint32_t cnt) {
        if (threadIdx.x < cnt) o[base + threadIdx.x] = wbuf[threadIdx.x];
    });
}

cudaError_t launch_lfg_words(uint64_t seed, uint64_t stream0, uint32_t pools,
                             uint64_t count, uint64_t* out, cudaStream_t st) {
    k_lfg_words<<<pools, 256, 0, st>>>(seed, stream0, count, out);
    return cudaGetLastError();
}

}  // namespace wg
