// Device helpers shared by the engines: bit-exact scalar restatements of the
// reference, the CTA-cooperative lagged-Fibonacci generator and the device
// Box-Muller initialisation.
//
// Reference (paths relative to /root/reference/proj):
//   uniform generator      src/uniform.cpp:13-51
//   Box-Muller             src/reference.cpp:9-22, 41-58
//   pass parameters        src/wallace.cpp:27-70
//   init_pool              src/wallace.cpp:158-167
//
// Compiled with -fmad=false: every floating-point expression is evaluated
// exactly as written (one rounding per operation), matching the reference's
// FMA-free Release build.  sqrt and / are IEEE-rounded on
// the device; log/cos/sin appear only in the device Box-Muller path.
#pragma once

#include "internal.h"

namespace wg {

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) {
    return a < b ? a : b;
}
__device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

__device__ __forceinline__ double u53(uint64_t w) {
    // next_uniform (uniform.cpp:42-45): top 53 bits * 2^-53
    return (double)(w >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ uint32_t nib(uint64_t w, uint32_t m) {
    // next_int_below (uniform.cpp:47-51)
    return (uint32_t)(u53(w) * (double)m);
}
// next_int_below(2^k): (w >> 11) * 2^-53 * 2^k is exact, so its floor is the
// integer w >> (64 - k) — identical to nib(w, 2^k) for 1 <= k <= 20.
__device__ __forceinline__ uint32_t nib_pow2(uint64_t w, uint32_t log2m) {
    return (uint32_t)(w >> (64 - log2m));
}
__device__ __forceinline__ double chi2_target(double r, uint32_t nu) {
    // wallace.cpp:27-31
    double t = r + sqrt(2.0 * (double)nu - 1.0);
    return 0.5 * t * t;
}
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t x) {
    // uniform.cpp:13-19 in counter form: output i = mix(s0 + (i + 1) * golden)
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ bool crossed(uint64_t before, uint64_t after, uint64_t period) {
    // wallace.cpp:182-184
    return period > 0 && after / period > before / period;
}

// Uniform words consumed by one pass: n = 2: alpha, beta, gamma, delta, u,
// region (wallace.cpp:54-58, 44-49); n = 4: 4 strides, 4 offsets, variant
// (docs/n4_spec.md §2).
template <int NA>
struct PassWords {
    static constexpr int K = NA == 2 ? 6 : 9;
};

// The uniform-generator part of a pass's parameters.
struct LfgParams {
    uint32_t stride[4];
    uint32_t offset[4];
    uint32_t variant;
    uint32_t pad_;
    double c, s;  // n = 2 rotation
};

template <int NA>
__device__ __forceinline__ void lfg_params(const uint64_t* w, uint32_t N, LfgParams& p) {
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
        const double kTanSpan = 0x1.3cd3a2c8198e2p-2;  // kTanHi - kTanLo, rounded
        double t = kTanLo + kTanSpan * u53(w[4]);
        uint32_t region = nib(w[5], 3);
        double t2 = t * t;
        double c = (1.0 - t2) / (1.0 + t2);
        double s = 2.0 * t / (1.0 + t2);
        if (region == 0) {
            p.c = c;
            p.s = s;
        } else if (region == 1) {
            p.c = c;
            p.s = -s;
        } else {
            p.c = -c;
            p.s = s;
        }
    } else {
        // strides from {3,5}, {7,11}, {13,17}, {19,23} (docs/n4_spec.md §2)
        const uint32_t lo[4] = {3, 7, 13, 19}, hi[4] = {5, 11, 17, 23};
#pragma unroll
        for (int m = 0; m < 4; ++m) p.stride[m] = nib(w[m], 2) == 0 ? lo[m] : hi[m];
#pragma unroll
        for (int m = 0; m < 4; ++m) p.offset[m] = nib(w[4 + m], N);
        p.variant = nib(w[8], 2);
        p.c = 0.0;
        p.s = 0.0;
    }
    p.pad_ = 0;
}

// Scale part of select_pass_params (wallace.cpp:59-69): 0 or ECORRUPT.
__device__ __forceinline__ int pass_scale(double tracked, double withheld, uint32_t nu,
                                          uint32_t mode, double& scale, double& target) {
    if (!(tracked > 0.0)) return WRNG_GPU_ECORRUPT;
    if (mode == WRNG_GPU_CHISQ) {
        target = chi2_target(withheld, nu);
        scale = sqrt(target / tracked);
    } else {
        scale = 1.0;
        target = tracked;
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

// Output element mu + sigma * v (wallace.cpp:209-212) in double, narrowed
// for f32 outputs; `unit` (mu = 0, sigma = 1) keeps the reference's
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

// Shared-memory control block of one pool.
struct Ctl {
    LfgParams cur;   // uniform-generator part of the next pass's parameters
    LfgParams cur2;  // second slot: the smem engine double-buffers (cur, cur2)
    double c0d, c1d; // coefficients: n=2 (c*scale, s*scale); n=4 (scale/2, scale)
    float c0f, c1f;
    double target;
    double scale;
    double tracked;  // pool scalars of the live buffer
    double withheld;
    double prev_tracked, prev_withheld;
    uint64_t draws;
    uint32_t r;
    uint32_t active;
    int32_t error;
    uint32_t have_prev;
    uint32_t rot;  // smem engine: pool arrays stored rotated by rot (bulk emission)
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

// UniformState(seed, stream) (uniform.cpp:23-32): table[i] = splitmix64
// output i of seed ^ rotl(stream, 32), then 6070 discarded words, draws = 0.
__device__ inline void lfg_seed(uint64_t* tab, Ctl* ctl, uint64_t* wbuf, uint64_t seed,
                                uint64_t stream, uint32_t step) {
    const uint64_t s0 = seed ^ ((stream << 32) | (stream >> 32));
    for (uint32_t i = threadIdx.x; i < kTable; i += blockDim.x)
        tab[i] = splitmix64_at(s0 + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull);
    if (threadIdx.x == 0) {
        ctl->r = 0;
        ctl->draws = 0;
    }
    __syncthreads();
    lfg_bulk(tab, ctl, wbuf, kWarmup, step, [](uint64_t, uint32_t) {});
    if (threadIdx.x == 0) ctl->draws = 0;
    __syncthreads();
}

// Warp 0 (all 32 lanes): draw one pass's K words and derive its uniform-
// generator parameters into ctl->cur (draw order of wallace.cpp:54-58).
// Lane k owns word k and writes the field that word decides, so the serial
// part is one table step.
template <int NA>
__device__ __forceinline__ void draw_pass_params_warp(uint64_t* tab, Ctl* ctl, uint64_t*,
                                                      uint32_t N, int slot = 0) {
    constexpr int K = PassWords<NA>::K;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t r = ctl->r;
    const uint64_t w = lane < (uint32_t)K ? lfg_word_at(tab, r, lane) : 0ull;
    const uint64_t w_next = __shfl_down_sync(0xffffffffu, w, 1);
    LfgParams& p = slot ? ctl->cur2 : ctl->cur;
    if (NA == 2) {
        const uint32_t lg = (uint32_t)__ffs(N) - 1;
        if (lane == 0) p.stride[0] = nib_pow2(w, 1) == 0 ? 3 : 5;
        if (lane == 1) p.stride[1] = nib_pow2(w, 1) == 0 ? 7 : 11;
        if (lane == 2) p.offset[0] = nib_pow2(w, lg);
        if (lane == 3) p.offset[1] = nib_pow2(w, lg);
        if (lane == 4) {
            // rotation_from_uniform: t from word 4, region from word 5
            // (wallace.cpp:44-49), rotation_from_t (wallace.cpp:33-42)
            const double kTanLo = 0x1.126145e9ecd56p-2;    // 0.26794919243112270
            const double kTanSpan = 0x1.3cd3a2c8198e2p-2;  // kTanHi - kTanLo, rounded
            const double t = kTanLo + kTanSpan * u53(w);
            const uint32_t region = nib(w_next, 3);
            const double t2 = t * t;
            const double c = (1.0 - t2) / (1.0 + t2);
            const double s = 2.0 * t / (1.0 + t2);
            p.c = region == 2 ? -c : c;
            p.s = region == 1 ? -s : s;
        }
        if (lane == 6) {
            p.stride[2] = p.stride[3] = 0;
            p.offset[2] = p.offset[3] = 0;
            p.variant = 0;
            p.pad_ = 0;
        }
    } else {
        // strides from {3,5}, {7,11}, {13,17}, {19,23} (docs/n4_spec.md §2)
        if (lane < 4) {
            const uint32_t lo = (0x130D0703u >> (8u * lane)) & 0xFFu;  // 3, 7, 13, 19
            p.stride[lane] = nib_pow2(w, 1) == 0 ? lo : lo + (lane == 0 ? 2 : 4);
        } else if (lane < 8) {
            p.offset[lane - 4] = nib_pow2(w, (uint32_t)__ffs(N) - 1);
        } else if (lane == 8) {
            p.variant = nib_pow2(w, 1);
        } else if (lane == 9) {
            p.c = 0.0;
            p.s = 0.0;
            p.pad_ = 0;
        }
    }
    if (lane == 31) {
        const uint32_t nr = r + K;
        ctl->r = nr >= kTable ? nr - kTable : nr;
        ctl->draws += K;
    }
    __syncwarp();
}

// Same draw for n = 4, executed branch-free by EVERY warp of the CTA with
// only `writer` (warp 0) storing: all warps run an identical instruction
// stream, so the draw's latency does not unbalance the pass barrier.  The
// uint32 fields stride[0..3], offset[0..3], variant of LfgParams are words
// 0..8, i.e. lane k writes word k.
template <int NA>
__device__ __forceinline__ void draw_pass_params_all(uint64_t* tab, Ctl* ctl, uint32_t N,
                                                     int slot, bool writer) {
    if constexpr (NA == 2) {
        if (writer) draw_pass_params_warp<2>(tab, ctl, nullptr, N, slot);
    } else {
        constexpr uint32_t K = PassWords<4>::K;
        const uint32_t lane = threadIdx.x & 31u;
        const uint32_t r = ctl->r;
        uint32_t i = r + lane;
        i = i >= kTable ? i - kTable : i;
        uint32_t s = i + kGap;
        s = s >= kTable ? s - kTable : s;
        const bool mine = lane < K;
        const uint64_t w = mine ? tab[i] + tab[s] : 0ull;
        if (writer && mine) tab[i] = w;
        // 3, 7, 13, 19 for lanes 0..3 without a per-lane jump table
        const uint32_t lo = (0x130D0703u >> (8u * (lane & 3u))) & 0xFFu;
        const uint32_t strd = (w >> 63) ? lo + (lane == 0 ? 2u : 4u) : lo;
        const uint32_t offs = (uint32_t)(w >> (64 - ((uint32_t)__ffs(N) - 1)));
        const uint32_t val = lane < 4 ? strd : lane < 8 ? offs : (uint32_t)(w >> 63);
        LfgParams& p = slot ? ctl->cur2 : ctl->cur;
        if (writer && mine) reinterpret_cast<uint32_t*>(&p)[lane] = val;
        if (writer && lane == 31) {
            const uint32_t nr = r + K;
            ctl->r = nr >= kTable ? nr - kTable : nr;
            ctl->draws += K;
        }
    }
}

// Sequential sum of squares in Pool::direct_sumsq order (wallace.cpp:13-18).
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

// ---------------------------------------------------------------------------
// Exact parallel reproduction of the reference's left-to-right sum of squares
// (Pool::direct_sumsq, wallace.cpp:13-18: q <- fl(q + v*v), arrays in order).
//
// While q stays in one binade [2^E, 2^(E+1)), q is a multiple of
// u = 2^(E-52) and fl(q + p) = q + u * R with R = p/u rounded to nearest,
// ties to the even value of q/u + R.  So a chunk of terms adds an INTEGER
// K = sum R to Q = q/u, exactly, as long as Q + K < 2^53.  R depends on the
// running parity of Q only at exact ties, and after a tie Q is even whatever
// came before; hence a chunk's effect is fully described by (K, parity out)
// for each of the two possible start parities.  These "segment functions"
// compose associatively.  A single thread then walks the chunks in order,
// applying each in O(1) when the exact running q is in the chunk's guessed
// binade and stays there, and adding that chunk's terms one by one
// otherwise (only near powers of two).  The result is bit-identical to the
// sequential loop for any inputs (all terms are >= 0).
// ---------------------------------------------------------------------------
struct SumSeg {
    long long s[2];    // K for start parity 0 / 1
    uint32_t par[2];   // parity after the chunk for start parity 0 / 1
    uint32_t valid;    // every term satisfied p/u < 2^53
    int32_t e;         // binade exponent the chunk was evaluated in
};

__device__ __forceinline__ double pow2d(int e) {  // 2^e for normal e
    return __longlong_as_double((long long)(e + 1023) << 52);
}
__device__ __forceinline__ int exp2_of(double q) {  // floor(log2 q), q normal > 0
    return (int)((__double_as_longlong(q) >> 52) & 0x7FF) - 1023;
}

__device__ __forceinline__ void seg_init(SumSeg& g, int e) {
    g.s[0] = g.s[1] = 0;
    g.par[0] = 0;
    g.par[1] = 1;
    g.valid = 1;
    g.e = e;
}

// Appends one term p (>= 0); sc = 2^(52 - e).
__device__ __forceinline__ void seg_push(SumSeg& g, double p, double sc) {
    const double x = p * sc;  // exact: scaling by a power of two
    if (!(x < 0x1.0p53)) {
        g.valid = 0;
        return;
    }
    const long long k = (long long)x;
    const double f = x - (double)k;  // exact
    if (f != 0.5) {
        const long long r = k + (f > 0.5 ? 1 : 0);
        g.s[0] += r;
        g.s[1] += r;
        g.par[0] ^= (uint32_t)(r & 1);
        g.par[1] ^= (uint32_t)(r & 1);
    } else {  // tie: round Q + k + 1/2 to even
        g.s[0] += k + ((g.par[0] ^ (uint32_t)k) & 1u);
        g.s[1] += k + ((g.par[1] ^ (uint32_t)k) & 1u);
        g.par[0] = g.par[1] = 0;
    }
}

// a then b (both evaluated in the same binade).
__device__ __forceinline__ SumSeg seg_compose(const SumSeg& a, const SumSeg& b) {
    SumSeg c;
    c.e = a.e;
    c.valid = a.valid & b.valid & (a.e == b.e ? 1u : 0u);
    // (selects, not b.s[a.par[h]]: a dynamically indexed member array sends the
    // whole struct to local memory)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const bool odd = a.par[h] != 0;
        c.s[h] = a.s[h] + (odd ? b.s[1] : b.s[0]);
        c.par[h] = odd ? b.par[1] : b.par[0];
    }
    return c;
}

// After all compositions: store the two increments as the bit patterns of
// doubles (exact below 2^53; anything larger can only fail to apply), so the
// serial walk below needs no int <-> double conversion.
__device__ __forceinline__ void seg_finalize(SumSeg& g) {
    g.s[0] = __double_as_longlong((double)g.s[0]);
    g.s[1] = __double_as_longlong((double)g.s[1]);
}

// Applies a finalized chunk to the exact running sum q; false when it cannot
// (q not in the chunk's binade, an invalid term, or the binade would be left).
// Q = q / u is an integer-valued double in [2^52, 2^53): its parity is the
// lowest mantissa bit and Q + K is exact while below 2^53.
__device__ __forceinline__ bool seg_apply(double& q, const SumSeg& g) {
    if (!g.valid || !(q > 0.0) || exp2_of(q) != g.e) return false;
    const double Q = q * pow2d(52 - g.e);
    const double Qn =
        Q + __longlong_as_double((__double_as_longlong(Q) & 1) ? g.s[1] : g.s[0]);
    if (!(Qn < 0x1.0p53)) return false;
    q = Qn * pow2d(g.e - 52);
    return true;
}

// Undo seg_finalize (increments are exact below 2^53; a larger one can only
// make every prefix containing it fail to apply).
__device__ __forceinline__ SumSeg seg_unfinalize(SumSeg g) {
    g.s[0] = (long long)__longlong_as_double(g.s[0]);
    g.s[1] = (long long)__longlong_as_double(g.s[1]);
    return g;
}

__device__ __forceinline__ SumSeg seg_shfl_up(const SumSeg& g, uint32_t o) {
    SumSeg r;
    r.s[0] = __shfl_up_sync(0xffffffffu, g.s[0], o);
    r.s[1] = __shfl_up_sync(0xffffffffu, g.s[1], o);
    r.par[0] = __shfl_up_sync(0xffffffffu, g.par[0], o);
    r.par[1] = __shfl_up_sync(0xffffffffu, g.par[1], o);
    r.valid = __shfl_up_sync(0xffffffffu, g.valid, o);
    r.e = __shfl_up_sync(0xffffffffu, g.e, o);
    return r;
}

// Warp-cooperative walk over long runs of segments in one binade (the HBM
// drift walk's blocks): applies the longest prefix of the (not finalized)
// segments load(0 .. n-1) to the exact running sum q, 32 at a time — lane k
// composes f_0 ... f_k by a shuffle scan and all lanes try their prefix on q
// at once; the applicable prefixes form an initial run (once a segment is
// invalid, changes binade or pushes Q past 2^53, every longer prefix fails
// too).  Returns the number applied; q (warp-uniform) moves past them.
// All 32 lanes call.  (Slower than one thread where the binade changes
// every few segments: DESIGN.md §4.)
template <typename Load>
__device__ __forceinline__ uint32_t warp_seg_walk(double& q, uint32_t n, Load&& load) {
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t done = 0;
    while (done < n) {
        const uint32_t k = done + lane;
        SumSeg g;
        if (k < n) {
            g = load(k);
        } else {
            seg_init(g, 0);
            g.valid = 0;
        }
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const SumSeg y = seg_shfl_up(g, o);
            if (lane >= o) g = seg_compose(y, g);
        }
        seg_finalize(g);
        double qk = q;
        const bool ok = seg_apply(qk, g);
        const uint32_t m = __ballot_sync(0xffffffffu, ok);
        const uint32_t cnt = ~m == 0u ? 32u : (uint32_t)__ffs(~m) - 1u;  // leading run
        if (cnt) q = __shfl_sync(0xffffffffu, qk, cnt - 1);
        done += cnt;
        if (cnt < 32) break;
    }
    return done < n ? done : n;
}

template <typename T>
__device__ __forceinline__ double sq_term(T v) {
    const double d = (double)v;
    return d * d;
}

// CTA-cooperative exact direct_sumsq of v[0, n) (shared or global memory).
// Chunks: up to min(blockDim, max_chunks) (one per thread), guessed binades
// from a block scan of approximate chunk sums; blocks of kSumBlk chunks are
// pre-composed in parallel, so the serial walk is O(chunks / kSumBlk) plus a
// chunk- or term-level fallback only where a guess fails (near powers of
// two).  `scratch` (shared) needs sum_scratch_bytes(max_chunks) bytes.
// Must be called by all threads; returns the sum to all.
constexpr uint32_t kSumBlk = 16;
__host__ __device__ constexpr uint32_t sum_scratch_bytes(uint32_t max_chunks) {
    return (uint32_t)sizeof(SumSeg) * (max_chunks + (max_chunks + kSumBlk - 1) / kSumBlk);
}
constexpr uint32_t kSumSmallChunks = 60;  // 60 + 4 segments: the 2 KiB word buffer
static_assert(sum_scratch_bytes(kSumSmallChunks) <= 2048, "word buffer");

// A pool whose arrays (length mask + 1) are each stored rotated by `rot`:
// value i lives at (i & ~mask) | ((i + rot) & mask).
template <typename T>
struct RotView {
    const T* p;
    uint32_t mask, rot;
    __device__ __forceinline__ T operator[](uint32_t i) const {
        return p[(i & ~mask) | ((i + rot) & mask)];
    }
};

template <typename T, typename V = const T*>
__device__ double exact_sumsq_cta(V v, uint32_t n, void* scratch,
                                  uint32_t max_chunks = kSumSmallChunks) {
    uint32_t nch = blockDim.x < max_chunks ? blockDim.x : max_chunks;
    if (nch > n) nch = n > 0 ? n : 1;
    // balanced chunks of c = ceil(n / nch) values, rounded up to odd (lane
    // stride c: conflict-free shared reads); the last chunk takes the rest
    uint32_t c = (n + nch - 1) / nch;
    if (c > 1 && (c & 1) == 0) c += 1;
    nch = (n + c - 1) / c;
    const uint32_t nblk = (nch + kSumBlk - 1) / kSumBlk;
    SumSeg* seg = static_cast<SumSeg*>(scratch);
    SumSeg* blk = seg + nch;
    double* wsum = static_cast<double*>(scratch);  // warp totals, before seg[] is written
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    const uint32_t lo = t * c, hi = t + 1 == nch ? n : (t + 1) * c;  // used for t < nch
    // pass 1: approximate chunk sums -> exclusive block scan (binade guesses)
    double a = 0.0;
    if (t < nch)
        for (uint32_t i = lo; i < hi; ++i) a += sq_term(v[i]);
    double x = a;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = (blockDim.x + 31) / 32;
        double w = lane < nw ? wsum[lane] : 0.0;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    const double pre = x - a + (warp > 0 ? wsum[warp - 1] : 0.0);
    const int e = (t < nch && pre > 0.0) ? exp2_of(pre) : -2000;
    __syncthreads();  // wsum aliases seg[]
    // pass 2: segment function of the chunk in its guessed binade
    SumSeg g;
    seg_init(g, e);
    if (t < nch && e > -1000) {
        const double sc = pow2d(52 - e);
        for (uint32_t i = lo; i < hi; ++i) seg_push(g, sq_term(v[i]), sc);
    } else {
        g.valid = 0;
    }
    if (t < nch) seg[t] = g;
    __syncthreads();
    // blocks of kSumBlk chunks composed in parallel (valid only within one binade)
    if (t < nblk) {
        SumSeg b = seg[t * kSumBlk];
        const uint32_t kend = (t + 1) * kSumBlk < nch ? (t + 1) * kSumBlk : nch;
        for (uint32_t k = t * kSumBlk + 1; k < kend; ++k) b = seg_compose(b, seg[k]);
        seg_finalize(b);
        blk[t] = b;
    }
    __syncthreads();
    // walk (one thread): per block, else per chunk, else term by term
    if (t == 0) {
        double q = 0.0;
        for (uint32_t bi = 0; bi < nblk; ++bi) {
            if (seg_apply(q, blk[bi])) continue;
            const uint32_t kend = (bi + 1) * kSumBlk < nch ? (bi + 1) * kSumBlk : nch;
            for (uint32_t k = bi * kSumBlk; k < kend; ++k) {
                SumSeg gk = seg[k];
                seg_finalize(gk);
                if (seg_apply(q, gk)) continue;
                const uint32_t l2 = k * c, h2 = k + 1 == nch ? n : (k + 1) * c;
                for (uint32_t i = l2; i < h2; ++i) q = q + sq_term(v[i]);
            }
        }
        *reinterpret_cast<double*>(blk) = q;
    }
    __syncthreads();
    const double q = *reinterpret_cast<const double*>(blk);
    __syncthreads();
    return q;
}

// init_pool (wallace.cpp:158-167) into `pool` (shared or global): Box-Muller
// pairs fill arrays 0..n-1 in order, then withheld = .x of one more pair;
// tracked = sequential sum.  Consumes n*N + 2 uniforms.
template <typename T>
__device__ void init_pool_dev(T* pool, uint64_t nvals, uint64_t* tab, Ctl* ctl,
                              uint64_t* wbuf, uint32_t step, void* sum_scratch = nullptr,
                              uint32_t sum_chunks = kSumSmallChunks) {
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
    // tracked = direct_sumsq (exact left-to-right value, computed in parallel)
    const double q = exact_sumsq_cta<T>(pool, (uint32_t)nvals, sum_scratch ? sum_scratch : wbuf,
                                        sum_scratch ? sum_chunks : kSumSmallChunks);
    if (threadIdx.x == 0) {
        ctl->draws += nvals + 2;
        ctl->tracked = q;
    }
    __syncthreads();
}

// Passes-until-boundary bookkeeping without divisions in the refill loop:
// crossed(before, before + f, P) (wallace.cpp:182-184) <=> (before mod P) + f >= P.
struct PeriodCounter {
    uint64_t period, rem;
    __device__ __forceinline__ void init(uint64_t P, uint64_t pc) {
        period = P;
        rem = P ? pc % P : 0;
    }
    __device__ __forceinline__ bool will_cross(uint64_t f) const {
        return period > 0 && rem + f >= period;
    }
    __device__ __forceinline__ void advance(uint64_t f) {
        if (!period) return;
        rem += f;
        while (rem >= period) rem -= period;
    }
};

}  // namespace wg
