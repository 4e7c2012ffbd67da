// The reference's free functions for value-type pools and host uniform
// states (proj/include/wrng/{wallace,uniform,reference,stats}.hpp), behind
// the C ABI so include/wrng_gpu/wallace.hpp can offer every name a reference
// caller uses.  The regeneration pass itself runs on the GPU (k_regenerate);
// the rest is scalar host work on the caller's UniformState / host arrays,
// compiled here with -ffp-contract=off so no multiply-add is fused no matter
// how the caller builds (rotation_from_uniform's
// lo + (hi - lo) * u and moments' s4 += v2 * v2 would contract under FMA).
//
// None of this is on the generator's hot path (WallaceState fills run the
// device engines); it is the drop-in for callers that drive passes on their
// own pools, as the reference's tests and acceptance suite do.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "internal.h"

namespace {

constexpr uint32_t kMaxIntBound = 1u << 20;  // uniform.hpp:19

// UniformState::next_word / next_uniform / next_int_below (uniform.cpp:34-51)
uint64_t u_word(wrng_gpu_uniform* us) {
    const uint64_t w = us->lag_table[us->cursor_r] + us->lag_table[us->cursor_s];
    us->lag_table[us->cursor_r] = w;
    if (++us->cursor_r == wg::kTable) us->cursor_r = 0;
    if (++us->cursor_s == wg::kTable) us->cursor_s = 0;
    return w;
}
double u_uniform(wrng_gpu_uniform* us) {
    ++us->draws;
    return (double)(u_word(us) >> 11) * 0x1.0p-53;
}
uint32_t u_int_below(wrng_gpu_uniform* us, uint32_t m) {
    return (uint32_t)(u_uniform(us) * m);
}

void box_muller(double u1, double u2, double* x, double* y) {  // reference.cpp:9-15
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.141592653589793 * u2;
    *x = radius * std::cos(angle);
    *y = radius * std::sin(angle);
}

// One regeneration pass (wallace.cpp:113-137; n = 4: docs/n4_spec.md §3)
// on natural-order fp64 arrays, one thread per output index j.  The source
// index (stride * j + offset) mod N is the segment plan's (pinned equal by
// test_wallace_core.cpp:203-217), computed with a mask because N = 2^p.
// Built with -fmad=false: every product is rounded before its sum, as the
// reference's default (FMA-free) build does.
__global__ void k_regenerate(const double* __restrict__ src, double* __restrict__ dst,
                             uint32_t na, uint32_t N, wrng_gpu_params p) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const uint64_t mask = N - 1;
    if (na == 2) {
        const double kc = p.c * p.scale, ks = p.s * p.scale;
        const double xs = src[((uint64_t)p.stride[0] * j + p.offset[0]) & mask];
        const double ys = src[N + (((uint64_t)p.stride[1] * j + p.offset[1]) & mask)];
        dst[j] = kc * xs + ks * ys;
        dst[N + j] = kc * ys - ks * xs;
        return;
    }
    double x[4];
#pragma unroll
    for (int m = 0; m < 4; ++m)
        x[m] = src[(uint64_t)m * N + (((uint64_t)p.stride[m] * j + p.offset[m]) & mask)];
    double y[4];
    if (p.variant == 0) {
        const double k = 0.5 * p.scale;
        const double ps = x[0] + x[1], qs = x[0] - x[1], rs = x[2] + x[3], ss = x[2] - x[3];
        y[0] = k * (ps + rs);
        y[1] = k * (qs + ss);
        y[2] = k * (ps - rs);
        y[3] = k * (qs - ss);
    } else {
        const double t = 0.5 * ((x[0] + x[1]) + (x[2] + x[3]));
#pragma unroll
        for (int m = 0; m < 4; ++m) y[m] = p.scale * (t - x[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) dst[(uint64_t)m * N + j] = y[m];
}

struct DevicePick {
    int prev = -1;
    explicit DevicePick(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevicePick() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Per-thread scratch of wrng_gpu_regenerate: device arrays grown on demand
// and a stream, so repeated small passes pay no allocation.
struct RegenScratch {
    int device = -1;
    double* d = nullptr;
    size_t cap = 0;  // doubles per half
    cudaStream_t s = nullptr;
    void release() {
        if (device >= 0) {
            DevicePick dp(device);
            if (d) cudaFree(d);
            if (s) cudaStreamDestroy(s);
        }
        device = -1;
        d = nullptr;
        cap = 0;
        s = nullptr;
    }
    ~RegenScratch() { release(); }
};
thread_local RegenScratch t_regen;

}  // namespace

extern "C" {

void wrng_gpu_uniform_seed(wrng_gpu_uniform* us, uint64_t seed, uint64_t stream_id) {
    // UniformState::UniformState (uniform.cpp:23-32): splitmix64 counter
    // sequence from seed ^ rotl(stream_id, 32), cursors (0, 334), 6070
    // warm-up words, draws reset.
    uint64_t s = seed ^ ((stream_id << 32) | (stream_id >> 32));
    for (uint32_t i = 0; i < wg::kTable; ++i) {
        s += 0x9E3779B97F4A7C15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        us->lag_table[i] = z ^ (z >> 31);
    }
    us->cursor_r = 0;
    us->cursor_s = wg::kGap;
    us->seed = seed;
    us->stream_id = stream_id;
    for (uint32_t i = 0; i < wg::kWarmup; ++i) u_word(us);
    us->draws = 0;
}

double wrng_gpu_sumsq_continue(double q, const double* v, uint64_t n) {
    // Pool::direct_sumsq's loop (wallace.cpp:13-18), continued from q
    for (uint64_t i = 0; i < n; ++i) q += v[i] * v[i];
    return q;
}

double wrng_gpu_chi2_target(double r, uint32_t nu) {  // wallace.cpp:27-31
    const double t = r + std::sqrt(2.0 * nu - 1.0);
    return 0.5 * t * t;
}

void wrng_gpu_rotation_from_t(double t, uint32_t region, double* c, double* s) {
    // wallace.cpp:33-42: C = (1 - t^2)/(1 + t^2), S = 2t/(1 + t^2); region
    // 0 -> (C, S), 1 -> (C, -S), else (-C, S)
    const double t2 = t * t;
    const double cc = (1.0 - t2) / (1.0 + t2);
    const double ss = 2.0 * t / (1.0 + t2);
    switch (region) {
        case 0: *c = cc; *s = ss; break;
        case 1: *c = cc; *s = -ss; break;
        default: *c = -cc; *s = ss; break;
    }
}

void wrng_gpu_rotation_from_uniform(wrng_gpu_uniform* us, double* c, double* s) {
    // wallace.cpp:44-49: t = tan(pi/12) + (tan(pi/6) - tan(pi/12)) * u, then
    // the region from next_int_below(3)
    const double lo = 0.26794919243112270, hi = 0.57735026918962576;
    const double t = lo + (hi - lo) * u_uniform(us);
    wrng_gpu_rotation_from_t(t, u_int_below(us, 3), c, s);
}

wrng_gpu_status wrng_gpu_select_pass_params(wrng_gpu_uniform* us, uint32_t n_arrays, uint32_t N,
                                            uint32_t scale_mode, double tracked_sumsq,
                                            double withheld, wrng_gpu_params* out) {
    // wallace.cpp:51-70 (n = 2) and docs/n4_spec.md §2 (n = 4): every draw
    // happens before the tracked > 0 check, which then raises ECORRUPT.
    if (!us || !out || (n_arrays != 2 && n_arrays != 4) || N < 1 || N > kMaxIntBound)
        return WRNG_GPU_EINVAL;
    wrng_gpu_params p{};
    if (n_arrays == 2) {
        p.stride[0] = u_int_below(us, 2) == 0 ? 3 : 5;
        p.stride[1] = u_int_below(us, 2) == 0 ? 7 : 11;
        p.offset[0] = u_int_below(us, N);
        p.offset[1] = u_int_below(us, N);
        wrng_gpu_rotation_from_uniform(us, &p.c, &p.s);
    } else {
        static const uint32_t kSet[4][2] = {{3, 5}, {7, 11}, {13, 17}, {19, 23}};
        for (int m = 0; m < 4; ++m) p.stride[m] = kSet[m][u_int_below(us, 2)];
        for (int m = 0; m < 4; ++m) p.offset[m] = u_int_below(us, N);
        p.variant = u_int_below(us, 2);
    }
    if (!(tracked_sumsq > 0.0)) {
        *out = p;
        return WRNG_GPU_ECORRUPT;
    }
    if (scale_mode == WRNG_GPU_CHISQ) {
        p.target_sumsq = wrng_gpu_chi2_target(withheld, n_arrays * N);
        p.scale = std::sqrt(p.target_sumsq / tracked_sumsq);
    } else {
        p.scale = 1.0;
        p.target_sumsq = tracked_sumsq;
    }
    *out = p;
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_regenerate(const double* src, double* dst, uint32_t n_arrays, uint32_t N,
                                    const wrng_gpu_params* p, double* withheld_out,
                                    int32_t device) {
    // regenerate (wallace.cpp:113-137): plan_segments' argument contract
    // (strides coprime to N, offsets in [0, N); wallace.cpp:75-80) is kept
    // as EINVAL, then the pass runs on the GPU.
    if (!src || !dst || !p || (n_arrays != 2 && n_arrays != 4) || N == 0 || (N & (N - 1)))
        return WRNG_GPU_EINVAL;
    for (uint32_t m = 0; m < n_arrays; ++m) {
        if (p->stride[m] == 0 || std::gcd<uint64_t>(p->stride[m], N) != 1) return WRNG_GPU_EINVAL;
        if (p->offset[m] >= N) return WRNG_GPU_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return WRNG_GPU_ENODEV;
    if (device < 0 || device >= ndev) return WRNG_GPU_ENODEV;
    DevicePick dp(device);
    RegenScratch& r = t_regen;
    const size_t nv = (size_t)n_arrays * N;
    if (r.device != device) {
        r.release();
        r.device = device;
        if (cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking) != cudaSuccess)
            return WRNG_GPU_ECUDA;
    }
    if (r.cap < nv) {
        if (r.d) cudaFree(r.d);
        r.d = nullptr;
        r.cap = 0;
        if (cudaMalloc(&r.d, 2 * nv * sizeof(double)) != cudaSuccess) return WRNG_GPU_ENOMEM;
        r.cap = nv;
    }
    double* dsrc = r.d;
    double* ddst = r.d + nv;
    cudaError_t e = cudaMemcpyAsync(dsrc, src, nv * sizeof(double), cudaMemcpyHostToDevice, r.s);
    if (e == cudaSuccess) {
        k_regenerate<<<(N + 255) / 256, 256, 0, r.s>>>(dsrc, ddst, n_arrays, N, *p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dst, ddst, nv * sizeof(double), cudaMemcpyDeviceToHost, r.s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(r.s);
    if (e != cudaSuccess) return WRNG_GPU_ECUDA;
    if (withheld_out) *withheld_out = dst[nv - 1];  // wallace.cpp:136
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_plan_segments(const wrng_gpu_params* p, uint32_t N,
                                       wrng_gpu_segment* out, uint32_t cap, uint32_t* count) {
    // plan_segments (wallace.cpp:72-111): the loop j in [0, N) splits where
    // either strided index alpha*j + gamma or beta*j + delta reaches a
    // multiple of N; on each piece the index is affine, j*stride + (off - wN).
    if (!p || !count) return WRNG_GPU_EINVAL;
    const uint64_t a = p->stride[0], b = p->stride[1];
    if (N == 0 || a == 0 || b == 0 || std::gcd<uint64_t>(a, N) != 1 ||
        std::gcd<uint64_t>(b, N) != 1)
        return WRNG_GPU_EINVAL;
    if (p->offset[0] >= N || p->offset[1] >= N) return WRNG_GPU_EINVAL;
    std::vector<uint32_t> cuts;
    auto add_cuts = [&](uint64_t stride, uint64_t off) {
        // the first j of each wrap k: smallest j with stride*j + off >= k*N
        for (uint64_t k = 1;; ++k) {
            const uint64_t need = k * (uint64_t)N - off;
            const uint64_t j = (need + stride - 1) / stride;
            if (j >= N) break;
            cuts.push_back((uint32_t)j);
        }
    };
    add_cuts(a, p->offset[0]);
    add_cuts(b, p->offset[1]);
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    cuts.push_back(N);
    *count = (uint32_t)cuts.size();
    if (!out) return WRNG_GPU_OK;
    if (cap < cuts.size()) return WRNG_GPU_EINVAL;
    uint32_t lo = 0;
    for (size_t i = 0; i < cuts.size(); ++i) {
        const int64_t wx = ((int64_t)a * lo + p->offset[0]) / N;
        const int64_t wy = ((int64_t)b * lo + p->offset[1]) / N;
        out[i].low = lo;
        out[i].high = cuts[i] - 1;
        out[i].jx = (int64_t)p->offset[0] - wx * (int64_t)N;
        out[i].jy = (int64_t)p->offset[1] - wy * (int64_t)N;
        lo = cuts[i];
    }
    return WRNG_GPU_OK;
}

// ---- reference normals (reference.cpp:9-63) -----------------------------
wrng_gpu_status wrng_gpu_box_muller_pair(double u1, double u2, double* x, double* y) {
    if (!(u1 > 0.0 && u1 < 1.0)) return WRNG_GPU_EINVAL;  // reference.cpp:10-11
    box_muller(u1, u2, x, y);
    return WRNG_GPU_OK;
}

void wrng_gpu_box_muller_next(wrng_gpu_uniform* us, double* x, double* y) {
    double u1 = u_uniform(us);  // reference.cpp:17-22
    if (u1 == 0.0) u1 = 0x1.0p-53;
    const double u2 = u_uniform(us);
    box_muller(u1, u2, x, y);
}

void wrng_gpu_polar_transform(double v1, double v2, double* x, double* y) {
    const double s = v1 * v1 + v2 * v2;  // reference.cpp:24-29
    const double f = std::sqrt(-2.0 * std::log(s) / s);
    *x = v1 * f;
    *y = v2 * f;
}

void wrng_gpu_polar_next(wrng_gpu_uniform* us, double* x, double* y) {
    for (;;) {  // reference.cpp:31-37
        const double v1 = 2.0 * u_uniform(us) - 1.0;
        const double v2 = 2.0 * u_uniform(us) - 1.0;
        const double s = v1 * v1 + v2 * v2;
        if (s > 0.0 && s < 1.0) {
            wrng_gpu_polar_transform(v1, v2, x, y);
            return;
        }
    }
}

void wrng_gpu_normal_fill(int32_t method, wrng_gpu_uniform* us, double* out, uint64_t n,
                          double mu, double sigma) {
    // fill_from_pairs (reference.cpp:41-51): pairs in order, an odd count
    // takes the .x of one more pair
    auto next = [&](double* x, double* y) {
        if (method == 0)
            wrng_gpu_box_muller_next(us, x, y);
        else
            wrng_gpu_polar_next(us, x, y);
    };
    uint64_t i = 0;
    double x, y;
    while (i + 1 < n) {
        next(&x, &y);
        out[i++] = mu + sigma * x;
        out[i++] = mu + sigma * y;
    }
    if (i < n) {
        next(&x, &y);
        out[i] = mu + sigma * x;
    }
}

// ---- statistics on host arrays (stats.cpp:10-146) ------------------------
void wrng_gpu_to_uv(double x, double y, double* u, double* v, int32_t* skip) {
    if (x == 0.0 && y == 0.0) {  // stats.cpp:10-16
        *u = 0.0;
        *v = 0.0;
        *skip = 1;
        return;
    }
    *u = std::exp(-0.5 * (x * x + y * y));
    *v = y == 0.0 ? std::copysign(3.141592653589793 / 2, x) : std::atan(x / y);
    *skip = 0;
}

wrng_gpu_status wrng_gpu_chi2_bins(const double* values, uint64_t n, uint32_t k, double lo,
                                   double hi, double* statistic) {
    // stats.cpp:18-38: k equal bins on [lo, hi], hi in the top bin
    if (k < 2 || !(lo < hi) || (!values && n)) return WRNG_GPU_EINVAL;
    std::vector<uint64_t> counts(k, 0);
    const double width = hi - lo;
    for (uint64_t i = 0; i < n; ++i) {
        const double v = values[i];
        if (!(v >= lo && v <= hi)) return WRNG_GPU_EINVAL;
        uint32_t bin = (uint32_t)((v - lo) / width * k);
        if (bin >= k) bin = k - 1;
        ++counts[bin];
    }
    const double expected = (double)n / k;
    double st = 0.0;
    for (uint64_t c : counts) {
        const double d = (double)c - expected;
        st += d * d / expected;
    }
    *statistic = st;
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_moments_host(const double* values, uint64_t n, double* out7) {
    // stats.cpp:89-108 (sequential s1, s2, s4) + m3 in the same pass:
    // out7 = {m1, m2, m3, m4, z1, z2, z4}
    if (!values || n == 0 || !out7) return WRNG_GPU_EINVAL;
    const double dn = (double)n;
    double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double v = values[i], v2 = v * v;
        s1 += v;
        s2 += v2;
        s3 += v2 * v;
        s4 += v2 * v2;
    }
    out7[0] = s1 / dn;
    out7[1] = s2 / dn;
    out7[2] = s3 / dn;
    out7[3] = s4 / dn;
    out7[4] = out7[0] * std::sqrt(dn / 1.0);
    out7[5] = (out7[1] - 1.0) * std::sqrt(dn / 2.0);
    out7[6] = (out7[3] - 3.0) * std::sqrt(dn / 96.0);
    return WRNG_GPU_OK;
}

wrng_gpu_status wrng_gpu_autocorr_host(const double* values, uint64_t n, uint64_t lag,
                                       double* r) {
    // stats.cpp:110-127: mean over all n, sums over t in [0, n - lag)
    if (!values || !r || n < lag + 2) return WRNG_GPU_EINVAL;
    double mean = 0.0;
    for (uint64_t i = 0; i < n; ++i) mean += values[i];
    mean /= (double)n;
    double num = 0.0, den = 0.0;
    for (uint64_t t = 0; t + lag < n; ++t) {
        const double a = values[t] - mean;
        num += a * (values[t + lag] - mean);
        den += a * a;
    }
    if (den == 0.0) return WRNG_GPU_EINVAL;
    *r = num / den;
    return WRNG_GPU_OK;
}

void wrng_gpu_target_stats(const double* s, uint64_t n, double* mean_var) {
    // sumsq_distribution_check's reduction (stats.cpp:136-145): sum and sum of
    // squares in order, population variance clamped at 0
    double sum = 0.0, sumsq = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        sum += s[i];
        sumsq += s[i] * s[i];
    }
    const double dn = (double)n;
    const double mean = sum / dn;
    const double var = sumsq / dn - mean * mean;
    mean_var[0] = mean;
    mean_var[1] = var < 0.0 ? 0.0 : var;
}

}  // extern "C"
