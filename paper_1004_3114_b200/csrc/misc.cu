// Validation reductions and raw uniform-generator words (test support).
#include "common.cuh"

namespace wg {

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
// Uniformity and serial-correlation checks on device:
// stats.cpp:10-38 (to_uv, chi2_bins), 110-127 (autocorr_at_lag), with the
// CLI's pairing (tools/main.cpp:160-193).  The data is a "window" of P
// streams: stream q occupies v[q * pitch, q * pitch + len); a plain array
// is P = 1.  Pairs are (2i, 2i+1) within each stream window (len even, or
// the last value unpaired).
// ---------------------------------------------------------------------------
constexpr double kHalfPi = 1.5707963267948966;  // tools/main.cpp:162

template <typename T>
__global__ void k_uv_counts(const T* v, uint32_t P, uint64_t pitch, uint64_t len, uint32_t k,
                            unsigned long long* cu, unsigned long long* cv,
                            unsigned long long* skipped) {
    extern __shared__ uint32_t hist[];  // [2k]: u bins, then v bins
    for (uint32_t i = threadIdx.x; i < 2 * k; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t per = len / 2, total = per * P;
    const double kd = (double)k, vlo = -kHalfPi, vwidth = kHalfPi - (-kHalfPi);
    uint32_t sk = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = i / per, j = i - q * per;
        const T* w = v + q * pitch + 2 * j;
        const double x = (double)w[0], y = (double)w[1];
        if (x == 0.0 && y == 0.0) {  // stats.cpp:11
            ++sk;
            continue;
        }
        const double u = exp(-0.5 * (x * x + y * y));                // stats.cpp:12
        const double a = y == 0.0 ? copysign(kHalfPi, x) : atan(x / y);  // stats.cpp:13-14
        uint32_t bu = (uint32_t)((u - 0.0) / 1.0 * kd);               // stats.cpp:27-28
        uint32_t bv = (uint32_t)((a - vlo) / vwidth * kd);
        bu = bu >= k ? k - 1 : bu;
        bv = bv >= k ? k - 1 : bv;
        atomicAdd(&hist[bu], 1u);
        atomicAdd(&hist[k + bv], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 2 * k; i += blockDim.x) {
        const uint32_t c = hist[i];
        if (c) atomicAdd(i < k ? &cu[i] : &cv[i - k], (unsigned long long)c);
    }
    for (int o = 16; o > 0; o >>= 1) sk += __shfl_xor_sync(0xffffffffu, sk, o);
    if ((threadIdx.x & 31) == 0 && sk) atomicAdd(skipped, (unsigned long long)sk);
}

cudaError_t launch_uv_counts(const void* v, int is_f32, uint32_t P, uint64_t pitch,
                             uint64_t len, uint32_t k, unsigned long long* cu,
                             unsigned long long* cv, unsigned long long* skipped,
                             cudaStream_t st) {
    const uint32_t smem = 2 * k * 4;
    const uint32_t nb = 148 * 4;
    if (is_f32) {
        cudaFuncSetAttribute(k_uv_counts<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem);
        k_uv_counts<float><<<nb, 256, smem, st>>>(static_cast<const float*>(v), P, pitch, len,
                                                  k, cu, cv, skipped);
    } else {
        cudaFuncSetAttribute(k_uv_counts<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem);
        k_uv_counts<double><<<nb, 256, smem, st>>>(static_cast<const double*>(v), P, pitch, len,
                                                   k, cu, cv, skipped);
    }
    return cudaGetLastError();
}

// Raw lag sums of P stream windows, each continuing `lag` tail values of
// the same stream from the previous window (tail[q * lag ..], `have` of
// them valid).  Per block: Sxy = sum z_t z_{t+lag}, Sa = sum z_t,
// Sb = sum z_{t+lag}, Saa = sum z_t^2 over the pairs (t, t + lag) whose
// second element lies in this window; pairs counted in `pairs`.
template <typename T>
__device__ __forceinline__ double win_at(const T* v, const T* tail, uint64_t q, uint64_t pitch,
                                         uint64_t lag, uint64_t have, uint64_t i) {
    // virtual stream q: [tail (have values) | window (len values)]
    return i < have ? (double)tail[q * lag + (lag - have) + i]
                    : (double)v[q * pitch + (i - have)];
}

template <typename T>
__global__ void k_ac_sums(const T* v, const T* tail, uint32_t P, uint64_t pitch, uint64_t len,
                          uint64_t lag, uint64_t have, double* part) {
    __shared__ double red[4][256];
    double s[4] = {0, 0, 0, 0};
    const uint64_t vlen = have + len;                     // virtual length per stream
    const uint64_t per = vlen > lag ? vlen - lag : 0;     // pairs per stream
    const uint64_t total = per * P;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
        const uint64_t q = i / per, t = i - q * per;
        const double a = win_at(v, tail, q, pitch, lag, have, t);
        const double b = win_at(v, tail, q, pitch, lag, have, t + lag);
        s[0] += a * b;
        s[1] += a;
        s[2] += b;
        s[3] += a * a;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) red[c][threadIdx.x] = s[c];
    __syncthreads();
    for (uint32_t o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
#pragma unroll
            for (int c = 0; c < 4; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

// acc[0..3] += block partials (in block order, one thread: deterministic)
__global__ void k_sum4_into(const double* part, uint32_t nb, double* acc) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s[4] = {0, 0, 0, 0};
    for (uint32_t b = 0; b < nb; ++b)
        for (int c = 0; c < 4; ++c) s[c] += part[b * 4 + c];
    for (int c = 0; c < 4; ++c) acc[c] += s[c];
}

// Next tail = the last `lag` values of [old tail (have) | window (len)] of
// each stream (fewer when the stream is still shorter than lag: right-
// aligned, like the old tail).  Old and new tails are distinct buffers.
template <typename T>
__global__ void k_ac_tail(const T* v, const T* told, T* tnew, uint32_t P, uint64_t pitch,
                          uint64_t len, uint64_t lag, uint64_t have) {
    const uint64_t vlen = have + len;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)P * lag;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = i / lag, j = i - q * lag;
        if (vlen + j < lag) continue;            // slot not yet filled
        const uint64_t src = vlen + j - lag;     // index into the virtual stream
        tnew[q * lag + j] =
            src < have ? told[q * lag + (lag - have) + src] : v[q * pitch + (src - have)];
    }
}

cudaError_t launch_ac_sums(const void* v, const void* tail, int is_f32, uint32_t P,
                           uint64_t pitch, uint64_t len, uint64_t lag, uint64_t have,
                           double* part, uint32_t nb, double* acc, cudaStream_t st) {
    if (is_f32)
        k_ac_sums<float><<<nb, 256, 0, st>>>(static_cast<const float*>(v),
                                             static_cast<const float*>(tail), P, pitch, len, lag,
                                             have, part);
    else
        k_ac_sums<double><<<nb, 256, 0, st>>>(static_cast<const double*>(v),
                                              static_cast<const double*>(tail), P, pitch, len,
                                              lag, have, part);
    k_sum4_into<<<1, 32, 0, st>>>(part, nb, acc);
    return cudaGetLastError();
}

// Moment sums s1..s4 of P stream windows added into acc[0..3]
// (per-block partials summed in block order: deterministic).
template <typename T>
__global__ void k_moments_win(const T* v, uint32_t P, uint64_t pitch, uint64_t len,
                              double* part) {
    __shared__ double red[4][256];
    double s[4] = {0, 0, 0, 0};
    const uint64_t total = len * P;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
        const uint64_t q = i / len, j = i - q * len;
        const double x = (double)v[q * pitch + j], x2 = x * x;
        s[0] += x;
        s[1] += x2;
        s[2] += x2 * x;
        s[3] += x2 * x2;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) red[c][threadIdx.x] = s[c];
    __syncthreads();
    for (uint32_t o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
#pragma unroll
            for (int c = 0; c < 4; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

cudaError_t launch_moment_sums(const void* v, int is_f32, uint32_t P, uint64_t pitch,
                               uint64_t len, double* part, uint32_t nb, double* acc,
                               cudaStream_t st) {
    if (is_f32)
        k_moments_win<float><<<nb, 256, 0, st>>>(static_cast<const float*>(v), P, pitch, len,
                                                 part);
    else
        k_moments_win<double><<<nb, 256, 0, st>>>(static_cast<const double*>(v), P, pitch, len,
                                                  part);
    k_sum4_into<<<1, 32, 0, st>>>(part, nb, acc);
    return cudaGetLastError();
}

cudaError_t launch_ac_tail(const void* v, const void* told, void* tnew, int is_f32, uint32_t P,
                           uint64_t pitch, uint64_t len, uint64_t lag, uint64_t have,
                           cudaStream_t st) {
    if (is_f32)
        k_ac_tail<float><<<64, 256, 0, st>>>(static_cast<const float*>(v),
                                             static_cast<const float*>(told),
                                             static_cast<float*>(tnew), P, pitch, len, lag, have);
    else
        k_ac_tail<double><<<64, 256, 0, st>>>(static_cast<const double*>(v),
                                              static_cast<const double*>(told),
                                              static_cast<double*>(tnew), P, pitch, len, lag,
                                              have);
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
