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
