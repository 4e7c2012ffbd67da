// GPU Box-Muller and polar generators (reference.cpp:9-63): the methods the
// paper measures Wallace against, so the speed-up claim
// can be restated on B200.  Stream p = UniformState(seed,
// stream_id + p) on CTA p (lag table in shared memory, 256 words per step
// via lfg_bulk's recurrence), each stream a fresh fill_from_pairs
// (reference.cpp:46-55): pairs in order, an odd length takes the final
// pair's x.  Output is pool-major like a bank fill.
//
// F64 math follows the reference expression by expression (CUDA libm
// log/sqrt/cos/sin: within a few ulp of glibc, the same tolerance as the
// device pool init).  The F32 variant (logf, sqrtf, sincospif) is the
// throughput baseline a GPU user would write; it is not parity-checked
// beyond fp32 tolerance.
#include "common.cuh"

namespace wg {

enum Method : int { M_BOXMULLER = 0, M_POLAR = 1 };

template <bool F64M>
__device__ __forceinline__ void bm_pair(uint64_t w1, uint64_t w2, double& x, double& y) {
    if constexpr (F64M) {
        box_muller(w1, w2, x, y);  // reference.cpp:9-22
    } else {
        double d1 = u53(w1);
        if (d1 == 0.0) d1 = 0x1.0p-53;
        const float u1 = (float)d1, u2 = (float)u53(w2);
        const float r = sqrtf(-2.0f * logf(u1));
        float s, c;
        sincospif(2.0f * u2, &s, &c);
        x = (double)(r * c);
        y = (double)(r * s);
    }
}

// polar_next's test and transform (reference.cpp:24-39); returns accept.
template <bool F64M>
__device__ __forceinline__ bool polar_pair(uint64_t w1, uint64_t w2, double& x, double& y) {
    const double v1 = 2.0 * u53(w1) - 1.0, v2 = 2.0 * u53(w2) - 1.0;
    const double s = v1 * v1 + v2 * v2;
    if (!(s > 0.0 && s < 1.0)) return false;
    if constexpr (F64M) {
        const double f = sqrt(-2.0 * log(s) / s);
        x = v1 * f;
        y = v2 * f;
    } else {
        const float sf = (float)s;
        const float f = sqrtf(-2.0f * logf(sf) / sf);
        x = (double)((float)v1 * f);
        y = (double)((float)v2 * f);
    }
    return true;
}

template <int METHOD, bool F64M>
__global__ void __launch_bounds__(256) k_method_fill(uint64_t seed, uint64_t stream0,
                                                     OutLayout lay, double mu, double sigma,
                                                     uint32_t out_f32, uint32_t unit,
                                                     void* out) {
    __shared__ uint64_t tab[608];
    __shared__ uint64_t wbuf[256];
    __shared__ Ctl ctl;
    __shared__ uint32_t wcnt[8];
    const uint32_t p = blockIdx.x, tid = threadIdx.x;
    const uint64_t len = lay.len_base + (p < lay.len_extra ? 1 : 0);
    const uint64_t off =
        (uint64_t)p * lay.off_stride + (p < lay.off_extra ? p : lay.off_extra);
    char* o = static_cast<char*>(out) + off * (out_f32 ? 4 : 8);
    lfg_seed(tab, &ctl, wbuf, seed, stream0 + p, 256);
    const uint64_t npairs = (len + 1) / 2;
    if (npairs == 0) return;
    if constexpr (METHOD == M_BOXMULLER) {
        // two words per pair, every pair used (reference.cpp:17-22)
        lfg_bulk(tab, &ctl, wbuf, 2 * npairs, 256, [&](uint64_t base, uint32_t cnt) {
            if (2 * tid + 1 < cnt) {
                double x, y;
                bm_pair<F64M>(wbuf[2 * tid], wbuf[2 * tid + 1], x, y);
                const uint64_t i = base + 2 * tid;  // = 2 * pair index
                put_out(o, i, x, out_f32, unit, mu, sigma);
                if (i + 1 < len) put_out(o, i + 1, y, out_f32, unit, mu, sigma);
            }
        });
    } else {
        // rejection: the accepted pairs of each 128-candidate step keep
        // their order (block prefix over the accept flags)
        uint32_t r = ctl.r;
        uint64_t produced = 0;
        while (produced < npairs) {
            wbuf[tid] = lfg_word_at(tab, r, tid);
            r += 256;
            r = r >= kTable ? r - kTable : r;
            __syncthreads();
            double x = 0.0, y = 0.0;
            const bool acc = tid < 128 && polar_pair<F64M>(wbuf[2 * tid], wbuf[2 * tid + 1], x, y);
            const uint32_t bal = __ballot_sync(0xffffffffu, acc);
            const uint32_t lane = tid & 31, warp = tid >> 5;
            if (lane == 0) wcnt[warp] = __popc(bal);
            __syncthreads();
            uint32_t before = 0, total = 0;
#pragma unroll
            for (uint32_t w = 0; w < 4; ++w) {
                const uint32_t c = wcnt[w];
                before += w < warp ? c : 0;
                total += c;
            }
            if (acc) {
                const uint64_t k = produced + before + __popc(bal & ((1u << lane) - 1u));
                if (k < npairs) {
                    const uint64_t i = 2 * k;
                    put_out(o, i, x, out_f32, unit, mu, sigma);
                    if (i + 1 < len) put_out(o, i + 1, y, out_f32, unit, mu, sigma);
                }
            }
            produced += total;
            __syncthreads();
        }
    }
}

cudaError_t launch_method_fill(int method, int f64_math, uint64_t seed, uint64_t stream0,
                               uint32_t pools, const OutLayout& lay, double mu, double sigma,
                               uint32_t out_f32, void* out, cudaStream_t st) {
    const uint32_t unit = mu == 0.0 && sigma == 1.0;
    if (method == M_BOXMULLER) {
        if (f64_math)
            k_method_fill<M_BOXMULLER, true><<<pools, 256, 0, st>>>(seed, stream0, lay, mu, sigma,
                                                                    out_f32, unit, out);
        else
            k_method_fill<M_BOXMULLER, false><<<pools, 256, 0, st>>>(seed, stream0, lay, mu,
                                                                     sigma, out_f32, unit, out);
    } else {
        if (f64_math)
            k_method_fill<M_POLAR, true><<<pools, 256, 0, st>>>(seed, stream0, lay, mu, sigma,
                                                                out_f32, unit, out);
        else
            k_method_fill<M_POLAR, false><<<pools, 256, 0, st>>>(seed, stream0, lay, mu, sigma,
                                                                 out_f32, unit, out);
    }
    return cudaGetLastError();
}

}  // namespace wg
