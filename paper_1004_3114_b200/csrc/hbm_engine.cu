// HBM engine: pools too large for shared memory (BASELINE.json config C2,
// one 4 x 2^20 fp64 pool).  Double-buffered in global memory (the 2 x 32 MiB
// of C2 stay L2-resident on the 126 MB L2), one grid-wide launch per pass,
// host-driven control flow (capi.cu plan_fill) mirroring wallace.cpp:169-216.
#include "common.cuh"

namespace wg {

// ---------------------------------------------------------------------------
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
            LfgParams lp;
            lfg_params<NA>(w, N, lp);
            wrng_gpu_params p;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                p.stride[m] = lp.stride[m];
                p.offset[m] = lp.offset[m];
            }
            p.variant = lp.variant;
            p.pad_ = 0;
            p.c = lp.c;
            p.s = lp.s;
            p.scale = 0.0;         // derived in the pass kernel from the
            p.target_sumsq = 0.0;  // previous pass's withheld value
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

// drift_check on an HBM pool (wallace.cpp:225-234).  Default: the exact
// value of the left-to-right Pool::direct_sumsq (wallace.cpp:13-18) through
// the binade segment functions of common.cuh, in four launches:
//   1 chunk sums (approximate)   2 exclusive scan -> binade guess per chunk
//   3 segment function per chunk, composed per block of 32 chunks
//   4 one thread walks blocks, then chunks, then terms where needed.
// tree != 0: blocked parallel reduction instead (documented deviation,
// relative error ~1e-16 * log n).
constexpr uint32_t kSumChunk = 128;

template <typename T>
__global__ void k_sum_chunks(KernelArgs a, uint32_t buf, uint64_t nvals, double* approx,
                             uint32_t nch) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch || a.meta->error) return;
    const T* v = static_cast<const T*>(a.buf[buf]);
    const uint64_t lo = (uint64_t)c * kSumChunk, hi = umin64(lo + kSumChunk, nvals);
    double s = 0.0;
    for (uint64_t i = lo; i < hi; ++i) s += sq_term(v[i]);
    approx[c] = s;
}

__global__ void __launch_bounds__(1024) k_sum_scan(const double* approx, uint32_t nch,
                                                   int* e_out, double* pref_scratch) {
    // approximate exclusive prefix: per-thread serial runs + one block scan
    __shared__ double part[1024];
    const uint32_t t = threadIdx.x, per = (nch + 1023) / 1024;
    const uint32_t lo = t * per, hi = lo + per < nch ? lo + per : nch;
    double s = 0.0;
    for (uint32_t i = lo; i < hi; ++i) s += approx[i];
    part[t] = s;
    __syncthreads();
    for (uint32_t off = 1; off < 1024; off <<= 1) {
        double x = t >= off ? part[t - off] : 0.0;
        __syncthreads();
        part[t] += x;
        __syncthreads();
    }
    double pre = t ? part[t - 1] : 0.0;
    for (uint32_t i = lo; i < hi; ++i) {
        pref_scratch[i] = pre;
        e_out[i] = pre > 0.0 ? exp2_of(pre) : -2000;
        pre += approx[i];
    }
}

template <typename T>
__global__ void k_sum_segs(KernelArgs a, uint32_t buf, uint64_t nvals, const int* e_in,
                           SumSeg* segs, SumSeg* blocks, uint32_t nch) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const T* v = static_cast<const T*>(a.buf[buf]);
    SumSeg g;
    const int e = c < nch ? e_in[c] : -2000;
    seg_init(g, e);
    if (c < nch && e > -1000) {
        const double sc = pow2d(52 - e);
        const uint64_t lo = (uint64_t)c * kSumChunk, hi = umin64(lo + kSumChunk, nvals);
        for (uint64_t i = lo; i < hi; ++i) seg_push(g, sq_term(v[i]), sc);
    } else {
        g.valid = 0;
    }
    if (c < nch) segs[c] = g;
    // compose 32 consecutive chunks (lane order) into one block function
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t off = 1; off < 32; off <<= 1) {
        SumSeg o;
        o.s[0] = __shfl_down_sync(0xffffffffu, g.s[0], off);
        o.s[1] = __shfl_down_sync(0xffffffffu, g.s[1], off);
        o.par[0] = __shfl_down_sync(0xffffffffu, g.par[0], off);
        o.par[1] = __shfl_down_sync(0xffffffffu, g.par[1], off);
        o.valid = __shfl_down_sync(0xffffffffu, g.valid, off);
        o.e = __shfl_down_sync(0xffffffffu, g.e, off);
        if ((lane & (2 * off - 1)) == 0) g = seg_compose(g, o);
    }
    if (lane == 0 && c < nch) blocks[c / 32] = g;
}

template <typename T>
__global__ void k_sum_walk(KernelArgs a, uint32_t buf, uint64_t nvals, const SumSeg* segs,
                           const SumSeg* blocks, uint32_t nch) {
    if (threadIdx.x != 0 || a.meta->error) return;
    const T* v = static_cast<const T*>(a.buf[buf]);
    double q = 0.0;
    const uint32_t nblk = (nch + 31) / 32;
    for (uint32_t b = 0; b < nblk; ++b) {
        if (b * 32 + 32 <= nch && seg_apply(q, blocks[b])) continue;
        const uint32_t cend = b * 32 + 32 < nch ? b * 32 + 32 : nch;
        for (uint32_t c = b * 32; c < cend; ++c) {
            if (seg_apply(q, segs[c])) continue;
            const uint64_t lo = (uint64_t)c * kSumChunk, hi = umin64(lo + kSumChunk, nvals);
            for (uint64_t i = lo; i < hi; ++i) q = q + sq_term(v[i]);
        }
    }
    const double rel = fabs(q / a.meta->tracked[buf] - 1.0);
    if (!(rel <= 1e-3))
        a.meta->error = WRNG_GPU_ECORRUPT;
    else
        a.meta->tracked[buf] = q;
}

size_t hbm_drift_scratch_bytes(uint64_t nvals) {
    const uint64_t nch = (nvals + kSumChunk - 1) / kSumChunk;
    return nch * (2 * sizeof(double) + sizeof(int) + sizeof(SumSeg)) +
           ((nch + 31) / 32) * sizeof(SumSeg) + 1024;
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
        const uint32_t nch = (uint32_t)((nvals + kSumChunk - 1) / kSumChunk);
        char* p = reinterpret_cast<char*>(scratch);
        double* approx = reinterpret_cast<double*>(p);
        double* pref = approx + nch;
        int* e = reinterpret_cast<int*>(pref + nch);
        SumSeg* segs = reinterpret_cast<SumSeg*>(
            (reinterpret_cast<uintptr_t>(e + nch) + 63) & ~uintptr_t(63));
        SumSeg* blocks = segs + nch;
        const uint32_t g = (nch + 255) / 256;
        if (dtype == WRNG_GPU_F64) {
            k_sum_chunks<double><<<g, 256, 0, st>>>(a, buf, nvals, approx, nch);
            k_sum_scan<<<1, 1024, 0, st>>>(approx, nch, e, pref);
            k_sum_segs<double><<<g, 256, 0, st>>>(a, buf, nvals, e, segs, blocks, nch);
            k_sum_walk<double><<<1, 32, 0, st>>>(a, buf, nvals, segs, blocks, nch);
        } else {
            k_sum_chunks<float><<<g, 256, 0, st>>>(a, buf, nvals, approx, nch);
            k_sum_scan<<<1, 1024, 0, st>>>(approx, nch, e, pref);
            k_sum_segs<float><<<g, 256, 0, st>>>(a, buf, nvals, e, segs, blocks, nch);
            k_sum_walk<float><<<1, 32, 0, st>>>(a, buf, nvals, segs, blocks, nch);
        }
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

}  // namespace wg
