// HBM engine: pools too large for shared memory (BASELINE.json config C2,
// one 4 x 2^20 fp64 pool).  Double-buffered in global memory, one grid-wide
// launch per pass, host-driven control flow (capi.cu plan_fill) mirroring
// wallace.cpp:169-216.
//
// Transposed storage.  Each array of N = C * R values (R = min(512, N)) is
// stored as C rows of R: value i lives at (i mod C) * R + i / C
// (hbm_pos, internal.h).  For output columns j = j_hi * C + j_lo with a fixed
// j_lo, the sources (a j + g) mod N of one array all lie in ONE stored row,
// (a j_lo + g) mod C, at positions (a j_hi + (a j_lo + g) / C) mod R.  So a
// CTA owning a few output rows j_lo loads whole source rows with coalesced
// loads, gathers from shared memory with an odd stride (conflict-free), and
// writes its output rows with coalesced stores; the natural-order output
// stream gets JLO consecutive values per thread and array.  Every gathered
// byte is used, instead of one 8-byte value per 32-byte sector of a direct
// strided gather.
#include <utility>

#include <cstdlib>

#include "common.cuh"

namespace wg {

// ---------------------------------------------------------------------------
// pass parameters: the uniform-generator part of `npass` consecutive passes;
// the scale needs the previous pass's withheld value and is derived inside
// each pass kernel.  One CTA: the words of up to kParTile passes are produced
// in one parallel table step (x[i] += x[i+334] is hazard-free for 273
// consecutive words, common.cuh), then one thread per pass decodes its words
// (draw order of wallace.cpp:54-58).  (One warp drawing pass after pass took
// 29 us per 64-pass batch, 3 % of a C2 step.)
// ---------------------------------------------------------------------------
constexpr uint32_t kParThreads = 256;
template <int NA>
__global__ void __launch_bounds__(kParThreads)
    k_hbm_params(uint32_t N, LfgState* lfg, wrng_gpu_params* params, uint32_t npass,
                 PoolMeta* meta) {
    constexpr uint32_t K = NA == 2 ? 6 : 9;
    constexpr uint32_t kParTile = 252 / K;  // passes per table step (<= 256 words)
    __shared__ uint64_t tab[kTable];
    __shared__ uint64_t w[kParTile * K];
    LfgState* lg = lfg + blockIdx.x;
    if (meta[blockIdx.x].error) return;
    const uint32_t t = threadIdx.x;
    for (uint32_t i = t; i < kTable; i += kParThreads) tab[i] = lg->table[i];
    uint32_t r = lg->r;
    __syncthreads();
    for (uint32_t ps0 = 0; ps0 < npass; ps0 += kParTile) {
        const uint32_t np = npass - ps0 < kParTile ? npass - ps0 : kParTile;
        if (t < np * K) w[t] = lfg_word_at(tab, r, t);
        r = (r + np * K) % kTable;
        __syncthreads();
        if (t < np) {
            LfgParams lp;
            lfg_params<NA>(w + t * K, N, lp);
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
            p.scale = 0.0;
            p.target_sumsq = 0.0;
            params[(uint64_t)blockIdx.x * npass + ps0 + t] = p;
        }
        __syncthreads();
    }
    for (uint32_t i = t; i < kTable; i += kParThreads) lg->table[i] = tab[i];
    if (t == 0) {
        lg->r = r;
        lg->draws += (uint64_t)K * npass;
    }
}

cudaError_t launch_hbm_params(uint32_t n_arrays, uint32_t N, LfgState* lfg,
                              wrng_gpu_params* params, uint32_t npass, PoolMeta* meta,
                              cudaStream_t st) {
    if (n_arrays == 2)
        k_hbm_params<2><<<1, kParThreads, 0, st>>>(N, lfg, params, npass, meta);
    else
        k_hbm_params<4><<<1, kParThreads, 0, st>>>(N, lfg, params, npass, meta);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// one regeneration pass (wallace.cpp:113-137) on transposed storage
// ---------------------------------------------------------------------------
#ifndef WG_HBM_JLO
#define WG_HBM_JLO 4
#endif
#ifndef WG_EMIT_TS
#define WG_EMIT_TS 64
#endif
constexpr uint32_t kJlo = WG_HBM_JLO;  // output rows per CTA

// Output element with an evict-first (streaming) store, so the write-once
// output stream does not push the pool buffers out of L2.
template <typename T>
__device__ __forceinline__ void put_out_cs(void* out, uint64_t i, T v, uint32_t out_f32,
                                           uint32_t unit, double mu, double sigma) {
    double o = unit ? (double)v + 0.0 : mu + sigma * (double)v;
    if (unit && out_f32) {
        __stcs(static_cast<float*>(out) + i, (float)v + 0.0f);
        return;
    }
    if (out_f32)
        __stcs(static_cast<float*>(out) + i, (float)o);
    else
        __stcs(static_cast<double*>(out) + i, o);
}

template <typename T, int NA, int JL>
__global__ void __launch_bounds__(512, 3) k_hbm_pass(KernelArgs a, wrng_gpu_params* params,
                                                  HbmPass ps) {
    extern __shared__ __align__(16) unsigned char hsm[];
    T* rows = reinterpret_cast<T*>(hsm);  // [NA][R]
    __shared__ double s_c0, s_c1, s_target, s_scale;
    __shared__ int s_err;
    const uint32_t N = a.N;
    const HbmSplit sp = hbm_split(N);
    const uint32_t R = 1u << sp.lr, C = 1u << sp.lc;
    PoolMeta* meta = a.meta;
    const uint32_t src = ps.src, dst = src ^ 1u;
    const wrng_gpu_params prm = params[ps.param_idx];
    const uint32_t t = threadIdx.x;
    const T* spool = static_cast<const T*>(a.buf[src]);
    T* dpool = static_cast<T*>(a.buf[dst]);
    const uint32_t jlo0 = blockIdx.x * JL;

    // software pipeline: sources of row r + 1 load while row r computes
    T nxt[NA];
    uint32_t shift[JL][NA];
#pragma unroll
    for (int r = 0; r < JL; ++r)
#pragma unroll
        for (int m = 0; m < NA; ++m)
            shift[r][m] = ((prm.stride[m] * (jlo0 + r) + prm.offset[m]) >> sp.lc) & (R - 1);
    auto load_row = [&](int r) {
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            const uint32_t srow = (prm.stride[m] * (jlo0 + r) + prm.offset[m]) & (C - 1);
            nxt[m] = __ldg(spool + (uint64_t)m * N + (uint64_t)srow * R + t);
        }
    };
    load_row(0);
    if (t == 0) {
        int err = meta->error ? -1 : 0;
        const double tracked = meta->tracked[src], withheld = meta->withheld[src];
        if (!err) {
            double scale, target;
            err = pass_scale(tracked, withheld, NA * N, a.mode, scale, target);
            if (!err) {
                s_target = target;
                s_scale = scale;
                // regenerate folds the scale into the matrix (wallace.cpp:116-117)
                s_c0 = NA == 2 ? prm.c * scale : (prm.variant ? scale : 0.5 * scale);
                s_c1 = NA == 2 ? prm.s * scale : scale;
            }
        }
        s_err = err;
    }
    __syncthreads();
    if (s_err) {
        if (s_err > 0 && blockIdx.x == 0 && t == 0) meta->error = s_err;
        return;
    }
    const T c0 = (T)s_c0, c1 = (T)s_c1;  // fp32 pools: rounded once
    const uint32_t variant = prm.variant;
#pragma unroll
    for (int r = 0; r < JL; ++r) {
        const uint32_t jlo = jlo0 + r;
#pragma unroll
        for (int m = 0; m < NA; ++m) rows[m * R + t] = nxt[m];
        __syncthreads();
        if (r + 1 < JL) load_row(r + 1);
        T g[NA];
#pragma unroll
        for (int m = 0; m < NA; ++m)
            g[m] = rows[m * R + ((prm.stride[m] * t + shift[r][m]) & (R - 1))];
        T y[NA];
        if (NA == 2) {
            y[0] = c0 * g[0] + c1 * g[NA > 1 ? 1 : 0];
            y[NA > 1 ? 1 : 0] = c0 * g[NA > 1 ? 1 : 0] - c1 * g[0];
        } else {
            const T a0 = g[0], a1 = g[NA > 1 ? 1 : 0], a2 = g[NA > 2 ? 2 : 0],
                    a3 = g[NA > 3 ? 3 : 0];
            if (variant == 0) {
                const T pp = a0 + a1, q = a0 - a1, rr = a2 + a3, s = a2 - a3;
                y[0] = c0 * (pp + rr);
                y[NA > 1 ? 1 : 0] = c0 * (q + s);
                y[NA > 2 ? 2 : 0] = c0 * (pp - rr);
                y[NA > 3 ? 3 : 0] = c0 * (q - s);
            } else {
                const T tt = (T)0.5 * ((a0 + a1) + (a2 + a3));
                y[0] = c0 * (tt - a0);
                y[NA > 1 ? 1 : 0] = c0 * (tt - a1);
                y[NA > 2 ? 2 : 0] = c0 * (tt - a2);
                y[NA > 3 ? 3 : 0] = c0 * (tt - a3);
            }
        }
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            dpool[(uint64_t)m * N + (uint64_t)jlo * R + t] = y[m];  // row jlo, coalesced
        }
        if (jlo == C - 1 && t == R - 1) meta->withheld[dst] = (double)y[NA - 1];
        __syncthreads();
    }
    // the exposed window is streamed by k_hbm_emit_t (coalesced transpose)
    if (blockIdx.x == 0 && t == 0) {
        params[ps.param_idx].scale = s_scale;
        params[ps.param_idx].target_sumsq = s_target;
        meta->tracked[dst] = s_target;
        meta->active = dst;
        meta->pass_count += 1;
        meta->avail = ps.end_refill ? (uint64_t)NA * N - 1 - ps.emit_n : 0;
    }
}

// Launch with the handle's persisting-L2 window (pool buffers), if any.
template <typename... KP, typename... Args>
static cudaError_t launch_l2(void (*kern)(KP...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, const KernelArgs& a, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    cfg.numAttrs = 0;
    if (a.l2_bytes) {
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = a.l2_base;
        attr[0].val.accessPolicyWindow.num_bytes = a.l2_bytes;
        attr[0].val.accessPolicyWindow.hitRatio = a.l2_hit;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename T, int NA>
static void hbm_pass_go(const KernelArgs& a, wrng_gpu_params* params, const HbmPass& ps,
                        uint32_t R, uint32_t C, size_t smem, cudaStream_t st) {
    if (C >= kJlo)
        launch_l2(k_hbm_pass<T, NA, kJlo>, dim3(C / kJlo), dim3(R), smem, st, a, a, params, ps);
    else if (C == 2)
        launch_l2(k_hbm_pass<T, NA, 2>, dim3(1), dim3(R), smem, st, a, a, params, ps);
    else
        launch_l2(k_hbm_pass<T, NA, 1>, dim3(1), dim3(R), smem, st, a, a, params, ps);
}

cudaError_t launch_hbm_pass(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                            wrng_gpu_params* params, const HbmPass& ps, cudaStream_t st) {
    const HbmSplit sp = hbm_split(a.N);
    const uint32_t R = 1u << sp.lr, C = 1u << sp.lc;
    const size_t smem = (size_t)n_arrays * R * (dtype == WRNG_GPU_F64 ? 8 : 4);
    if (dtype == WRNG_GPU_F64) {
        if (n_arrays == 2)
            hbm_pass_go<double, 2>(a, params, ps, R, C, smem, st);
        else
            hbm_pass_go<double, 4>(a, params, ps, R, C, smem, st);
    } else {
        if (n_arrays == 2)
            hbm_pass_go<float, 2>(a, params, ps, R, C, smem, st);
        else
            hbm_pass_go<float, 4>(a, params, ps, R, C, smem, st);
    }
    return cudaGetLastError();
}

// Exposed window of a freshly regenerated pool (wallace.cpp:206-213):
// natural index m*N + j_hi*C + j_lo is stored at m*N + j_lo*R + j_hi, i.e.
// a (C x R) -> (R x C) transpose per array, done in 32 x 32 shared-memory
// tiles so both the pool reads and the output writes are coalesced; output
// stores are evict-first.  Flat indices >= emit_n are not written.
template <typename T>
__global__ void __launch_bounds__(256) k_hbm_emit_t(KernelArgs a, uint32_t buf,
                                                    uint64_t emit_n, uint64_t out_off) {
    constexpr uint32_t TS = WG_EMIT_TS;  // TS x TS tile, TS^2/256 loads + stores per thread
    __shared__ T tile[TS][TS + 1];
    if (a.meta->error) return;
    const uint32_t N = a.N;
    const HbmSplit sp = hbm_split(N);
    const uint32_t R = 1u << sp.lr, C = 1u << sp.lc;
    const T* pool = static_cast<const T*>(a.buf[buf]) + (uint64_t)blockIdx.z * N;
    const uint32_t jh0 = blockIdx.x * TS, jl0 = blockIdx.y * TS;
    const uint32_t tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
    for (uint32_t k = 0; k < TS; k += 8) {
        const uint32_t jl = jl0 + ty + k;  // stored row
        if (jl < C) {
#pragma unroll
            for (uint32_t h = 0; h < TS; h += 32)
                tile[ty + k][tx + h] = pool[(uint64_t)jl * R + jh0 + tx + h];
        }
    }
    __syncthreads();
    char* outc = static_cast<char*>(a.out) + out_off * (a.out_f32 ? 4 : 8);
    const uint64_t mbase = (uint64_t)blockIdx.z * N;
#pragma unroll
    for (uint32_t k = 0; k < TS; k += 8) {
        const uint32_t jh = jh0 + ty + k;
#pragma unroll
        for (uint32_t h = 0; h < TS; h += 32) {
            const uint32_t jl = jl0 + tx + h;
            const uint64_t flat = mbase + (uint64_t)jh * C + jl;
            if (jl < C && flat < emit_n)
                put_out_cs(outc, flat, tile[tx + h][ty + k], a.out_f32, a.unit, a.mu, a.sigma);
        }
    }
}

cudaError_t launch_hbm_emit_t(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                              uint32_t buf, uint64_t emit_n, uint64_t out_off, cudaStream_t st) {
    const HbmSplit sp = hbm_split(a.N);
    const uint32_t R = 1u << sp.lr, C = 1u << sp.lc;
    const dim3 grid(R / WG_EMIT_TS, (C + WG_EMIT_TS - 1) / WG_EMIT_TS, n_arrays), block(32, 8);
    if (dtype == WRNG_GPU_F64)
        return launch_l2(k_hbm_emit_t<double>, grid, block, 0, st, a, a, buf, emit_n, out_off);
    return launch_l2(k_hbm_emit_t<float>, grid, block, 0, st, a, a, buf, emit_n, out_off);
    return cudaGetLastError();
}

// leftover emission of the live pool: flat [pos, pos + take)
template <typename T>
__global__ void k_hbm_emit(KernelArgs a, uint32_t buf, uint64_t pos, uint64_t take,
                           uint64_t out_off) {
    if (a.meta->error) return;
    const T* pool = static_cast<const T*>(a.buf[buf]);
    const HbmSplit sp = hbm_split(a.N);
    char* o = static_cast<char*>(a.out) + out_off * (a.out_f32 ? 4 : 8);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < take;
         i += (uint64_t)gridDim.x * blockDim.x)
        put_out(o, i, pool[hbm_pos(pos + i, a.N, sp)], a.out_f32, a.unit, a.mu, a.sigma);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.meta->avail -= take;
}

cudaError_t launch_hbm_emit(uint32_t, uint32_t dtype, const KernelArgs& a, uint32_t buf,
                            uint64_t pos, uint64_t take, uint64_t out_off, cudaStream_t st) {
    uint32_t grid = (uint32_t)umin64((take + 255) / 256, 148 * 8);
    if (grid == 0) grid = 1;
    if (dtype == WRNG_GPU_F64)
        k_hbm_emit<double><<<grid, 256, 0, st>>>(a, buf, pos, take, out_off);
    else
        k_hbm_emit<float><<<grid, 256, 0, st>>>(a, buf, pos, take, out_off);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// drift_check / init tracked sum on an HBM pool (wallace.cpp:225-234).
// Default: the exact value of the left-to-right Pool::direct_sumsq
// (wallace.cpp:13-18) through the binade segment functions of common.cuh:
//   1 k_sum_chunks: approximate chunk sums, CTA-local exclusive scan, CTA sums;
//   2 k_sum_segs:   binade guess per chunk from that prefix, segment function
//                   per chunk, composed per block of 32 chunks;
//   3 k_sum_walk:   one CTA composes 32-block super-blocks in shared memory;
//                   thread 0 walks super-blocks, descending into blocks and
//                   (with the CTA staging data) chunks and terms only where a
//                   function cannot be applied (~log2 n places).
// tree != 0: blocked parallel reduction (documented deviation, relative
// error ~1e-16 * log n).
// ---------------------------------------------------------------------------
#ifndef WG_SUM_CHUNK
#define WG_SUM_CHUNK 64  // terms per chunk (C2: 64 -> 9.36 ms/step, 128 -> 9.59, 32 -> 9.43)
#endif
constexpr uint32_t kSumChunk = WG_SUM_CHUNK;
constexpr uint32_t kSumCta = 256;  // chunks per CTA of kernels 1-2

template <typename T>
__device__ __forceinline__ double pool_term(const T* v, uint64_t i, uint32_t N,
                                            const HbmSplit& sp) {
    return sq_term(v[hbm_pos(i, N, sp)]);
}

// Which chunk of its CTA's kSumCta consecutive chunks thread t evaluates.  A
// chunk is kSumChunk consecutive natural indices jh*C + jl .. (one jh, a run
// of jl), stored kSumChunk rows apart — storage position jl*R + jh — so with
// thread = chunk a warp's load touches 32 rows: 32 sectors for 256 bytes.
// When a natural row holds CPR = C / kSumChunk whole chunks and the CTA covers
// JH = kSumCta / CPR whole rows, thread t takes chunk (t % JH) * CPR + t / JH:
// JH consecutive lanes then read JH consecutive jh of one storage row (64
// contiguous bytes for C2's JH = 8; a quarter of the sectors).  The results
// change hands through shared memory, so everything after the term loops
// (the scan, the 32-chunk compositions, the stores) stays in natural order.
__device__ __forceinline__ uint32_t sum_chunk_of_thread(uint32_t t, uint32_t N) {
    const HbmSplit sp = hbm_split(N);
    const uint32_t C = 1u << sp.lc;
    const uint32_t cpr = C / kSumChunk;
    if (cpr < 1 || C % kSumChunk || cpr * 2 > kSumCta || kSumCta % cpr ||
        (N / kSumChunk) % kSumCta)
        return t;
    const uint32_t jhn = kSumCta / cpr;
    return (t % jhn) * cpr + t / jhn;
}

template <typename T>
__global__ void __launch_bounds__(kSumCta) k_sum_chunks(KernelArgs a, uint32_t buf,
                                                        uint64_t nvals, double* pre_local,
                                                        double* cta_sum, uint32_t nch) {
    __shared__ double part[kSumCta];
    const uint32_t t = threadIdx.x;
    const uint32_t cl = sum_chunk_of_thread(t, a.N), c = blockIdx.x * kSumCta + cl;
    const T* v = static_cast<const T*>(a.buf[buf]);
    const HbmSplit sp = hbm_split(a.N);
    double s = 0.0;
    if (c < nch) {
        const uint64_t lo = (uint64_t)c * kSumChunk, hi = umin64(lo + kSumChunk, nvals);
        for (uint64_t i = lo; i < hi; ++i) s += pool_term(v, i, a.N, sp);
    }
    part[cl] = s;
    __syncthreads();
    for (uint32_t off = 1; off < kSumCta; off <<= 1) {  // inclusive scan (approximate)
        const double x = t >= off ? part[t - off] : 0.0;
        __syncthreads();
        part[t] += x;
        __syncthreads();
    }
    // thread t now writes chunk t's exclusive prefix
    if (blockIdx.x * kSumCta + t < nch) pre_local[blockIdx.x * kSumCta + t] = t ? part[t - 1] : 0.0;
    if (t == kSumCta - 1) cta_sum[blockIdx.x] = part[t];
}

template <typename T>
__global__ void __launch_bounds__(kSumCta) k_sum_segs(KernelArgs a, uint32_t buf, uint64_t nvals,
                                                      const double* pre_local,
                                                      const double* cta_sum, SumSeg* segs,
                                                      SumSeg* blocks, uint32_t nch) {
    __shared__ double s_base;
    __shared__ SumSeg s_seg[kSumCta];
    const uint32_t t = threadIdx.x;
    const uint32_t cl = sum_chunk_of_thread(t, a.N);
    if (t < 32) {  // prefix of the previous CTAs' sums (approximate)
        double x = 0.0;
        for (uint32_t b = t; b < blockIdx.x; b += 32) x += cta_sum[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (t == 0) s_base = x;
    }
    __syncthreads();
    const T* v = static_cast<const T*>(a.buf[buf]);
    const HbmSplit sp = hbm_split(a.N);
    {
        const uint32_t c = blockIdx.x * kSumCta + cl;  // the chunk this thread evaluates
        const double pre = c < nch ? s_base + pre_local[c] : 0.0;
        const int e = pre > 0.0 ? exp2_of(pre) : -2000;
        SumSeg g;
        seg_init(g, e);
        if (c < nch && e > -1000) {
            const double sc = pow2d(52 - e);
            const uint64_t lo = (uint64_t)c * kSumChunk, hi = umin64(lo + kSumChunk, nvals);
            // the terms 16 at a time: the loads of a batch are in flight together
            // (seg_push branches, so the compiler does not hoist them itself)
            for (uint64_t i0 = lo; i0 < hi; i0 += 16) {
                double tm[16];
#pragma unroll
                for (uint32_t k = 0; k < 16; ++k)
                    tm[k] = i0 + k < hi ? pool_term(v, i0 + k, a.N, sp) : 0.0;
#pragma unroll
                for (uint32_t k = 0; k < 16; ++k)
                    if (i0 + k < hi) seg_push(g, tm[k], sc);
            }
        } else {
            g.valid = 0;
        }
        s_seg[cl] = g;
    }
    __syncthreads();
    // from here thread t holds chunk t (natural order)
    const uint32_t c = blockIdx.x * kSumCta + t;
    SumSeg g = s_seg[t];
    if (c < nch) {
        SumSeg f = g;
        seg_finalize(f);
        segs[c] = f;
    }
    // compose 32 consecutive chunks (lane order) into one block function
    const uint32_t lane = t & 31u;
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
    if (lane == 0 && c < nch) {
        if (c + 32 > nch) g.valid = 0;  // partial block
        blocks[c / 32] = g;             // not finalized: composed again
    }
}

constexpr uint32_t kWalkThreads = 256;
constexpr uint32_t kMaxPreBlk = 64;    // blocks whose chunk functions the walk pre-stages
constexpr uint32_t kMaxPreChk = 128;   // chunks whose terms the walk pre-stages

// The serial walk of the exact sum (one CTA).  Warp 0 applies the 32-chunk
// block functions 32 at a time (warp_seg_walk); where a block cannot be
// applied it walks the block's chunk functions, and where a chunk cannot be
// applied lane 0 adds its 64 terms one by one.  Those places are predictable:
// a block or chunk whose function is invalid (its guessed binade changes
// inside it) — about one per power of two the sum crosses.  So before the
// walk the whole CTA pre-stages, in one burst, the chunk functions of every
// invalid block and the terms of every invalid chunk in them (64 terms each);
// anything else that fails (a guess off by one binade) is fetched by warp 0
// on demand: 32 chunk functions or 64 terms, one round trip.
// mode 0: drift_check (compare, adopt or flag ECORRUPT); mode 1: set tracked.
template <typename T>
__global__ void __launch_bounds__(kWalkThreads) k_sum_walk(KernelArgs a, uint32_t buf,
                                                           uint64_t nvals, const SumSeg* segs,
                                                           const SumSeg* blocks, uint32_t nch,
                                                           int mode, uint32_t maxpb,
                                                           uint32_t maxpc) {
    extern __shared__ __align__(16) unsigned char wsm[];
    const uint32_t nblk = (nch + 31) / 32;
    SumSeg* sblk = reinterpret_cast<SumSeg*>(wsm);                     // [nblk]
    SumSeg* spchk = sblk + nblk;                                       // [maxpb][32]
    SumSeg* schk = spchk + (size_t)maxpb * 32;                         // [32] on demand
    double* spre = reinterpret_cast<double*>(schk + 32);               // [maxpc][kSumChunk]
    double* sterm = spre + (size_t)maxpc * kSumChunk;                  // [kSumChunk] on demand
    SumSeg* srun = reinterpret_cast<SumSeg*>(sterm + kSumChunk);       // [maxpb + 1]
    __shared__ uint32_t s_pb[kMaxPreBlk], s_pc[kMaxPreChk], s_npb, s_npc;
    __shared__ uint32_t s_wcnt[kWalkThreads / 32];
    if (a.meta->error) return;
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    const T* v = static_cast<const T*>(a.buf[buf]);
    const HbmSplit sp = hbm_split(a.N);
    for (uint32_t b = t; b < nblk; b += kWalkThreads) sblk[b] = blocks[b];
    if (t == 0) s_npb = s_npc = 0;
    __syncthreads();
    // ballot compaction of candidates in index order into list[<= cap]
    auto compact = [&](uint32_t n, uint32_t cap, uint32_t* list, uint32_t& count, auto&& cand_of,
                       auto&& id_of) {
        for (uint32_t base = 0; base < n && count < cap; base += kWalkThreads) {
            const uint32_t i = base + t;
            const bool cand = i < n && cand_of(i);
            const uint32_t m = __ballot_sync(0xffffffffu, cand);
            if (lane == 0) s_wcnt[warp] = __popc(m);
            __syncthreads();
            uint32_t off = count;
            for (uint32_t w = 0; w < warp; ++w) off += s_wcnt[w];
            const uint32_t pos = off + __popc(m & ((1u << lane) - 1u));
            if (cand && pos < cap) list[pos] = id_of(i);
            __syncthreads();
            if (t == 0) {
                uint32_t tot = count;
                for (uint32_t w = 0; w < kWalkThreads / 32; ++w) tot += s_wcnt[w];
                count = tot < cap ? tot : cap;
            }
            __syncthreads();
        }
    };
    compact(nblk, maxpb, s_pb, s_npb, [&](uint32_t b) { return !sblk[b].valid; },
            [](uint32_t b) { return b; });
    const uint32_t npb = s_npb;
    for (uint32_t i = t; i < npb * 32; i += kWalkThreads) {
        const uint32_t c = s_pb[i / 32] * 32 + (i & 31u);
        if (c < nch) {
            spchk[i] = segs[c];
        } else {
            seg_init(spchk[i], 0);
            spchk[i].valid = 0;
        }
    }
    __syncthreads();
    compact(npb * 32, maxpc, s_pc, s_npc,
            [&](uint32_t i) { return s_pb[i / 32] * 32 + (i & 31u) < nch && !spchk[i].valid; },
            [&](uint32_t i) { return s_pb[i / 32] * 32 + (i & 31u); });
    const uint32_t npc = s_npc;
    for (uint32_t i = t; i < npc * kSumChunk; i += kWalkThreads) {
        const uint64_t term = (uint64_t)s_pc[i / kSumChunk] * kSumChunk + i % kSumChunk;
        spre[i] = term < nvals ? pool_term(v, term, a.N, sp) : 0.0;
    }
    // Runs of blocks between consecutive pre-staged (invalid) blocks, each
    // composed into one function in parallel (a warp per run, 32 blocks per
    // step by a shuffle scan), so the serial walk applies a whole run at once.
    for (uint32_t r = warp; r <= npb; r += kWalkThreads / 32) {
        const uint32_t lo = r == 0 ? 0u : s_pb[r - 1] + 1, hi = r < npb ? s_pb[r] : nblk;
        SumSeg acc;
        seg_init(acc, lo < hi ? sblk[lo].e : 0);
        for (uint32_t base = lo; base < hi; base += 32) {
            SumSeg g;
            if (base + lane < hi) {
                g = sblk[base + lane];
            } else {
                seg_init(g, acc.e);  // identity in the run's binade
            }
#pragma unroll
            for (uint32_t o = 1; o < 32; o <<= 1) {
                const SumSeg y = seg_shfl_up(g, o);
                if (lane >= o) g = seg_compose(y, g);
            }
            SumSeg tot;
            tot.s[0] = __shfl_sync(0xffffffffu, g.s[0], 31);
            tot.s[1] = __shfl_sync(0xffffffffu, g.s[1], 31);
            tot.par[0] = __shfl_sync(0xffffffffu, g.par[0], 31);
            tot.par[1] = __shfl_sync(0xffffffffu, g.par[1], 31);
            tot.valid = __shfl_sync(0xffffffffu, g.valid, 31);
            tot.e = __shfl_sync(0xffffffffu, g.e, 31);
            acc = seg_compose(acc, tot);
        }
        if (lane == 0) {
            seg_finalize(acc);
            srun[r] = acc;
        }
    }
    __syncthreads();
    for (uint32_t b = t; b < nblk; b += kWalkThreads) seg_finalize(sblk[b]);
    __syncthreads();
    if (warp != 0) return;
    // ---- warp 0: the serial walk --------------------------------------
    // index of `id` in list[0, n), or n (lanes search 32 entries at a time)
    auto find = [&](const uint32_t* list, uint32_t n, uint32_t id) -> uint32_t {
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t m =
                __ballot_sync(0xffffffffu, base + lane < n && list[base + lane] == id);
            if (m) return base + (uint32_t)__ffs(m) - 1u;
        }
        return n;
    };
    double q = 0.0;
    // blocks [b, hi) one at a time where a run function does not apply
    auto walk_blocks = [&](uint32_t b, uint32_t hi) {
      while (b < hi) {
        b += warp_seg_walk(q, hi - b, [&](uint32_t k) { return seg_unfinalize(sblk[b + k]); });
        if (b >= hi) break;
        // block b cannot be applied: its chunk functions
        const uint32_t c0 = b * 32, cend = c0 + 32 < nch ? c0 + 32 : nch;
        const uint32_t jb = find(s_pb, npb, b);
        const SumSeg* ck = spchk + (size_t)jb * 32;
        if (jb >= npb) {
            if (c0 + lane < cend) schk[lane] = segs[c0 + lane];
            __syncwarp();
            ck = schk;
        }
        uint32_t c = c0;
        while (c < cend) {
            const uint32_t cs = c;
            c += warp_seg_walk(q, cend - cs, [&](uint32_t k) { return seg_unfinalize(ck[cs - c0 + k]); });
            if (c >= cend) break;
            // chunk c cannot be applied: its terms, one by one
            const uint64_t l2 = (uint64_t)c * kSumChunk, h2 = umin64(l2 + kSumChunk, nvals);
            const uint32_t jc = find(s_pc, npc, c);
            const double* tm = spre + (size_t)jc * kSumChunk;
            if (jc >= npc) {
#pragma unroll
                for (uint32_t h = 0; h < kSumChunk; h += 32)
                    if (l2 + h + lane < h2) sterm[h + lane] = pool_term(v, l2 + h + lane, a.N, sp);
                __syncwarp();
                tm = sterm;
            }
            if (lane == 0)
                for (uint64_t i = l2; i < h2; ++i) q = q + tm[i - l2];
            q = __shfl_sync(0xffffffffu, q, 0);
            __syncwarp();  // sterm / schk reused
            ++c;
        }
        ++b;
      }
    };
    for (uint32_t r = 0; r <= npb; ++r) {
        const uint32_t lo = r == 0 ? 0u : s_pb[r - 1] + 1, hi = r < npb ? s_pb[r] : nblk;
        if (hi > lo && !seg_apply(q, srun[r])) walk_blocks(lo, hi);
        if (r < npb) walk_blocks(hi, hi + 1);  // the invalid block itself
    }
    if (lane != 0) return;
    if (mode == 1) {
        a.meta->tracked[buf] = q;
        return;
    }
    const double rel = fabs(q / a.meta->tracked[buf] - 1.0);
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
        double d = (double)v[i];  // any order: a storage permutation is irrelevant
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

size_t hbm_drift_scratch_bytes(uint64_t nvals) {
    const uint64_t nch = (nvals + kSumChunk - 1) / kSumChunk;
    const uint64_t ncta = (nch + kSumCta - 1) / kSumCta;
    const size_t sum = (nch + ncta) * sizeof(double) + 128 +
                       (nch + (nch + 31) / 32) * sizeof(SumSeg) + 1024;
    const size_t words = (nvals + 2) * sizeof(uint64_t);  // init: uniform words
    return sum > words ? sum : words;
}

static cudaError_t exact_sum(uint32_t dtype, const KernelArgs& a, uint32_t buf, int mode,
                             void* scratch, uint64_t nvals, cudaStream_t st) {
    const uint32_t nch = (uint32_t)((nvals + kSumChunk - 1) / kSumChunk);
    const uint32_t ncta = (nch + kSumCta - 1) / kSumCta;
    double* pre_local = static_cast<double*>(scratch);
    double* cta_sum = pre_local + nch;
    SumSeg* segs = reinterpret_cast<SumSeg*>(
        (reinterpret_cast<uintptr_t>(cta_sum + ncta) + 63) & ~uintptr_t(63));
    SumSeg* blocks = segs + nch;
    const uint32_t nblk = (nch + 31) / 32;
    const size_t wbase = (nblk + 32) * sizeof(SumSeg) + kSumChunk * sizeof(double);
    // pre-staged block functions (32 chunks each) and chunk terms, two
    // chunks per block, as many as fit next to the block functions
    const size_t kWalkSmemMax = 200 * 1024;
    const size_t pre_pair = 33 * sizeof(SumSeg) + 2 * kSumChunk * sizeof(double);
    const uint32_t maxpb =
        wbase + pre_pair > kWalkSmemMax
            ? 0u
            : (uint32_t)std::min<size_t>(kMaxPreBlk, (kWalkSmemMax - wbase) / pre_pair);
    const uint32_t maxpc = std::min<uint32_t>(kMaxPreChk, 2 * maxpb);
    const size_t wsm = wbase + (size_t)maxpb * 32 * sizeof(SumSeg) +
                       (size_t)maxpc * kSumChunk * sizeof(double) + (maxpb + 1) * sizeof(SumSeg);
    cudaFuncSetAttribute(k_sum_walk<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)wsm);
    cudaFuncSetAttribute(k_sum_walk<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)wsm);
    if (dtype == WRNG_GPU_F64) {
        k_sum_chunks<double><<<ncta, kSumCta, 0, st>>>(a, buf, nvals, pre_local, cta_sum, nch);
        k_sum_segs<double><<<ncta, kSumCta, 0, st>>>(a, buf, nvals, pre_local, cta_sum, segs,
                                                     blocks, nch);
        k_sum_walk<double><<<1, kWalkThreads, wsm, st>>>(a, buf, nvals, segs, blocks, nch, mode,
                                                         maxpb, maxpc);
    } else {
        k_sum_chunks<float><<<ncta, kSumCta, 0, st>>>(a, buf, nvals, pre_local, cta_sum, nch);
        k_sum_segs<float><<<ncta, kSumCta, 0, st>>>(a, buf, nvals, pre_local, cta_sum, segs,
                                                    blocks, nch);
        k_sum_walk<float><<<1, kWalkThreads, wsm, st>>>(a, buf, nvals, segs, blocks, nch, mode,
                                                        maxpb, maxpc);
    }
    return cudaGetLastError();
}

cudaError_t launch_hbm_drift(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                             uint32_t buf, int tree, double* scratch, cudaStream_t st) {
    const uint64_t nvals = (uint64_t)n_arrays * a.N;
    if (!tree) return exact_sum(dtype, a, buf, 0, scratch, nvals, st);
    const uint32_t nb = 296;
    if (dtype == WRNG_GPU_F64)
        k_hbm_drift_tree_partial<double><<<nb, 256, 0, st>>>(a, buf, nvals, scratch);
    else
        k_hbm_drift_tree_partial<float><<<nb, 256, 0, st>>>(a, buf, nvals, scratch);
    k_hbm_drift_tree_final<<<1, 32, 0, st>>>(a, buf, scratch, nb);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// init_pool / restart of an HBM pool (wallace.cpp:158-167, 236):
//   1 one CTA seeds (or loads) the uniform generator and writes the n*N + 2
//     uniform words of the pool to scratch, 256 per step;
//   2 a grid applies Box-Muller to the word pairs (pool values, withheld);
//   3 tracked = exact direct_sumsq (the sum kernels, mode 1).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_init_words(KernelArgs a, uint64_t nwords, int seed_lfg,
                                                    uint64_t* words) {
    __shared__ uint64_t tab[608];
    __shared__ uint64_t wbuf[256];
    __shared__ Ctl ctl;
    LfgState* lg = a.lfg;
    if (!seed_lfg && a.meta->error) return;
    if (seed_lfg) {
        lfg_seed(tab, &ctl, wbuf, a.seed, a.stream0, 256);
    } else {
        for (uint32_t i = threadIdx.x; i < kTable; i += 256) tab[i] = lg->table[i];
        if (threadIdx.x == 0) {
            ctl.r = lg->r;
            ctl.draws = lg->draws;
        }
        __syncthreads();
    }
    lfg_bulk(tab, &ctl, wbuf, nwords, 256, [&](uint64_t base, uint32_t cnt) {
        if (threadIdx.x < cnt) words[base + threadIdx.x] = wbuf[threadIdx.x];
    });
    for (uint32_t i = threadIdx.x; i < kTable; i += 256) lg->table[i] = tab[i];
    if (threadIdx.x == 0) {
        lg->r = ctl.r;
        lg->draws = ctl.draws + nwords;
    }
}

template <typename T>
__global__ void k_init_bm(KernelArgs a, uint32_t buf, uint64_t nvals, const uint64_t* words,
                          int seed_lfg) {
    if (!seed_lfg && a.meta->error) return;
    T* pool = static_cast<T*>(a.buf[buf]);
    const HbmSplit sp = hbm_split(a.N);
    const uint64_t npairs = nvals / 2 + 1;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < npairs;
         k += (uint64_t)gridDim.x * blockDim.x) {
        double x, y;
        box_muller(words[2 * k], words[2 * k + 1], x, y);
        const uint64_t i = 2 * k;
        if (i < nvals) {
            // fill_from_pairs: out = mu + sigma * z with mu = 0, sigma = 1
            pool[hbm_pos(i, a.N, sp)] = (T)(x + 0.0);
            pool[hbm_pos(i + 1, a.N, sp)] = (T)(y + 0.0);
        } else {
            a.meta->withheld[buf] = x;
        }
    }
}

__global__ void k_init_meta(PoolMeta* meta, uint32_t buf, int seed_lfg) {
    if (!seed_lfg && meta->error) return;
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

cudaError_t launch_hbm_init(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                            uint32_t buf, int seed_lfg, void* scratch, cudaStream_t st) {
    const uint64_t nvals = (uint64_t)n_arrays * a.N;
    uint64_t* words = static_cast<uint64_t*>(scratch);
    k_init_meta<<<1, 1, 0, st>>>(a.meta, buf, seed_lfg);
    k_init_words<<<1, 256, 0, st>>>(a, nvals + 2, seed_lfg, words);
    const uint32_t grid = 148 * 4;
    if (dtype == WRNG_GPU_F64)
        k_init_bm<double><<<grid, 256, 0, st>>>(a, buf, nvals, words, seed_lfg);
    else
        k_init_bm<float><<<grid, 256, 0, st>>>(a, buf, nvals, words, seed_lfg);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return exact_sum(dtype, a, buf, 1, scratch, nvals, st);
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
// Persistent run of passes (C2): one launch executes up to kRunMax passes of
// one pool with a grid-wide barrier between passes, instead of one pass
// launch (+ one emission launch) each.  Every CTA stays resident (grid =
// SMs x occupancy, cooperative launch), walks the stored rows
// jlo = blockIdx.x, + gridDim.x, ... of each pass exactly as k_hbm_pass does
// for its kJlo rows, and after an emitting pass streams 64 x 64 transpose
// tiles of the new pool to the output (as k_hbm_emit_t).  Emission and the
// next pass only READ the new pool, so they share one barrier interval; the
// pass after that (which overwrites the emitted buffer) is behind the next
// barrier.  Same arithmetic, same op order, bit-identical to the per-pass
// kernels (wallace.cpp:113-137, 206-213).
// ---------------------------------------------------------------------------

// Grid barrier on a monotone arrival counter (zeroed before each launch):
// barrier e (1, 2, ...) completes when the counter reaches e * gridDim.x.
// Arrival is a fire-and-forget release reduction; no reset round trip.
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long& epoch) {
    __syncthreads();
    epoch += gridDim.x;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(bar), "l"(1ull)
                     : "memory");
        // relaxed polling (an acquire load invalidates L1 on every poll),
        // then one acquire fence
        unsigned long long v;
        do {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < epoch);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

#ifndef WG_RUN_EMIT_MODE
// where a refill's emission runs: 0 right after the barrier, 1 after the
// next pass's row loads are issued, 2 after the next pass's rows, tiles
// claimed dynamically (CTAs with fewer rows take more tiles)
#define WG_RUN_EMIT_MODE 0
#endif
constexpr uint32_t kRunThreads = 512;
constexpr uint32_t kRunTile = 64;
#ifndef WG_RUN_TILE_H
// k_hbm_run's emission tiles are kRunTile (jl: 512 B output runs) x kRunTileH
// (jh).  64 x 64 gives C2 1024 tiles = 3.46 per CTA (4 rounds, 86 % balance);
// 64 x 32 balances better (6.9 per CTA) but doubles the per-tile barriers and
// index work: C2 8.96 ms per step against 8.74-8.82 ms, so 64 stays.
#define WG_RUN_TILE_H 64
#endif
constexpr uint32_t kRunTileH = WG_RUN_TILE_H;
constexpr uint32_t kRunStages = 3;  // source-row buffers in flight per CTA

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
#ifndef WG_RUN_L2HINT  // 1: source rows evict_first, new pool rows evict_last
#define WG_RUN_L2HINT 0
#endif
// global -> shared bulk copy completing on an mbarrier (TMA, 1-D), with an
// L2 cache policy
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes,
                                              uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
template <typename T>
__device__ __forceinline__ void st_hint(T* p, T v, uint64_t pol) {
    if constexpr (sizeof(T) == 8)
        asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
                     : "memory");
    else
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol)
                     : "memory");
}
// global -> shared bulk copy completing on an mbarrier (TMA, 1-D)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

template <typename T, int NA>
__global__ void __launch_bounds__(kRunThreads, 2)
    k_hbm_run(KernelArgs a, wrng_gpu_params* params, HbmRun run, unsigned long long* gbar) {
    extern __shared__ __align__(128) unsigned char hsm[];
    const uint32_t N = a.N;
    const HbmSplit sp = hbm_split(N);
    const uint32_t R = 1u << sp.lr, C = 1u << sp.lc;
    T* stage = reinterpret_cast<T*>(hsm);                          // [S][NA][R]
    T(*tile)[kRunTile + 1] = reinterpret_cast<T(*)[kRunTile + 1]>(  // [64][65]
        hsm + (size_t)kRunStages * NA * R * sizeof(T));
    __shared__ __align__(8) uint64_t full[kRunStages];
    __shared__ double s_c0, s_c1, s_target, s_scale;
    __shared__ int s_err;
    __shared__ uint32_t s_tile[2];
    PoolMeta* meta = a.meta;
    const uint32_t t = threadIdx.x;
    const bool active_t = t < R;  // R < 512 only for forced-HBM small pools
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
    const uint32_t full_s = (uint32_t)__cvta_generic_to_shared(full);
    const uint32_t row_bytes = R * (uint32_t)sizeof(T);
    if (t == 0) {
        for (uint32_t k = 0; k < kRunStages; ++k) mbar_init(full_s + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint64_t pol_first = 0, pol_last = 0;
    if (WG_RUN_L2HINT) {
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    }
    uint32_t q = 0;  // source rows consumed by this CTA so far (stage q % S)
    unsigned long long epoch = 0;  // grid barrier target
    // Emission of a freshly regenerated pool (wallace.cpp:206-213), streamed
    // by all CTAs in 64 x 64 transpose tiles, the next tile's values loaded
    // while the current one is stored.  Where it runs: WG_RUN_EMIT_MODE
    // (default: right after the barrier that completes the pool).  `ctr`:
    // tiles claimed from an atomic counter instead of blockIdx-strided.
    auto emit = [&](const T* e_pool, uint64_t e_n, uint64_t e_off, unsigned* ctr) {
        // natural index m*N + jh*C + jl is stored at m*N + jl*R + jh
        const uint32_t tiles_h = (R + kRunTileH - 1) / kRunTileH;
        const uint32_t tiles_l = (C + kRunTile - 1) / kRunTile;
        const uint32_t ntiles = tiles_h * tiles_l * NA;
        char* outc = static_cast<char*>(a.out) + e_off * (a.out_f32 ? 4 : 8);
        const uint32_t tx = t & 31u, ty = t >> 5;  // 32 x 16
        // the next tile's values (4 or 8 per thread) load while this one is stored
        auto tile_at = [&](uint32_t tl, uint32_t& m, uint32_t& jh0, uint32_t& jl0) {
            m = tl / (tiles_h * tiles_l);
            const uint32_t rem = tl - m * tiles_h * tiles_l;
            jh0 = (rem % tiles_h) * kRunTileH;
            jl0 = (rem / tiles_h) * kRunTile;
        };
        constexpr uint32_t HN = kRunTileH / 32;  // 32-wide column groups of a tile
        auto load_tile = [&](uint32_t tl, T (&v)[4 * HN]) {
            uint32_t m, jh0, jl0;
            tile_at(tl, m, jh0, jl0);
            const T* pool = e_pool + (uint64_t)m * N;
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
#pragma unroll
                for (uint32_t h = 0; h < HN; ++h) {
                    const uint32_t jl = jl0 + ty + 16 * k, jh = jh0 + tx + 32 * h;
                    v[HN * k + h] = jl < C && jh < R ? pool[(uint64_t)jl * R + jh] : (T)0;
                }
        };
        // tiles: static (tl = blockIdx.x + k gridDim.x) or claimed from *ctr
        auto next = [&](uint32_t cur, int slot) -> uint32_t {
            if (!ctr) return cur + gridDim.x;
            if (t == 0) s_tile[slot] = atomicAdd(ctr, 1u);
            __syncthreads();
            return s_tile[slot];
        };
        int slot = 0;
        uint32_t tl = ctr ? next(0, slot) : blockIdx.x;
        T v[4 * HN];
        if (tl < ntiles) load_tile(tl, v);
        while (tl < ntiles) {
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
#pragma unroll
                for (uint32_t h = 0; h < HN; ++h) tile[ty + 16 * k][tx + 32 * h] = v[HN * k + h];
            __syncthreads();
            slot ^= 1;
            const uint32_t nt = next(tl, slot);
            if (nt < ntiles) load_tile(nt, v);
            uint32_t m, jh0, jl0;
            tile_at(tl, m, jh0, jl0);
            const uint64_t mbase = (uint64_t)m * N;
#pragma unroll
            for (uint32_t k = 0; k < kRunTileH; k += 16) {
                const uint32_t jh = jh0 + ty + k;
#pragma unroll
                for (uint32_t h = 0; h < kRunTile; h += 32) {
                    const uint32_t jl = jl0 + tx + h;
                    const uint64_t flat = mbase + (uint64_t)jh * C + jl;
                    if (jl < C && jh < R && flat < e_n)
                        put_out_cs(outc, flat, tile[tx + h][ty + k], a.out_f32, a.unit,
                                   a.mu, a.sigma);
                }
            }
            __syncthreads();
            tl = nt;
        }
    };
    const T* pend_pool = nullptr;  // emission owed by the previous pass
    uint64_t pend_n = 0, pend_off = 0;
    unsigned* pend_ctr = nullptr;
    unsigned* tile_ctr = reinterpret_cast<unsigned*>(gbar + 1);  // [kRunMax], zeroed per launch

    for (uint32_t i = 0; i < run.npass; ++i) {
        if (WG_RUN_EMIT_MODE == 0 && pend_n) {
            emit(pend_pool, pend_n, pend_off, nullptr);
            pend_n = 0;
        }
        const uint32_t src = run.src0 ^ (i & 1u), dst = src ^ 1u;
        const wrng_gpu_params prm = params[run.param0 + i];
        const T* spool = static_cast<const T*>(a.buf[src]);
        T* dpool = static_cast<T*>(a.buf[dst]);
        const uint32_t nrows = blockIdx.x < C ? (C - 1 - blockIdx.x) / gridDim.x + 1 : 0;
        const uint32_t q0 = q;
        // thread 0: the sources of this CTA's k-th row of the pass -> stage (q0 + k) % S
        auto issue = [&](uint32_t k) {
            const uint32_t jlo = blockIdx.x + k * gridDim.x;
            const uint32_t sb = (q0 + k) % kRunStages;
            const uint32_t bar = full_s + 8 * sb;
            mbar_expect_tx(bar, NA * row_bytes);
#pragma unroll
            for (int m = 0; m < NA; ++m) {
                const uint32_t srow = (prm.stride[m] * jlo + prm.offset[m]) & (C - 1);
                if (WG_RUN_L2HINT)
                    bulk_g2s_hint(stage_s + (sb * NA + m) * row_bytes,
                                  spool + (uint64_t)m * N + (uint64_t)srow * R, row_bytes, bar,
                                  pol_first);
                else
                    bulk_g2s(stage_s + (sb * NA + m) * row_bytes,
                             spool + (uint64_t)m * N + (uint64_t)srow * R, row_bytes, bar);
            }
        };
        if (t == 0) {
            // the previous pass's pool was written by other CTAs' generic
            // stores (ordered by the grid barrier); the async proxy reads it
            asm volatile("fence.proxy.async.global;" ::: "memory");
            for (uint32_t k = 0; k < nrows && k < kRunStages; ++k) issue(k);
            int err = meta->error ? -1 : 0;
            const double tracked = meta->tracked[src], withheld = meta->withheld[src];
            if (!err) {
                double scale, target;
                err = pass_scale(tracked, withheld, NA * N, a.mode, scale, target);
                if (!err) {
                    s_target = target;
                    s_scale = scale;
                    // regenerate folds the scale into the matrix (wallace.cpp:116-117)
                    s_c0 = NA == 2 ? prm.c * scale : (prm.variant ? scale : 0.5 * scale);
                    s_c1 = NA == 2 ? prm.s * scale : scale;
                }
            }
            s_err = err;
        }
        if (WG_RUN_EMIT_MODE == 1 && pend_n) {
            emit(pend_pool, pend_n, pend_off, nullptr);
            pend_n = 0;
        }
        __syncthreads();
        if (s_err) {  // every CTA reads the same state: all leave here together
            if (pend_n) emit(pend_pool, pend_n, pend_off, pend_ctr);  // the refill before stands
            // (rows already in flight complete into shared memory we abandon)
            if (t == 0)
                for (uint32_t k = 0; k < nrows && k < kRunStages; ++k)
                    mbar_wait(full_s + 8 * ((q + k) % kRunStages), ((q + k) / kRunStages) & 1u);
            if (s_err > 0 && blockIdx.x == 0 && t == 0) meta->error = s_err;
            return;
        }
        const T c0 = (T)s_c0, c1 = (T)s_c1;  // fp32 pools: rounded once
        const uint32_t variant = prm.variant;
        for (uint32_t k = 0; k < nrows; ++k, ++q) {
            const uint32_t jlo = blockIdx.x + k * gridDim.x;
            const uint32_t sb = q % kRunStages;
            mbar_wait(full_s + 8 * sb, (q / kRunStages) & 1u);
            if (active_t) {
                const T* rows = stage + (size_t)sb * NA * R;
                T g[NA];
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    const uint32_t sh = ((prm.stride[m] * jlo + prm.offset[m]) >> sp.lc) & (R - 1);
                    g[m] = rows[m * R + ((prm.stride[m] * t + sh) & (R - 1))];
                }
                T y[NA];
                if (NA == 2) {
                    y[0] = c0 * g[0] + c1 * g[NA > 1 ? 1 : 0];
                    y[NA > 1 ? 1 : 0] = c0 * g[NA > 1 ? 1 : 0] - c1 * g[0];
                } else {
                    const T a0 = g[0], a1 = g[NA > 1 ? 1 : 0], a2 = g[NA > 2 ? 2 : 0],
                            a3 = g[NA > 3 ? 3 : 0];
                    if (variant == 0) {
                        const T pp = a0 + a1, qq = a0 - a1, rr = a2 + a3, s = a2 - a3;
                        y[0] = c0 * (pp + rr);
                        y[NA > 1 ? 1 : 0] = c0 * (qq + s);
                        y[NA > 2 ? 2 : 0] = c0 * (pp - rr);
                        y[NA > 3 ? 3 : 0] = c0 * (qq - s);
                    } else {
                        const T tt = (T)0.5 * ((a0 + a1) + (a2 + a3));
                        y[0] = c0 * (tt - a0);
                        y[NA > 1 ? 1 : 0] = c0 * (tt - a1);
                        y[NA > 2 ? 2 : 0] = c0 * (tt - a2);
                        y[NA > 3 ? 3 : 0] = c0 * (tt - a3);
                    }
                }
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    if (WG_RUN_L2HINT)
                        st_hint(dpool + (uint64_t)m * N + (uint64_t)jlo * R + t, y[m], pol_last);
                    else
                        dpool[(uint64_t)m * N + (uint64_t)jlo * R + t] = y[m];
                }
                if (jlo == C - 1 && t == R - 1) meta->withheld[dst] = (double)y[NA - 1];
            }
            __syncthreads();  // stage sb fully read
            if (t == 0 && k + kRunStages < nrows) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(k + kRunStages);
            }
        }
        if (WG_RUN_EMIT_MODE == 2 && pend_n) {
            emit(pend_pool, pend_n, pend_off, pend_ctr);
            pend_n = 0;
        }
        const bool end = (run.end_mask >> i) & 1u;
        const uint64_t emit_n = run.emit_n[i];
        if (blockIdx.x == 0 && t == 0) {
            params[run.param0 + i].scale = s_scale;
            params[run.param0 + i].target_sumsq = s_target;
            meta->tracked[dst] = s_target;
            meta->active = dst;
            meta->pass_count += 1;
            meta->avail = end ? (uint64_t)NA * N - 1 - emit_n : 0;
        }
        grid_barrier(gbar, epoch);
        if (emit_n) {
            pend_pool = dpool;
            pend_n = emit_n;
            pend_off = run.out_off[i];
            pend_ctr = WG_RUN_EMIT_MODE == 2 ? tile_ctr + i : nullptr;
        }
    }
    if (pend_n) emit(pend_pool, pend_n, pend_off, pend_ctr);
}

// ---------------------------------------------------------------------------
// Dataflow variant of the persistent run (WRNG_GPU_HBM_FLOW=1): the same
// passes, rows, arithmetic and emission tiles as k_hbm_run, but no grid
// barrier.  In the transposed storage, destination row c of pass i reads
// exactly one storage row per array, s_m(c) = (a_m c + g_m) mod C, of pass
// i-1's output; and the buffer row c it overwrites was read in pass i-1 by
// exactly the rows c'_m with s_m(c'_m) = c.  So each row waits only for
// those 8 rows of the previous pass (per-row epoch flags, release/acquire),
// and for the emission tiles that read its buffer slot two passes earlier
// (per 64-row group counters).  A CTA emits its tiles of an emitting pass
// after its rows of the NEXT pass, when those tiles' rows are long done.
// Deadlock-free: a CTA enters pass i+1 only after its rows of pass i, so the
// least advanced CTA only waits for rows of passes every CTA has finished.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void flag_release(unsigned* f, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ void flag_add_release(unsigned* f, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ void flag_wait(const unsigned* f, unsigned v) {
    unsigned x;
    do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
    } while (x < v);
}
// inverse of an odd a modulo 2^32 (Newton: 5 steps from 3 correct bits)
__device__ __forceinline__ uint32_t inv_odd(uint32_t a) {
    uint32_t x = a;
#pragma unroll
    for (int k = 0; k < 5; ++k) x *= 2u - a * x;
    return x;
}

template <typename T, int NA>
__global__ void __launch_bounds__(kRunThreads, 2)
    k_hbm_flow(KernelArgs a, wrng_gpu_params* params, HbmRun run, unsigned long long* gbar) {
    extern __shared__ __align__(128) unsigned char hsm[];
    const uint32_t N = a.N;
    const HbmSplit sp = hbm_split(N);
    const uint32_t R = 1u << sp.lr, C = 1u << sp.lc;
    T* stage = reinterpret_cast<T*>(hsm);                          // [S][NA][R]
    T(*tile)[kRunTile + 1] = reinterpret_cast<T(*)[kRunTile + 1]>(  // [64][65]
        hsm + (size_t)kRunStages * NA * R * sizeof(T));
    __shared__ __align__(8) uint64_t full[kRunStages];
    __shared__ double s_c0, s_c1, s_target, s_scale, s_tracked;
    __shared__ int s_err;
    PoolMeta* meta = a.meta;
    unsigned* rowflag = reinterpret_cast<unsigned*>(gbar + kRunBarWords);  // [C]: passes done
    unsigned* emitcnt = rowflag + C;  // [ceil(C/64)]: emission tiles read, per 64-row group
    // withheld value of each pass of the launch (a later pass of the same
    // buffer may overwrite meta->withheld before a slow CTA has read it)
    double* whslot = reinterpret_cast<double*>(gbar + kRunBarWords + kRunFlowRowWords);
    const uint32_t t = threadIdx.x;
    const bool active_t = t < R;
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
    const uint32_t full_s = (uint32_t)__cvta_generic_to_shared(full);
    const uint32_t row_bytes = R * (uint32_t)sizeof(T);
    const uint32_t tiles_h = (R + kRunTile - 1) / kRunTile;
    const uint32_t tiles_per_group = tiles_h * NA;  // tiles reading one 64-row group
    if (t == 0) {
        for (uint32_t k = 0; k < kRunStages; ++k) mbar_init(full_s + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_tracked = meta->tracked[run.src0];
    }
    __syncthreads();
    uint32_t q = 0;
    // tiles of the emission of pass `ip` (pool e_pool), this CTA's share;
    // `eidx` counts the emissions of this launch before it
    auto emit = [&](const T* e_pool, uint64_t e_n, uint64_t e_off, uint32_t e_pass) {
        const uint32_t tiles_l = (C + kRunTile - 1) / kRunTile;
        const uint32_t ntiles = tiles_h * tiles_l * NA;
        char* outc = static_cast<char*>(a.out) + e_off * (a.out_f32 ? 4 : 8);
        const uint32_t tx = t & 31u, ty = t >> 5;
        for (uint32_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
            const uint32_t m = tl / (tiles_h * tiles_l);
            const uint32_t rem = tl - m * tiles_h * tiles_l;
            const uint32_t jh0 = (rem % tiles_h) * kRunTile, jl0 = (rem / tiles_h) * kRunTile;
            const T* pool = e_pool + (uint64_t)m * N;
            if (t < kRunTile && jl0 + t < C) {  // the tile's 64 rows of the emitted pass
                flag_wait(rowflag + jl0 + t, e_pass + 1);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            __syncthreads();
            T v[8];
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
#pragma unroll
                for (uint32_t h = 0; h < 2; ++h) {
                    const uint32_t jl = jl0 + ty + 16 * k, jh = jh0 + tx + 32 * h;
                    v[2 * k + h] = jl < C && jh < R ? pool[(uint64_t)jl * R + jh] : (T)0;
                }
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
#pragma unroll
                for (uint32_t h = 0; h < 2; ++h) tile[ty + 16 * k][tx + 32 * h] = v[2 * k + h];
            __syncthreads();
            if (t == 0) flag_add_release(emitcnt + jl0 / kRunTile, 1u);  // the tile's reads are done
            const uint64_t mbase = (uint64_t)m * N;
#pragma unroll
            for (uint32_t k = 0; k < kRunTile; k += 16) {
                const uint32_t jh = jh0 + ty + k;
#pragma unroll
                for (uint32_t h = 0; h < kRunTile; h += 32) {
                    const uint32_t jl = jl0 + tx + h;
                    const uint64_t flat = mbase + (uint64_t)jh * C + jl;
                    if (jl < C && jh < R && flat < e_n)
                        put_out_cs(outc, flat, tile[tx + h][ty + k], a.out_f32, a.unit,
                                   a.mu, a.sigma);
                }
            }
            __syncthreads();
        }
    };
    const T* pend_pool = nullptr;  // emission owed (pass before the current one)
    uint64_t pend_n = 0, pend_off = 0;
    uint32_t pend_pass = 0;
    uint32_t emissions = 0;     // emissions of this launch so far (any CTA's schedule)
    uint32_t emit_of[2] = {0xFFFFFFFFu, 0xFFFFFFFFu};  // per buffer: index of the emission reading it

    for (uint32_t i = 0; i < run.npass; ++i) {
        const uint32_t src = run.src0 ^ (i & 1u), dst = src ^ 1u;
        const wrng_gpu_params prm = params[run.param0 + i];
        const wrng_gpu_params pprev = i ? params[run.param0 + i - 1] : prm;
        const T* spool = static_cast<const T*>(a.buf[src]);
        T* dpool = static_cast<T*>(a.buf[dst]);
        const uint32_t nrows = blockIdx.x < C ? (C - 1 - blockIdx.x) / gridDim.x + 1 : 0;
        const uint32_t q0 = q;
        // buffer dst was last read by an emission (of pass i-2): wait for its tiles
        const uint32_t e_dst = emit_of[dst];
        uint32_t ainv[NA];
#pragma unroll
        for (int m = 0; m < NA; ++m) ainv[m] = inv_odd(pprev.stride[m]);
        // thread 0: row k's dependencies, then its sources -> stage (q0 + k) % S
        auto issue = [&](uint32_t k) {
            const uint32_t jlo = blockIdx.x + k * gridDim.x;
            // RAW: the source rows of pass i-1; WAR: the pass i-1 rows that
            // read row jlo of dst, and the emission tiles that read its group.
            // All polled together: one round trip once they are done.
            const unsigned* fa[2 * NA + 1];
            unsigned ft[2 * NA + 1];
            int nf = 0;
            if (i > 0) {
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    fa[nf] = rowflag + ((prm.stride[m] * jlo + prm.offset[m]) & (C - 1));
                    ft[nf++] = i;
                    fa[nf] = rowflag + ((ainv[m] * (jlo - pprev.offset[m])) & (C - 1));
                    ft[nf++] = i;
                }
            }
            if (e_dst != 0xFFFFFFFFu) {
                fa[nf] = emitcnt + jlo / kRunTile;
                ft[nf++] = (e_dst + 1) * tiles_per_group;
            }
            for (bool ok = nf == 0; !ok;) {
                unsigned x[2 * NA + 1];
#pragma unroll
                for (int f = 0; f < 2 * NA + 1; ++f)
                    if (f < nf)
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];"
                                     : "=r"(x[f])
                                     : "l"(fa[f])
                                     : "memory");
                ok = true;
#pragma unroll
                for (int f = 0; f < 2 * NA + 1; ++f)
                    if (f < nf) ok = ok && x[f] >= ft[f];
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const uint32_t sb = (q0 + k) % kRunStages;
            const uint32_t bar = full_s + 8 * sb;
            mbar_expect_tx(bar, NA * row_bytes);
#pragma unroll
            for (int m = 0; m < NA; ++m) {
                const uint32_t srow = (prm.stride[m] * jlo + prm.offset[m]) & (C - 1);
                bulk_g2s(stage_s + (sb * NA + m) * row_bytes,
                         spool + (uint64_t)m * N + (uint64_t)srow * R, row_bytes, bar);
            }
        };
        if (t == 0) {
            int err = meta->error ? -1 : 0;
            // the pool's withheld value comes from pass i-1's last row
            if (i > 0) {
                flag_wait(rowflag + (C - 1), i);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            const double tracked = s_tracked;
            double withheld;
            asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];"
                         : "=d"(withheld)
                         : "l"(i > 0 ? &whslot[i - 1] : &meta->withheld[src])
                         : "memory");
            if (!err) {
                double scale, target;
                err = pass_scale(tracked, withheld, NA * N, a.mode, scale, target);
                if (!err) {
                    s_target = target;
                    s_scale = scale;
                    s_c0 = NA == 2 ? prm.c * scale : (prm.variant ? scale : 0.5 * scale);
                    s_c1 = NA == 2 ? prm.s * scale : scale;
                }
            }
            s_err = err;
            if (!err)
                for (uint32_t k = 0; k < nrows && k < kRunStages; ++k) issue(k);
        }
        __syncthreads();
        if (s_err) {
            if (pend_n) emit(pend_pool, pend_n, pend_off, pend_pass);
            if (s_err > 0 && blockIdx.x == 0 && t == 0) meta->error = s_err;
            return;
        }
        const T c0 = (T)s_c0, c1 = (T)s_c1;
        const uint32_t variant = prm.variant;
        for (uint32_t k = 0; k < nrows; ++k, ++q) {
            const uint32_t jlo = blockIdx.x + k * gridDim.x;
            const uint32_t sb = q % kRunStages;
            mbar_wait(full_s + 8 * sb, (q / kRunStages) & 1u);
            if (active_t) {
                const T* rows = stage + (size_t)sb * NA * R;
                T g[NA];
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    const uint32_t sh = ((prm.stride[m] * jlo + prm.offset[m]) >> sp.lc) & (R - 1);
                    g[m] = rows[m * R + ((prm.stride[m] * t + sh) & (R - 1))];
                }
                T y[NA];
                if (NA == 2) {
                    y[0] = c0 * g[0] + c1 * g[NA > 1 ? 1 : 0];
                    y[NA > 1 ? 1 : 0] = c0 * g[NA > 1 ? 1 : 0] - c1 * g[0];
                } else {
                    const T a0 = g[0], a1 = g[NA > 1 ? 1 : 0], a2 = g[NA > 2 ? 2 : 0],
                            a3 = g[NA > 3 ? 3 : 0];
                    if (variant == 0) {
                        const T pp = a0 + a1, qq = a0 - a1, rr = a2 + a3, s = a2 - a3;
                        y[0] = c0 * (pp + rr);
                        y[NA > 1 ? 1 : 0] = c0 * (qq + s);
                        y[NA > 2 ? 2 : 0] = c0 * (pp - rr);
                        y[NA > 3 ? 3 : 0] = c0 * (qq - s);
                    } else {
                        const T tt = (T)0.5 * ((a0 + a1) + (a2 + a3));
                        y[0] = c0 * (tt - a0);
                        y[NA > 1 ? 1 : 0] = c0 * (tt - a1);
                        y[NA > 2 ? 2 : 0] = c0 * (tt - a2);
                        y[NA > 3 ? 3 : 0] = c0 * (tt - a3);
                    }
                }
#pragma unroll
                for (int m = 0; m < NA; ++m) dpool[(uint64_t)m * N + (uint64_t)jlo * R + t] = y[m];
                if (jlo == C - 1 && t == R - 1) {
                    meta->withheld[dst] = (double)y[NA - 1];
                    whslot[i] = (double)y[NA - 1];
                }
            }
            __syncthreads();  // stage sb fully read, row jlo stored
            if (t == 0) {
                flag_release(rowflag + jlo, i + 1);  // row done: its reads and writes
                if (k + kRunStages < nrows) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(k + kRunStages);
                }
            }
        }
        // the previous emitting pass's tiles: its rows are done by now
        if (pend_n) {
            emit(pend_pool, pend_n, pend_off, pend_pass);
            pend_n = 0;
        }
        const bool end = (run.end_mask >> i) & 1u;
        const uint64_t emit_n = run.emit_n[i];
        if (blockIdx.x == 0 && t == 0) {
            params[run.param0 + i].scale = s_scale;
            params[run.param0 + i].target_sumsq = s_target;
            meta->tracked[dst] = s_target;
            meta->active = dst;
            meta->pass_count += 1;
            meta->avail = end ? (uint64_t)NA * N - 1 - emit_n : 0;
        }
        if (t == 0) s_tracked = s_target;  // regenerate sets tracked = target
        if (emit_n) {
            pend_pool = dpool;
            pend_n = emit_n;
            pend_off = run.out_off[i];
            pend_pass = i;
            emit_of[dst] = emissions++;
        } else {
            emit_of[dst] = 0xFFFFFFFFu;
        }
        __syncthreads();
    }
    if (pend_n) emit(pend_pool, pend_n, pend_off, pend_pass);
}

static const bool g_hbm_flow = std::getenv("WRNG_GPU_HBM_FLOW") != nullptr;

template <typename T, int NA>
static cudaError_t hbm_run_go(const KernelArgs& a, wrng_gpu_params* params, const HbmRun& run,
                              unsigned long long* gbar, cudaStream_t st) {
    const HbmSplit sp = hbm_split(a.N);
    const uint32_t R = 1u << sp.lr;
    const size_t smem = (size_t)kRunStages * NA * R * sizeof(T) +
                        (size_t)kRunTile * (kRunTile + 1) * sizeof(T);
    // attribute and occupancy for the largest row length (R = 512), so one
    // cached grid size is co-resident for every pool size
    const size_t smem_max = (size_t)kRunStages * NA * 512 * sizeof(T) +
                            (size_t)kRunTile * (kRunTile + 1) * sizeof(T);
    auto kern = g_hbm_flow ? k_hbm_flow<T, NA> : k_hbm_run<T, NA>;
    static int occ_cache[2][2][2][64] = {};  // [flow][dtype][n4][device] CTAs in the grid
    int dev = 0;
    cudaGetDevice(&dev);
    int& occ = occ_cache[g_hbm_flow][sizeof(T) == 8][NA == 4][dev & 63];
    if (occ == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem_max);
        if (e != cudaSuccess) return e;
        int nb = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kRunThreads, smem_max);
        if (e != cudaSuccess) return e;
        int sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        occ = nb * sms;
        if (occ <= 0) return cudaErrorLaunchOutOfResources;
    }
    // barrier counter + the emission tile counters of this launch
    cudaError_t e = cudaMemsetAsync(
        gbar, 0, (kRunBarWords + (g_hbm_flow ? kRunFlowWords : 0)) * sizeof(unsigned long long),
        st);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)occ);
    cfg.blockDim = dim3(kRunThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeCooperative;  // co-residency for grid_barrier
    attr[na].val.cooperative = 1;
    ++na;
    if (a.l2_bytes) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = a.l2_base;
        attr[na].val.accessPolicyWindow.num_bytes = a.l2_bytes;
        attr[na].val.accessPolicyWindow.hitRatio = a.l2_hit;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, a, params, run, gbar);
}

cudaError_t launch_hbm_run(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                           wrng_gpu_params* params, const HbmRun& run, unsigned long long* gbar,
                           cudaStream_t st) {
    if (run.npass == 0) return cudaSuccess;
    if (dtype == WRNG_GPU_F64)
        return n_arrays == 2 ? hbm_run_go<double, 2>(a, params, run, gbar, st)
                             : hbm_run_go<double, 4>(a, params, run, gbar, st);
    return n_arrays == 2 ? hbm_run_go<float, 2>(a, params, run, gbar, st)
                         : hbm_run_go<float, 4>(a, params, run, gbar, st);
}

}  // namespace wg

