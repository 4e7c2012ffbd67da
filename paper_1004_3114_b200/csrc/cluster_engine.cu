// Cluster engine: ONE pool spread over a thread-block cluster of K CTAs on K
// SMs (BASELINE.json C1: the reference's single 4 x 4096 fp64 pool, where a
// single CTA is latency-bound).  CTA r of the cluster owns columns
// [r*NC, (r+1)*NC) of every array (NC = N / K): it keeps them in its shared
// memory, gathers x_m[(a_m j + g_m) mod N] for its columns from whichever
// CTA owns them through distributed shared memory (ld.shared::cluster), and
// writes its new columns in place after a cluster barrier.  The arithmetic
// is the smem engine's, operation for operation (wallace.cpp:113-137,
// docs/n4_spec.md §3), so the stream is bit-identical.
//
// Per pass:  params (drawn one pass ahead by warp 0 of rank 0, read by all
// ranks from rank 0's control block) -> gathers (DSMEM) + unscaled
// transform -> cluster barrier -> scale, store, emit (warp stores) ->
// cluster barrier.  The previous withheld value lives in the control block
// of rank K-1 (it owns column N-1 of the last array); every rank derives
// the chi-squared scale from (tracked, withheld) itself (wallace.cpp:59-69).
// Drift audits (wallace.cpp:225-234) gather the pool into rank 0's staging
// buffer in flat order and run the exact ordered sum there (common.cuh).
//
// Only fills (OP_FILL) without restarts take this path; every other
// operation runs on the single-CTA smem engine over the same device state.
//
// Opt-in (WRNG_GPU_CLUSTER=1): measured on C1 it is SLOWER than one CTA
// (4.9 vs 3.6 ms per 2^24): the per-lane 8-byte DSMEM gathers are
// request-bound (~4 B/clk per SM against 17-21 B/clk for coalesced DSMEM
// traffic), and a release cluster barrier waits for the emission stores.
#include "common.cuh"

namespace wg {

template <typename T, int NA, int LOGN, int K>
struct CShape {
    static constexpr uint32_t N = 1u << LOGN;
    static constexpr uint32_t NC = N / K;                  // columns per CTA
    static constexpr uint32_t NTH = NC < 256 ? NC : 256;   // threads per CTA
    static constexpr uint32_t JC = NC / NTH;               // columns per thread
    static constexpr uint32_t LOGNC = LOGN - (K == 2 ? 1 : K == 4 ? 2 : K == 8 ? 3 : 4);
    static constexpr uint64_t NVALS = (uint64_t)NA * N;
    static constexpr uint64_t CAP = NVALS - 1;
    static constexpr uint32_t TAB_OFF = 0;
    static constexpr uint32_t WBUF_OFF = 608 * 8;
    static constexpr uint32_t CTL_OFF = WBUF_OFF + 256 * 8;
    static constexpr uint32_t SHARE_OFF = CTL_OFF + 256;
    static constexpr uint32_t SHARE_BYTES = NA * NC * (uint32_t)sizeof(T);
    static constexpr uint32_t STAGE_OFF = SHARE_OFF + SHARE_BYTES;
    static constexpr uint32_t SCR_OFF = STAGE_OFF + (uint32_t)(NVALS * sizeof(T));
    static constexpr uint32_t SUM_CHUNKS = NTH;
    static constexpr uint32_t BYTES = SCR_OFF + sum_scratch_bytes(SUM_CHUNKS);
    static_assert(sizeof(Ctl) <= 256, "control block");
    static_assert((1u << LOGNC) == NC, "K is a power of two");
};

extern __shared__ __align__(16) unsigned char c_sm[];

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
#ifndef WG_CL_SYNC
#define WG_CL_SYNC 0
#endif
__device__ __forceinline__ void cluster_sync() {
#if WG_CL_SYNC == 1
    asm volatile(
        "fence.acq_rel.cluster;\n\t"
        "barrier.cluster.arrive.relaxed.aligned;\n\t"
        "barrier.cluster.wait.aligned;" ::: "memory");
#elif WG_CL_SYNC == 2
    asm volatile(
        "barrier.cluster.arrive.relaxed.aligned;\n\t"
        "barrier.cluster.wait.aligned;" ::: "memory");
#else
    asm volatile(
        "barrier.cluster.arrive.release.aligned;\n\t"
        "barrier.cluster.wait.acquire.aligned;" ::: "memory");
#endif
}
template <typename T>
__device__ __forceinline__ T ld_cl(uint32_t a) {
    T v;
    if constexpr (sizeof(T) == 8)
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    else
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_cl_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ double ld_cl_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
template <typename T>
__device__ __forceinline__ void st_cl(uint32_t a, T v) {
    if constexpr (sizeof(T) == 8)
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
    else
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

template <typename T, int NA, int LOGN, int K>
__global__ void __launch_bounds__(CShape<T, NA, LOGN, K>::NTH, 1)
    k_cluster_fill(const KernelArgs a) {
    using S = CShape<T, NA, LOGN, K>;
    constexpr uint32_t N = S::N, NC = S::NC, NTH = S::NTH, JC = S::JC;
    constexpr uint64_t NVALS = S::NVALS, CAP = S::CAP;

    uint64_t* tab = reinterpret_cast<uint64_t*>(c_sm + S::TAB_OFF);
    uint64_t* wbuf = reinterpret_cast<uint64_t*>(c_sm + S::WBUF_OFF);
    Ctl* ctl = reinterpret_cast<Ctl*>(c_sm + S::CTL_OFF);
    T* share = reinterpret_cast<T*>(c_sm + S::SHARE_OFF);
    T* stage = reinterpret_cast<T*>(c_sm + S::STAGE_OFF);
    const uint32_t sm_base = (uint32_t)__cvta_generic_to_shared(c_sm);
    const uint32_t share_s = sm_base + S::SHARE_OFF;
    const uint32_t ctl_s = sm_base + S::CTL_OFF;

    const uint32_t tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const uint32_t p = blockIdx.x / K;  // pool
    const uint32_t col0 = rank * NC;
    PoolMeta* meta = a.meta + p;
    LfgState* lg = a.lfg + p;
    // remote addresses: rank 0's control block (params, tracked, error) and
    // rank K-1's (withheld)
    const uint32_t ctl0 = mapa(ctl_s, 0), ctlw = mapa(ctl_s, K - 1);
    const uint32_t off_cur = (uint32_t)offsetof(Ctl, cur), off_cur2 = (uint32_t)offsetof(Ctl, cur2);
    const uint32_t off_tr = (uint32_t)offsetof(Ctl, tracked);
    const uint32_t off_wh = (uint32_t)offsetof(Ctl, withheld);
    const uint32_t off_err = (uint32_t)offsetof(Ctl, error);

    if (meta->error) return;  // sticky device error (all ranks agree)

    // ---- load state ----------------------------------------------------------
    uint64_t pc = meta->pass_count, avail = meta->avail, emitted = meta->emitted;
    uint32_t act = meta->active;
    if (rank == 0)
        for (uint32_t i = tid; i < kTable; i += NTH) tab[i] = lg->table[i];
    if (tid == 0) {
        ctl->r = lg->r;
        ctl->draws = lg->draws;
        ctl->tracked = meta->tracked[act];
        ctl->withheld = meta->withheld[act];
        ctl->error = 0;
    }
    {
        const T* src = static_cast<const T*>(a.buf[act]) + (uint64_t)p * NVALS;
        for (uint32_t i = tid; i < NA * NC; i += NTH) {
            const uint32_t m = i / NC, jl = i - m * NC;
            share[i] = src[(uint64_t)m * N + col0 + jl];
        }
    }
    __syncthreads();
    cluster_sync();

    const uint64_t len = a.lay.len_base + (p < a.lay.len_extra ? 1 : 0);
    const uint64_t out_base =
        (uint64_t)p * a.lay.off_stride + (p < a.lay.off_extra ? p : a.lay.off_extra);
    const uint32_t f = a.f, mode = a.mode;
    const uint32_t esz = a.out_f32 ? 4u : 8u;
    char* outc = static_cast<char*>(a.out);
    PeriodCounter drift;
    drift.init(a.drift, pc);
    double tracked = ctl->tracked;
    int err = 0;

    uint64_t done = 0;
    if (avail > 0 && len > 0) {  // leftover of the live pool: flat [pos, pos + take)
        const uint64_t take = umin64(len, avail), pos = CAP - avail;
        char* o = outc + out_base * esz;
        for (uint32_t i = tid; i < NA * NC; i += NTH) {
            const uint32_t m = i / NC, jl = i - m * NC;
            const uint64_t flat = (uint64_t)m * N + col0 + jl;
            if (flat >= pos && flat < pos + take)
                put_out(o, flat - pos, share[i], a.out_f32, a.unit, a.mu, a.sigma);
        }
        done = take;
        avail -= take;
    }
    uint64_t rem = len - done;
    const uint64_t total_passes = (rem + CAP - 1) / CAP * f;
    uint64_t pass_i = 0;
    int slot = 0;
    // rank 0 draws the first pass's words
    if (rank == 0 && tid < 32 && total_passes) draw_pass_params_warp<NA>(tab, ctl, wbuf, N, 0);
    cluster_sync();

    while (!err && done < len) {
        const bool will_drift = drift.will_cross(f);
        const uint32_t emit_n = (uint32_t)umin64(len - done, CAP);
        char* out_p = outc + (out_base + done) * esz;
        for (uint32_t it = 0; it < f; ++it) {
            ++pass_i;
            const bool lastp = it + 1 == f, last_launch = pass_i == total_passes;
            const uint32_t en = lastp ? emit_n : 0u;
            // ---- parameters and scale (every rank, identical inputs) ----------
            const uint32_t pb = ctl0 + (slot ? off_cur2 : off_cur);
            uint32_t stride[NA], offset[NA];
#pragma unroll
            for (int m = 0; m < NA; ++m) {
                stride[m] = ld_cl_u32(pb + 4u * m);
                offset[m] = ld_cl_u32(pb + 16u + 4u * m);
            }
            const uint32_t variant = ld_cl_u32(pb + 32u);
            const double pc_c = ld_cl_f64(pb + 40u), pc_s = ld_cl_f64(pb + 48u);
            const double withheld = ld_cl_f64(ctlw + off_wh);
            double scale = 0.0, target = 0.0;
            const int e = pass_scale(tracked, withheld, (uint32_t)NVALS, mode, scale, target);
            if (e) {
                err = e;
                break;
            }
            const double c0d = NA == 2 ? pc_c * scale : (variant ? scale : 0.5 * scale);
            const double c1d = NA == 2 ? pc_s * scale : scale;
            const T c0 = (T)c0d, c1 = (T)c1d;  // fp32 pools: rounded once (n4_spec §4)
            if (last_launch) {
                // the pre-pass pool becomes the inactive buffer (wallace.cpp:170-174)
                T* prev = static_cast<T*>(a.buf[act]) + (uint64_t)p * NVALS;
                for (uint32_t i = tid; i < NA * NC; i += NTH) {
                    const uint32_t m = i / NC, jl = i - m * NC;
                    prev[(uint64_t)m * N + col0 + jl] = share[i];
                }
                if (rank == 0 && tid == 0) {
                    meta->tracked[act] = tracked;
                    meta->withheld[act] = withheld;
                }
            }
            // rank 0 draws the next pass's words into the other slot
            if (rank == 0 && tid < 32 && !last_launch)
                draw_pass_params_warp<NA>(tab, ctl, wbuf, N, slot ^ 1);
            // ---- gathers (DSMEM) + unscaled transform --------------------------
            T u[NA][JC];
#pragma unroll
            for (uint32_t q = 0; q < JC; ++q) {
                const uint32_t j = col0 + tid + q * NTH;
                T g[NA];
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    const uint32_t i = (stride[m] * j + offset[m]) & (N - 1);
                    const uint32_t own = i >> S::LOGNC, off = i & (NC - 1);
                    g[m] = ld_cl<T>(mapa(share_s + (m * NC + off) * (uint32_t)sizeof(T), own));
                }
                if constexpr (NA == 4) {
                    if (variant == 0) {  // (1/2) H4
                        const T pp = g[0] + g[1], qq = g[0] - g[1], r = g[2] + g[3],
                                s = g[2] - g[3];
                        u[0][q] = pp + r;
                        u[1][q] = qq + s;
                        u[2][q] = pp - r;
                        u[3][q] = qq - s;
                    } else {  // (1/2) J - I
                        const T t = (T)0.5 * ((g[0] + g[1]) + (g[2] + g[3]));
                        u[0][q] = t - g[0];
                        u[1][q] = t - g[1];
                        u[2][q] = t - g[2];
                        u[3][q] = t - g[3];
                    }
                } else {
                    u[0][q] = g[0];
                    u[1][q] = g[1];
                }
            }
            cluster_sync();  // every rank's gathers are done: rewrite in place
            // ---- scale, store, emit ------------------------------------------
#pragma unroll
            for (uint32_t q = 0; q < JC; ++q) {
                const uint32_t jl = tid + q * NTH, j = col0 + jl;
                T y[NA];
                if constexpr (NA == 4) {
#pragma unroll
                    for (int m = 0; m < NA; ++m) y[m] = c0 * u[m][q];
                } else {
                    // dst.x = kc*xs + ks*ys ; dst.y = kc*ys - ks*xs (wallace.cpp:130-131)
                    const T xs = u[0][q], ys = u[1][q];
                    y[0] = c0 * xs + c1 * ys;
                    y[1] = c0 * ys - c1 * xs;
                }
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    share[m * NC + jl] = y[m];
                    const uint64_t flat = (uint64_t)m * N + j;
#if !WG_EXP_NOSTG
                    if (flat < en) put_out(out_p, flat, y[m], a.out_f32, a.unit, a.mu, a.sigma);
#endif
                }
                if (j == N - 1) ctl->withheld = (double)y[NA - 1];  // rank K-1 (wallace.cpp:136)
            }
            tracked = target;  // wallace.cpp:135
            act ^= 1u;
            slot ^= 1;
            ++pc;
            cluster_sync();
        }
        if (err) break;
        drift.advance(f);
        avail = CAP;
        if (will_drift) {
            // Pool::direct_sumsq over the flat pool (wallace.cpp:13-18, 225-234)
            const uint32_t stage0 = mapa(sm_base + S::STAGE_OFF, 0);
            for (uint32_t i = tid; i < NA * NC; i += NTH) {
                const uint32_t m = i / NC, jl = i - m * NC;
                st_cl<T>(stage0 + (uint32_t)(((uint64_t)m * N + col0 + jl) * sizeof(T)), share[i]);
            }
            cluster_sync();
            if (rank == 0) {
                const double rec = exact_sumsq_cta<T>(stage, (uint32_t)NVALS,
                                                      c_sm + S::SCR_OFF, S::SUM_CHUNKS);
                if (tid == 0) {
                    const double rel = fabs(rec / tracked - 1.0);
                    if (!(rel <= 1e-3))
                        ctl->error = WRNG_GPU_ECORRUPT;
                    else
                        ctl->tracked = rec;
                }
            }
            cluster_sync();
            err = (int)ld_cl_u32(ctl0 + off_err);
            if (!err) tracked = ld_cl_f64(ctl0 + off_tr);
            cluster_sync();  // rank 0's control block is rewritten later
            if (err) break;
        }
        done += emit_n;
        avail -= emit_n;
    }
    if (!err) emitted += len;

    // ---- write back ------------------------------------------------------------
    {
        T* dst = static_cast<T*>(a.buf[act]) + (uint64_t)p * NVALS;
        for (uint32_t i = tid; i < NA * NC; i += NTH) {
            const uint32_t m = i / NC, jl = i - m * NC;
            dst[(uint64_t)m * N + col0 + jl] = share[i];
        }
    }
    const double wh_final = ld_cl_f64(ctlw + off_wh);
    if (rank == 0) {
        for (uint32_t i = tid; i < kTable; i += NTH) lg->table[i] = tab[i];
        if (tid == 0) {
            lg->r = ctl->r;
            lg->draws = ctl->draws;
            meta->tracked[act] = tracked;
            meta->withheld[act] = wh_final;
            meta->active = act;
            meta->pass_count = pc;
            meta->avail = avail;
            meta->emitted = emitted;
            meta->error = (uint32_t)err;
        }
    }
    cluster_sync();  // no rank exits while others may still read its memory
}

template <typename T, int NA, int LOGN>
static cudaError_t go_cluster(const KernelArgs& a, cudaStream_t st) {
    constexpr int K = 8;
    using S = CShape<T, NA, LOGN, K>;
    auto kern = k_cluster_fill<T, NA, LOGN, K>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.pools * K);
    cfg.blockDim = dim3(S::NTH);
    cfg.dynamicSmemBytes = S::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename T, int NA>
static cudaError_t dispatch_cluster(const KernelArgs& a, cudaStream_t st) {
    switch (a.N) {
        case 1u << 11: return go_cluster<T, NA, 11>(a, st);
        case 1u << 12: return go_cluster<T, NA, 12>(a, st);
        case 1u << 13:
            if constexpr (NA * (1u << 13) * sizeof(T) <= 128 * 1024) return go_cluster<T, NA, 13>(a, st);
            return cudaErrorInvalidValue;
        case 1u << 14:
            if constexpr (NA * (1u << 14) * sizeof(T) <= 128 * 1024) return go_cluster<T, NA, 14>(a, st);
            return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

bool cluster_engine_fits(uint32_t n_arrays, uint32_t dtype, uint32_t N, uint32_t pools) {
    const uint32_t es = dtype == WRNG_GPU_F64 ? 8 : 4;
    return pools <= 18 && N >= (1u << 11) && N <= (1u << 14) &&
           (uint64_t)n_arrays * N * es <= 128 * 1024;
}

cudaError_t launch_cluster(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                           cudaStream_t st) {
    if (dtype == WRNG_GPU_F64)
        return n_arrays == 2 ? dispatch_cluster<double, 2>(a, st)
                             : dispatch_cluster<double, 4>(a, st);
    return n_arrays == 2 ? dispatch_cluster<float, 2>(a, st) : dispatch_cluster<float, 4>(a, st);
}

}  // namespace wg
