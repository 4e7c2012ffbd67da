// Shared-memory engine: one CTA per pool, the pool resident in shared memory
// for the whole fill call (BASELINE.json configs C1, C3, C4, C5).
//
// One regeneration pass (wallace.cpp:113-137, in the naive modular form the
// reference pins bit-identical to its segmented loop,
// tests/test_wallace_core.cpp:203-217) runs IN PLACE in two phases separated
// by one barrier:
//   B  gather x_m[(a_m j + g_m) mod N] for this thread's columns j = tid +
//      k*NTH (lane-consecutive: odd strides hit 32 distinct banks) and form
//      the unscaled transform — for n = 4 the scale multiply is the last
//      rounding of every element (docs/n4_spec.md §3), so the Hadamard /
//      (J/2 - I) sums need no scale.  Every thread derives this pass's
//      chi-squared scale from the broadcast (tracked, withheld)
//      (wallace.cpp:62-65); warp 0 (all warps compute, warp 0 stores) draws
//      the next pass's uniform words (wallace.cpp:54-58).
//   C  multiply by the scale and store back in place.  On the last pass of
//      a full refill the pool in shared memory is the emitted sequence, and
//      thread 0 hands it to the bulk-copy engine (cp.async.bulk) after the
//      pass's final barrier (wallace.cpp:206-213); partial windows and
//      non-unit outputs use warp stores.  See "bulk-copy emission" below.
//
// Addressing: pool accesses are 32-bit shared-window addresses.  When one
// pool array (N * sizeof(T) bytes) is at most 8 KiB the pool is placed on an
// N*sizeof(T)-aligned shared address, so a gather address is a single LOP3
// ((idx & mask) | base) plus an immediate array offset in the LDS; the
// alignment assumption is probed once per device (smem_base_probe) and the
// IADD form is used otherwise.
#pragma once
#include <type_traits>

#include "common.cuh"

#ifndef WG_EXP_NOSTG
#define WG_EXP_NOSTG 0
#endif
#ifndef WG_EXP_NORAGGED  // experiment only: drop the ragged-end warp stores
#define WG_EXP_NORAGGED 0
#endif
#ifndef WG_EXP_NOBULK  // experiment only: drop the bulk copies
#define WG_EXP_NOBULK 0
#endif
#ifndef WG_DATA_REGS
// registers holding one thread's columns of a pass.  128: a 4x1024 fp32 pool
// (C3/C4) is one warp of 32 columns per thread, so the per-pass scalar work
// (parameter draw, chi-squared scale, loop control) is amortised over 128
// values per thread instead of 64 (C3 12.07 -> 11.70 ms; C1 3.60 -> 3.53 ms)
#define WG_DATA_REGS 128
#endif

// Each translation unit instantiates the engine in its own namespace, so a
// second register budget (WG_DATA_REGS, e.g. 64 in smem_*_r64.cu) can live
// beside the default one.
#ifndef WG_SMEM_NS
#define WG_SMEM_NS r128
#endif

namespace wg {
namespace WG_SMEM_NS {

static constexpr uint32_t kSmemPoolMax = 128 * 1024;  // largest pool kept on chip

extern __shared__ __align__(16) unsigned char g_sm[];

// EM_STATS: generic emission that also accumulates the moment sums of every
// emitted value (wrng_gpu_validate: s1..s4 fused into the emitting pass)
enum EmitMode : int { EM_UNIT = 0, EM_GENERIC = 1, EM_STATS = 2 };

#ifndef WG_RBUDGET_MIN  // smallest per-thread register budget of a shape.  255 here: the
                        // f = 1 fills of small pools are bound by their output pattern and
                        // ran best at 8 CTAs per SM (fp64 4x256: 82 % at 8, 70 % at 16); the
                        // f >= 2 engine (smem_r64.cu) sets 128 for 16 warps per SM
#define WG_RBUDGET_MIN 255
#endif

constexpr uint32_t pick_j(uint32_t N, uint32_t regs_per_col, uint32_t data_regs) {
    uint32_t j = data_regs / regs_per_col;
    if (j > 32) j = 32;
    while (N / j < 32 && j > 1) j /= 2;
    while (N / j > 1024) j *= 2;
    return j;
}

// The dynamic shared-memory window of a CTA starts 1 KiB in (reserved
// system area); smem_base_probe() checks this once per device.
constexpr uint32_t kDynSmemBase = 0x400;

template <typename T, int NA, int LOGN>
struct SmemShape {
    static constexpr uint32_t N = 1u << LOGN;
    static constexpr uint32_t DREGS = WG_DATA_REGS;
    static constexpr uint32_t J = pick_j(N, NA * (uint32_t)sizeof(T) / 4, DREGS);  // columns/thread
    static constexpr uint32_t NTH = N / J;                                         // CTA size
    // CTAs per SM the register budget must allow: twice the data registers
    // J * (regs per column), at least WG_RBUDGET_MIN and at most 255 per
    // thread (C3: 32 threads x 8 CTAs).
    static constexpr uint32_t DATA = J * (NA * (uint32_t)sizeof(T) / 4);
    // fp32 pools of >= 2 warps with 128 data registers (4x2048, 4x4096): as many
    // CTAs per SM as shared memory holds, the register budget cut to match —
    // f = 1 fills overlap one CTA's emission with the others' passes, and 2
    // CTAs per SM left the SM idle while both waited for their bulk copies
    // (4x4096: 3 CTAs per SM at 168 registers 87.3 % of the HBM roofline
    // against 80.7 % at 2; 4x2048: 5 at 200 registers 90.5 % against 89.0 %;
    // the fp64 shapes, at 95 %, gain nothing: 4x1024 91.8 % at 5 against 96.2 %)
    static constexpr uint32_t POOLB = NA * N * (uint32_t)sizeof(T);
    static constexpr uint32_t SMEM_CTAS = (227u * 1024u) / (POOLB + 9u * 1024u);
    static constexpr uint32_t RB_OCC = SMEM_CTAS ? (65536u / (NTH * SMEM_CTAS)) & ~7u : 255u;
    static constexpr bool OCC_TUNE = sizeof(T) == 4 && NTH >= 64 && 2 * DATA > 255 &&
                                     RB_OCC < 255 && RB_OCC >= DATA + 30;
    static constexpr uint32_t RBUDGET = OCC_TUNE                      ? RB_OCC
                                        : 2 * DATA > 255             ? 255
                                        : 2 * DATA < WG_RBUDGET_MIN ? WG_RBUDGET_MIN
                                                                      : 2 * DATA;
    static constexpr uint32_t MINB_R = 65536 / (NTH * RBUDGET);
    static constexpr uint32_t MINB = MINB_R < 1 ? 1 : MINB_R > 32 ? 32 : MINB_R;
    static constexpr uint32_t MASK = N - 1;
    static constexpr uint32_t ABYTES = N * (uint32_t)sizeof(T);  // one array
    static constexpr uint32_t MASKB = MASK * (uint32_t)sizeof(T);
    static constexpr uint64_t NVALS = (uint64_t)NA * N;
    static constexpr uint64_t CAP = NVALS - 1;
    static constexpr uint32_t STEP = NTH < 256 ? NTH : 256;  // uniform words per bulk step
    // shared layout: lag table | word staging | control block | pool
    static constexpr uint32_t TAB_OFF = 0;
    static constexpr uint32_t WBUF_OFF = 608 * 8;
    static constexpr uint32_t CTL_OFF = WBUF_OFF + 256 * 8;
    static constexpr uint32_t HEAD = CTL_OFF + 256;
    static_assert(sizeof(Ctl) <= 256, "control block");
    static constexpr bool CAN_ALIGN = ABYTES <= 8192;
    static constexpr uint32_t POOL_OFF =
        CAN_ALIGN ? ((kDynSmemBase + HEAD + ABYTES - 1) / ABYTES) * ABYTES - kDynSmemBase
                  : HEAD;
    static constexpr uint32_t POOL_END = POOL_OFF + (uint32_t)(NVALS * sizeof(T));
    // exact-sum scratch: pools of >= 96 KiB run one CTA per SM anyway, so the
    // drift audit gets up to 512 chunks (short serial chains); smaller pools
    // reuse the 2 KiB word buffer (60 chunks) to keep their occupancy
    static constexpr bool BIGSUM = NVALS * sizeof(T) >= 96 * 1024;
    static constexpr uint32_t SUM_CHUNKS = BIGSUM ? (NTH < 512 ? NTH : 512) : kSumSmallChunks;
    static constexpr uint32_t SCR_OFF = BIGSUM ? ((POOL_END + 15) & ~15u) : WBUF_OFF;
    static constexpr uint32_t BYTES = BIGSUM ? SCR_OFF + sum_scratch_bytes(SUM_CHUNKS) : POOL_END;
};

template <int B, int E, typename F>
__device__ __forceinline__ void sfor(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        sfor<B + 1, E>(f);
    }
}

template <typename T, uint32_t OFF>
__device__ __forceinline__ T lds(uint32_t a) {
    T v;
    if constexpr (sizeof(T) == 4)
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
    else
        asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF));
    return v;
}

template <typename T, uint32_t OFF>
__device__ __forceinline__ void sts(uint32_t a, T v) {
    if constexpr (sizeof(T) == 4)
        asm volatile("st.shared.f32 [%0+%1], %2;" ::"r"(a), "n"(OFF), "f"(v) : "memory");
    else
        asm volatile("st.shared.f64 [%0+%1], %2;" ::"r"(a), "n"(OFF), "d"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T& sm_at(uint32_t off) {
    return *reinterpret_cast<T*>(g_sm + off);
}

template <typename T, int EM>
__device__ __forceinline__ void emit_one(void* out, uint64_t i, T v, uint32_t out_f32,
                                         uint32_t unit, double mu, double sigma) {
    if (EM == EM_UNIT)
        static_cast<T*>(out)[i] = v + (T)0;  // 0 + 1 * v: -0.0 -> +0.0
    else
        put_out(out, i, v, out_f32, unit, mu, sigma);
}

struct EmitCfg {  // per-launch constants of the output stream
    double mu, sigma;
    uint32_t out_f32, unit;
    // EM_STATS: this thread's sums of v, v^2, v^3, v^4 over its emitted values
    mutable double st[4] = {0.0, 0.0, 0.0, 0.0};
    __device__ __forceinline__ void add(double v) const {
        const double v2 = v * v;
        st[0] += v;
        st[1] += v2;
        st[2] += v2 * v;
        st[3] += v2 * v2;
    }
};

// ---- bulk-copy emission of full refills (unit output) ---------------------
// Phase C writes the new pool into shared memory anyway, and on a full refill
// the pool IS the emitted sequence (array-major, wallace.cpp:206-213).  Thread
// 0 hands it to the bulk-copy engine after the pass's final barrier, so the
// warps issue no per-value global stores.  cp.async.bulk needs 16-byte
// alignment on both sides, while a refill's output offset moves by 4N-1
// values per refill; so the pool is kept ROTATED in shared memory: value j
// of every array sits at position (j + rot) mod N, with rot chosen on each
// emitting pass to match the output address modulo 16 bytes.  Gathers fold
// rot into their offsets (free), phase C stores shift by rot (only the last
// column group can wrap), and the <= 2*VEC ragged values at each array's
// ends leave through ordinary stores.  Before the next phase C overwrites
// the pool, thread 0 waits for the engine's shared-memory reads.
#ifndef WG_EXP_BULK_HINT  // experiment: L2 policy of the output copies (1 evict_first, 2 evict_last):
                          // both measured 2 % slower on C3 (92.6 / 92.8 % against 94.9 %)
#define WG_EXP_BULK_HINT 0
#endif
__device__ __forceinline__ void bulk_store(uint64_t dst, uint32_t src_s, uint32_t bytes) {
#if WG_EXP_BULK_HINT
    uint64_t pol;
#if WG_EXP_BULK_HINT == 1
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                     dst),
                 "r"(src_s), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(src_s), "r"(bytes)
                 : "memory");
#endif
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read_n() {  // <= N groups still reading
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Where phase C stores and what it emits itself.  my_s: shared address of
// this thread's column 0 at the new rotation; last_s: of its last column
// (k = J - 1, the only one that can wrap).  MD 3: values j < j0 and
// j >= jend[m] (j < N, the withheld slot excluded) are stored by the warps,
// [j0, jend[m]) by the bulk engine.
struct PhaseC {
    uint32_t my_s, last_s;
    uint32_t j0, jend, jend_last;
    uint32_t src0;  // shared address of array 0's bulk span (value j0)
};

// Experiment (off): one-warp fp32 n = 4 pools issue their bulk copies array
// by array from phase C (phase_c2_split) instead of once per pass.  Measured
// slower on C3 (11.95-11.99 ms vs 11.62-11.70 ms per step).
#ifndef WG_EXP_SPLIT
#define WG_EXP_SPLIT 0
#endif
template <typename T, int NA, int LOGN>
constexpr bool kSplitC = WG_EXP_SPLIT && sizeof(T) == 4 && NA == 4 &&
                         SmemShape<T, NA, LOGN>::NTH == 32 &&
                         SmemShape<T, NA, LOGN>::J % 2 == 0;

// Phase B: gather + unscaled transform (VAR = n=4 matrix variant; AL =
// aligned pool base, gather address = (idx & mask) | base).
template <typename T, int NA, int LOGN, int VAR, bool AL>
__device__ __forceinline__ void phase_b(uint32_t pool_s, uint32_t (&ixb)[NA],
                                        const uint32_t (&stepb)[NA],
                                        T (&u)[NA][SmemShape<T, NA, LOGN>::J]) {
    using S = SmemShape<T, NA, LOGN>;
    sfor<0, (int)S::J>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        T g[NA];
        sfor<0, NA>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            const uint32_t a =
                AL ? ((ixb[m] & S::MASKB) | pool_s) : ((ixb[m] & S::MASKB) + pool_s);
            g[m] = lds<T, (uint32_t)m * S::ABYTES>(a);
            ixb[m] += stepb[m];
        });
        if constexpr (NA == 4) {
            if constexpr (VAR == 0) {
                // (1/2) H4: y = k * {(p+r), (q+s), (p-r), (q-s)}
                const T pp = g[0] + g[1], q = g[0] - g[1], r = g[2] + g[3], s = g[2] - g[3];
                u[0][k] = pp + r;
                u[1][k] = q + s;
                u[2][k] = pp - r;
                u[3][k] = q - s;
            } else {
                // (1/2) J - I: y_i = scale * (t - x_i)
                const T t = (T)0.5 * ((g[0] + g[1]) + (g[2] + g[3]));
                u[0][k] = t - g[0];
                u[1][k] = t - g[1];
                u[2][k] = t - g[2];
                u[3][k] = t - g[3];
            }
        } else {
            u[0][k] = g[0];
            u[1][k] = g[1];
        }
    });
}

// ---- packed fp32 path (n = 4, fp32 pools): Blackwell FADD2 / FMUL2 ------
// add/sub/mul.rn.f32x2 round each lane exactly like the scalar op, so two
// columns (k, k+1) of a thread are transformed by one instruction.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float a, float b) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
    f2_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
    f2_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

template <int LOGN, int VAR, bool AL>
__device__ __forceinline__ void phase_b2(uint32_t pool_s, uint32_t (&ixb)[4],
                                         const uint32_t (&stepb)[4],
                                         f2_t (&u)[4][SmemShape<float, 4, LOGN>::J / 2]) {
    using S = SmemShape<float, 4, LOGN>;
    static_assert(S::J % 2 == 0, "column pairs");
    sfor<0, (int)S::J / 2>([&](auto kc) {
        constexpr int kp = decltype(kc)::value;
        float g[4][2];
        sfor<0, 2>([&](auto hc) {
            constexpr int h = decltype(hc)::value;
            sfor<0, 4>([&](auto mc) {
                constexpr int m = decltype(mc)::value;
                const uint32_t a =
                    AL ? ((ixb[m] & S::MASKB) | pool_s) : ((ixb[m] & S::MASKB) + pool_s);
                g[m][h] = lds<float, (uint32_t)m * S::ABYTES>(a);
                ixb[m] += stepb[m];
            });
        });
        const f2_t G0 = f2_pack(g[0][0], g[0][1]), G1 = f2_pack(g[1][0], g[1][1]);
        const f2_t G2 = f2_pack(g[2][0], g[2][1]), G3 = f2_pack(g[3][0], g[3][1]);
        if constexpr (VAR == 0) {
            const f2_t PP = f2_add(G0, G1), Q = f2_sub(G0, G1);
            const f2_t R = f2_add(G2, G3), Sd = f2_sub(G2, G3);
            u[0][kp] = f2_add(PP, R);
            u[1][kp] = f2_add(Q, Sd);
            u[2][kp] = f2_sub(PP, R);
            u[3][kp] = f2_sub(Q, Sd);
        } else {
            const f2_t T = f2_mul(f2_pack(0.5f, 0.5f), f2_add(f2_add(G0, G1), f2_add(G2, G3)));
            u[0][kp] = f2_sub(T, G0);
            u[1][kp] = f2_sub(T, G1);
            u[2][kp] = f2_sub(T, G2);
            u[3][kp] = f2_sub(T, G3);
        }
    });
}

#ifndef WG_SCALE_LANE0  // 1: the pass's fp64 scale chain on one lane per warp (power)
#define WG_SCALE_LANE0 1
#endif
#ifndef WG_GATHER_FIRST  // 1: gather all columns, then one small per-variant transform
#define WG_GATHER_FIRST 1
#endif
// Variant-independent gathers of phase B (packed fp32, n = 4): u[m][kp]
// holds the sources of columns (2kp, 2kp+1) of array m; the transform then
// runs in place, so only ~130 instructions differ between the variants
// (hot code shrinks by one copy of the 128 gathers).
template <int LOGN, bool AL>
__device__ __forceinline__ void gather_b2(uint32_t pool_s, uint32_t (&ixb)[4],
                                          const uint32_t (&stepb)[4],
                                          f2_t (&u)[4][SmemShape<float, 4, LOGN>::J / 2]) {
    using S = SmemShape<float, 4, LOGN>;
    sfor<0, (int)S::J / 2>([&](auto kc) {
        constexpr int kp = decltype(kc)::value;
        float g[4][2];
        sfor<0, 2>([&](auto hc) {
            constexpr int h = decltype(hc)::value;
            sfor<0, 4>([&](auto mc) {
                constexpr int m = decltype(mc)::value;
                const uint32_t a =
                    AL ? ((ixb[m] & S::MASKB) | pool_s) : ((ixb[m] & S::MASKB) + pool_s);
                g[m][h] = lds<float, (uint32_t)m * S::ABYTES>(a);
                ixb[m] += stepb[m];
            });
        });
        sfor<0, 4>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            u[m][kp] = f2_pack(g[m][0], g[m][1]);
        });
    });
}
template <int LOGN, int VAR>
__device__ __forceinline__ void transform_b2(f2_t (&u)[4][SmemShape<float, 4, LOGN>::J / 2]) {
    using S = SmemShape<float, 4, LOGN>;
    sfor<0, (int)S::J / 2>([&](auto kc) {
        constexpr int kp = decltype(kc)::value;
        const f2_t G0 = u[0][kp], G1 = u[1][kp], G2 = u[2][kp], G3 = u[3][kp];
        if constexpr (VAR == 0) {
            const f2_t PP = f2_add(G0, G1), Q = f2_sub(G0, G1);
            const f2_t R = f2_add(G2, G3), Sd = f2_sub(G2, G3);
            u[0][kp] = f2_add(PP, R);
            u[1][kp] = f2_add(Q, Sd);
            u[2][kp] = f2_sub(PP, R);
            u[3][kp] = f2_sub(Q, Sd);
        } else {
            const f2_t T = f2_mul(f2_pack(0.5f, 0.5f), f2_add(f2_add(G0, G1), f2_add(G2, G3)));
            u[0][kp] = f2_sub(T, G0);
            u[1][kp] = f2_sub(T, G1);
            u[2][kp] = f2_sub(T, G2);
            u[3][kp] = f2_sub(T, G3);
        }
    });
}

// Generic (fp64 / n = 2) counterpart: gathers into u, then the n = 4
// transform in place (op order of phase_b).
template <typename T, int NA, int LOGN, bool AL>
__device__ __forceinline__ void gather_b(uint32_t pool_s, uint32_t (&ixb)[NA],
                                         const uint32_t (&stepb)[NA],
                                         T (&u)[NA][SmemShape<T, NA, LOGN>::J]) {
    using S = SmemShape<T, NA, LOGN>;
    sfor<0, (int)S::J>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        sfor<0, NA>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            const uint32_t a =
                AL ? ((ixb[m] & S::MASKB) | pool_s) : ((ixb[m] & S::MASKB) + pool_s);
            u[m][k] = lds<T, (uint32_t)m * S::ABYTES>(a);
            ixb[m] += stepb[m];
        });
    });
}
template <typename T, int LOGN, int VAR>
__device__ __forceinline__ void transform_b(T (&u)[4][SmemShape<T, 4, LOGN>::J]) {
    using S = SmemShape<T, 4, LOGN>;
    sfor<0, (int)S::J>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        const T g0 = u[0][k], g1 = u[1][k], g2 = u[2][k], g3 = u[3][k];
        if constexpr (VAR == 0) {
            const T pp = g0 + g1, q = g0 - g1, r = g2 + g3, s = g2 - g3;
            u[0][k] = pp + r;
            u[1][k] = q + s;
            u[2][k] = pp - r;
            u[3][k] = q - s;
        } else {
            const T t = (T)0.5 * ((g0 + g1) + (g2 + g3));
            u[0][k] = t - g0;
            u[1][k] = t - g1;
            u[2][k] = t - g2;
            u[3][k] = t - g3;
        }
    });
}

// Store of value (m, column group k) into the rotated pool.
template <typename T, int NA, int LOGN, int M, int K>
__device__ __forceinline__ void sts_rot(const PhaseC& pc, T v) {
    using S = SmemShape<T, NA, LOGN>;
    if constexpr (K == (int)S::J - 1)
        sts<T, (uint32_t)M * S::ABYTES>(pc.last_s, v);
    else
        sts<T, (uint32_t)M * S::ABYTES + (uint32_t)K * S::NTH * (uint32_t)sizeof(T)>(pc.my_s, v);
}

// MD 3: does this thread store value (m, k) itself (ragged ends)?
template <typename T, int NA, int LOGN, int M, int K>
__device__ __forceinline__ bool md3_own(const PhaseC& pc, uint32_t tid) {
    using S = SmemShape<T, NA, LOGN>;
    bool own = false;
    if constexpr (K == 0) own = tid < pc.j0;
    if constexpr (K == (int)S::J - 1) {  // the ragged tail lies in the last column group
        const uint32_t j = (uint32_t)K * S::NTH + tid;
        if constexpr (M == NA - 1)
            own = own || (j >= pc.jend_last && j != S::N - 1);
        else
            own = own || j >= pc.jend;
    }
    return own;
}

// Phase C (packed fp32, n = 4): scale, store in place, emit.  MD 0: no
// emission; 1: full refill, unit output, warp stores at immediate offsets;
// 2: partial window / generic output; 3: full refill through the bulk-copy
// engine (the pool holds the emitted form 0 + v, which differs from v only
// for v = -0.0; the warps store only the ragged ends).
// MD 3 on a one-warp pool (NTH == 32): array-major, so each array's bulk
// copy leaves as soon as the array is written (lane 0 issues it after a
// __syncwarp), and before rewriting array m lane 0 waits only for the
// previous refill's copy of array m (bulk groups retire in order).
template <int LOGN>
__device__ __forceinline__ void phase_c2_split(
    const f2_t (&u)[4][SmemShape<float, 4, LOGN>::J / 2], float c0, const PhaseC& pc,
    char* out_p, double& withheld_out) {
    using S = SmemShape<float, 4, LOGN>;
    static_assert(S::NTH == 32, "one-warp pools");
    const uint32_t tid = threadIdx.x;
    float* ob = reinterpret_cast<float*>(out_p) + tid;
    const f2_t C = f2_pack(c0, c0), Z = f2_pack(0.0f, 0.0f);
    sfor<0, 4>([&](auto mc) {
        constexpr int m = decltype(mc)::value;
        if (tid == 0) bulk_wait_read_n<3 - m>();
        __syncwarp();
        sfor<0, (int)S::J / 2>([&](auto kc) {
            constexpr int kp = decltype(kc)::value;
            const f2_t Y = f2_mul(C, u[m][kp]);
            float e[2];
            f2_unpack(f2_add(Y, Z), e[0], e[1]);  // 0 + 1 * v
            sfor<0, 2>([&](auto hc) {
                constexpr int h = decltype(hc)::value;
                constexpr int k = 2 * kp + h;
                constexpr uint32_t col = m * S::N + k * S::NTH;
                sts_rot<float, 4, LOGN, m, k>(pc, e[h]);
                if constexpr (k == 0 || k == (int)S::J - 1) {
                    if (!WG_EXP_NORAGGED && md3_own<float, 4, LOGN, m, k>(pc, tid))
                        ob[col] = e[h];
                }
                if constexpr (m == 3 && k == (int)S::J - 1) {
                    if (tid == S::NTH - 1) {
                        float y[2];
                        f2_unpack(Y, y[0], y[1]);
                        withheld_out = (double)y[h];
                    }
                }
            });
        });
        fence_async_smem();
        __syncwarp();
        if (tid == 0) {
            const uint32_t je = m == 3 ? pc.jend_last : pc.jend;
            if (je > pc.j0 && !WG_EXP_NOBULK)
                bulk_store(reinterpret_cast<uint64_t>(out_p) + ((uint64_t)m * S::N + pc.j0) * 4,
                           pc.src0 + (uint32_t)m * S::ABYTES, (je - pc.j0) * 4);
            bulk_commit();
        }
    });
}

template <int LOGN, int EM, int MD>
__device__ __forceinline__ void phase_c2(const f2_t (&u)[4][SmemShape<float, 4, LOGN>::J / 2],
                                         float c0, const PhaseC& pc, char* out_p, uint32_t en,
                                         const EmitCfg& ec, double& withheld_out) {
    using S = SmemShape<float, 4, LOGN>;
    const uint32_t tid = threadIdx.x;
    float* ob = (MD == 1 || MD == 3) ? reinterpret_cast<float*>(out_p) + tid : nullptr;
    const f2_t C = f2_pack(c0, c0), Z = f2_pack(0.0f, 0.0f);
    sfor<0, (int)S::J / 2>([&](auto kc) {
        constexpr int kp = decltype(kc)::value;
        sfor<0, 4>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            const f2_t Y = f2_mul(C, u[m][kp]);
            float y[2];
            f2_unpack(Y, y[0], y[1]);
            float e[2];
            if constexpr (MD == 1 || MD == 3) f2_unpack(f2_add(Y, Z), e[0], e[1]);  // 0 + 1 * v
            sfor<0, 2>([&](auto hc) {
                constexpr int h = decltype(hc)::value;
                constexpr int k = 2 * kp + h;
                constexpr uint32_t col = m * S::N + k * S::NTH;
                sts_rot<float, 4, LOGN, m, k>(pc, MD == 3 ? e[h] : y[h]);
                if constexpr (MD == 3) {
                    if constexpr (k == 0 || k == (int)S::J - 1) {
                        if (!WG_EXP_NORAGGED && md3_own<float, 4, LOGN, m, k>(pc, tid))
                            ob[col] = e[h];
                    }
                } else if constexpr (MD == 1) {
#if !WG_EXP_NOSTG  // experiment only: drop the output stores to bound their cost
                    if (!(m == 3 && k == (int)S::J - 1) || tid != S::NTH - 1) ob[col] = e[h];
#endif
                } else if constexpr (MD == 2) {
                    const uint32_t flat = col + tid;
                    if (flat < en) {
                        emit_one<float, EM>(out_p, flat, y[h], ec.out_f32, ec.unit, ec.mu,
                                            ec.sigma);
                        if constexpr (EM == EM_STATS) ec.add((double)y[h]);
                    }
                }
                if (m == 3 && k == (int)S::J - 1 && tid == S::NTH - 1)
                    withheld_out = (double)y[h];
            });
        });
    });
    if constexpr (MD == 3) fence_async_smem();  // generic -> async proxy
}

// Phase C, generic (fp64 pools, n = 2, odd J): as phase_c2.
template <typename T, int NA, int LOGN, int EM, int MD>
__device__ __forceinline__ void phase_c(const T (&u)[NA][SmemShape<T, NA, LOGN>::J], T c0, T c1,
                                        const PhaseC& pc, char* out_p, uint32_t en,
                                        const EmitCfg& ec, double& withheld_out) {
    using S = SmemShape<T, NA, LOGN>;
    const uint32_t tid = threadIdx.x;
    T* ob = (MD == 1 || MD == 3) ? reinterpret_cast<T*>(out_p) + tid : nullptr;
    sfor<0, (int)S::J>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        T y[NA];
        if constexpr (NA == 4) {
#pragma unroll
            for (int m = 0; m < NA; ++m) y[m] = c0 * u[m][k];
        } else {
            // dst.x = kc*xs + ks*ys ; dst.y = kc*ys - ks*xs (wallace.cpp:130-131)
            const T xs = u[0][k], ys = u[1][k];
            y[0] = c0 * xs + c1 * ys;
            y[1] = c0 * ys - c1 * xs;
        }
        sfor<0, NA>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            constexpr uint32_t col = m * S::N + k * S::NTH;
            if constexpr (MD == 3) {
                const T e = y[m] + (T)0;  // 0 + 1 * v: the pool is the bulk source
                sts_rot<T, NA, LOGN, m, k>(pc, e);
                if constexpr (k == 0 || k == (int)S::J - 1) {
                    if (md3_own<T, NA, LOGN, m, k>(pc, tid)) ob[col] = e;
                }
            } else {
                sts_rot<T, NA, LOGN, m, k>(pc, y[m]);
            }
            if constexpr (MD == 1) {
                if (!(m == NA - 1 && k == (int)S::J - 1) || tid != S::NTH - 1)
                    ob[col] = y[m] + (T)0;  // 0 + 1 * v
            } else if constexpr (MD == 2) {
                const uint32_t flat = col + tid;
                if (flat < en) {
                    emit_one<T, EM>(out_p, flat, y[m], ec.out_f32, ec.unit, ec.mu, ec.sigma);
                    if constexpr (EM == EM_STATS) ec.add((double)y[m]);
                }
            }
        });
        if (k == (int)S::J - 1 && tid == S::NTH - 1) withheld_out = (double)y[NA - 1];
    });
    if constexpr (MD == 3) fence_async_smem();
}

template <int LOGN, int EM>
__device__ __forceinline__ void phase_c2_any(uint32_t md,
                                             const f2_t (&u)[4][SmemShape<float, 4, LOGN>::J / 2],
                                             float c0, const PhaseC& pc, char* out_p, uint32_t en,
                                             const EmitCfg& ec, double& wh) {
    if (md == 0)
        phase_c2<LOGN, EM, 0>(u, c0, pc, out_p, 0, ec, wh);
    else if (EM == EM_UNIT && md == 3) {
        if constexpr (kSplitC<float, 4, LOGN>)
            phase_c2_split<LOGN>(u, c0, pc, out_p, wh);
        else
            phase_c2<LOGN, EM, 3>(u, c0, pc, out_p, en, ec, wh);
    }
    else if (EM == EM_UNIT && md == 1)
        phase_c2<LOGN, EM, 1>(u, c0, pc, out_p, en, ec, wh);
    else
        phase_c2<LOGN, EM, 2>(u, c0, pc, out_p, en, ec, wh);
}

template <typename T, int NA, int LOGN, int EM>
__device__ __forceinline__ void phase_c_any(uint32_t md,
                                            const T (&u)[NA][SmemShape<T, NA, LOGN>::J], T c0,
                                            T c1, const PhaseC& pc, char* out_p, uint32_t en,
                                            const EmitCfg& ec, double& wh) {
    if (md == 0)
        phase_c<T, NA, LOGN, EM, 0>(u, c0, c1, pc, out_p, 0, ec, wh);
    else if (EM == EM_UNIT && md == 3)
        phase_c<T, NA, LOGN, EM, 3>(u, c0, c1, pc, out_p, en, ec, wh);
    else if (EM == EM_UNIT && md == 1)
        phase_c<T, NA, LOGN, EM, 1>(u, c0, c1, pc, out_p, en, ec, wh);
    else
        phase_c<T, NA, LOGN, EM, 2>(u, c0, c1, pc, out_p, en, ec, wh);
}

// The phase B -> C barrier; with bulk emission on, thread 0 first waits
// until the previous refill's bulk copies have read the pool (phase C
// rewrites it).
template <int EM>
__device__ __forceinline__ void bc_barrier(bool bulk_on) {
    if constexpr (EM == EM_UNIT) {
        if (bulk_on && threadIdx.x == 0) bulk_wait_read();
    }
    __syncthreads();
}

// One in-place regeneration pass.  Preconditions (after a barrier): the
// parameter slot `slot` (ctl->cur / ctl->cur2) holds this pass's uniform-
// generator parameters.  prefetch: warp 0 draws the next pass's words into
// the other slot during phase B.  prev: when non-null, the pre-pass pool is
// copied there (it becomes the inactive buffer).  Returns false on a
// device-detected error (ctl->error set); every thread returns the same.
//
// The chi-squared scale (wallace.cpp:59-69) is derived by EVERY thread from
// the broadcast (tracked, withheld): warp-uniform, so its fp64 div/sqrt
// chain overlaps the gathers instead of serialising one lane of warp 0.
template <typename T, int NA, int LOGN, int EM, bool AL, bool COLD>
__device__ __forceinline__ bool smem_pass(uint32_t pool_s, uint32_t mode, uint32_t emit_n,
                                          char* out_p, const EmitCfg& ec, wrng_gpu_params* rec,
                                          bool prefetch, T* prev, int slot, uint32_t bvec) {
    using S = SmemShape<T, NA, LOGN>;
    const bool bulk_on = bvec != 0;
    constexpr uint32_t N = S::N, NTH = S::NTH;
    const uint32_t tid = threadIdx.x;
    Ctl* ctl = &sm_at<Ctl>(S::CTL_OFF);
    const LfgParams& cp = slot ? ctl->cur2 : ctl->cur;
    constexpr uint32_t ES = (uint32_t)sizeof(T);
    const uint32_t rot = ctl->rot;  // value j of each array sits at (j + rot) mod N

    uint32_t ixb[NA], stepb[NA];
#pragma unroll
    for (int m = 0; m < NA; ++m) {
        const uint32_t st = cp.stride[m];
        ixb[m] = (st * tid + cp.offset[m] + rot) * ES;
        stepb[m] = st * NTH * ES;
    }
    const uint32_t variant = cp.variant;
    const double tracked = ctl->tracked, withheld = ctl->withheld;
    double scale = 0.0, target = 0.0;
    int e = 0;
    double c0d = 0.0, c1d = 0.0;
#if WG_SCALE_LANE0
    // lane 0 of every warp runs the fp64 div/sqrt chain and broadcasts the two
    // coefficients: the same issue slots, but 1/32 of the fp64 datapath energy
    T c0 = (T)0, c1 = (T)0;
    if ((tid & 31u) == 0) {
        e = pass_scale(tracked, withheld, (uint32_t)S::NVALS, mode, scale, target);
        // regenerate folds the scale into the matrix (wallace.cpp:116-117)
        c0d = NA == 2 ? cp.c * scale : (variant ? scale : 0.5 * scale);
        c1d = NA == 2 ? cp.s * scale : scale;
        c0 = (T)c0d;  // fp32 pools: rounded once (docs/n4_spec.md §4)
        c1 = (T)c1d;
    }
    e = __shfl_sync(0xffffffffu, e, 0);
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    if (NA == 2) c1 = __shfl_sync(0xffffffffu, c1, 0);
#else
    e = pass_scale(tracked, withheld, (uint32_t)S::NVALS, mode, scale, target);
    // regenerate folds the scale into the matrix (wallace.cpp:116-117)
    c0d = NA == 2 ? cp.c * scale : (variant ? scale : 0.5 * scale);
    c1d = NA == 2 ? cp.s * scale : scale;
#endif
    if (e) {  // every thread sees the same e (wallace.cpp:59-61)
        if (tid == 0) ctl->error = e;
        __syncthreads();
        return false;
    }
    if (COLD && tid == 0) {
        if (rec) {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                rec->stride[m] = cp.stride[m];
                rec->offset[m] = cp.offset[m];
            }
            rec->variant = cp.variant;
            rec->pad_ = 0;
            rec->c = cp.c;
            rec->s = cp.s;
            rec->scale = scale;
            rec->target_sumsq = target;
        }
        if (prev) {
            ctl->prev_tracked = tracked;
            ctl->prev_withheld = withheld;
            ctl->have_prev = 1;
        }
    }
    if (COLD && prev) {
        // the pre-pass pool becomes the inactive buffer (wallace.cpp:170-174)
        const RotView<T> v{&sm_at<T>(S::POOL_OFF), S::MASK, rot};
        for (uint32_t i = tid; i < (uint32_t)S::NVALS; i += NTH) prev[i] = v[i];
    }
    if (prefetch)
        draw_pass_params_all<NA>(&sm_at<uint64_t>(S::TAB_OFF), ctl, N, slot ^ 1, tid < 32);
#if !WG_SCALE_LANE0
    const T c0 = (T)c0d, c1 = (T)c1d;  // fp32 pools: rounded once (docs/n4_spec.md §4)
#endif
    double wh = 0.0;
    const uint32_t md = emit_n == 0                                    ? 0u
                        : (EM == EM_UNIT && emit_n == (uint32_t)S::CAP) ? (bulk_on ? 3u : 1u)
                                                                        : 2u;
    // new rotation: on a bulk-emitting pass, the output's 16-byte phase
    constexpr uint32_t VEC = 16 / ES;
    const uint32_t rot2 =
        md == 3 ? (uint32_t)(reinterpret_cast<uintptr_t>(out_p) / ES) & (VEC - 1) : rot;
    PhaseC pc;
    pc.my_s = pool_s + (tid + rot2) * ES;
    {
        const uint32_t lastb = (((uint32_t)(S::J - 1) * NTH + tid + rot2) * ES) & S::MASKB;
        pc.last_s = AL ? (lastb | pool_s) : (lastb + pool_s);
    }
    // bulk-copied span [j0, jend): starts and ends on a bvec-element boundary
    // of the output (bvec >= VEC, a power of 2; 128 B lines by default)
    {
        const uint32_t bv = bulk_on ? bvec : VEC;
        const uint32_t ph = (uint32_t)(reinterpret_cast<uintptr_t>(out_p) / ES) & (bv - 1);
        pc.j0 = (bv - ph) & (bv - 1);
        pc.jend = pc.j0 + ((N - rot2 - pc.j0) & ~(bv - 1));
        pc.jend_last = pc.j0 + ((umin32(N - rot2, N - 1) - pc.j0) & ~(bv - 1));
    }
    pc.src0 = pool_s + (pc.j0 + rot2) * ES;
    if constexpr (sizeof(T) == 4 && NA == 4 && S::J % 2 == 0) {
        f2_t u[4][S::J / 2];
        if (WG_GATHER_FIRST) {
            gather_b2<LOGN, AL>(pool_s, ixb, stepb, u);
            if (variant == 0)
                transform_b2<LOGN, 0>(u);
            else
                transform_b2<LOGN, 1>(u);
        } else if (variant == 0) {
            phase_b2<LOGN, 0, AL>(pool_s, ixb, stepb, u);
        } else {
            phase_b2<LOGN, 1, AL>(pool_s, ixb, stepb, u);
        }
        bc_barrier<EM>(bulk_on && !(kSplitC<T, NA, LOGN> && md == 3));
        phase_c2_any<LOGN, EM>(md, u, c0, pc, out_p, emit_n, ec, wh);
    } else {
        T u[NA][S::J];
        if constexpr (NA == 4 && WG_GATHER_FIRST) {
            gather_b<T, NA, LOGN, AL>(pool_s, ixb, stepb, u);
            if (variant == 0)
                transform_b<T, LOGN, 0>(u);
            else
                transform_b<T, LOGN, 1>(u);
        } else if (NA == 2 || variant == 0) {
            phase_b<T, NA, LOGN, 0, AL>(pool_s, ixb, stepb, u);
        } else {
            phase_b<T, NA, LOGN, 1, AL>(pool_s, ixb, stepb, u);
        }
        bc_barrier<EM>(bulk_on);
        phase_c_any<T, NA, LOGN, EM>(md, u, c0, c1, pc, out_p, emit_n, ec, wh);
    }
    if (tid == NTH - 1) ctl->withheld = wh;  // wallace.cpp:136
    if (tid == 0) {
        ctl->tracked = target;  // wallace.cpp:135
        ctl->active ^= 1u;
        ctl->rot = rot2;
    }
    __syncthreads();
    if (md == 3 && !kSplitC<T, NA, LOGN> && tid == 0) {
        // [j0, jend) of every array (last: jend_last) -> output, 16-byte aligned
        const uint64_t ob = reinterpret_cast<uint64_t>(out_p);
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            const uint32_t je = m == NA - 1 ? pc.jend_last : pc.jend;
            if (je > pc.j0 && !WG_EXP_NOBULK)
                bulk_store(ob + ((uint64_t)m * N + pc.j0) * ES, pc.src0 + (uint32_t)m * S::ABYTES,
                           (je - pc.j0) * ES);
        }
        bulk_commit();
    }
    return true;
}

template <typename T, int NA, int LOGN>
__device__ __forceinline__ bool smem_drift_check() {
    // wallace.cpp:225-234 with Pool::direct_sumsq order (wallace.cpp:13-18)
    using S = SmemShape<T, NA, LOGN>;
    Ctl* ctl = &sm_at<Ctl>(S::CTL_OFF);
    const RotView<T> v{&sm_at<T>(S::POOL_OFF), S::MASK, ctl->rot};
    const double rec =
        exact_sumsq_cta<T>(v, (uint32_t)S::NVALS, &sm_at<uint64_t>(S::SCR_OFF), S::SUM_CHUNKS);
    if (threadIdx.x == 0) {
        const double rel = fabs(rec / ctl->tracked - 1.0);
        if (!(rel <= 1e-3))
            ctl->error = WRNG_GPU_ECORRUPT;
        else
            ctl->tracked = rec;
    }
    __syncthreads();
    return ctl->error == 0;
}

template <typename T, int NA, int LOGN>
__device__ __forceinline__ void smem_restart() {
    using S = SmemShape<T, NA, LOGN>;
    init_pool_dev(&sm_at<T>(S::POOL_OFF), S::NVALS, &sm_at<uint64_t>(S::TAB_OFF),
                  &sm_at<Ctl>(S::CTL_OFF), &sm_at<uint64_t>(S::WBUF_OFF), S::STEP,
                  &sm_at<uint64_t>(S::SCR_OFF), S::SUM_CHUNKS);
    if (threadIdx.x == 0) sm_at<Ctl>(S::CTL_OFF).rot = 0;  // natural order again
    __syncthreads();
}

template <typename T, int NA, int LOGN, int EM, bool AL>
__global__ void __launch_bounds__(SmemShape<T, NA, LOGN>::NTH, SmemShape<T, NA, LOGN>::MINB)
    k_smem(const KernelArgs a) {
    using S = SmemShape<T, NA, LOGN>;
    constexpr uint32_t N = S::N, NTH = S::NTH;
    constexpr uint64_t NVALS = S::NVALS, CAP = S::CAP;

    uint64_t* tab = &sm_at<uint64_t>(S::TAB_OFF);
    uint64_t* wbuf = &sm_at<uint64_t>(S::WBUF_OFF);
    Ctl* ctl = &sm_at<Ctl>(S::CTL_OFF);
    const uint32_t pool_s = (uint32_t)__cvta_generic_to_shared(g_sm) + S::POOL_OFF;

    const uint32_t tid = threadIdx.x;
    const uint32_t p = blockIdx.x;
    PoolMeta* meta = a.meta + p;
    LfgState* lg = a.lfg + p;
    const uint32_t op = a.op;
    // A device-raised error is sticky until the host observes it: the pool
    // stays frozen at the failure point.
    if (op != OP_INIT && meta->error) return;
    // Host-restart resume launch: only the pools the host just restarted
    // continue (PoolMeta::restart_pending == 2), from their fill_done.
    const bool resume = a.resume != 0 && op == OP_FILL;
    if (resume && meta->restart_pending != 2) return;

    // ---- load state -------------------------------------------------------
    uint64_t pc, avail, emitted;
    if (op == OP_INIT) {
        pc = avail = emitted = 0;
        if (tid == 0) {
            ctl->active = 0;
            ctl->error = 0;
            ctl->have_prev = 0;
            ctl->cur.c = ctl->cur.s = ctl->cur2.c = ctl->cur2.s = 0.0;
            ctl->cur.pad_ = ctl->cur2.pad_ = 0;
            ctl->rot = 0;
        }
        lfg_seed(tab, ctl, wbuf, a.seed, a.stream0 + p, S::STEP);
    } else {
        pc = meta->pass_count;
        avail = meta->avail;
        emitted = meta->emitted;
        const uint32_t act = meta->active;
        for (uint32_t i = tid; i < kTable; i += NTH) tab[i] = lg->table[i];
        if (tid == 0) {
            ctl->r = lg->r;
            ctl->draws = lg->draws;
            ctl->active = act;
            ctl->tracked = meta->tracked[act];
            ctl->withheld = meta->withheld[act];
            ctl->error = 0;
            ctl->have_prev = 0;
            ctl->cur.c = ctl->cur.s = ctl->cur2.c = ctl->cur2.s = 0.0;
            ctl->cur.pad_ = ctl->cur2.pad_ = 0;
            ctl->rot = 0;
        }
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const T*>(a.buf[act]) +
                                                          (uint64_t)p * NVALS);
        constexpr uint32_t NVEC = (uint32_t)(NVALS * sizeof(T) / 16);
        for (uint32_t i = tid; i < NVEC; i += NTH) sm_at<uint4>(S::POOL_OFF + i * 16) = src[i];
    }
    __syncthreads();

    const uint64_t len = a.lay.len_base + (p < a.lay.len_extra ? 1 : 0);
    const uint64_t out_base =
        (uint64_t)p * a.lay.off_stride + (p < a.lay.off_extra ? p : a.lay.off_extra);
    const uint32_t f = a.f;
    const uint32_t mode = a.mode;
    const EmitCfg ec{a.mu, a.sigma, a.out_f32, a.unit};
    const bool bulk_on = EM == EM_UNIT && op == OP_FILL && a.bulk_emit != 0;
    // bulk span alignment in elements: the ragged head (< bvec) must stay
    // inside column group 0 and the tail (< bvec + VEC) inside the last one
    constexpr uint32_t kVec = 16 / (uint32_t)sizeof(T);
    constexpr uint32_t kTailCols = NTH;  // warp-stored tail: last column group only
    uint32_t bvec = 0;
    if (bulk_on) {
        bvec = kVec;
        const uint32_t want = a.bulk_emit / (uint32_t)sizeof(T);
        while (bvec * 2 <= want && bvec * 2 <= NTH && bvec * 2 + kVec <= kTailCols + 2) bvec *= 2;
    }
    PeriodCounter drift, restart;
    drift.init(a.drift, pc);
    restart.init(a.restart, pc);

    // ---- passes in this launch (the last one keeps its source pool as the
    // inactive buffer, as advance_pass's swap does, wallace.cpp:170-174) ---
    uint64_t total_passes = 0;
    const uint64_t done0 = resume ? meta->fill_done : 0;
    if (op == OP_FILL) {
        uint64_t rem = len - umin64(len, done0);
        if (avail > 0 && rem > 0) rem -= umin64(rem, avail);
        if (a.restart == 0) {
            total_passes = (rem + CAP - 1) / CAP * f;
        } else {
            PeriodCounter r2 = restart;
            while (rem > 0) {
                const bool rs = r2.will_cross(f);
                r2.advance(f);
                total_passes += f;
                if (rs) continue;
                rem -= umin64(rem, CAP);
            }
        }
    } else if (op == OP_PASSES) {
        total_passes = a.npasses;
    } else if (op == OP_REFILL) {
        total_passes = f;
    }

    uint64_t pass_i = 0;
    bool primed = false;  // parameter slot `slot` holds the next pass's parameters
    int slot = 0;
    int err = 0;
    char* outc = static_cast<char*>(a.out);
    const uint32_t esz = EM == EM_UNIT ? (uint32_t)sizeof(T) : (a.out_f32 ? 4u : 8u);

    auto prev_buf = [&]() -> T* {
        return static_cast<T*>(a.buf[ctl->active]) + (uint64_t)p * NVALS;
    };

    uint64_t done = done0;
    bool pending = false;  // stopped at a restart the host performs
    if (op == OP_FILL && avail > 0 && len > 0) {
        // leftover of the live pool: flat [pos, pos + take)
        const uint64_t take = umin64(len, avail);
        const uint64_t pos = CAP - avail;
        char* o = outc + out_base * esz;
        const T* pl = &sm_at<T>(S::POOL_OFF);
        for (uint64_t i = tid; i < take; i += NTH) {
            emit_one<T, EM>(o, i, pl[pos + i], ec.out_f32, ec.unit, ec.mu, ec.sigma);
            if constexpr (EM == EM_STATS) ec.add((double)pl[pos + i]);
        }
        done = take;
        avail -= take;
    }
    bool once = op == OP_REFILL;
    while (!err && ((op == OP_FILL && done < len) || once)) {
        once = false;
        // refill (wallace.cpp:188-196), the exposed window fused into the
        // last pass.
        const bool will_restart = restart.will_cross(f);
        const bool will_drift = drift.will_cross(f);
        const uint64_t want = op == OP_FILL ? umin64(len - done, CAP) : 0;
        const uint32_t emit_n = will_restart ? 0u : (uint32_t)want;
        char* out_p = outc + (out_base + done) * esz;
        for (uint32_t i = 0; i < f; ++i) {
            const bool lastp = i + 1 == f;
            if (!primed) {
                if (tid < 32) draw_pass_params_warp<NA>(tab, ctl, wbuf, N, slot);
                __syncthreads();
            }
            ++pass_i;
            const bool last_launch = pass_i == total_passes;
            // no prefetch across a restart (it draws the Box-Muller uniforms
            // first) or an audit (a failing audit leaves the uniform state
            // where the reference's exception leaves it, wallace.cpp:192)
            const bool prefetch = !last_launch && !(lastp && (will_restart || will_drift));
            const uint32_t en = lastp ? emit_n : 0u;
            const bool ok =
                last_launch
                    ? smem_pass<T, NA, LOGN, EM, AL, true>(pool_s, mode, en, out_p, ec, nullptr,
                                                           prefetch, prev_buf(), slot, bvec)
                    : smem_pass<T, NA, LOGN, EM, AL, false>(pool_s, mode, en, out_p, ec, nullptr,
                                                            prefetch, nullptr, slot, bvec);
            if (!ok) {
                err = ctl->error;
                break;
            }
            primed = prefetch;
            if (prefetch) slot ^= 1;
            ++pc;
        }
        if (err) break;
        restart.advance(f);
        drift.advance(f);
        avail = CAP;
        if (will_drift && !smem_drift_check<T, NA, LOGN>()) {
            err = ctl->error;
            break;
        }
        if (will_restart) {
            avail = 0;
            primed = false;
            if (a.host_restart) {  // glibc Box-Muller on the host (capi.cu)
                pending = true;
                break;
            }
            smem_restart<T, NA, LOGN>();
            continue;
        }
        done += emit_n;
        avail -= emit_n;
    }
    if (op == OP_FILL && !err && !pending) emitted += len;
    if (op == OP_PASSES) {
        for (uint32_t i = 0; i < a.npasses && !err; ++i) {
            // advance_pass (wallace.cpp:169-178)
            if (!primed) {
                if (tid < 32) draw_pass_params_warp<NA>(tab, ctl, wbuf, N, slot);
                __syncthreads();
            }
            ++pass_i;
            const bool last_launch = pass_i == total_passes;
            wrng_gpu_params* rec = (a.params_out && last_launch) ? a.params_out + p : nullptr;
            if (!smem_pass<T, NA, LOGN, EM, AL, true>(pool_s, mode, 0u, nullptr, ec, rec,
                                                      !last_launch,
                                                      last_launch ? prev_buf() : nullptr, slot,
                                                      0u)) {
                err = ctl->error;
                break;
            }
            primed = !last_launch;
            if (primed) slot ^= 1;
            ++pc;
            avail = 0;
        }
    }
    if (op == OP_DRIFT) {
        if (!smem_drift_check<T, NA, LOGN>()) err = ctl->error;
    } else if (op == OP_RESTART || op == OP_INIT) {
        smem_restart<T, NA, LOGN>();
        avail = 0;
    }

    // ---- write back -------------------------------------------------------
    if (bulk_on && tid == 0) bulk_wait_all();  // bulk copies complete before exit
    __syncthreads();
    if constexpr (EM == EM_STATS) {
        // this pool's moment sums: lanes, then warps, in a fixed order
        double* red = &sm_at<double>(S::WBUF_OFF);  // [warps][4]
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            double x = ec.st[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
            if ((tid & 31u) == 0) red[(tid >> 5) * 4 + k] = x;
        }
        __syncthreads();
        if (tid < 4 && a.stats) {
            double x = 0.0;
            for (uint32_t w = 0; w < NTH / 32; ++w) x += red[w * 4 + tid];
            a.stats[(uint64_t)p * 4 + tid] += x;
        }
        __syncthreads();
    }
    const uint32_t act = ctl->active;
    if (ctl->rot == 0) {
        uint4* dst =
            reinterpret_cast<uint4*>(static_cast<T*>(a.buf[act]) + (uint64_t)p * NVALS);
        constexpr uint32_t NVEC = (uint32_t)(NVALS * sizeof(T) / 16);
        for (uint32_t i = tid; i < NVEC; i += NTH) dst[i] = sm_at<uint4>(S::POOL_OFF + i * 16);
    } else {  // back to natural order
        T* dst = static_cast<T*>(a.buf[act]) + (uint64_t)p * NVALS;
        const RotView<T> v{&sm_at<T>(S::POOL_OFF), S::MASK, ctl->rot};
        for (uint32_t i = tid; i < (uint32_t)NVALS; i += NTH) dst[i] = v[i];
    }
    for (uint32_t i = tid; i < kTable; i += NTH) lg->table[i] = tab[i];
    if (tid == 0) {
        lg->r = ctl->r;
        lg->draws = ctl->draws;
        meta->tracked[act] = ctl->tracked;
        meta->withheld[act] = ctl->withheld;
        if (ctl->have_prev) {
            meta->tracked[act ^ 1u] = ctl->prev_tracked;
            meta->withheld[act ^ 1u] = ctl->prev_withheld;
        }
        if (op == OP_INIT) {
            meta->tracked[1] = 0.0;
            meta->withheld[1] = 0.0;
        }
        meta->active = act;
        meta->pass_count = pc;
        meta->avail = avail;
        meta->emitted = emitted;
        meta->error = (uint32_t)err;
        meta->restart_pending = pending ? 1u : 0u;
        meta->fill_done = done;
    }
}

template <typename T, int NA, int LOGN, int EM, bool AL>
static cudaError_t go(const KernelArgs& a, cudaStream_t st) {
    using S = SmemShape<T, NA, LOGN>;
    auto kern = k_smem<T, NA, LOGN, EM, AL>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e != cudaSuccess) return e;
    if (a.op == OP_QUERY)
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(static_cast<int*>(a.out), kern,
                                                             (int)S::NTH, S::BYTES);
    kern<<<a.pools, S::NTH, S::BYTES, st>>>(a);
    return cudaGetLastError();
}

template <typename T, int NA, int LOGN>
static cudaError_t go_em(const KernelArgs& a, cudaStream_t st, bool unit_same, bool al) {
    using S = SmemShape<T, NA, LOGN>;
    if constexpr (S::CAN_ALIGN) {
        if (al)
            return a.stats      ? go<T, NA, LOGN, EM_STATS, true>(a, st)
                   : unit_same ? go<T, NA, LOGN, EM_UNIT, true>(a, st)
                               : go<T, NA, LOGN, EM_GENERIC, true>(a, st);
    }
    return a.stats      ? go<T, NA, LOGN, EM_STATS, false>(a, st)
           : unit_same ? go<T, NA, LOGN, EM_UNIT, false>(a, st)
                       : go<T, NA, LOGN, EM_GENERIC, false>(a, st);
}

template <typename T, int NA>
static cudaError_t dispatch(const KernelArgs& a, cudaStream_t st, bool unit_same, bool al) {
    constexpr uint32_t es = sizeof(T);
    switch (a.N) {
        case 1u << 8: return go_em<T, NA, 8>(a, st, unit_same, al);
        case 1u << 9: return go_em<T, NA, 9>(a, st, unit_same, al);
        case 1u << 10: return go_em<T, NA, 10>(a, st, unit_same, al);
        case 1u << 11: return go_em<T, NA, 11>(a, st, unit_same, al);
        case 1u << 12: return go_em<T, NA, 12>(a, st, unit_same, al);
        case 1u << 13:
            if constexpr (NA * (1u << 13) * es <= kSmemPoolMax)
                return go_em<T, NA, 13>(a, st, unit_same, al);
            else
                return cudaErrorInvalidValue;
        case 1u << 14:
            if constexpr (NA * (1u << 14) * es <= kSmemPoolMax)
                return go_em<T, NA, 14>(a, st, unit_same, al);
            else
                return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace WG_SMEM_NS
using namespace WG_SMEM_NS;
}  // namespace wg
