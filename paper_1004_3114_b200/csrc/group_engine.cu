// Group engine: TWO small pools per warp (BASELINE.json configs[4]: the 4x256
// shapes, and fp32 4x512).  A 4x256 pool gives one warp only 8 columns per
// thread, so in the one-CTA-per-pool engine (smem_impl.cuh) two thirds of a
// pass's instructions are its per-pass scalar work (parameter decode, fp64
// chi-squared scale, emission bookkeeping).  Here a pool belongs to a GROUP of
// G = N / J = 16 lanes (J = 16 columns per lane; fp32 4x512: 32), a warp — one
// CTA — carries 2 pools side by side, and every lane runs its own pool's
// scalar work: the fixed cost of a pass is paid once per warp for 2 pools.
// Groups synchronise with __syncwarp(group mask) only and never depend on one
// another, so a group whose control flow differs (another matrix variant, an
// error, one refill more) just diverges for that stretch.
//
// Same algorithm, state and results as k_smem (bit-identical, tested):
//   pass            wallace.cpp:113-137 in the modular form (a*j + g) & (N-1)
//   parameters      wallace.cpp:54-58 / docs/n4_spec.md §2 (9 words per pass)
//   scale           wallace.cpp:59-69
//   refill / fill   wallace.cpp:188-216
//   drift audit     wallace.cpp:225-234 with Pool::direct_sumsq (13-18)
// Differences in mechanism only:
//   * the lag table stays in global memory (LfgState::table, L2-resident):
//     a group produces the words of up to 28 passes at a time — the step
//     x[i] += x[i+334] is hazard-free for up to 273 consecutive words
//     (common.cuh) — into a 2 KiB shared word buffer; words a failing pass
//     leaves unconsumed are un-drawn (x[i] -= x[i+334]), so the generator
//     state after an error is the reference's;
//   * the drift audit of a 1024-term pool is the plain sequential loop on
//     lane 0 of each group (all groups of a warp audit on the same pass);
//   * the pool is ONE linear image in shared memory (flat index m*N + j at
//     position m*N + j + rot, rot < 16 bytes), so a full refill leaves as one
//     bulk copy whose source is 16-byte aligned whatever the output phase;
//     the < 16 ragged values at either end leave through warp stores;
//   * thread-to-column maps (k_group, "thread-to-column map") chosen per
//     dtype so that the groups of a warp do not collide on shared-memory
//     banks.
// Measured and not kept: the pools of a warp interleaved
// element by element (conflict-free, but no bulk-copy source: per-value warp
// stores of 32-byte segments cost 4.8 LSU cycles each, 1.49 ms per 2^30
// against 1.04 ms); 4 fp32 pools per warp at 8 warps per SM (64 % of the HBM
// roofline against 74-79 % for 2 pools per warp at 16 warps per SM).
// Fills only (unit output of the pool's dtype, no restarts); every other
// operation on such a handle runs on k_smem over the same device state.
#include <type_traits>

#include "common.cuh"

namespace wg {
namespace grp {

extern __shared__ __align__(16) unsigned char g_gsm[];

constexpr uint32_t kWPass = 28;                // passes per word batch
constexpr uint32_t kWWords = kWPass * 9;       // 252 <= 273: hazard-free step
constexpr uint32_t kWBytes = 2048;             // word buffer per pool
static_assert(kWWords * 8 <= kWBytes && kWWords <= kShortLag, "word batch");

template <typename T, int LOGN>
struct Shape {
    static constexpr uint32_t N = 1u << LOGN;
    static constexpr uint32_t ES = (uint32_t)sizeof(T);
    // columns per lane: 16 (64 data registers fp32, 128 fp64); fp32 4x512: 32.
    // (fp32 4x256 with J = 32 — 4 pools per warp, 8 warps per SM — measured 64 %.)
    static constexpr uint32_t J = ES == 4 ? (LOGN == 8 ? 16 : 32) : 16;
    static constexpr uint32_t G = N / J;              // lanes per pool
    static constexpr uint32_t PPW = 32 / G;           // pools per warp
    static_assert(G == 16 && PPW == 2, "group engine shapes: 2 pools per warp");
    static constexpr uint32_t ABYTES = N * ES;
    // a pool in shared memory: flat index i = m*N + j at position i + rot,
    // rot < VEC (one linear image, so a full refill is ONE bulk copy)
    static constexpr uint32_t PBYTES = 4 * ABYTES + 16;
    static constexpr uint32_t MASK = N - 1;
    static constexpr uint32_t MASKB = MASK * ES;
    static constexpr uint32_t NVALS = 4 * N;
    static constexpr uint32_t CAP = NVALS - 1;
    static constexpr uint32_t VEC = 16 / ES;
    // CTAs per SM the register budget must allow: 16 at 64 data registers (12
    // at 166 registers measured 72 % against 74.8 %), else 8
    static constexpr uint32_t MINB = (J * ES <= 64) ? 16 : 8;
    // fp32: residue-class thread-to-column map (k_group, "thread-to-column map")
    static constexpr bool R4 = ES == 4;
    // shared layout: word buffers | pools
    static constexpr uint32_t BYTES = PPW * kWBytes + PPW * PBYTES;
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

// L2 policy of the output copies (0 none, 1 evict_first, 2 evict_last).  With
// thousands of 4 KiB output streams evict_first measured +2 % (fp32 4x256 R = 1:
// 78.6-78.9 % against 76.7-77.1 %; evict_last 75.1 %); on C3's 16 KiB refills
// (smem_impl.cuh) both hints cost 2 % (92.6 % against 94.9 %), so k_smem has none.
#ifndef WG_EXP_BULK_HINT
#define WG_EXP_BULK_HINT 1
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
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Packed fp32 (Blackwell add/sub/mul.rn.f32x2: each half rounds like the
// scalar operation).
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

// One thread's columns of a pass: fp32 as packed pairs of columns (2kp, 2kp+1).
template <typename T, uint32_t J>
struct Cols {
    T v[4][J];
};
template <uint32_t J>
struct Cols<float, J> {
    f2_t v[4][J / 2];
};

// Unscaled n = 4 transform in place (docs/n4_spec.md §3; operation order of
// smem_impl.cuh's transform_b / transform_b2).
template <typename T, uint32_t J>
__device__ __forceinline__ void transform(Cols<T, J>& u, uint32_t variant) {
    if constexpr (sizeof(T) == 4) {
        if (variant == 0) {
            sfor<0, (int)J / 2>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                const f2_t G0 = u.v[0][k], G1 = u.v[1][k], G2 = u.v[2][k], G3 = u.v[3][k];
                const f2_t PP = f2_add(G0, G1), Q = f2_sub(G0, G1);
                const f2_t R = f2_add(G2, G3), Sd = f2_sub(G2, G3);
                u.v[0][k] = f2_add(PP, R);
                u.v[1][k] = f2_add(Q, Sd);
                u.v[2][k] = f2_sub(PP, R);
                u.v[3][k] = f2_sub(Q, Sd);
            });
        } else {
            const f2_t H = f2_pack(0.5f, 0.5f);
            sfor<0, (int)J / 2>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                const f2_t G0 = u.v[0][k], G1 = u.v[1][k], G2 = u.v[2][k], G3 = u.v[3][k];
                const f2_t Tt = f2_mul(H, f2_add(f2_add(G0, G1), f2_add(G2, G3)));
                u.v[0][k] = f2_sub(Tt, G0);
                u.v[1][k] = f2_sub(Tt, G1);
                u.v[2][k] = f2_sub(Tt, G2);
                u.v[3][k] = f2_sub(Tt, G3);
            });
        }
    } else {
        if (variant == 0) {
            sfor<0, (int)J>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                const T g0 = u.v[0][k], g1 = u.v[1][k], g2 = u.v[2][k], g3 = u.v[3][k];
                const T pp = g0 + g1, q = g0 - g1, r = g2 + g3, s = g2 - g3;
                u.v[0][k] = pp + r;
                u.v[1][k] = q + s;
                u.v[2][k] = pp - r;
                u.v[3][k] = q - s;
            });
        } else {
            sfor<0, (int)J>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                const T g0 = u.v[0][k], g1 = u.v[1][k], g2 = u.v[2][k], g3 = u.v[3][k];
                const T t = (T)0.5 * ((g0 + g1) + (g2 + g3));
                u.v[0][k] = t - g0;
                u.v[1][k] = t - g1;
                u.v[2][k] = t - g2;
                u.v[3][k] = t - g3;
            });
        }
    }
}

// Phase C bookkeeping of a bulk-emitting pass (smem_impl.cuh's PhaseC with
// the group for the CTA).
struct PhaseC {
    uint32_t j0;    // flat [0, j0): ragged head, stored by the lanes holding it
    uint32_t jend;  // flat [j0, jend): the bulk copy; [jend, 4N - 1): ragged tail
};

template <typename T, int LOGN>
__global__ void __launch_bounds__(32, Shape<T, LOGN>::MINB) k_group(const KernelArgs a) {
    using S = Shape<T, LOGN>;
    constexpr uint32_t N = S::N, G = S::G, J = S::J, ES = S::ES, VEC = S::VEC, PPW = S::PPW;
    constexpr bool R4 = S::R4;
    constexpr uint32_t NT = J / PPW;  // R4: slots k = t*PPW + r, t < NT
    constexpr uint64_t CAP = S::CAP;
    const uint32_t lane = threadIdx.x;
    const uint32_t q = lane / G, gl = lane % G;
    const uint32_t gmask = ((1u << G) - 1u) << (q * G);
    const uint32_t p = blockIdx.x * PPW + q;
    if (p >= a.pools) return;  // the other groups never wait for this one
    PoolMeta* meta = a.meta + p;
    LfgState* lg = a.lfg + p;
    // a device-raised error is sticky until the host observes it
    if (meta->error) return;

    const uint32_t base_s = (uint32_t)__cvta_generic_to_shared(g_gsm);
    uint64_t* wbuf = reinterpret_cast<uint64_t*>(g_gsm + q * kWBytes);
    const uint32_t pool_s = base_s + PPW * kWBytes + q * S::PBYTES;  // 16-byte aligned
    T* const pool = reinterpret_cast<T*>(g_gsm + (pool_s - base_s));
    uint64_t* tab = lg->table;

    // ---- load state -------------------------------------------------------
    // (loop state is kept in 32-bit counters: the host sends a fill here only
    // when every pool's passes in the call stay below 2^31)
    uint32_t avail = (uint32_t)meta->avail;  // <= CAP
    uint32_t act = meta->active;
    double tracked = meta->tracked[act], withheld = meta->withheld[act];
    uint32_t r = lg->r;  // cursor at the start of the current word batch
    {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const T*>(a.buf[act]) +
                                                          (uint64_t)p * S::NVALS);
        uint4* dst = reinterpret_cast<uint4*>(pool);
        constexpr uint32_t NVEC = S::NVALS * ES / 16;
        for (uint32_t i = gl; i < NVEC; i += G) dst[i] = src[i];
    }
    __syncwarp(gmask);

    const uint64_t len = a.lay.len_base + (p < a.lay.len_extra ? 1 : 0);
    const uint64_t out_base =
        (uint64_t)p * a.lay.off_stride + (p < a.lay.off_extra ? p : a.lay.off_extra);
    T* const outv = static_cast<T*>(a.out) + out_base;
    const uint32_t f = a.f, mode = a.mode;
    // bulk span alignment in elements (a power of two, 16 bytes to 16
    // elements).  The ragged head (< bvec values of array 0) and tail (< bvec
    // values of array 3) leave through warp stores from the slots that hold
    // the first / last 16 columns.
    uint32_t bvec = VEC;
    {
        const uint32_t want = a.bulk_emit / ES;
        while (bvec * 2 <= want && bvec * 2 <= 16) bvec *= 2;
    }
    // passes until the next drift audit (wallace.cpp:182-184: the refill that
    // moves pass_count across a multiple of the period); ~0u: none in this call
    uint32_t dper = 0, dleft = ~0u;
    if (a.drift) {
        const uint64_t until = a.drift - meta->pass_count % a.drift;
        if (a.drift <= 0x7fffffffull) dper = (uint32_t)a.drift;
        if (until <= 0x7fffffffull) dleft = (uint32_t)until;
    }

    uint32_t take = 0;
    if (avail > 0 && len > 0) {
        // leftover of the live pool: flat [pos, pos + take)
        take = (uint32_t)umin64(len, avail);
        const uint32_t pos = (uint32_t)CAP - avail;
        for (uint32_t i = gl; i < take; i += G) outv[i] = pool[pos + i] + (T)0;
        avail -= take;
    }
    // refills of this call: all full but the last, which exposes last_n values
    const uint32_t nref = (uint32_t)((len - take + CAP - 1) / CAP);
    const uint32_t last_n = nref ? (uint32_t)(len - take - (uint64_t)(nref - 1) * CAP) : 0u;
    uint32_t ref_left = nref;
    uint32_t passes_left = nref * a.f;
    T* out_p = outv + take;

    // ---- thread-to-column map ------------------------------------------------
    // R4 (fp32): slot (t, r) of lane gl holds column j = 32 t + PPW gl + rr[r],
    //   rr[r] = (r + cq) mod PPW.  The G lanes of a group then touch, in one
    //   instruction, columns PPW apart: gathers (odd stride a) and stores hit G
    //   distinct banks of ONE residue class mod PPW, so two groups collide
    //   only when their classes coincide (whole-or-nothing: 2.1 wavefronts per
    //   gather on average against 3.1 for consecutive columns) and never on
    //   stores: cq = q - (output phase of the group's first refill), which
    //   keeps (rr[r] + rot) mod PPW distinct across the groups for as long as
    //   they refill in step.
    // else (fp64: a group is a half-warp, which 64-bit accesses serve
    //   separately): slot k holds column (k G + lane) mod N — lane of the
    //   WARP, so the stores of a warp spread over all banks; the last PPW
    //   slots can wrap.
    uint32_t rr[PPW], jr[PPW];
    if constexpr (R4) {
        const uint32_t d0 = (uint32_t)(reinterpret_cast<uintptr_t>(out_p) / ES);
        const uint32_t cq = q - d0;
#pragma unroll
        for (uint32_t x = 0; x < PPW; ++x) {
            rr[x] = (x + cq) & (PPW - 1);
            jr[x] = PPW * gl + rr[x];
        }
    }

    uint32_t nstart = 0;  // passes whose words were consumed
    uint32_t rot = 0;     // value j of each array sits at (j + rot) mod N
    uint32_t wleft = 0;   // passes whose words are still in wbuf
    uint32_t wpos = 0;    // next word in wbuf
    uint32_t wcnt = 0;    // words of the current batch
    int err = 0;
    bool scale_err = false;
    bool bulk_pending = false;

    while (ref_left > 0) {
        // refill (wallace.cpp:188-196), the exposed window fused into its last pass
        const bool will_drift = f >= dleft;
        const uint32_t emit_n = ref_left == 1 ? last_n : (uint32_t)CAP;
        for (uint32_t i = 0; i < f; ++i) {
            if (wleft == 0) {
                // next batch of uniform words, straight from the global lag table
                r += wcnt;
                r = r >= kTable ? r - kTable : r;
                wleft = passes_left < kWPass ? passes_left : kWPass;
                wcnt = wleft * 9;
                wpos = 0;
#pragma unroll 4
                for (uint32_t k = gl; k < wcnt; k += G) {
                    uint32_t ii = r + k;
                    ii = ii >= kTable ? ii - kTable : ii;
                    uint32_t ss = ii + kGap;
                    ss = ss >= kTable ? ss - kTable : ss;
                    const uint64_t w = __ldcg(tab + ii) + __ldcg(tab + ss);
                    __stcg(tab + ii, w);
                    wbuf[k] = w;
                }
                __syncwarp(gmask);
            }
            --passes_left;
            const bool last_launch = passes_left == 0;
            const uint32_t en = i + 1 == f ? emit_n : 0u;

            // ---- this pass's parameters (docs/n4_spec.md §2) --------------
            uint32_t strd[4], offs[4];
            uint32_t variant;
            {
                const uint64_t* w = wbuf + wpos;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const uint32_t lo = m == 0 ? 3u : m == 1 ? 7u : m == 2 ? 13u : 19u;
                    strd[m] = (w[m] >> 63) ? lo + (m == 0 ? 2u : 4u) : lo;
                    offs[m] = (uint32_t)(w[4 + m] >> (64 - LOGN));
                }
                variant = (uint32_t)(w[8] >> 63);
            }
            wpos += 9;
            --wleft;
            ++nstart;
            // (every lane runs the fp64 scale chain: on lane 0 of the group with a
            // broadcast — 1.1 % faster for C3 in smem_impl.cuh — the f >= 2 fills
            // here lost 3 %, the f = 1 fills nothing)
            double scale = 0.0, target = 0.0;
            if (pass_scale(tracked, withheld, S::NVALS, mode, scale, target)) {
                err = WRNG_GPU_ECORRUPT;  // wallace.cpp:59-61, after the draws
                scale_err = true;
                break;
            }
            // regenerate folds the scale into the matrix (wallace.cpp:116-117)
            const T c0 = (T)(variant ? scale : 0.5 * scale);
            if (last_launch) {
                // the pre-pass pool becomes the inactive buffer (wallace.cpp:170-174)
                T* prev = static_cast<T*>(a.buf[act]) + (uint64_t)p * S::NVALS;
                for (uint32_t k = gl; k < S::NVALS; k += G) prev[k] = pool[k + rot];
                if (gl == 0) {
                    meta->tracked[act] = tracked;
                    meta->withheld[act] = withheld;
                }
            }
            // emission mode: 0 none, 2 warp stores of the window [0, en),
            // 3 full refill through the bulk-copy engine
            const uint32_t md = en == 0 ? 0u : en == (uint32_t)CAP ? 3u : 2u;
            // new rotation: on a bulk-emitting pass, the output's 16-byte phase
            const uint32_t ophase = (uint32_t)(reinterpret_cast<uintptr_t>(out_p) / ES);
            const uint32_t rot2 = md == 3 ? ophase & (VEC - 1) : rot;
            PhaseC c;
            {
                const uint32_t ph = ophase & (bvec - 1);
                c.j0 = (bvec - ph) & (bvec - 1);
                c.jend = c.j0 + (((uint32_t)CAP - c.j0) & ~(bvec - 1));
            }
            // store addresses: sb[x] + immediate; wj[x]: the columns of the
            // last PPW slots (fp64 map: they can wrap)
            uint32_t sb[R4 ? PPW : 1], wj[PPW], wa[PPW];
            if constexpr (R4) {
#pragma unroll
                for (uint32_t x = 0; x < PPW; ++x) {
                    sb[x] = pool_s + (jr[x] + rot2) * ES;
                    wj[x] = (NT - 1) * 32 + jr[x];
                    wa[x] = sb[x] + (NT - 1) * 32 * ES;
                }
            } else {
                sb[0] = pool_s + (lane + rot2) * ES;
#pragma unroll
                for (uint32_t x = 0; x < PPW; ++x) {
                    wj[x] = ((J - PPW + x) * G + lane) & S::MASK;
                    wa[x] = pool_s + (wj[x] + rot2) * ES;
                }
            }
            const uint32_t gbase = pool_s + rot * ES;  // gather base: value i at i + rot

            // ---- phase B: gather every column, then the transform ---------
            Cols<T, J> u;
            if constexpr (R4) {
                // pairs of residues outside, t inside: 2 x 4 running indices
                sfor<0, (int)PPW / 2>([&](auto rpc) {
                    constexpr int rp = decltype(rpc)::value;
                    uint32_t ix[2][4], stp[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const uint32_t bs = strd[m] * PPW * gl + offs[m];
                        ix[0][m] = (bs + strd[m] * rr[2 * rp]) * ES;
                        ix[1][m] = (bs + strd[m] * rr[2 * rp + 1]) * ES;
                        stp[m] = strd[m] * 32 * ES;
                    }
                    sfor<0, (int)NT>([&](auto tc) {
                        constexpr int t = decltype(tc)::value;
                        constexpr int kp = (t * (int)PPW + 2 * rp) / 2;
                        float g[4][2];
                        sfor<0, 2>([&](auto hc) {
                            constexpr int h = decltype(hc)::value;
                            sfor<0, 4>([&](auto mc) {
                                constexpr int m = decltype(mc)::value;
                                g[m][h] = lds<float, (uint32_t)m * S::ABYTES>(
                                    (ix[h][m] & S::MASKB) + gbase);
                                ix[h][m] += stp[m];
                            });
                        });
                        sfor<0, 4>([&](auto mc) {
                            constexpr int m = decltype(mc)::value;
                            u.v[m][kp] = f2_pack(g[m][0], g[m][1]);
                        });
                    });
                });
            } else {
                uint32_t ixb[4], stepb[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    ixb[m] = (strd[m] * lane + offs[m]) * ES;  // slot 0: column lane
                    stepb[m] = strd[m] * G * ES;
                }
                sfor<0, (int)J>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    sfor<0, 4>([&](auto mc) {
                        constexpr int m = decltype(mc)::value;
                        u.v[m][k] =
                            lds<T, (uint32_t)m * S::ABYTES>((ixb[m] & S::MASKB) + gbase);
                        ixb[m] += stepb[m];
                    });
                });
            }
            transform<T, J>(u, variant);
            // phase C rewrites the pool: the group's gathers are done, and the
            // previous refill's bulk copies have read it
            if (bulk_pending && gl == 0) bulk_wait_read();
            __syncwarp(gmask);

            // ---- phase C: scale, store in place (rotated), emit -----------
            double wh = 0.0;
            // one instantiation per emission mode MD
            auto phase_c = [&](auto mdc) {
                constexpr uint32_t MD = decltype(mdc)::value;
                // value y of array m in slot k: into the pool, and to the output
                // where this lane emits it itself
                auto put = [&](auto mc, auto kc, T y) {
                    constexpr int m = decltype(mc)::value;
                    constexpr int k = decltype(kc)::value;
                    // emitted form 0 + 1 * v (-0.0 -> +0.0); on MD 3 the pool
                    // holds it, being the bulk source
                    const T e = MD == 0 ? y : y + (T)0;
                    const T sv = MD == 3 ? e : y;
                    constexpr int x = R4 ? k % (int)PPW : k - (int)(J - PPW);
                    constexpr bool first = R4 ? k < (int)PPW : k == 0;
                    constexpr bool last = R4 ? k >= (int)(J - PPW) : k >= (int)(J - PPW);
                    if constexpr (!last) {
                        constexpr uint32_t o = R4 ? (uint32_t)(k / (int)PPW) * 32 : (uint32_t)k * G;
                        const uint32_t j = o + (R4 ? jr[x] : lane);  // no wrap
                        sts<T, (uint32_t)m * S::ABYTES + o * ES>(sb[R4 ? x : 0], sv);
                        if constexpr (MD == 3 && first && m == 0) {  // ragged head
                            if (j < c.j0) out_p[j] = e;
                        }
                        if constexpr (MD == 2) {
                            if ((uint32_t)m * N + j < en) out_p[(uint32_t)m * N + j] = e;
                        }
                    } else {
                        const uint32_t j = wj[x];
                        sts<T, (uint32_t)m * S::ABYTES>(wa[x], sv);
                        if constexpr (MD == 3 && !R4 && m == 0) {  // ragged head (fp64 map)
                            if (j < c.j0) out_p[j] = e;
                        }
                        if constexpr (MD == 3 && m == 3) {  // ragged tail, withheld slot excluded
                            if (3 * N + j >= c.jend && j != N - 1) out_p[3 * N + j] = e;
                        }
                        if constexpr (MD == 2) {
                            if ((uint32_t)m * N + j < en) out_p[(uint32_t)m * N + j] = e;
                        }
                        if constexpr (m == 3) {
                            if (j == N - 1) wh = (double)y;
                        }
                    }
                };
                if constexpr (ES == 4) {
                    const f2_t C = f2_pack(c0, c0), Z = f2_pack(0.0f, 0.0f);
                    sfor<0, (int)J / 2>([&](auto kc) {
                        constexpr int kp = decltype(kc)::value;
                        constexpr int k0 = 2 * kp;
                        sfor<0, 4>([&](auto mc) {
                            constexpr int m = decltype(mc)::value;
                            const f2_t Y = f2_mul(C, u.v[m][kp]);
                            float y0, y1;
                            if constexpr (MD == 3 && k0 >= (int)PPW && k0 + 1 < (int)(J - PPW)) {
                                // nothing to emit here: only the pool's emitted form
                                f2_unpack(f2_add(Y, Z), y0, y1);
                                constexpr uint32_t o = (uint32_t)m * S::ABYTES +
                                                       (uint32_t)(k0 / (int)PPW) * 32 * ES;
                                sts<T, o>(sb[k0 % (int)PPW], y0);
                                sts<T, o>(sb[(k0 + 1) % (int)PPW], y1);
                            } else {
                                f2_unpack(Y, y0, y1);
                                put(mc, std::integral_constant<int, k0>{}, y0);
                                put(mc, std::integral_constant<int, k0 + 1>{}, y1);
                            }
                        });
                    });
                } else {
                    sfor<0, (int)J>([&](auto kc) {
                        constexpr int k = decltype(kc)::value;
                        sfor<0, 4>([&](auto mc) {
                            constexpr int m = decltype(mc)::value;
                            put(mc, kc, c0 * u.v[m][k]);
                        });
                    });
                }
            };
            if (md == 0)
                phase_c(std::integral_constant<uint32_t, 0>{});
            else if (md == 3)
                phase_c(std::integral_constant<uint32_t, 3>{});
            else
                phase_c(std::integral_constant<uint32_t, 2>{});
            if (md == 3) fence_async_smem();  // generic -> async proxy
            tracked = target;                                  // wallace.cpp:135
            withheld = __shfl_sync(gmask, wh, G - 1, G);       // wallace.cpp:136
            act ^= 1u;
            rot = rot2;
            __syncwarp(gmask);
            if (md == 3) {
                if (gl == 0) {
                    // flat [j0, jend) -> output: one copy, 16-byte aligned on both sides
                    bulk_store(reinterpret_cast<uint64_t>(out_p + c.j0),
                               pool_s + (c.j0 + rot2) * ES, (c.jend - c.j0) * ES);
                    bulk_commit();
                }
                bulk_pending = true;
            }
        }
        if (err) break;
        if (will_drift) {
            const uint32_t over = f - dleft;
            dleft = dper ? dper - over % dper : ~0u;
        } else if (dleft != ~0u) {
            dleft -= f;
        }
        avail = (uint32_t)CAP;
        if (will_drift) {
            // wallace.cpp:225-234 with Pool::direct_sumsq order (wallace.cpp:13-18)
            double rec = 0.0;
            if (gl == 0) {
#pragma unroll 8
                for (uint32_t k = 0; k < S::NVALS; ++k) {
                    const double d = (double)pool[rot + k];
                    rec = rec + d * d;
                }
            }
            rec = __shfl_sync(gmask, rec, 0, G);
            const double rel = fabs(rec / tracked - 1.0);
            if (!(rel <= 1e-3)) {
                err = WRNG_GPU_ECORRUPT;
                break;
            }
            tracked = rec;
        }
        out_p += emit_n;
        avail -= emit_n;
        --ref_left;
    }

    // ---- write back -------------------------------------------------------
    if (bulk_pending && gl == 0) bulk_wait_all();  // bulk copies complete before exit
    // words drawn ahead of a failing pass are un-drawn (x[i] -= x[i+334]; the
    // slots a batch reads are not written by it)
    for (uint32_t k = wpos + gl; k < wcnt; k += G) {
        uint32_t ii = r + k;
        ii = ii >= kTable ? ii - kTable : ii;
        uint32_t ss = ii + kGap;
        ss = ss >= kTable ? ss - kTable : ss;
        __stcg(tab + ii, __ldcg(tab + ii) - __ldcg(tab + ss));
    }
    r += wpos;
    r = r >= kTable ? r - kTable : r;
    __syncwarp(gmask);
    if (nstart > 0) {
        T* dst = static_cast<T*>(a.buf[act]) + (uint64_t)p * S::NVALS;
        if (rot == 0) {
            constexpr uint32_t NVEC = S::NVALS * ES / 16;
            for (uint32_t i = gl; i < NVEC; i += G)
                reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(pool)[i];
        } else {  // unshifted
            for (uint32_t i = gl; i < S::NVALS; i += G) dst[i] = pool[i + rot];
        }
    }
    if (gl == 0) {
        lg->r = r;
        lg->draws += (uint64_t)nstart * 9;
        meta->tracked[act] = tracked;
        meta->withheld[act] = withheld;
        meta->active = act;
        meta->pass_count += nstart - (scale_err ? 1u : 0u);
        meta->avail = avail;
        if (!err) meta->emitted += len;
        meta->error = (uint32_t)err;
        meta->restart_pending = 0u;
        meta->fill_done = err ? take + (uint64_t)(nref - ref_left) * CAP : len;
    }
}

template <typename T, int LOGN>
static cudaError_t go(const KernelArgs& a, cudaStream_t st) {
    using S = Shape<T, LOGN>;
    auto kern = k_group<T, LOGN>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    if (e != cudaSuccess) return e;
    if (a.op == OP_QUERY) {  // pools per SM
        int ctas = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, kern, 32, S::BYTES);
        // f = 1 fills are bound by the output pattern, not by generation:
        // fewer, longer output streams measured faster — 3/4 of the occupancy
        // limit (fp32 4x256: 24 pools per SM 76-79 % of the HBM roofline, 32 per
        // SM 73 %; fp64 4x256: 12 per SM 87.6 %, 16 per SM 83.5 %)
        // (4x256 only: fp32 4x512 runs 83.5 % with all 16 pools per SM, 76 % with 12)
        if (a.f == 1 && S::N == 256) ctas = ctas * 3 / 4;
        *static_cast<int*>(a.out) = ctas * (int)S::PPW;
        return e;
    }
    kern<<<(a.pools + S::PPW - 1) / S::PPW, 32, S::BYTES, st>>>(a);
    return cudaGetLastError();
}

}  // namespace grp

// Shapes the group engine takes (measured against one CTA per pool, one wave
// of pools each, 2^32 normals, % of the HBM-store roofline):
// fp32 4x256 f = 1..4: 77-79 / 57 / 39 / 30 % against 44 / 25 / 18 / 14 %; fp32
// 4x512 f = 1, 2: 85 / 50 % against 71 / 39 %; fp64 4x256 f = 1..4: 85-88 / 70 /
// 49 / 38 % against 81 / 47 / 34 / 26 %.
bool group_engine_fits(uint32_t n_arrays, uint32_t dtype, uint32_t N, uint32_t f) {
    if (n_arrays != 4) return false;
    (void)f;
    return dtype == WRNG_GPU_F64 ? N == 256 : (N == 256 || N == 512);
}

cudaError_t launch_group(uint32_t dtype, const KernelArgs& a, cudaStream_t st) {
    if (dtype == WRNG_GPU_F64) {
        if (a.N == 256) return grp::go<double, 8>(a, st);
    } else {
        if (a.N == 256) return grp::go<float, 8>(a, st);
        if (a.N == 512) return grp::go<float, 9>(a, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace wg
