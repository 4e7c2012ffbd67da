// Internal declarations shared by the kernel translation units (smem_*.cu,
// hbm_engine.cu, cluster_engine.cu, misc.cu, baselines.cu) and capi.cu (the extern "C" ABI in include/wrng_gpu.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "wrng_gpu.h"

namespace wg {

constexpr uint32_t kTable = 607;          // lag table size (uniform.hpp:17)
constexpr uint32_t kShortLag = 273;       // (uniform.hpp:18)
constexpr uint32_t kGap = kTable - kShortLag;  // cursor_s - cursor_r = 334
constexpr uint32_t kWarmup = 10 * kTable;      // uniform.cpp:30

// Per-pool uniform generator, device resident (UniformState, uniform.hpp:16-29).
// cursor_s is implied: (r + 334) mod 607 (serialize.cpp:145-148 invariant).
struct LfgState {
    uint64_t table[kTable];
    uint32_t r;
    uint32_t pad_;
    uint64_t draws;
};

// Per-pool bookkeeping, device resident.  tracked/withheld per buffer as in
// Pool (wallace.hpp:36-40); counters as in WallaceState (wallace.hpp:167-172).
struct PoolMeta {
    double tracked[2];
    double withheld[2];
    uint64_t pass_count;
    uint64_t avail;
    uint64_t emitted;
    uint32_t active;
    uint32_t error;  // 0, or a wrng_gpu_status raised on the device
    // Host-side restarts (WRNG_GPU_INIT_HOST handles with restarts on): a
    // smem fill stops at a restart refill with restart_pending = 1 and
    // fill_done = values of the call already written; the host re-initialises
    // the pool with glibc's Box-Muller, sets restart_pending = 2 and relaunches
    // (KernelArgs::resume), which continues pools marked 2 from fill_done.
    uint64_t fill_done;
    uint32_t restart_pending;
    uint32_t pad_;
};

enum Op : uint32_t {
    OP_FILL = 0,     // WallaceState::fill
    OP_PASSES = 1,   // advance_pass x npasses
    OP_REFILL = 2,   // refill
    OP_DRIFT = 3,    // drift_check
    OP_RESTART = 4,  // restart
    OP_INIT = 5,     // seed uniform generators + init_pool
    OP_QUERY = 6,    // no launch: CTAs per SM of the fill kernel -> *(int*)out
};

// Output placement of a bank fill: pool p writes len_p values at
// out + p * off_stride + min(p, off_extra), len_p = len_base + (p < len_extra).
struct OutLayout {
    uint64_t off_stride;
    uint64_t off_extra;
    uint64_t len_base;
    uint64_t len_extra;
};

struct KernelArgs {
    void* buf[2];          // pool double buffer, pools * n_arrays * N each
    PoolMeta* meta;        // [pools]
    LfgState* lfg;         // [pools]
    void* out;             // output (device)
    OutLayout lay;
    double mu, sigma;
    uint32_t out_f32;      // 1: float output, 0: double output
    uint32_t unit;         // mu == 0 && sigma == 1
    uint32_t N;            // per-array length
    uint32_t f;            // throwaway_f
    uint32_t mode;         // scale mode
    uint32_t op;           // Op
    uint32_t npasses;      // OP_PASSES
    uint32_t pools;
    uint64_t restart;      // restart_interval_passes
    uint64_t drift;        // drift_check_period
    uint64_t seed, stream0;  // OP_INIT
    wrng_gpu_params* params_out;  // OP_PASSES: [pools], params of the last pass
    // HBM engine: persisting-L2 access window over both pool buffers
    void* l2_base;
    uint64_t l2_bytes;
    float l2_hit;
    // smem engine: full refills leave shared memory through the bulk-copy
    // engine (output must be aligned to its element size); the value is the
    // output alignment in bytes of each bulk span (0 = warp stores only)
    uint32_t bulk_emit;
    // 1: stop at a restart instead of running the device Box-Muller (the
    // host restarts the pool, PoolMeta::restart_pending); 1 with resume = 1:
    // continue the pools the host restarted
    uint32_t host_restart;
    uint32_t resume;
    // smem fills: non-null -> the emitting passes also add each pool's sums
    // of v, v^2, v^3, v^4 over its emitted values to stats[pool * 4 + k]
    double* stats;
};

struct EngineShape {
    uint32_t threads;   // CTA size
    uint32_t smem;      // dynamic shared memory bytes
    uint32_t j;         // pool columns per thread
};

// Shared-memory engine: one CTA per pool.
bool smem_engine_fits(uint32_t n_arrays, uint32_t dtype, uint32_t N);
EngineShape smem_engine_shape(uint32_t n_arrays, uint32_t dtype, uint32_t N);
cudaError_t launch_smem(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                        cudaStream_t st);
// Probes the dynamic shared-memory base of the current device once (the
// aligned pool layout needs its low bits to be 0x400).
void smem_engine_probe(cudaStream_t st);

// Group engine (group_engine.cu): 2 or 4 small n = 4 pools per warp; unit
// fills without restarts.  OP_QUERY writes the POOLS per SM to *(int*)out.
bool group_engine_fits(uint32_t n_arrays, uint32_t dtype, uint32_t N, uint32_t f);
cudaError_t launch_group(uint32_t dtype, const KernelArgs& a, cudaStream_t st);

// Cluster engine (cluster_engine.cu): one pool over a cluster of 8 CTAs,
// fills without restarts.
bool cluster_engine_fits(uint32_t n_arrays, uint32_t dtype, uint32_t N, uint32_t pools);
cudaError_t launch_cluster(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                           cudaStream_t st);

// HBM engine: one grid-wide launch per pass.
struct HbmPass {
    uint32_t src;        // buffer index read
    uint32_t param_idx;  // index into the per-pool params array
    uint64_t emit_n;     // emit flat [0, emit_n) of the new pool
    uint64_t out_off;    // ... to out + out_off
    uint32_t end_refill; // 1: last pass of a refill (sets avail = cap - emit_n)
};
// A run of consecutive passes (no drift audit, restart or leftover emission
// in between) executed by ONE persistent launch with grid-wide barriers
// between passes (k_hbm_run).  Pass i reads buffer src0 ^ (i & 1) and uses
// params[param0 + i]; emit_n[i] > 0 streams the new pool's flat [0, emit_n)
// to out + out_off[i].
constexpr uint32_t kRunMax = 64;
// k_hbm_run's device words: grid-barrier counter, then kRunMax 32-bit
// emission tile counters (packed two per word)
constexpr uint32_t kRunBarWords = 1 + kRunMax / 2;
// the dataflow run's per-row epoch flags (C <= 2048 rows) and per-64-row
// emission counters, after the barrier words
constexpr uint32_t kRunFlowRowWords = (2048 + 2048 / 64) / 2;
constexpr uint32_t kRunFlowWords = kRunFlowRowWords + kRunMax;  // + per-pass withheld slots
struct HbmRun {
    uint32_t npass, src0, param0, pad_;
    uint64_t end_mask;  // bit i: pass i ends a refill
    uint64_t emit_n[kRunMax];
    uint64_t out_off[kRunMax];
};
cudaError_t launch_hbm_run(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                           wrng_gpu_params* params, const HbmRun& run, unsigned long long* gbar,
                           cudaStream_t st);
cudaError_t launch_hbm_params(uint32_t n_arrays, uint32_t N, LfgState* lfg,
                              wrng_gpu_params* params, uint32_t npass, PoolMeta* meta,
                              cudaStream_t st);
cudaError_t launch_hbm_pass(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                            wrng_gpu_params* params, const HbmPass& ps,
                            cudaStream_t st);
cudaError_t launch_hbm_emit_t(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                              uint32_t buf, uint64_t emit_n, uint64_t out_off, cudaStream_t st);
cudaError_t launch_hbm_emit(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                            uint32_t buf, uint64_t pos, uint64_t take, uint64_t out_off,
                            cudaStream_t st);
size_t hbm_drift_scratch_bytes(uint64_t nvals);
cudaError_t launch_hbm_drift(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                             uint32_t buf, int tree, double* scratch,
                             cudaStream_t st);
cudaError_t launch_hbm_init(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                            uint32_t buf, int seed_lfg, void* scratch, cudaStream_t st);

// Transposed storage of HBM pools: array values i = 0..N-1 stored at
// (i mod C) * R + i / C with R = 2^lr = min(512, N), C = 2^lc = N / R.
struct HbmSplit {
    uint32_t lr, lc;
};
__host__ __device__ inline HbmSplit hbm_split(uint32_t N) {
    uint32_t L = 0;
    while ((1u << L) < N) ++L;
    HbmSplit s;
    s.lr = L < 9 ? L : 9;
    s.lc = L - s.lr;
    return s;
}
// storage position of flat pool index m*N + i
__host__ __device__ inline uint64_t hbm_pos(uint64_t flat, uint32_t N, HbmSplit s) {
    const uint32_t L = s.lr + s.lc;
    const uint64_t m = flat >> L, i = flat & (N - 1);
    return (m << L) + ((i & ((1ull << s.lc) - 1)) << s.lr) + (i >> s.lc);
}
cudaError_t launch_hbm_setmeta(PoolMeta* meta, uint64_t pass_count, uint64_t avail,
                               uint64_t emitted, uint32_t active, cudaStream_t st);

// Validation reductions.
cudaError_t launch_moments(const void* v, int is_f32, uint64_t n, double* partials,
                           uint32_t nblocks, double* out5_dev, cudaStream_t st);

// Uniformity / serial-correlation checks on P stream windows (misc.cu).
cudaError_t launch_uv_counts(const void* v, int is_f32, uint32_t P, uint64_t pitch,
                             uint64_t len, uint32_t k, unsigned long long* cu,
                             unsigned long long* cv, unsigned long long* skipped,
                             cudaStream_t st);
cudaError_t launch_ac_sums(const void* v, const void* tail, int is_f32, uint32_t P,
                           uint64_t pitch, uint64_t len, uint64_t lag, uint64_t have,
                           double* part, uint32_t nb, double* acc, cudaStream_t st);
cudaError_t launch_moment_sums(const void* v, int is_f32, uint32_t P, uint64_t pitch,
                               uint64_t len, double* part, uint32_t nb, double* acc,
                               cudaStream_t st);
cudaError_t launch_ac_tail(const void* v, const void* told, void* tnew, int is_f32, uint32_t P,
                           uint64_t pitch, uint64_t len, uint64_t lag, uint64_t have,
                           cudaStream_t st);

// Anderson-Darling A^2 vs N(0, 1) on the device (stats_ad.cu): scratch of
// ad_scratch_bytes(is_f32, n); keys of the sample's windows are added with
// ad_add_values, then ad_finish sorts them and writes A^2 to *out_dev.
size_t ad_scratch_bytes(int is_f32, uint64_t n);
cudaError_t ad_add_values(const void* v, int is_f32, uint32_t P, uint64_t pitch, uint64_t len,
                          void* scratch, uint64_t at, cudaStream_t st);
cudaError_t ad_finish(int is_f32, uint64_t n, void* scratch, double* out_dev, cudaStream_t st);

// Box-Muller / polar baselines (baselines.cu).
cudaError_t launch_method_fill(int method, int f64_math, uint64_t seed, uint64_t stream0,
                               uint32_t pools, const OutLayout& lay, double mu, double sigma,
                               uint32_t out_f32, void* out, cudaStream_t st);

// Device uniform generator words (tests).
cudaError_t launch_lfg_words(uint64_t seed, uint64_t stream0, uint32_t pools,
                             uint64_t count, uint64_t* out, cudaStream_t st);

}  // namespace wg
