// Shared-memory engine with 64 data registers per thread (two warps per
// 4x1024 fp32 pool): used for fills with f >= 2 on pools of <= 16 KiB, where
// no emission overlaps the non-emitting passes and twice the warps per SM
// win (BASELINE configs[4] sweep).
#define WG_DATA_REGS 64
// 128 registers per thread -> 8 CTAs (16 warps) per SM for a 4x1024 fp32 pool:
// f >= 2 fills are generation-bound, occupancy wins (C5 fp32 4x1024 R = 2:
// 50.9 % at 8 CTAs per SM against 39.7 % at the 255-register budget's 4).
// Larger pools gain nothing from this engine (shared memory, not registers,
// limits their CTAs per SM: fp32 4x4096 R = 2 42.7 % here against 45.3 %).
#define WG_RBUDGET_MIN 128
#define WG_SMEM_NS r64
#include "smem_impl.cuh"

namespace wg {

template <typename T>
static cudaError_t dispatch_small(const KernelArgs& a, cudaStream_t st, bool unit_same, bool al) {
    switch (a.N) {
        case 1u << 8: return r64::go_em<T, 4, 8>(a, st, unit_same, al);
        case 1u << 9: return r64::go_em<T, 4, 9>(a, st, unit_same, al);
        case 1u << 10:
            if constexpr (sizeof(T) == 4) return r64::go_em<T, 4, 10>(a, st, unit_same, al);
            return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

bool smem_r64_fits(uint32_t dtype, uint32_t N) {
    return N >= 256 && (uint64_t)4 * N * (dtype == WRNG_GPU_F64 ? 8 : 4) <= 16 * 1024;
}

cudaError_t smem_dispatch_n4_r64(uint32_t dtype, const KernelArgs& a, cudaStream_t st,
                                 bool unit_same, bool al) {
    return dtype == WRNG_GPU_F64 ? dispatch_small<double>(a, st, unit_same, al)
                                 : dispatch_small<float>(a, st, unit_same, al);
}

}  // namespace wg
