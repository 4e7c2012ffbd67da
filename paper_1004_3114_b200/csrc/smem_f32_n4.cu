// Shared-memory engine instantiations for float pools, n = 4 (split per
// dtype x n so the kernel variants compile in parallel).
#include "smem_impl.cuh"

namespace wg {

cudaError_t smem_dispatch_f32_n4(const KernelArgs& a, cudaStream_t st, bool unit_same, bool al) {
    return dispatch<float, 4>(a, st, unit_same, al);
}

}  // namespace wg
