// Shared-memory engine instantiations for double pools, n = 2 (split per
// dtype x n so the kernel variants compile in parallel).
#include "smem_impl.cuh"

namespace wg {

cudaError_t smem_dispatch_f64_n2(const KernelArgs& a, cudaStream_t st, bool unit_same, bool al) {
    return dispatch<double, 2>(a, st, unit_same, al);
}

}  // namespace wg
