// Shared-memory engine, host side: dispatch to the per-(dtype, n) kernel
// instantiations (smem_{f32,f64}_n{2,4}.cu; templates in smem_impl.cuh) and
// the once-per-device shared-window probe.
#include "smem_impl.cuh"

namespace wg {

cudaError_t smem_dispatch_f32_n2(const KernelArgs&, cudaStream_t, bool, bool);
cudaError_t smem_dispatch_f32_n4(const KernelArgs&, cudaStream_t, bool, bool);
cudaError_t smem_dispatch_f64_n2(const KernelArgs&, cudaStream_t, bool, bool);
cudaError_t smem_dispatch_f64_n4(const KernelArgs&, cudaStream_t, bool, bool);
bool smem_r64_fits(uint32_t dtype, uint32_t N);
cudaError_t smem_dispatch_n4_r64(uint32_t dtype, const KernelArgs&, cudaStream_t, bool, bool);

__global__ void k_smem_base_probe(uint32_t* out) {
    if (threadIdx.x == 0) *out = (uint32_t)__cvta_generic_to_shared(g_sm) & 0xFFFFFFu;
}

// ---------------------------------------------------------------------------
// Host-side dispatch
// ---------------------------------------------------------------------------

// Low 24 bits of the dynamic shared-memory base per device (-1: unknown).
static int64_t g_base_low[64];
static bool g_base_init = false;

void smem_engine_probe(cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (!g_base_init) {
        for (auto& v : g_base_low) v = -1;
        g_base_init = true;
    }
    if (dev < 0 || dev >= 64) return;
    if (g_base_low[dev] < 0) {
        uint32_t* d = nullptr;
        uint32_t h = 0xFFFFFFFFu;
        if (cudaMalloc(&d, 4) == cudaSuccess) {
            k_smem_base_probe<<<1, 32, 16, st>>>(d);
            if (cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, st) == cudaSuccess)
                cudaStreamSynchronize(st);
            cudaFree(d);
        }
        g_base_low[dev] = h;
    }
}

static bool aligned_layout_ok() {
    int dev = 0;
    cudaGetDevice(&dev);
    return g_base_init && dev >= 0 && dev < 64 && g_base_low[dev] == kDynSmemBase;
}

bool smem_engine_fits(uint32_t n_arrays, uint32_t dtype, uint32_t N) {
    const uint32_t es = dtype == WRNG_GPU_F64 ? 8 : 4;
    return (uint64_t)n_arrays * N * es <= kSmemPoolMax;
}

EngineShape smem_engine_shape(uint32_t n_arrays, uint32_t dtype, uint32_t N) {
    const uint32_t es = dtype == WRNG_GPU_F64 ? 8 : 4;
    EngineShape s;
    s.j = pick_j(N, n_arrays * es / 4, WG_DATA_REGS);
    s.threads = N / s.j;
    s.smem = 0;
    return s;
}

cudaError_t launch_smem(uint32_t n_arrays, uint32_t dtype, const KernelArgs& a,
                        cudaStream_t st) {
    const bool unit_same =
        a.op != OP_FILL || (a.unit && (a.out_f32 != 0) == (dtype == WRNG_GPU_F32));
    const bool al = aligned_layout_ok();
    // f >= 2 on small n = 4 pools: the 64-register engine (two warps per
    // 4x1024 fp32 pool) — non-emitting passes are generation-bound
    if (n_arrays == 4 && (a.op == OP_FILL || a.op == OP_QUERY) && a.f >= 2 &&
        smem_r64_fits(dtype, a.N))
        return smem_dispatch_n4_r64(dtype, a, st, unit_same, al);
    if (dtype == WRNG_GPU_F64)
        return n_arrays == 2 ? smem_dispatch_f64_n2(a, st, unit_same, al)
                             : smem_dispatch_f64_n4(a, st, unit_same, al);
    return n_arrays == 2 ? smem_dispatch_f32_n2(a, st, unit_same, al)
                         : smem_dispatch_f32_n4(a, st, unit_same, al);
}

}  // namespace wg
