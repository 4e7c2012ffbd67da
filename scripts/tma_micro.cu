// Micro test: 1-D TMA tensor stores from shared memory at element-granular
// coordinates, descriptor as __grid_constant__ parameter or in global memory.
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/tma_micro.cu -o /tmp/tma_micro
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct alignas(64) Desc {
    unsigned long long w[16];
};
struct P {
    Desc d[2];
    int n;
};

__device__ void store_box(const void* d, int x, unsigned src) {
    asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];" ::"l"(
                     reinterpret_cast<unsigned long long>(d)),
                 "r"(x), "r"(src)
                 : "memory");
}

__global__ void k_param(const __grid_constant__ P p, int x, int mode) {
    extern __shared__ __align__(1024) float sm[];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (float)(i + 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(sm);
        store_box(mode == 0 ? (const void*)&p.d[0] : (const void*)&p.d[1], x, s);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

__global__ void k_global(const Desc* d, int x) {
    extern __shared__ __align__(1024) float sm[];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (float)(i + 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(sm);
        store_box(d, x, s);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

static int check(const char* name, float* dout, int x, int n) {
    std::vector<float> h(n);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(h.data(), dout, n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) {
        float want = (i >= x && i < x + 256) ? (float)(i - x + 1) : 0.f;
        bad += h[i] != want;
    }
    printf("%s x=%d: %s (%d bad)\n", name, x, bad ? "MISMATCH" : "OK", bad);
    return bad != 0;
}

int main(int argc, char** argv) {
    const int which = argc > 1 ? atoi(argv[1]) : -1;  // 0 global, 1 param d0, 2 param d1
    const int xsel = argc > 2 ? atoi(argv[2]) : 0;
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q);
    EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(fp);
    if (!enc) {
        printf("no encode fn\n");
        return 1;
    }
    const int n = 4096;
    float* dout = nullptr;
    cudaMalloc(&dout, n * 4);
    CUtensorMap m;
    cuuint64_t dim = n, strd = 0;
    cuuint32_t box = 256, es = 1;
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, dout, &dim, &strd, &box, &es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    P p;
    memset(&p, 0, sizeof(p));
    memcpy(&p.d[0], &m, sizeof(m));
    memcpy(&p.d[1], &m, sizeof(m));
    Desc* dg = nullptr;
    cudaMalloc(&dg, sizeof(Desc));
    cudaMemcpy(dg, &m, sizeof(m), cudaMemcpyHostToDevice);
    int fails = 0;
    cudaFuncSetAttribute(k_param, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    cudaFuncSetAttribute(k_global, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    const int x = xsel;
    cudaMemset(dout, 0, n * 4);
    if (which == 0) {
        k_global<<<1, 128, 8192>>>(dg, x);
        fails += check("global", dout, x, n);
    } else {
        k_param<<<1, 128, 8192>>>(p, x, which - 1);
        fails += check(which == 1 ? "param d0" : "param d1", dout, x, n);
    }
    printf(fails ? "FAIL\n" : "PASS\n");
    return fails;
}
