// Write-bandwidth ceiling of the C3 OUTPUT PATTERN without any generation
// work: P = 1184 CTAs (8 per SM), CTA p streams its own contiguous segment of
// 2^34 / P fp32 values in refill-sized chunks (4095 values, so successive
// chunks start 4 bytes off 16-byte alignment, as in the real fill).
//   mode 0: warp stores (64 threads, 1 STG per value, 128 B per warp store)
//   mode 1: bulk-copy engine (thread 0: cp.async.bulk from a 16 KiB shared
//           buffer, 16-byte aligned part only; ragged ends skipped)
//   mode 2: plain fill over the whole range, 1184 x 256 threads, float4
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/seg_write_peak.cu -o scripts/seg_write_peak.bin
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

constexpr int kChunk = 4095;

__global__ void __launch_bounds__(64) k_warp(float* out, uint64_t seg) {
    float* o = out + (uint64_t)blockIdx.x * seg;
    const float v = (float)blockIdx.x;
    for (uint64_t done = 0; done < seg; done += kChunk) {
        const uint64_t n = seg - done < kChunk ? seg - done : kChunk;
        for (uint32_t i = threadIdx.x; i < n; i += 64) o[done + i] = v;
    }
}

__global__ void __launch_bounds__(64) k_bulk(float* out, uint64_t seg) {
    extern __shared__ __align__(1024) float sm[];
    for (int i = threadIdx.x; i < 4096; i += 64) sm[i] = (float)blockIdx.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    float* o = out + (uint64_t)blockIdx.x * seg;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    for (uint64_t done = 0; done < seg; done += kChunk) {
        const uint64_t n = seg - done < kChunk ? seg - done : kChunk;
        uint64_t a = reinterpret_cast<uint64_t>(o + done);
        const uint64_t e = reinterpret_cast<uint64_t>(o + done + n) & ~15ull;
        a = (a + 15) & ~15ull;
        if (e > a) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a),
                         "r"(s), "r"((uint32_t)(e - a))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_fill(float4* out, uint64_t n4) {
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = v;
}

int main(int argc, char** argv) {
    const int P = 1184;
    const uint64_t total = 1ull << (argc > 1 ? atoi(argv[1]) : 34);
    const uint64_t seg = total / P;
    float* out = nullptr;
    if (cudaMalloc(&out, total * 4) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k_warp<<<P, 64>>>(out, seg);
            if (mode == 1) k_bulk<<<P, 64, 16384>>>(out, seg);
            if (mode == 2) k_fill<<<P, 256>>>(reinterpret_cast<float4*>(out), total / 4);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("{\"mode\": %d, \"ms\": %.3f, \"gbs\": %.1f, \"err\": \"%s\"}\n", mode, best,
               (double)(P * seg) * 4 / (best / 1e3) / 1e9, cudaGetErrorString(e));
    }
    return 0;
}
