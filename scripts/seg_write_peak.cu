// Write-bandwidth ceiling of the C3 OUTPUT PATTERN without any generation
// work: P = 1184 CTAs (8 per SM), CTA p streams its own contiguous segment of
// 2^34 / P fp32 values in refill-sized chunks (4095 values, so successive
// chunks start 4 bytes off 16-byte alignment, as in the real fill).
//   mode 0: warp stores (64 threads, 1 STG per value, 128 B per warp store)
//   mode 1: bulk-copy engine (thread 0: cp.async.bulk from a 16 KiB shared
//           buffer, 16-byte aligned part only; ragged ends skipped)
//   mode 2: plain fill over the whole range, 1184 x 256 threads, float4
//   mode 3: as 2 with 256-bit stores (st.global.v8.f32)
//   mode 4: as 2, float4 with the streaming hint (st.global.cs)
//   mode 5: as 1 with 8 bulk groups in flight per CTA
//   mode 6: one-shot grid, 128 threads x 16 float4 per block (32 KiB chunk)
//   mode 7: as 1 but CTA p starts at chunk (37 p) mod nchunks (decorrelated)
//   mode 8+: bulk, aligned chunks of CB bytes, P2 CTAs, queue Q, optional
//            L2 evict_first hint (see table in main)
//   mode 23: C3's actual emission: per refill 4 bulk copies (one per 1024-value
//            array, 64 B-aligned spans) + warp stores of the ragged values
//   mode 24: as 23 but ONE bulk copy per refill (64 B-aligned interior of
//            the whole 4095-value window) + warp stores of its ragged ends
//   mode 16+: C3's exact segments and refill boundaries (4095 values), but
//            each refill's copy is [first U-aligned byte of the not yet
//            written part, last U-aligned byte of the refill): what a
//            CTA-side carry buffer of U bytes would emit (U = 128 .. 16384)
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

__global__ void __launch_bounds__(64) k_bulk8(float* out, uint64_t seg) {
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
            asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(64) k_bulk_rot(float* out, uint64_t seg) {
    extern __shared__ __align__(1024) float sm[];
    for (int i = threadIdx.x; i < 4096; i += 64) sm[i] = (float)blockIdx.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    float* o = out + (uint64_t)blockIdx.x * seg;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    const uint64_t nch = seg / kChunk;
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t done = ((c + 37ull * blockIdx.x) % nch) * kChunk;
        uint64_t a = reinterpret_cast<uint64_t>(o + done);
        const uint64_t e = reinterpret_cast<uint64_t>(o + done + kChunk) & ~15ull;
        a = (a + 15) & ~15ull;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a),
                     "r"(s), "r"((uint32_t)(e - a))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int HINT>
__global__ void __launch_bounds__(32) k_bulk_gen(char* out, uint64_t seg, uint32_t cb, int q) {
    extern __shared__ __align__(1024) float sm[];
    for (uint32_t i = threadIdx.x; i < cb / 4; i += 32) sm[i] = (float)blockIdx.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    char* o = out + (uint64_t)blockIdx.x * seg;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    uint64_t pol = 0;
    if (HINT) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (uint64_t done = 0; done + cb <= seg; done += cb) {
        if (HINT)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                         ::"l"(o + done), "r"(s), "r"(cb), "l"(pol) : "memory");
        else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o + done),
                         "r"(s), "r"(cb) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (q <= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(64) k_bulk_carry(float* out, uint64_t seg, uint32_t ub) {
    extern __shared__ __align__(1024) float sm[];
    for (int i = threadIdx.x; i < (ub <= 4096 ? 6144 : 9216); i += 64) sm[i] = (float)blockIdx.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    float* o = out + (uint64_t)blockIdx.x * seg;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    const uint64_t end = reinterpret_cast<uint64_t>(o + seg);
    uint64_t from = reinterpret_cast<uint64_t>(o) & ~15ull;  // written up to here
    for (uint64_t done = 0; done < seg; done += kChunk) {
        const uint64_t n = seg - done < kChunk ? seg - done : kChunk;
        uint64_t e = reinterpret_cast<uint64_t>(o + done + n);
        e = e >= end ? (e & ~15ull) : (e & ~(uint64_t)(ub - 1));
        if (e > from) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(from),
                         "r"(s), "r"((uint32_t)(e - from))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            from = e;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// one warp per CTA, like the one-warp C3 pools
template <int ONE>
__global__ void __launch_bounds__(32) k_c3_emit(float* out, uint64_t seg) {
    extern __shared__ __align__(1024) float sm[];
    for (int i = threadIdx.x; i < 4096 + 64; i += 32) sm[i] = (float)blockIdx.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    float* o = out + (uint64_t)blockIdx.x * seg;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t lane = threadIdx.x;
    for (uint64_t done = 0; done < seg; done += kChunk) {
        const uint64_t n = seg - done < kChunk ? seg - done : kChunk;
        float* w = o + done;
        const uint32_t nspan = ONE ? 1 : 4;
        for (uint32_t m = 0; m < nspan; ++m) {
            const uint64_t lo = ONE ? 0 : m * 1024ull;
            const uint64_t hi = ONE || m == 3 || (m + 1) * 1024ull > n ? n : (m + 1) * 1024ull;
            if (hi <= lo) continue;
            uint64_t a = reinterpret_cast<uint64_t>(w + lo);
            uint64_t e = reinterpret_cast<uint64_t>(w + hi);
            const uint64_t a64 = (a + 63) & ~63ull, e64 = e & ~63ull;
            // ragged head [a, a64) and tail [e64, e): warp stores
            const uint32_t nh = (uint32_t)((a64 > e ? e : a64) - a) / 4;
            if (lane < nh) w[lo + lane] = 1.0f;
            if (e64 > a64) {
                const uint32_t nt = (uint32_t)(e - e64) / 4;
                if (lane < nt) reinterpret_cast<float*>(e64)[lane] = 1.0f;
                if (lane == 0) {
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a64),
                                 "r"(s), "r"((uint32_t)(e64 - a64))
                                 : "memory");
                }
            }
        }
        if (lane == 0) {
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_fill8(float* out, uint64_t n8) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n8;
         i += (uint64_t)gridDim.x * blockDim.x)
        asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(out + 8 * i),
                     "f"(1.0f)
                     : "memory");
}

__global__ void k_fill_cs(float4* out, uint64_t n4) {
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
         i += (uint64_t)gridDim.x * blockDim.x)
        __stcs(out + i, v);
}

__global__ void __launch_bounds__(128) k_chunk(float4* out) {
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    float4* o = out + (uint64_t)blockIdx.x * 2048 + threadIdx.x;
#pragma unroll
    for (int i = 0; i < 16; ++i) o[128 * i] = v;
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
    cudaFuncSetAttribute(k_bulk8, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaFuncSetAttribute(k_bulk_rot, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaFuncSetAttribute(k_bulk_gen<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k_bulk_gen<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    // mode 8..: {chunk bytes, CTAs per SM, queue, hint}
    const int gen[][4] = {{16384, 8, 4, 0}, {4096, 8, 4, 0}, {65536, 2, 4, 0}, {16384, 8, 4, 1},
                          {16384, 4, 4, 0}, {16384, 14, 4, 0}, {32768, 6, 4, 0}, {16384, 8, 1, 0}};
    cudaFuncSetAttribute(k_bulk_carry, cudaFuncAttributeMaxDynamicSharedMemorySize, 36864);
    const int nmodes = argc > 2 ? atoi(argv[2]) : 16;
    const uint32_t carry_u[] = {16, 128, 512, 1024, 2048, 4096, 16384};
    cudaFuncSetAttribute(k_c3_emit<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 17000);
    cudaFuncSetAttribute(k_c3_emit<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 17000);
    const int first = argc > 3 ? atoi(argv[3]) : 0;
    for (int mode = first; mode < nmodes; ++mode) {
        if (mode >= 23) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                if (mode == 23) k_c3_emit<0><<<P, 32, 17000>>>(out, seg);
                else k_c3_emit<1><<<P, 32, 17000>>>(out, seg);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            cudaError_t e = cudaGetLastError();
            printf("{\"mode\": %d, \"ms\": %.3f, \"gbs\": %.1f, \"err\": \"%s\"}\n", mode, best,
                   (double)(P * seg) * 4 / (best / 1e3) / 1e9, cudaGetErrorString(e));
            continue;
        }
        if (mode >= 16) {
            const uint32_t ub = carry_u[(mode - 16) % 7];
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                k_bulk_carry<<<P, 64, ub <= 4096 ? 24576 : 36864>>>(out, seg, ub);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            cudaError_t e = cudaGetLastError();
            printf("{\"mode\": %d, \"carry_bytes\": %u, \"ms\": %.3f, \"gbs\": %.1f, \"err\": \"%s\"}\n",
                   mode, ub, best, (double)(P * seg) * 4 / (best / 1e3) / 1e9, cudaGetErrorString(e));
            continue;
        }
        if (mode >= 8) {
            const int* gcfg = gen[mode - 8];
            const int P2 = 148 * gcfg[1];
            const uint64_t seg2 = (total * 4 / P2) & ~65535ull;
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(a);
                if (gcfg[3]) k_bulk_gen<1><<<P2, 32, gcfg[0]>>>((char*)out, seg2, gcfg[0], gcfg[2]);
                else k_bulk_gen<0><<<P2, 32, gcfg[0]>>>((char*)out, seg2, gcfg[0], gcfg[2]);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms < best) best = ms;
            }
            cudaError_t e = cudaGetLastError();
            printf("{\"mode\": %d, \"chunk\": %d, \"ctas_per_sm\": %d, \"queue\": %d, \"hint\": %d, \"ms\": %.3f, \"gbs\": %.1f, \"err\": \"%s\"}\n",
                   mode, gcfg[0], gcfg[1], gcfg[2], gcfg[3], best,
                   (double)(P2 * (seg2 / gcfg[0]) * gcfg[0]) / (best / 1e3) / 1e9, cudaGetErrorString(e));
            continue;
        }
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k_warp<<<P, 64>>>(out, seg);
            if (mode == 1) k_bulk<<<P, 64, 16384>>>(out, seg);
            if (mode == 2) k_fill<<<P, 256>>>(reinterpret_cast<float4*>(out), total / 4);
            if (mode == 3) k_fill8<<<P, 256>>>(out, total / 8);
            if (mode == 4) k_fill_cs<<<P, 256>>>(reinterpret_cast<float4*>(out), total / 4);
            if (mode == 5) k_bulk8<<<P, 64, 16384>>>(out, seg);
            if (mode == 7) k_bulk_rot<<<P, 64, 16384>>>(out, seg);
            if (mode == 6) k_chunk<<<(unsigned)(total / 8192), 128>>>(reinterpret_cast<float4*>(out));
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
