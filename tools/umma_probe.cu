// Throughput probe of tcgen05.mma kind::f16 (bf16 -> fp32) at the decode
// GEMM's shapes: M = 128 weight rows, N = tokens (16..256), K = 16 per
// instruction; operands resident (no memory traffic), one CTA per SM, one
// thread issuing back-to-back MMAs into one TMEM accumulator.  A from shared
// memory (SS, the gemm_tc raw / codec-1 path) or from tensor memory (TS, the
// codec-3 path).  Reports ns per MMA and the bf16-weight bytes per second the
// chip could consume at that rate (128 x 16 x 2 B of A per MMA).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2411_11217_b200/csrc tools/umma_probe.cu -o tools/umma_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels/common.cuh"

using namespace mltk;

// warp-uniform issue: the whole warp runs the loop (descriptors stay in
// uniform registers), one elected lane executes each tcgen05.mma
__device__ __forceinline__ void umma_ss_elect(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc));
}
__device__ __forceinline__ void umma_ts_elect(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d), "r"(a), "l"(bd), "r"(idesc));
}

__global__ void __launch_bounds__(128, 1) probe(int N, int iters, int ts, int chains, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;             // 16 KiB: 128 x 64 bf16, SW128
    uint8_t* B = smem + 16384;     // N x 64 bf16, SW128
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, chains >= 100 ? chains - 100 : 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tbase, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t ta = tmem + 256;  // A in TMEM: 32 columns (64 bf16 per lane)
    if (ts) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0x3c003c00u + i;
        tmem_st32(tmem + ((warp * 32u) << 16) + 256, v);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t idesc = idesc_bf16(128, N);
    unsigned long long t0 = 0, t1 = 0;
    if (chains < 0 && warp == 0) {  // warp-uniform issue
        chains = -chains;
        t0 = globaltimer();
        const uint32_t sa = smem_u32(A), sb = smem_u32(B);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t d = tmem + (k % chains) * N;
                if (ts)
                    umma_ts_elect(d, ta + k * 8, sdesc_sw128(sb + k * 32), idesc);
                else
                    umma_ss_elect(d, sdesc_sw128(sa + k * 32), sdesc_sw128(sb + k * 32), idesc);
            }
        }
        if (elect_one()) umma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        t1 = globaltimer();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    } else if (chains >= 100) {  // (chains - 100) warps issue concurrently, each its own accumulator
        const int nw = chains - 100;
        if (warp < nw && (threadIdx.x & 31) == 0) {
            t0 = globaltimer();
            const uint32_t sa = smem_u32(A), sb = smem_u32(B);
            const uint32_t d = tmem + warp * N;
            for (int it = 0; it < iters; ++it)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_bf16(d, sdesc_sw128(sa + k * 32), sdesc_sw128(sb + k * 32), idesc, 1u);
            umma_commit(&bar);
        }
        if (threadIdx.x == 0) {
            mbar_wait(&bar, 0);
            t1 = globaltimer();
            out[blockIdx.x] = t1 - t0;
        }
    } else if (chains > 0 && threadIdx.x == 0) {
        t0 = globaltimer();
        const uint32_t sa = smem_u32(A), sb = smem_u32(B);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // independent accumulators: MMA k goes to chain k % chains (N columns each)
                const uint32_t d = tmem + (k % chains) * N;
                if (ts)
                    umma_bf16_ts(d, ta + k * 8, sdesc_sw128(sb + k * 32), idesc, 1u);
                else
                    umma_bf16(d, sdesc_sw128(sa + k * 32), sdesc_sw128(sb + k * 32), idesc, 1u);
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = globaltimer();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, sms * sizeof(unsigned long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 2000;
    for (int nw : {1, 2, 4}) {
        const int N = 16, smem = 1024 + 16384 + N * 128;
        probe<<<sms, 128, smem>>>(N, 10, 0, 100 + nw, d);
        probe<<<sms, 128, smem>>>(N, iters, 0, 100 + nw, d);
        cudaDeviceSynchronize();
        unsigned long long h[1024];
        cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("SS %d issuing warps N=16: %7.1f ns per MMA (all warps)\n", nw, double(mx) / (iters * 4.0 * nw));
    }
    for (int ts = 0; ts < 2; ++ts)
        for (int chains : {1, -1})
        for (int N : {16, 32, 64, 128, 256}) {
            if (abs(chains) * N > 256) continue;
            const int smem = 1024 + 16384 + N * 128;
            probe<<<sms, 128, smem>>>(N, 10, ts, chains, d);
            probe<<<sms, 128, smem>>>(N, iters, ts, chains, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            unsigned long long h[1024];
            cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
            const double ns = double(mx) / (iters * 4.0);
            const double a_bytes = 128.0 * 16 * 2 * iters * 4 * sms;
            const double flops = 2.0 * 128 * N * 16 * iters * 4 * sms;
            printf("%s chains=%d N=%3d: %7.1f ns/MMA  A-stream %7.0f GB/s  %6.1f TFLOP/s\n", ts ? "TS" : "SS", chains, N, ns,
                   a_bytes / (mx * 1e-9) / 1e9, flops / (mx * 1e-9) / 1e12);
        }
    return 0;
}
