// mma_bench.cu -- microbenchmark: tcgen05.mma (kind::f16, bf16 -> fp32) dispatch rate per SM by
// operand source and tile shape, all 148 SMs busy, one issuing thread per CTA, no other work.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_05503_b200/csrc
//        scripts/mma_bench.cu -o /tmp/mma_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace csa;

// mode: 0 SS N128, 1 SS N256, 2 TS N128, 3 TS N256, 4 SS N64, 5 SS N128 (B MN-major)
__global__ void __launch_bounds__(128, 1) mma_loop(int mode, int tiles, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_ptr;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&tmem_ptr);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_ptr;
    const int N = (mode == 1 || mode == 3) ? 256 : (mode == 4 ? 64 : 128);
    const bool ts = mode == 2 || mode == 3 || mode == 7;
    // 6: SS N128 into alternating accumulators [0,128) / [128,256); 7: TS N128 alternating;
    // 8: FA-style mix per tile: SS QK (N128) into S[t&1], then TS P.V (N128) into O;
    // 9: same mix with QK as TS (Q in TMEM); 10: 2 Q tiles: SS QK0, SS QK1, TS PV0, TS PV1.
    const uint32_t b_mn = mode == 5 ? 1u : 0u;
    const uint32_t idesc = umma_idesc_bf16(128, N, 0, b_mn);
    const uint32_t a_base = smem_u32(smem);              // 128 x 128 bf16, K-major SW128 (32 KB)
    const uint32_t b_base = smem_u32(smem + 32768);      // N x 128 bf16 (<= 64 KB)
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        if (elect_one()) {
            t0 = clock64();
            for (int t = 0; t < tiles; ++t) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk & 3) * 32;
                    if (mode >= 8) {
                        const uint32_t idqk = umma_idesc_bf16(128, 128, 0, 0);
                        const uint32_t idpv = umma_idesc_bf16(128, 128, 0, 1);
                        const uint64_t kd = umma_desc_sw128(b_base + (kk >> 2) * 128 * 128 + off, 16, 1024);
                        const uint64_t ad = umma_desc_sw128(a_base + (kk >> 2) * 16384 + off, 16, 1024);
                        const uint64_t vd = umma_desc_sw128(b_base + kk * 16 * 128, 128 * 128, 1024);
                        const uint32_t sb = (t & 1) * 128;
                        if (mode == 8) {
                            mma_ss(tmem + sb, ad, kd, idqk, kk > 0 ? 1u : 0u);
                        } else if (mode == 9) {
                            mma_ts(tmem + sb, tmem + 448 + kk * 8, kd, idqk, kk > 0 ? 1u : 0u);
                        } else {
                            mma_ss(tmem + 0, ad, kd, idqk, kk > 0 ? 1u : 0u);
                        }
                        continue;
                    }
                    const uint64_t bd = b_mn ? umma_desc_sw128(b_base + kk * 16 * 128, N * 128, 1024)
                                             : umma_desc_sw128(b_base + (kk >> 2) * N * 128 + off,
                                                               16, 1024);
                    const uint32_t dd = (mode == 6 || mode == 7) ? (t & 1) * 128 : 0;
                    if (ts) {
                        mma_ts(tmem + dd, tmem + 448 + kk * 8, bd, idesc, kk > 0 ? 1u : 0u);
                    } else {
                        const uint64_t ad = umma_desc_sw128(a_base + (kk >> 2) * 16384 + off, 16, 1024);
                        mma_ss(tmem + dd, ad, bd, idesc, kk > 0 ? 1u : 0u);
                    }
                }
                if (mode >= 8) {
                    const uint32_t idqk = umma_idesc_bf16(128, 128, 0, 0);
                    const uint32_t idpv = umma_idesc_bf16(128, 128, 0, 1);
                    if (mode == 10) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint32_t off = (kk & 3) * 32;
                            const uint64_t kd = umma_desc_sw128(b_base + (kk >> 2) * 128 * 128 + off, 16, 1024);
                            const uint64_t ad = umma_desc_sw128(a_base + (kk >> 2) * 16384 + off, 16, 1024);
                            mma_ss(tmem + 128, ad, kd, idqk, kk > 0 ? 1u : 0u);
                        }
                    }
                    const int npv = mode == 10 ? 2 : 1;
                    for (int q = 0; q < npv; ++q) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t vd = umma_desc_sw128(b_base + kk * 16 * 128, 128 * 128, 1024);
                            mma_ts(tmem + 256 + q * 128, tmem + (q * 128 + 64) + kk * 8, vd, idpv, 1u);
                        }
                    }
                }
            }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        t1 = clock64();
        if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d_cyc;
    cudaMalloc(&d_cyc, sms * sizeof(long long));
    const int smem = 32768 + 65536;
    cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"SS M128 N128", "SS M128 N256", "TS M128 N128", "TS M128 N256",
                           "SS M128 N64", "SS M128 N128 B-MN", "SS N128 alt D", "TS N128 alt D",
                           "mix SS-QK + TS-PV", "mix TS-QK + TS-PV", "2Q: 2xSS-QK + 2xTS-PV"};
    const int ns[] = {128, 256, 128, 256, 64, 128, 128, 128, 256, 256, 512};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 11; ++mode) {
        const int tiles = 4000;
        mma_loop<<<sms, 128, smem>>>(mode, 100, d_cyc);
        cudaEventRecord(e0);
        mma_loop<<<sms, 128, smem>>>(mode, tiles, d_cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) { printf("%s: %s\n", names[mode], cudaGetErrorString(err)); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[256];
        cudaMemcpy(h, d_cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += h[i];
        avg /= sms;
        const double flop = 2.0 * 128 * ns[mode] * 128 * tiles * sms;
        printf("%-20s cyc/dispatch %7.1f  (floor %5.1f)  %7.1f TFLOP/s\n", names[mode],
               avg / (tiles * 8.0 * (ns[mode] > 256 ? ns[mode] / 128 : (mode >= 8 ? 2 : 1))), mode >= 8 ? 64.0 : 128.0 * ns[mode] / 256.0, flop / (ms * 1e-3) / 1e12);
    }
    return 0;
}
