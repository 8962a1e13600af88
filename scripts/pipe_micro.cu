// pipe_micro.cu -- microbenchmark of the K-stream pipeline shared by the calibration and
// attention kernels: TMA producer -> smem ring -> tcgen05.mma (Q from TMEM or smem) -> commit,
// no softmax.  Measures cycles per 128x128x128 tile on all 148 SMs, by ring depth and MMA form.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_05503_b200/csrc
//        scripts/pipe_micro.cu -o /tmp/pipe_micro -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace csa;

constexpr int N = 75600, H = 40, D = 128, BK = 128;
constexpr int kTile = BK * D * 2;  // 32 KB

__global__ void __launch_bounds__(128, 1)
    pipe(const __grid_constant__ CUtensorMap map, int slots, int ts, int tiles, int nbuf,
         long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_ptr;
    __shared__ __align__(8) uint64_t full[8], empty[8], sdone[2];
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 2) tmem_alloc<512>(&tmem_ptr);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        for (int i = 0; i < 2; ++i) mbar_init(sdone + i, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_ptr;
    uint8_t* ring = smem + 32768;  // Q (smem form) at 0
    const uint32_t q_base = smem_u32(smem), k_base = smem_u32(ring);
    const uint32_t idesc = umma_idesc_bf16(128, 128, 0, 0);
    const uint64_t pol = policy_evict_last();
    long long t0 = clock64();
    if (warp == 0) {
        for (int t = 0; t < tiles; ++t) {
            const int s = t % slots;
            mbar_wait(empty + s, ((t / slots) & 1) ^ 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(full + s, kTile);
                const int n0 = ((t + blockIdx.x * 7) % (N / BK)) * BK;
                for (int x = 0; x < 2; ++x)
                    tma_load_4d(ring + s * kTile + x * BK * 128, &map, full + s, x * 64, 0, n0, 0, pol);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        for (int t = 0; t < tiles; ++t) {
            const int s = t % slots;
            mbar_wait(full + s, (t / slots) & 1);
            tc_fence_after();
            const uint32_t d = tmem + (nbuf == 2 ? (t & 1) * 128 : 0);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk & 3) * 32;
                    const uint64_t bd = umma_desc_sw128(k_base + s * kTile + (kk >> 2) * BK * 128 + off, 16, 1024);
                    if (ts) {
                        mma_ts(d, tmem + 448 + kk * 8, bd, idesc, kk > 0 ? 1u : 0u);
                    } else {
                        const uint64_t ad = umma_desc_sw128(q_base + (kk >> 2) * BK * 128 + off, 16, 1024);
                        mma_ss(d, ad, bd, idesc, kk > 0 ? 1u : 0u);
                    }
                }
                mma_commit(empty + s);
                if (t == tiles - 1) mma_commit(sdone);
            }
            __syncwarp();
        }
        mbar_wait(sdone, 0);
        if (threadIdx.x == 32) cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// CTA pair, cta_group::2: M = 256 (128 Q rows per CTA, Q in TMEM), N = 128 keys per tile of which
// each CTA loads and holds 64 (16 KB); the leader issues, commits multicast to both CTAs' slots.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pipe_pair(const __grid_constant__ CUtensorMap map64, int slots, int tiles, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_ptr;
    __shared__ __align__(8) uint64_t full[8], empty[8], sdone[2];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    if (warp == 2) tmem_alloc_pair<512>(&tmem_ptr);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) { mbar_init(full + i, 2); mbar_init(empty + i, 1); }
        for (int i = 0; i < 2; ++i) mbar_init(sdone + i, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tmem_ptr;
    uint8_t* ring = smem + 32768;
    const uint32_t k_base = smem_u32(ring);
    constexpr int kHalf = 64 * D * 2;  // 16 KB
    const uint32_t idesc = umma_idesc_bf16(256, 128, 0, 0);
    const uint64_t pol = policy_evict_last();
    long long t0 = clock64();
    if (warp == 0) {
        for (int t = 0; t < tiles; ++t) {
            const int s = t % slots;
            mbar_wait(empty + s, ((t / slots) & 1) ^ 1);
            if (elect_one()) {
                const uint32_t lb = mapa_shared(smem_u32(full + s), 0);
                mbar_arrive_expect_tx_cluster(lb, kHalf);
                const int n0 = ((t + (blockIdx.x >> 1) * 7) % (N / BK)) * BK + rank * 64;
                for (int x = 0; x < 2; ++x)
                    tma_load_4d_pair(ring + s * kHalf + x * 64 * 128, &map64, lb, x * 64, 0, n0, 0, pol);
            }
            __syncwarp();
        }
    } else if (warp == 1 && rank == 0) {
        for (int t = 0; t < tiles; ++t) {
            const int s = t % slots;
            mbar_wait(full + s, (t / slots) & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk & 3) * 32;
                    const uint64_t bd = umma_desc_sw128(k_base + s * kHalf + (kk >> 2) * 64 * 128 + off, 16, 1024);
                    mma_ts_pair(tmem, tmem + 448 + kk * 8, bd, idesc, kk > 0 ? 1u : 0u);
                }
                mma_commit_pair(empty + s);
                if (t == tiles - 1) mma_commit_pair(sdone);
            }
            __syncwarp();
        }
        mbar_wait(sdone, 0);
        if (threadIdx.x == 32) cycles[blockIdx.x >> 1] = clock64() - t0;
    } else if (warp == 1) {
        mbar_wait(sdone, 0);
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem);
    }
}

int main() {
    void* buf;
    const size_t bytes = (size_t)N * H * D * 2;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d_cyc;
    cudaMalloc(&d_cyc, sms * sizeof(long long));
    CUtensorMap map;
    cuuint64_t dims[4] = {D, H, N, 1};
    cuuint64_t strides[3] = {D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)N * H * D * 2};
    cuuint32_t box[4] = {64, 1, BK, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 32768 + 6 * kTile;
    cudaFuncSetAttribute(pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int ts = 0; ts < 2; ++ts)
        for (int slots : {2, 3, 4, 6})
            for (int grid : {sms, sms / 2}) {
                const int tiles = 3000;
                pipe<<<grid, 128, smem>>>(map, slots, ts, 50, 1, d_cyc);
                pipe<<<grid, 128, smem>>>(map, slots, ts, tiles, 1, d_cyc);
                cudaError_t err = cudaDeviceSynchronize();
                if (err != cudaSuccess) { printf("%s\n", cudaGetErrorString(err)); return 1; }
                long long h[256];
                cudaMemcpy(h, d_cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
                double avg = 0;
                for (int i = 0; i < grid; ++i) avg += h[i];
                avg /= grid;
                printf("%s slots %d grid %3d: %7.1f cyc/tile (%5.1f per dispatch)\n",
                       ts ? "TS" : "SS", slots, grid, avg / tiles, avg / tiles / 8);
            }
        CUtensorMap map64;
    cuuint32_t box64[4] = {64, 1, 64, 1};
    cuTensorMapEncodeTiled(&map64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box64, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(pipe_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int slots : {2, 4, 6}) {
        const int tiles = 3000;
        pipe_pair<<<sms, 128, smem>>>(map64, slots, 50, d_cyc);
        pipe_pair<<<sms, 128, smem>>>(map64, slots, tiles, d_cyc);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("pair: %s\n", cudaGetErrorString(err)); return 1; }
        long long h[256];
        cudaMemcpy(h, d_cyc, sms / 2 * sizeof(long long), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms / 2; ++i) avg += h[i];
        avg /= sms / 2;
        printf("PAIR TS slots %d: %7.1f cyc per 256x128x128 tile (= %5.1f per SM-tile of 128x128x128)\n",
               slots, avg / tiles, avg / tiles / 2);
    }
    return 0;
}
