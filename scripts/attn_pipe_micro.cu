// attn_pipe_micro.cu -- microbenchmark of the attention MMA pipeline without softmax: per 128-key
// tile, S = Q K^T then O += P V (P read from TMEM), K/V streamed by TMA through a smem ring.
//   single: one CTA per 128 query rows, full K and V tiles (32 KB each), QK SS or TS
//   pair:   cta_group::2 (M = 256): each CTA loads half of K (64 keys) and half of V (64 d-cols)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_05503_b200/csrc
//        scripts/attn_pipe_micro.cu -o /tmp/attn_pipe_micro -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace csa;

constexpr int N = 75600, H = 40, D = 128, BK = 128;

// single CTA: ring slot = 32 KB (K tile or V tile); order K0, K1, V0, K2, V1, ...
__global__ void __launch_bounds__(128, 1)
    single(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv, int ts,
           int tiles, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_ptr;
    __shared__ __align__(8) uint64_t full[8], empty[8], done;
    constexpr int kSlots = 5, kSlot = 32768;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 2) tmem_alloc<512>(&tmem_ptr);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_ptr;
    uint8_t* ring = smem + 32768;
    const uint32_t q_base = smem_u32(smem), r_base = smem_u32(ring);
    const uint32_t id_qk = umma_idesc_bf16(128, 128, 0, 0), id_pv = umma_idesc_bf16(128, D, 0, 1);
    const uint64_t pol = policy_evict_last();
    const long long t0 = clock64();
    const int nb = N / BK;
    if (warp == 0) {
        int ld = 0;
        for (int step = 0; step <= tiles; ++step)
            for (int kv = 0; kv < 2; ++kv) {
                if ((kv == 0 && step >= tiles) || (kv == 1 && step == 0)) continue;
                const int j = kv == 0 ? step : step - 1;
                const int s = ld % kSlots, ph = (ld / kSlots) & 1;
                ++ld;
                mbar_wait(empty + s, ph ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(full + s, kSlot);
                    const int n0 = ((j + blockIdx.x * 7) % nb) * BK;
                    for (int x = 0; x < 2; ++x)
                        tma_load_4d(ring + s * kSlot + x * BK * 128, kv ? &tv : &tk, full + s,
                                    x * 64, 0, n0, 0, pol);
                }
                __syncwarp();
            }
    } else if (warp == 1) {
        int cons = 0;
        auto pv = [&](int t) {
            const int s = cons % kSlots, ph = (cons / kSlots) & 1;
            ++cons;
            mbar_wait(full + s, ph);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts(tmem + 256, tmem + (t & 1) * 128 + kk * 8,
                           umma_desc_sw128(r_base + s * kSlot + kk * 16 * 128, BK * 128, 1024),
                           id_pv, 1u);
                mma_commit(empty + s);
            }
            __syncwarp();
        };
        for (int t = 0; t < tiles; ++t) {
            const int s = cons % kSlots, ph = (cons / kSlots) & 1;
            ++cons;
            mbar_wait(full + s, ph);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk & 3) * 32;
                    const uint64_t bd = umma_desc_sw128(r_base + s * kSlot + (kk >> 2) * BK * 128 + off, 16, 1024);
                    if (ts)
                        mma_ts(tmem + (t & 1) * 128, tmem + 448 + kk * 8, bd, id_qk, kk > 0);
                    else
                        mma_ss(tmem + (t & 1) * 128,
                               umma_desc_sw128(q_base + (kk >> 2) * BK * 128 + off, 16, 1024), bd,
                               id_qk, kk > 0);
                }
                mma_commit(empty + s);
            }
            __syncwarp();
            if (t >= 1) pv(t - 1);
        }
        pv(tiles - 1);
        if (elect_one()) mma_commit(&done);
        __syncwarp();
        mbar_wait(&done, 0);
        if (threadIdx.x == 32) cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// pair: ring slot = 16 KB (K half: 64 keys x 128 d, or V half: 128 keys x 64 d-cols)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair(const __grid_constant__ CUtensorMap tk64, const __grid_constant__ CUtensorMap tv, int ts,
         int tiles, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_ptr;
    __shared__ __align__(8) uint64_t full[12], empty[12], done;
    constexpr int kSlots = 10, kSlot = 16384;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    if (warp == 2) tmem_alloc_pair<512>(&tmem_ptr);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 12; ++i) { mbar_init(full + i, 2); mbar_init(empty + i, 1); }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tmem_ptr;
    uint8_t* ring = smem + 32768;
    const uint32_t q_base = smem_u32(smem), r_base = smem_u32(ring);
    const uint32_t id_qk = umma_idesc_bf16(256, 128, 0, 0), id_pv = umma_idesc_bf16(256, D, 0, 1);
    const uint64_t pol = policy_evict_last();
    const long long t0 = clock64();
    const int nb = N / BK;
    if (warp == 0) {
        int ld = 0;
        for (int step = 0; step <= tiles; ++step)
            for (int kv = 0; kv < 2; ++kv) {
                if ((kv == 0 && step >= tiles) || (kv == 1 && step == 0)) continue;
                const int j = kv == 0 ? step : step - 1;
                const int s = ld % kSlots, ph = (ld / kSlots) & 1;
                ++ld;
                mbar_wait(empty + s, ph ^ 1);
                if (elect_one()) {
                    const uint32_t lb = mapa_shared(smem_u32(full + s), 0);
                    mbar_arrive_expect_tx_cluster(lb, kSlot);
                    const int n0 = ((j + (blockIdx.x >> 1) * 7) % nb) * BK;
                    if (kv == 0) {
                        for (int x = 0; x < 2; ++x)
                            tma_load_4d_pair(ring + s * kSlot + x * 64 * 128, &tk64, lb, x * 64, 0,
                                             n0 + 64 * rank, 0, pol);
                    } else {
                        tma_load_4d_pair(ring + s * kSlot, &tv, lb, 64 * rank, 0, n0, 0, pol);
                    }
                }
                __syncwarp();
            }
    } else if (warp == 1 && rank == 0) {
        int cons = 0;
        auto pv = [&](int t) {
            const int s = cons % kSlots, ph = (cons / kSlots) & 1;
            ++cons;
            mbar_wait(full + s, ph);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts_pair(tmem + 256, tmem + 384 + (t & 1) * 32 + kk * 8,
                                umma_desc_sw128(r_base + s * kSlot + kk * 16 * 128, 16384, 1024),
                                id_pv, 1u);
                mma_commit_pair(empty + s);
            }
            __syncwarp();
        };
        for (int t = 0; t < tiles; ++t) {
            const int s = cons % kSlots, ph = (cons / kSlots) & 1;
            ++cons;
            mbar_wait(full + s, ph);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk & 3) * 32;
                    const uint64_t bd = umma_desc_sw128(r_base + s * kSlot + (kk >> 2) * 64 * 128 + off, 16, 1024);
                    if (ts)
                        mma_ts_pair(tmem + (t & 1) * 128, tmem + 448 + kk * 8, bd, id_qk, kk > 0);
                    else
                        mma_ss_pair(tmem + (t & 1) * 128,
                                    umma_desc_sw128(q_base + (kk >> 2) * BK * 128 + off, 16, 1024),
                                    bd, id_qk, kk > 0);
                }
                mma_commit_pair(empty + s);
            }
            __syncwarp();
            if (t >= 1) pv(t - 1);
        }
        pv(tiles - 1);
        if (elect_one()) mma_commit_pair(&done);
        __syncwarp();
        mbar_wait(&done, 0);
        if (threadIdx.x == 32) cycles[blockIdx.x >> 1] = clock64() - t0;
    } else if (warp == 1) {
        mbar_wait(&done, 0);
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem);
    }
}

static CUtensorMap make(void* buf, int rows, int cols) {
    CUtensorMap map;
    cuuint64_t dims[4] = {D, H, N, 1};
    cuuint64_t strides[3] = {D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)N * H * D * 2};
    cuuint32_t box[4] = {(cuuint32_t)cols, 1, (cuuint32_t)rows, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return map;
}

int main() {
    void *kb, *vb;
    const size_t bytes = (size_t)N * H * D * 2;
    cudaMalloc(&kb, bytes);
    cudaMalloc(&vb, bytes);
    cudaMemset(kb, 0, bytes);
    cudaMemset(vb, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d_cyc;
    cudaMalloc(&d_cyc, sms * sizeof(long long));
    const CUtensorMap tk = make(kb, 128, 64), tv = make(vb, 128, 64), tk64 = make(kb, 64, 64);
    const int tiles = 3000;
    long long h[256];
    {
        const int smem = 32768 + 5 * 32768;
        cudaFuncSetAttribute(single, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int ts = 0; ts < 2; ++ts) {
            single<<<sms, 128, smem>>>(tk, tv, ts, 50, d_cyc);
            single<<<sms, 128, smem>>>(tk, tv, ts, tiles, d_cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("single: %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, d_cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < sms; ++i) avg += h[i];
            avg /= sms;
            printf("single QK-%s + PV-TS: %7.1f cyc/tile (floor 1024) -> %6.0f TFLOP/s @1.9GHz\n",
                   ts ? "TS" : "SS", avg / tiles, 8.39e6 * sms * 1.9e9 / (avg / tiles) / 1e12);
        }
    }
    {
        const int smem = 32768 + 10 * 16384;
        cudaFuncSetAttribute(pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int ts = 0; ts < 2; ++ts) {
            pair<<<sms, 128, smem>>>(tk64, tv, ts, 50, d_cyc);
            pair<<<sms, 128, smem>>>(tk64, tv, ts, tiles, d_cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("pair: %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, d_cyc, sms / 2 * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < sms / 2; ++i) avg += h[i];
            avg /= sms / 2;
            printf("pair   QK-%s + PV-TS: %7.1f cyc/pair-tile (floor 1024) -> %6.0f TFLOP/s @1.9GHz\n",
                   ts ? "TS" : "SS", avg / tiles, 2 * 8.39e6 * (sms / 2) * 1.9e9 / (avg / tiles) / 1e12);
        }
    }
    return 0;
}
