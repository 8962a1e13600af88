// tma_bench.cu -- microbenchmark: per-SM TMA ingest rate for the K-tile streams of the CSA
// kernels, by global layout, box height and ring depth (no math, consumer just frees slots).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_05503_b200/csrc
//        scripts/tma_bench.cu -o gpurun_out/tma_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace csa;

constexpr int N = 75600, H = 40, D = 128;

__global__ void __launch_bounds__(64, 1)
    tma_stream(const __grid_constant__ CUtensorMap map, int layout, int rows, int slots,
               int iters, int same_head) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 196608);
    uint64_t* empty = full + 8;
    const int tile_bytes = rows * D * 2;
    if (threadIdx.x == 0) {
        for (int i = 0; i < slots; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int h = same_head ? 0 : blockIdx.x % H;
    const int nb = N / rows;
    const uint64_t pol = policy_evict_last();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % slots;
            mbar_wait(empty + s, ((it / slots) & 1) ^ 1);
            mbar_arrive_expect_tx(full + s, tile_bytes);
            const int n0 = ((it + blockIdx.x * 7) % nb) * rows;
            uint8_t* dst = smem + s * tile_bytes;
            for (int x = 0; x < D / 64; ++x) {
                if (layout == 0)  // [N][H][D]: dims (d, h, n, 1)
                    tma_load_4d(dst + x * rows * 128, &map, full + s, x * 64, h, n0, 0, pol);
                else              // [H][N][D]: dims (d, n, h, 1)
                    tma_load_4d(dst + x * rows * 128, &map, full + s, x * 64, n0, h, 0, pol);
            }
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % slots;
            mbar_wait(full + s, (it / slots) & 1);
            mbar_arrive(empty + s);
        }
    }
}

int main() {
    void* buf;
    const size_t bytes = (size_t)N * H * D * 2;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("layout rows slots same_head grid | GB/s total  B/clk/SM(@1.9GHz)\n");
    for (int layout = 0; layout < 2; ++layout)
        for (int rows : {128, 256})
            for (int slots : {2, 3, 4, 6})
                for (int same : {0, 1})
                    for (int grid : {sms, sms / 2}) {
                        if (slots * rows * D * 2 > 196608) continue;
                        CUtensorMap map;
                        cuuint64_t dims[4], strides[3];
                        if (layout == 0) {
                            dims[0] = D; dims[1] = H; dims[2] = N; dims[3] = 1;
                            strides[0] = D * 2; strides[1] = (cuuint64_t)H * D * 2;
                            strides[2] = (cuuint64_t)N * H * D * 2;
                        } else {
                            dims[0] = D; dims[1] = N; dims[2] = H; dims[3] = 1;
                            strides[0] = D * 2; strides[1] = (cuuint64_t)N * D * 2;
                            strides[2] = (cuuint64_t)N * H * D * 2;
                        }
                        cuuint32_t box[4];
                        if (layout == 0) { box[0] = 64; box[1] = 1; box[2] = rows; box[3] = 1; }
                        else { box[0] = 64; box[1] = rows; box[2] = 1; box[3] = 1; }
                        cuuint32_t es[4] = {1, 1, 1, 1};
                        CUresult r = cuTensorMapEncodeTiled(
                            &map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
                        const int iters = 4000 * 128 / rows;
                        tma_stream<<<grid, 64, 196608 + 256>>>(map, layout, rows, slots, 200, same);
                        cudaEventRecord(e0);
                        tma_stream<<<grid, 64, 196608 + 256>>>(map, layout, rows, slots, iters, same);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        float ms = 0;
                        cudaEventElapsedTime(&ms, e0, e1);
                        cudaError_t err = cudaGetLastError();
                        if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
                        const double tot = (double)grid * iters * rows * D * 2;
                        const double gbs = tot / (ms * 1e-3) / 1e9;
                        printf("%6d %4d %5d %9d %4d | %10.0f  %6.1f\n", layout, rows, slots, same, grid,
                               gbs, gbs * 1e9 / grid / 1.9e9);
                    }
    return 0;
}
