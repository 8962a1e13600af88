// Throughput of the softmax's per-element instructions on one SM (4 warps per SMSP, independent
// chains): MUFU.EX2, F2FP (cvt.rn.bf16x2.f32), both interleaved, and integer packing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/xu scripts/xu_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
    float x[8];
    uint32_t u[8];
    for (int i = 0; i < 8; ++i) {
        x[i] = -0.001f * (threadIdx.x + i);
        u[i] = threadIdx.x * 7 + i;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0 || MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            if (MODE == 1 || MODE == 2) {
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
                u[i] ^= r;
            }
            if (MODE == 3) {  // round-half-up + byte permute packing: IADD3 + PRMT per pair
                uint32_t a = __float_as_uint(x[i]) + 0x8000u, b = __float_as_uint(x[(i + 1) & 7]) + 0x8000u;
                uint32_t r;
                asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
                u[i] ^= r;
                x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (r & 1u));
            }
            if (MODE == 4) {  // two ex2 per F2FP: the softmax's 2:1 ratio
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[(i + 4) & 7]));
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 4) & 7]));
                u[i] ^= r;
            }
            if (MODE == 5) {  // packed half-precision exp2: two elements per instruction
                uint32_t h = u[i];
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
                u[i] = h;
            }
            if (MODE == 6) {
                uint32_t h = u[i];
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h));
                u[i] = h;
            }
            if (MODE == 8) {  // F2FP in a dependent chain that cannot be folded away
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
                x[i] = __uint_as_float(r);
            }
            if (MODE == 9) {  // 7 EX2 + 4 F2FP: the attention softmax's per-octet mix
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
                if (i & 1) {
                    uint32_t r;
                    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[i ^ 1]));
                    u[i] ^= r;
                }
            }
            if (MODE == 7) {  // f32 pair -> f16x2 convert (cvt.rn.f16x2.f32)
                uint32_t r;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
                u[i] ^= r;
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i] + (float)u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int ops_per_iter, int threads = 512) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    int iters = 4096;
    k<MODE><<<148, threads>>>(out, cyc, iters);
    k<MODE><<<148, threads>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double warp_instr_per_smsp = threads / 128.0 * iters * 8 * ops_per_iter;  // warps / 4 SMSPs
    printf("%-28s %4d thr %8.2f cycles per warp-instruction per SMSP\n", name, threads,
           c / warp_instr_per_smsp);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0>("MUFU.EX2", 1);
    run<1>("F2FP bf16x2", 1);
    run<2>("EX2 + F2FP (per pair)", 2);
    run<3>("IADD+IADD+PRMT+LOP (pack)", 1);
    run<4>("2 EX2 + 1 F2FP", 3);
    run<5>("EX2 f16x2 (2 elements)", 1);
    run<6>("EX2 bf16x2 (2 elements)", 1);
    run<7>("F2FP f16x2", 1);
    run<8>("F2FP bf16x2 (dependent)", 1);
    run<9>("8 EX2 + 4 F2FP (per 12)", 1);
    for (int thr : {128, 256, 384, 512}) run<0>("MUFU.EX2 (warps per SMSP)", 1, thr);
    for (int thr : {128, 256, 512}) run<9>("8 EX2 + 4 F2FP (warps/SMSP)", 1, thr);
    return 0;
}
