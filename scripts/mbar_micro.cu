// Latency of waiting on an mbarrier whose phase has ALREADY completed: try_wait (the kernels'
// mbar_wait) vs test_wait, from one thread, and of the wait right after a remote arrive.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbar scripts/mbar_micro.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void wait_try(uint64_t* bar, uint32_t par) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}\n" ::"r"(su(bar)), "r"(par) : "memory");
}
__device__ __forceinline__ void wait_test(uint64_t* bar, uint32_t par) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}\n" ::"r"(su(bar)), "r"(par) : "memory");
}
__global__ void k(long long* out) {
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar[0])) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar[1])) : "memory");
        long long t0 = clock64();
        for (int i = 0; i < 100; ++i) wait_try(&bar[0], 0);
        long long t1 = clock64();
        for (int i = 0; i < 100; ++i) wait_test(&bar[1], 0);
        long long t2 = clock64();
        out[0] = (t1 - t0) / 100;
        out[1] = (t2 - t1) / 100;
    }
    __syncthreads();
    // producer (warp 1) arrives after a delay; consumer (warp 0) measures arrive -> wake
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[0])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    __shared__ long long t_arr;
    if (threadIdx.x == 32) {
        long long t = clock64();
        while (clock64() - t < 20000) {}
        t_arr = clock64();
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su(&bar[0])) : "memory");
    }
    if (threadIdx.x == 0) {
        wait_try(&bar[0], 0);
        long long t = clock64();
        out[2] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) out[2] -= t_arr;
}
int main() {
    long long* d;
    cudaMalloc(&d, 64);
    k<<<1, 64>>>(d);
    long long h[3];
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("completed phase: try_wait %lld cycles, test_wait %lld cycles; arrive->wake (try_wait) %lld cycles\n",
           h[0], h[1], h[2]);
    return 0;
}
