// mufu_peak.cu -- measured MUFU ex2 throughput of the whole B200 under load: the exp roofline
// denominator of the calibration pass (a2/a3, SURVEY 8.5 "exp throughput").
//
// Every SM runs 16 warps (4 per SMSP) of independent ex2.approx.ftz.f32 chains for ~2 s of
// back-to-back launches (sustained clocks, power cap active like in a long calibration run);
// ex2/s = executed ex2 / CUDA-event time.  The SM clock seen by the kernel is clock64 cycles /
// event time of the same launch.  Prints one JSON line (profiles/mufu_peak_b200.json).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mufu_peak_bin scripts/mufu_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __launch_bounds__(512, 1) ex2_loop(float* out, long long* cyc, int iters) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = -1e-3f * (float)(threadIdx.x + i);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, (size_t)sms * 512 * sizeof(float));
    cudaMalloc(&cyc, (size_t)sms * sizeof(long long));
    const int threads = 512, iters = 200000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ex2_loop<<<sms, threads>>>(out, cyc, 1000);  // warm-up
    cudaDeviceSynchronize();
    // ~2 s of load: repeat launches, time the last one
    float ms = 0.f;
    double best = 0.0, clk_at_best = 0.0, sum_rate = 0.0;
    int n = 0;
    for (int rep = 0; rep < 40; ++rep) {
        cudaEventRecord(e0);
        ex2_loop<<<sms, threads>>>(out, cyc, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[256];
        cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        double cmean = 0;
        for (int i = 0; i < sms; ++i) cmean += (double)h[i];
        cmean /= sms;
        const double ex2 = (double)sms * threads * iters * 16.0;
        const double rate = ex2 / (ms * 1e-3);
        if (rep >= 10) {  // steady state
            sum_rate += rate;
            ++n;
            if (rate > best) {
                best = rate;
                clk_at_best = cmean / (ms * 1e-3) / 1e6;
            }
        }
        if (rep == 39) {
            const double mean = sum_rate / n;
            printf("{\"ex2_per_s\": %.6e, \"ex2_per_s_best\": %.6e, \"sm_mhz_at_best\": %.1f, "
                   "\"sm_mhz_last\": %.1f, \"ex2_per_clk_per_sm\": %.3f, \"sms\": %d, "
                   "\"how\": \"scripts/mufu_peak.cu: %d SMs x 512 threads of independent "
                   "ex2.approx.ftz.f32 chains, 40 launches of %d x 16 ex2 per thread, mean of the "
                   "last 30 (sustained, clocks under load)\"}\n",
                   mean, best, clk_at_best, cmean / (ms * 1e-3) / 1e6,
                   best / (clk_at_best * 1e6) / sms, sms, sms, iters);
        }
    }
    return 0;
}
