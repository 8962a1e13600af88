// xu_mix_micro.cu -- exponential throughput of the fused calibration pass's inner-loop mix on
// register data (no TMEM / MMA / barriers): per pair of scores 2 FFMA2 (exp2 arguments of the
// row and its anchor row), 4 MUFU.EX2, then FADD2 (tile sum), FFMA2 (sum p^2), FADD2 (l_a),
// FFMA2 (sum p_a^2), FFMA2 (sum p p_a) -- csrc/calibsim.cu's loop body.  Modes: mix (that body),
// exp-only (the 4 MUFU per pair alone).  Warps per SM 8 / 16 (2 / 4 per SMSP).  Prints exps per
// clock per SM and the fraction of the 16 / clk / SM MUFU rate.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_05503_b200/csrc
//        scripts/xu_mix_micro.cu -o /tmp/xu_mix
#include <cuda_runtime.h>

#include <cstdio>

#include "attn_common.cuh"

using namespace csa;
using namespace csa::attn;

template <bool kMix>
__global__ void mix_loop(int iters, float* out, long long* cyc) {
    uint32_t so[32], sx[32];
#pragma unroll
    for (int x = 0; x < 32; ++x) {
        so[x] = __float_as_uint(-0.01f * (float)((threadIdx.x + x) & 63));
        sx[x] = __float_as_uint(-0.02f * (float)((threadIdx.x * 3 + x) & 63));
    }
    const uint64_t sl2x2 = f2(0.1275f, 0.1275f), negm = f2(-0.5f, -0.5f), negma = f2(-0.25f, -0.25f);
    uint64_t tt2 = 0, nn2 = 0, la2 = 0, na2 = 0, dd2 = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int x = 0; x < 32; x += 2) {
            const uint64_t to = ffma2(pk2(so[x], so[x + 1]), sl2x2, negm);
            const uint64_t ta = ffma2(pk2(sx[x], sx[x + 1]), sl2x2, negma);
            const uint64_t p = f2(ex2_approx(lo_f(to)), ex2_approx(hi_f(to)));
            const uint64_t pa = f2(ex2_approx(lo_f(ta)), ex2_approx(hi_f(ta)));
            if (kMix) {
                tt2 = fadd2(tt2, p);
                nn2 = ffma2(p, p, nn2);
                la2 = fadd2(la2, pa);
                na2 = ffma2(pa, pa, na2);
                dd2 = ffma2(p, pa, dd2);
            } else {
                tt2 = fadd2(tt2, p);
                la2 = fadd2(la2, pa);
            }
        }
        // keep the loads live across iterations without a dependency on the sums
        so[it & 31] ^= 1u;
        sx[it & 31] ^= 1u;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] =
        lo_f(tt2) + hi_f(nn2) + lo_f(la2) + hi_f(na2) + lo_f(dd2);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, (size_t)sms * 1024 * sizeof(float));
    cudaMalloc(&cyc, (size_t)sms * sizeof(long long));
    const int iters = 20000;
    for (int mix = 0; mix < 2; ++mix) {
        for (int warps : {8, 16}) {
            const int threads = warps * 32;
            for (int rep = 0; rep < 3; ++rep) {
                if (mix) mix_loop<true><<<sms, threads>>>(iters, out, cyc);
                else mix_loop<false><<<sms, threads>>>(iters, out, cyc);
            }
            cudaDeviceSynchronize();
            long long h[256];
            cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            double c = 0;
            for (int i = 0; i < sms; ++i) c += (double)h[i];
            c /= sms;
            const double exps_per_sm = (double)threads * iters * 64.0;  // 32 scores x 2 rows
            const double per_clk = exps_per_sm / c;
            printf("%-9s warps/SM %2d: %.2f exp/clk/SM (%.1f %% of 16)\n", mix ? "calib mix" : "exp only",
                   warps, per_clk, 100.0 * per_clk / 16.0);
        }
    }
    return 0;
}
