// sim.cu -- f1: the spatial-similarity statistic of the repetitive-head decision.
//
// "We compute the cosine similarity between each P^(f,i) and its nearest
// anchor row, then average over f, i, and the input prompts to obtain s^(t,l,h).  When s exceeds
// a threshold gamma, we mark the corresponding (t,l,h) to be computed as spatially repetitive."
// P^(f,i) = the rows of the dense map P = softmax(scale Q K^T) (Eq. eq:p, all N keys) of the W
// query tokens (f, i, 0..W-1).  Readings (Q23-Q25): Frobenius cosine of the two W x N
// blocks with query (f,i,j) paired to (f,a(i),j); the mean runs over every (f, i) including the
// anchor rows; a(i) is the nearest anchor of Q9.  The paper computes this in PyTorch; here
// it is fused into one pass over the key tiles per (head, query block), P never materialised:
//   kernel 1 (per head, query block): for each query token t and its anchor token t_a, over all
//     key tiles: p = 2^(s*scale*log2e - lse2_t), p_a likewise with lse2_{t_a};
//     dot_t = sum p p_a, nn_t = sum p^2, na_t = sum p_a^2   -> workspace [h][t] (fp32 x 3)
//   kernel 2 (per head): cos(f,i) = sum_j dot / sqrt(sum_j nn * sum_j na) (j ascending), and
//     sim_sum[h] += sum over (f,i) of cos (fixed-order reduction; one writer per head).
// The row LSE comes from the calibration pass (csa_calib_accumulate's lse_out) or the dense run.
// Roles of kernel 1 (persistent, 12 warps): warp 0 producer (own Q by TMA, anchor Q rows gathered
// into the swizzled tile, K ring), warp 1 MMA issuer (S = Q K^T and S_a = Q_a K^T per tile),
// warp 2 TMEM allocator, warps 4-7 / 8-11 two groups on alternate key tiles, merged at the end.
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kThreadsSim = 384;

template <int BK, int D>
struct SimSmem {
    using C = TileCfg<BK, D>;
    static constexpr int kQOff = 0;                        // own Q tile
    static constexpr int kQAOff = C::kQBytes;              // anchor Q tile (gathered)
    static constexpr int kKOff = 2 * C::kQBytes;
    static constexpr int kBudget = 224 * 1024 - kKOff;
    static constexpr int kSlots = kBudget / C::kKVBytes > 6 ? 6 : kBudget / C::kKVBytes;
    static constexpr int kBarOff = kKOff + kSlots * C::kKVBytes;
    // q_full q_empty | k_full[S] k_empty[S] | s_full[2] s_empty[2]
    static constexpr int kNumBars = 2 + 2 * kSlots + 4;
    static constexpr int kPartOff = kBarOff + kNumBars * 8;   // float [3][128] group-1 partials
    static constexpr int kLseOff = kPartOff + 3 * 128 * 4;    // float [2][128] lse2 own / anchor
    static constexpr int kTmemPtrOff = kLseOff + 2 * 128 * 4;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(kSlots >= 2, "K ring");
    static_assert(kBytes <= 232448, "smem");
};

__device__ __forceinline__ int64_t anchor_token(const Geo& g, int32_t kA, int64_t t) {
    const int64_t hw = (int64_t)g.H * g.W;
    const int64_t f = t / hw;
    const int32_t i = (int32_t)((t / g.W) % g.H);
    const int64_t j = t % g.W;
    // nearest anchor (Q9): a_m = floor((2m+1)H/(2k)), tie -> lower m
    int32_t best = 0, bestd = 0x7fffffff;
    for (int32_t m = 0; m < kA; ++m) {
        const int32_t am = anchor_row(g.H, kA, m);
        const int32_t dd = am > i ? am - i : i - am;
        if (dd < bestd) {
            best = am;
            bestd = dd;
        }
    }
    return f * hw + (int64_t)best * g.W + j;
}

template <int BK, int D>
__global__ void __launch_bounds__(kThreadsSim, 1)
    sim_partials_kernel(const SimArgs a, const __grid_constant__ CUtensorMap tq,
                        const __grid_constant__ CUtensorMap tk) {
    using C = TileCfg<BK, D>;
    using L = SimSmem<BK, D>;
    constexpr int S = L::kSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;
    uint64_t* k_empty = k_full + S;
    uint64_t* s_full = k_empty + S;  // [grp]
    uint64_t* s_empty = s_full + 2;  // [grp]
    float* part = reinterpret_cast<float*>(smem + L::kPartOff);
    float* lse_s = reinterpret_cast<float*>(smem + L::kLseOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    const Geo& g = a.g;
    const int32_t n_items = a.n_heads * g.NB;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 2);  // TMA (own rows, with tx) + the anchor gather
        mbar_init(q_empty, 1);
        for (int i = 0; i < S; ++i) {
            mbar_init(k_full + i, 1);
            mbar_init(k_empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(s_empty + i, 4);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_ptr);  // [grp][own | anchor] x BK fp32 columns
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_ptr;

    if (warp < 4) {
        set_maxnreg_dec56();
        if (warp == 0) {
            // ------------------------------------------------------------------- producer
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_k = policy_evict_last();
            const __nv_bfloat16* qh_base = a.q;
            uint32_t ld = 0;
            int32_t local = 0;
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                const int32_t h = item / g.NB, r = item % g.NB;
                mbar_wait(q_empty, (local & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(q_full, C::kBoxes * BK * 128);
                    tma_tile<D>(smem + L::kQOff, C::kQBox, &tq, q_full, h, r * BK, 0, pol_q);
                }
                __syncwarp();
                // anchor query rows t_a of the block's tokens, into the swizzled tile
                constexpr int kChunks = D / 8;  // 16-byte chunks per row
                const __nv_bfloat16* qb = qh_base + (int64_t)h * a.q_sh;
                for (int x = lane; x < BK * kChunks; x += 32) {
                    const int row = x / kChunks, ch = x % kChunks;
                    const int64_t t = (int64_t)r * BK + row;
                    uint4 val = make_uint4(0u, 0u, 0u, 0u);
                    if (t < g.N)
                        val = *reinterpret_cast<const uint4*>(
                            qb + anchor_token(g, a.anchor_k, t) * a.q_sn + ch * 8);
                    *reinterpret_cast<uint4*>(smem + L::kQAOff + (ch >> 3) * C::kQBox +
                                              sw128_offset(row, ch & 7)) = val;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(q_full);
                for (int32_t c = 0; c < g.NB; ++c) {
                    const uint32_t slot = ld % S, ph = (ld / S) & 1;
                    ++ld;
                    mbar_wait(k_empty + slot, ph ^ 1);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(k_full + slot, C::kKVBytes);
                        tma_tile<D>(smem + L::kKOff + slot * C::kKVBytes, C::kKBox, &tk,
                                    k_full + slot, h, c * BK, 0, pol_k);
                    }
                    __syncwarp();
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------------------------ MMA issuer
            uint32_t cons = 0, sused[2] = {0, 0};
            int32_t local = 0;
            const uint32_t q_base = smem_u32(smem + L::kQOff);
            const uint32_t qa_base = smem_u32(smem + L::kQAOff);
            const uint32_t k_base = smem_u32(smem + L::kKOff);
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                mbar_wait(q_full, local & 1);
                for (int32_t c = 0; c < g.NB; ++c) {
                    const int grp = c & 1;
                    mbar_wait(s_empty + grp, (sused[grp] & 1) ^ 1);
                    ++sused[grp];
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    mbar_wait(k_full + slot, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t kb = k_base + slot * C::kKVBytes;
                        issue_qk<BK, D>(tmem + grp * 2 * BK, q_base, kb);
                        issue_qk<BK, D>(tmem + grp * 2 * BK + BK, qa_base, kb);
                        mma_commit(s_full + grp);
                        mma_commit(k_empty + slot);
                        if (c == g.NB - 1) mma_commit(q_empty);
                    }
                    __syncwarp();
                }
            }
        }
        __syncwarp();
    } else {
        set_maxnreg_inc224();
        // ---------------------------------------------------------------- row groups
        const int grp = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16) + grp * 2 * BK;
        const float sl2 = a.scale_log2;
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;
        const uint64_t sl2x2 = f2(sl2, sl2);
        uint32_t scount = 0;
        int32_t local = 0;
        for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
            const int32_t h = item / g.NB, r = item % g.NB;
            const int64_t t = (int64_t)r * BK + row;
            const bool row_ok = row < BK && t < g.N;
            // log2-domain LSE of this row's token and of its anchor token
            float lo = 0.0f, la = 0.0f;
            if (row_ok) {
                const float* lh = a.lse + (int64_t)h * g.N;
                lo = lh[t] * 1.4426950408889634f;
                la = lh[anchor_token(g, a.anchor_k, t)] * 1.4426950408889634f;
            }
            const uint64_t nlo = f2(-lo, -lo), nla = f2(-la, -la);
            uint64_t dot2 = 0, nn2 = 0, na2 = 0;  // packed partial sums (even / odd columns)
            for (int32_t c = grp; c < g.NB; c += 2) {
                mbar_wait(s_full + grp, scount & 1);
                ++scount;
                tc_fence_after();
                const bool ragged = (c == g.NB - 1) && tail_valid < BK;
#pragma unroll
                for (int cc = 0; cc < BK; cc += 32) {
                    uint32_t so[32], sa[32];
                    tmem_ld32(lane_addr + cc, so);
                    tmem_ld32(lane_addr + BK + cc, sa);
                    tmem_ld_wait(so);
                    tmem_ld_wait(sa);
                    if (cc + 32 >= BK) {  // last chunk: S free for this group's next tile
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(s_empty + grp);
                    }
                    if (ragged) {
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if (cc + x >= tail_valid) {  // keys >= N do not exist (Q2)
                                so[x] = 0xff800000u;
                                sa[x] = 0xff800000u;
                            }
                    }
#pragma unroll
                    for (int x = 0; x < 32; x += 2) {
                        const uint64_t to = ffma2(pk2(so[x], so[x + 1]), sl2x2, nlo);
                        const uint64_t ta = ffma2(pk2(sa[x], sa[x + 1]), sl2x2, nla);
                        const uint64_t po = f2(ex2_approx(lo_f(to)), ex2_approx(hi_f(to)));
                        const uint64_t pa = f2(ex2_approx(lo_f(ta)), ex2_approx(hi_f(ta)));
                        dot2 = ffma2(po, pa, dot2);
                        nn2 = ffma2(po, po, nn2);
                        na2 = ffma2(pa, pa, na2);
                    }
                }
            }
            float dot = lo_f(dot2) + hi_f(dot2);
            float nn = lo_f(nn2) + hi_f(nn2);
            float na = lo_f(na2) + hi_f(na2);
            // merge the two groups (fixed order: group 0 + group 1) and publish the row
            if (grp == 1) {
                part[row] = dot;
                part[128 + row] = nn;
                part[256 + row] = na;
            }
            named_bar_sync(1, 256);
            if (grp == 0 && row_ok) {
                float* w = a.partials + ((int64_t)h * g.N + t) * 3;
                w[0] = dot + part[row];
                w[1] = nn + part[128 + row];
                w[2] = na + part[256 + row];
            }
            named_bar_sync(1, 256);  // part[] reused by the next item
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// One CTA per head: cos(f,i) over j ascending, then the fixed-order sum over (f, i).
__global__ void __launch_bounds__(256)
    sim_reduce_kernel(const SimArgs a) {
    const Geo& g = a.g;
    const int32_t h = blockIdx.x;
    const int32_t n_fi = g.F * g.H;
    const float* p = a.partials + (int64_t)h * g.N * 3;
    double acc = 0.0;
    for (int32_t u = threadIdx.x; u < n_fi; u += blockDim.x) {
        const int64_t t0 = (int64_t)u * g.W;  // tokens (f, i, 0..W-1) are contiguous
        double dot = 0.0, nn = 0.0, na = 0.0;
        for (int32_t j = 0; j < g.W; ++j) {
            dot += (double)p[(t0 + j) * 3 + 0];
            nn += (double)p[(t0 + j) * 3 + 1];
            na += (double)p[(t0 + j) * 3 + 2];
        }
        const double cs = dot / (sqrt(nn) * sqrt(na));
        if (a.cos_out) a.cos_out[(int64_t)h * n_fi + u] = (float)cs;
        acc += cs;
    }
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s2 = 128; s2 > 0; s2 >>= 1) {
        if ((int)threadIdx.x < s2) red[threadIdx.x] += red[threadIdx.x + s2];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.sim_sum[h] += red[0];
}

template <int BK, int D>
cudaError_t launch_t(const SimArgs& a, const CUtensorMap& tq, const CUtensorMap& tk, int grid,
                     cudaStream_t s) {
    auto kern = sim_partials_kernel<BK, D>;
    const int smem = SimSmem<BK, D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreadsSim, smem, s>>>(a, tq, tk);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    sim_reduce_kernel<<<a.n_heads, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_similarity_reduce(const SimArgs& a, cudaStream_t s) {
    sim_reduce_kernel<<<a.n_heads, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_similarity(const SimArgs& a, int head_dim, const CUtensorMap& tq,
                              const CUtensorMap& tk, int num_sms, cudaStream_t s) {
    const int64_t items = (int64_t)a.n_heads * a.g.NB;
    const int grid = (int)(items < num_sms ? items : num_sms);
    if (a.g.B == 128 && head_dim == 128) return launch_t<128, 128>(a, tq, tk, grid, s);
    if (a.g.B == 128 && head_dim == 64) return launch_t<128, 64>(a, tq, tk, grid, s);
    if (a.g.B == 64 && head_dim == 128) return launch_t<64, 128>(a, tq, tk, grid, s);
    if (a.g.B == 64 && head_dim == 64) return launch_t<64, 64>(a, tq, tk, grid, s);
    return cudaErrorInvalidValue;
}

}  // namespace csa
