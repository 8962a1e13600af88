// calib.cu -- a2..a5: calibration statistics of one prompt at one (t, l), all heads.
//
// PAPER.md P:486-571 + P:643 ("custom CUDA kernel that operates at block granularity and
// accumulates the required statistics without materializing the full attention matrix P"):
//   a2  lse_i = log sum_j exp(scale q_i.k_j)                    (pass A; skipped if lse_in given)
//   a3  E_{r,c} = (1/|I_r|) sum_{i in I_r} sum_{j in J_c} exp(s_ij - lse_i)   (pass B,
//       Eq. eq:block_energy; divides by the actual |I_r| -- reading Q2)
//   a4  shortest prefix of (E desc, c asc) whose fp64 sequential sum of the fp32 E values
//       reaches eps(t) (Eq. eq:row_energy_constraint; readings Q4, Q5)
//   a5  keep_count[h][r][c] += kept (numerator of Eq. eq:mask_mean)
// One work item = one (head, query block) pair; the CTA owns the row, so no atomics anywhere and
// every reduction runs in a fixed order (bit-reproducible).
//
// Roles (persistent, one CTA per SM, 12 warps): warp 0 TMA producer (Q, then every K tile of
// pass A and pass B), warp 1 MMA issuer (S_j = Q K_j^T into TMEM S[j&1]), warp 2 TMEM allocator,
// warps 4-7 / 8-11 two row groups taking alternate tiles.  Exp-bound (N^2 exp per pass).
#include <cstdint>

#include "csa_internal.cuh"
#include "tiles.cuh"

namespace csa {
namespace {

constexpr int kThreads = 384;

template <int BK, int D>
struct CalibSmem {
    using C = TileCfg<BK, D>;
    static constexpr int kBudget = 200 * 1024 - 2 * C::kQBytes - 2 * 2048 * 4 - 2048 * 8;
    static constexpr int kSlots = kBudget / C::kKVBytes > 8 ? 8 : kBudget / C::kKVBytes;
    static constexpr int kMaxBlocks1 = 2048;
    static constexpr int kQOff = 0;
    static constexpr int kKOff = 2 * C::kQBytes;
    static constexpr int kERowOff = kKOff + kSlots * C::kKVBytes;          // float [2][2048]
    static constexpr int kSortOff = kERowOff + 2 * kMaxBlocks1 * 4;         // u64 [2048]
    static constexpr int kBarOff = kSortOff + 2048 * 8;
    // q_full[2] q_empty[2] k_full[S] k_empty[S] s_full[2] s_empty[2]
    static constexpr int kNumBars = 8 + 2 * kSlots;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;                  // m[2][128] l[2][128]
    static constexpr int kPartOff = kRowOff + 4 * 128 * 4;                  // float [2][2][4]
    static constexpr int kTmemPtrOff = kPartOff + 16 * 4;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static constexpr int kAlloc = kBytes;  // base is 1 KiB aligned (__align__ on the extern)
    static_assert(kAlloc <= 232448, "smem");
};

template <int BK, int D>
__global__ void __launch_bounds__(kThreads, 1)
    calib_kernel(const CalibArgs a, const __grid_constant__ CUtensorMap tq,
                 const __grid_constant__ CUtensorMap tk) {
    using C = TileCfg<BK, D>;
    using L = CalibSmem<BK, D>;
    constexpr int S = L::kSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();  // SWIZZLE_128B atoms need 1 KiB alignment
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 2;
    uint64_t* k_full = bars + 4;
    uint64_t* k_empty = bars + 4 + S;
    uint64_t* s_full = bars + 4 + 2 * S;
    uint64_t* s_empty = bars + 6 + 2 * S;
    float* e_row = reinterpret_cast<float*>(smem + L::kERowOff);          // [2][2048]
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + L::kSortOff);     // [2048]
    float* row_m = reinterpret_cast<float*>(smem + L::kRowOff);
    float* row_l = row_m + 256;
    float* part = reinterpret_cast<float*>(smem + L::kPartOff);           // [grp][parity][4]
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    const Geo& g = a.g;
    const int32_t n_items = a.n_heads * g.NB;
    const int32_t passes = a.lse_in ? 1 : 2;
    const int32_t tiles_per_item = passes * g.NB;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full + i, 1);
            mbar_init(q_empty + i, 1);
            mbar_init(s_full + i, 1);
            mbar_init(s_empty + i, 4);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(k_full + i, 1);
            mbar_init(k_empty + i, 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<256>(tmem_ptr);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_ptr;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_k = policy_evict_last();
            uint32_t ld = 0;
            int32_t local = 0;
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                const int32_t h = item / g.NB, r = item % g.NB;
                const int qb = local & 1;
                mbar_wait(q_empty + qb, ((local >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(q_full + qb, C::kBoxes * BK * 128);
                tma_tile<D>(smem + L::kQOff + qb * C::kQBytes, C::kQBox, &tq, q_full + qb, h,
                            r * BK, 0, pol_q);
                for (int32_t j = 0; j < tiles_per_item; ++j) {
                    const int32_t c = j % g.NB;
                    const uint32_t slot = ld % S, ph = (ld / S) & 1;
                    ++ld;
                    mbar_wait(k_empty + slot, ph ^ 1);
                    mbar_arrive_expect_tx(k_full + slot, C::kKVBytes);
                    tma_tile<D>(smem + L::kKOff + slot * C::kKVBytes, C::kKBox, &tk, k_full + slot,
                                h, c * BK, 0, pol_k);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            uint32_t cons = 0;
            uint32_t sused[2] = {0, 0};
            int32_t local = 0;
            const uint32_t q_base = smem_u32(smem + L::kQOff);
            const uint32_t k_base = smem_u32(smem + L::kKOff);
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                const int qb = local & 1;
                mbar_wait(q_full + qb, (local >> 1) & 1);
                for (int32_t j = 0; j < tiles_per_item; ++j) {
                    const int grp = j & 1;
                    mbar_wait(s_empty + grp, (sused[grp] & 1) ^ 1);
                    ++sused[grp];
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    mbar_wait(k_full + slot, ph);
                    tc_fence_after();
                    issue_qk<BK, D>(tmem + grp * BK, q_base + qb * C::kQBytes,
                                    k_base + slot * C::kKVBytes);
                    mma_commit(s_full + grp);
                    mma_commit(k_empty + slot);
                    if (j == tiles_per_item - 1) mma_commit(q_empty + qb);
                }
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        const int grp = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t s_addr = tmem + ((uint32_t)(quarter * 32) << 16) + grp * BK;
        const float sl2 = a.scale_log2;
        uint32_t scount = 0;
        int32_t local = 0;
        for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
            const int32_t h = item / g.NB, r = item % g.NB;
            const int32_t rows_valid = min(BK, g.N - r * BK);
            const bool row_ok = row < rows_valid;
            float* erow = e_row + (local & 1) * 2048;
            float m_run = -INFINITY, l_run = 0.0f, lse2 = 0.0f;
            // load the S row of tile j (group grp owns every other tile), then free S[grp]
            auto load_s = [&](float (&s)[BK]) {
                mbar_wait(s_full + grp, scount & 1);
                ++scount;
                tc_fence_after();
                uint32_t rr[32];
#pragma unroll
                for (int cc = 0; cc < BK; cc += 32) {
                    tmem_ld32(s_addr + cc, rr);
                    tmem_ld_wait(rr);
#pragma unroll
                    for (int x = 0; x < 32; ++x) s[cc + x] = __uint_as_float(rr[x]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty + grp);
            };
            // ---------------- pass A: online row max / sum over all N keys (a2)
            if (passes == 2) {
                for (int32_t j = grp; j < g.NB; j += 2) {
                    float s[BK];
                    load_s(s);
                    const int32_t valid = g.N - j * BK;
                    float mx = -INFINITY;
#pragma unroll
                    for (int x = 0; x < BK; ++x)
                        if (x < valid) mx = fmaxf(mx, s[x]);
                    const float m_new = fmaxf(m_run, mx * sl2);
                    float acc = 0.0f;
#pragma unroll
                    for (int x = 0; x < BK; ++x)
                        if (x < valid) acc += ex2_approx(fmaf(s[x], sl2, -m_new));
                    l_run = l_run * ex2_approx(m_run - m_new) + acc;
                    m_run = m_new;
                }
                row_m[grp * 128 + row] = m_run;
                row_l[grp * 128 + row] = l_run;
            }
            named_bar_sync(1, 256);
            if (passes == 2) {
                const float m0 = row_m[row], m1 = row_m[128 + row];
                const float l0 = row_l[row], l1 = row_l[128 + row];
                const float M = fmaxf(m0, m1);
                const float l0s = l0 > 0.0f ? l0 * ex2_approx(m0 - M) : 0.0f;
                const float l1s = l1 > 0.0f ? l1 * ex2_approx(m1 - M) : 0.0f;
                lse2 = M + __log2f(l0s + l1s);
            } else {
                lse2 = row_ok ? a.lse_in[(int64_t)h * g.N + r * BK + row] * 1.4426950408889634f
                              : 0.0f;
            }
            if (grp == 0 && a.lse_out != nullptr && row_ok)
                a.lse_out[(int64_t)h * g.N + r * BK + row] = lse2 * 0.69314718055994531f;
            // ---------------- pass B: block energies E_{r,c} (a3)
            const int32_t first_b = passes == 2 ? g.NB : 0;
            int32_t nb_mine = 0;
            for (int32_t j = first_b + (((first_b & 1) != grp) ? 1 : 0); j < tiles_per_item;
                 j += 2, ++nb_mine) {
                float s[BK];
                load_s(s);
                const int32_t c = j - first_b;
                const int32_t valid = g.N - c * BK;
                float acc = 0.0f;
                if (row_ok) {
#pragma unroll
                    for (int x = 0; x < BK; ++x)
                        if (x < valid) acc += ex2_approx(fmaf(s[x], sl2, -lse2));
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                float* pp = part + (grp * 2 + (nb_mine & 1)) * 4;
                if (lane == 0) pp[quarter] = acc;
                named_bar_sync(2 + grp, 128);
                if (quarter == 0 && lane == 0)
                    erow[c] = (((pp[0] + pp[1]) + pp[2]) + pp[3]) / (float)rows_valid;
            }
            // ---------------------------------------------------- selection (group 0)
            named_bar_sync(1, 256);  // E row complete
            if (grp == 0) {
                const int t = row;  // 0..127
                float* eout = a.energy_out ? a.energy_out + ((int64_t)h * g.NB + r) * g.NB : nullptr;
                int32_t p2 = 1;
                while (p2 < g.NB) p2 <<= 1;
                for (int32_t x = t; x < p2; x += 128) {
                    uint64_t key = ~0ull;
                    if (x < g.NB) {
                        const float e = erow[x];
                        if (eout) eout[x] = e;
                        key = ((uint64_t)(0xFFFFFFFFu - __float_as_uint(e)) << 32) | (uint32_t)x;
                    }
                    keys[x] = key;
                }
                named_bar_sync(3, 128);
                for (int32_t k2 = 2; k2 <= p2; k2 <<= 1) {
                    for (int32_t jj = k2 >> 1; jj > 0; jj >>= 1) {
                        for (int32_t x = t; x < p2; x += 128) {
                            const int32_t y = x ^ jj;
                            if (y > x) {
                                const uint64_t ka = keys[x], kb = keys[y];
                                const bool up = (x & k2) == 0;
                                if ((ka > kb) == up) { keys[x] = kb; keys[y] = ka; }
                            }
                        }
                        named_bar_sync(3, 128);
                    }
                }
                __shared__ int32_t s_cnt;
                if (t == 0) {
                    double acc = 0.0;
                    int32_t cnt = 0;
                    for (int32_t x = 0; x < g.NB; ++x) {
                        const uint32_t c = (uint32_t)(keys[x] & 0xFFFFFFFFu);
                        ++cnt;
                        acc = __dadd_rn(acc, (double)erow[c]);
                        if (acc >= a.eps) break;
                    }
                    s_cnt = cnt;
                }
                named_bar_sync(3, 128);
                const int32_t cnt = s_cnt;
                uint16_t* kc = a.keep_count + ((int64_t)h * g.NB + r) * g.NB;
                for (int32_t x = t; x < cnt; x += 128) {
                    const uint32_t c = (uint32_t)(keys[x] & 0xFFFFFFFFu);
                    const uint16_t v = kc[c];
                    if (v != 0xFFFFu) kc[c] = (uint16_t)(v + 1);
                }
                named_bar_sync(3, 128);  // keys / s_cnt reused by the next item
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

template <int BK, int D>
cudaError_t launch_t(const CalibArgs& a, const CUtensorMap& tq, const CUtensorMap& tk, int grid,
                     cudaStream_t s) {
    auto kern = calib_kernel<BK, D>;
    const int smem = CalibSmem<BK, D>::kAlloc;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(a, tq, tk);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_calib(const CalibArgs& a, int head_dim, const CUtensorMap& tq,
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
