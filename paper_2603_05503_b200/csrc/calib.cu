// calib.cu -- a2..a5: calibration statistics of one prompt at one (t, l), all heads.
//
// PAPER.md P:486-571 + P:643 ("custom CUDA kernel that operates at block granularity and
// accumulates the required statistics without materializing the full attention matrix P"):
//   a2  lse_i = log sum_j exp(scale q_i.k_j)            (or taken from lse_in, the dense run's own)
//   a3  E_{r,c} = (1/|I_r|) sum_{i in I_r} sum_{j in J_c} exp(s_ij - lse_i)   (Eq. eq:block_energy;
//       divides by the actual |I_r| -- reading Q2)
//   a4  shortest prefix of (E desc, c asc) whose fp64 sequential sum of the fp32 E values
//       reaches eps(t) (Eq. eq:row_energy_constraint; readings Q4, Q5)
//   a5  keep_count[h][r][c] += kept (numerator of Eq. eq:mask_mean)
// One work item = one (head, query block); the CTA owns the row, so there are no atomics and
// every reduction runs in a fixed order (bit-reproducible).
//
// Passes over the N_B key tiles of an item (each tile: S = Q K^T by tcgen05 into TMEM):
//   lse_in given      one pass: per-row sums of exp(s - lse) reduced to E_{r,c} tile by tile.
//   scratch given     one pass: per (row, tile) the tile's log2-sum-exp u_ic = m_ic + log2(t_ic),
//                     t_ic = sum_j 2^(s_ij*l2e - m_ic) against the running max m_ic, goes to global
//                     scratch (4 bytes); after the pass lse is known and
//                     E_{r,c} = sum_i 2^(u_ic - lse2_i) / |I_r|.
//   neither           two passes (online LSE, then E) -- twice the exponentials.
// Roles (persistent, one CTA per SM, 12 warps): warp 0 TMA producer, warp 1 MMA issuer, warp 2
// TMEM allocator, warps 4-7 / 8-11 two row groups taking alternate tiles.  Exp-bound: packed
// f32x2 arithmetic and a polynomial exp2 for part of the elements offload the MUFU unit.
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

static __device__ unsigned long long* g_trace;  // csa_debug_trace (CTA 0, first item)
static __device__ int g_debug_mode;  // csa_debug_trace mode: 11 skip softmax math, 12 also skip ld

constexpr int kThreads = 384;
constexpr int kCalibEmuPerOctet = 0;  // pairs p with (p & 7) >= 8 - this -> exp2_poly5; A/B at Wan
                                      // 720p: 0 -> 78 ms, 1 -> 78, 2 -> 81, 3 -> 87 (issue-bound)

template <int BK, int D, int BKV = BK>
struct CalibSmem {
    using C = TileCfg<BK, D>;
    // key tiles of BKV rows (= BK for square blocks; B_q = 128 x B_kv, otherwise)
    static constexpr int kKBoxV = BKV * 128;
    static constexpr int kKVB = C::kBoxes * kKBoxV;
    static constexpr uint32_t kSB = (BKV + 31) / 32 * 32;  // TMEM columns per S buffer
    static constexpr uint32_t kIdescQKV = umma_idesc_bf16(128, BKV, 0, 0);
    // BK = 128: Q lives in TMEM (tcgen05.cp from the TMA'd tile) and S = Q K^T runs as a TS
    // MMA reading only K from shared memory -- measured 74 vs 107 cycles per 128x128x16
    // dispatch for the SS form (scripts/mma_bench.cu); S is then single-buffered per group
    // (TMEM: S[2] 256 + Q 64 columns).  BK = 64 (M = 64) keeps the SS form, S double-buffered.
    static constexpr bool kQT = BK == 128;
    static constexpr int kSBufs = kQT ? 1 : 2;
    static constexpr uint32_t kQCol = 2 * kSBufs * kSB;  // used when kQT
    // One Q buffer (the next item's Q waits for this item's last MMA: one bubble per N_B tiles);
    // everything else not in the K ring is small, so the ring gets 4 slots of 128x128 bf16 --
    // the pass streams K from L2 and needs that many loads in flight.
    static constexpr int kFixed = C::kQBytes + 2048 * 4 + 2048 * 8 + 4096;
    static constexpr int kQOff = 0;
    static constexpr int kKOff = C::kQBytes;
    static constexpr int kBudget = 232448 - kFixed;
    static constexpr int kSlots = kBudget / kKVB > 8 ? 8 : kBudget / kKVB;
    static constexpr int kERowOff = kKOff + kSlots * kKVB;  // float [2048]
    static constexpr int kSortOff = kERowOff + 2048 * 4;              // u64 [2048] (a4 sort)
    static constexpr int kBarOff = kSortOff + 2048 * 8;
    // q_full[2] q_empty[2] (entry 0 used) k_full[S] k_empty[S] s_full[2][2] s_empty[2][2]
    static constexpr int kNumBars = 12 + 2 * kSlots;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;  // m[2][128] l[2][128] lse2[128]
    static constexpr int kPartOff = kRowOff + 5 * 128 * 4;           // float [2][2][4]
    static constexpr int kMiscOff = kPartOff + 16 * 4;               // int32 s_cnt
    static constexpr int kTmemPtrOff = kMiscOff + 16;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static constexpr int kAlloc = kBytes;
    static_assert(kSlots >= 2, "K ring");
    static_assert(BKV == BK || (BK == 128 && BKV % 16 == 0 && kQCol + D / 2 <= 512), "B_kv");
    static_assert(kAlloc <= 232448, "smem");
};

// sum of 2^(s*sl2 - m) over the BK columns of a row (masked columns hold -inf)
template <int BK>
__device__ __forceinline__ float exp_sum(const uint32_t (&r)[BK], float sl2, float m) {
    const uint64_t sl2x2 = f2(sl2, sl2);
    const uint64_t negm = f2(-m, -m);
    uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int x = 0; x < BK; x += 2) {
        const uint64_t t = ffma2(pk2(r[x], r[x + 1]), sl2x2, negm);
        uint64_t p;
        if (((x / 2) & 7) >= 8 - kCalibEmuPerOctet) {
            p = exp2_poly5(t);
        } else {
            p = f2(ex2_approx(lo_f(t)), ex2_approx(hi_f(t)));
        }
        acc[(x / 2) & 3] = fadd2(acc[(x / 2) & 3], p);
    }
    const uint64_t s2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    return lo_f(s2) + hi_f(s2);
}

template <int BK, int D, int BKV = BK>
__global__ void __launch_bounds__(kThreads, 1)
    calib_kernel(const CalibArgs a, const __grid_constant__ CUtensorMap tq,
                 const __grid_constant__ CUtensorMap tk) {
    using C = TileCfg<BK, D>;
    using L = CalibSmem<BK, D, BKV>;
    constexpr int S = L::kSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 2;
    uint64_t* k_full = bars + 4;
    uint64_t* k_empty = bars + 4 + S;
    uint64_t* s_full = bars + 4 + 2 * S;   // [grp][buf]
    uint64_t* s_empty = bars + 8 + 2 * S;  // [grp][buf]
    float* e_row = reinterpret_cast<float*>(smem + L::kERowOff);        // [2048]
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + L::kSortOff);   // [2048]
    float* row_m = reinterpret_cast<float*>(smem + L::kRowOff);
    float* row_l = row_m + 256;
    float* row_lse2 = row_m + 512;
    float* part = reinterpret_cast<float*>(smem + L::kPartOff);         // [grp][parity][4]
    volatile int32_t* s_cnt = reinterpret_cast<int32_t*>(smem + L::kMiscOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    const Geo& g = a.g;
    const int32_t n_items = a.n_heads * g.NB;
    const bool have_lse = a.lse_in != nullptr;
    const bool use_scratch = !have_lse && a.scratch != nullptr;
    const int32_t passes = (have_lse || use_scratch) ? 1 : 2;
    const int32_t tiles_per_item = passes * g.NBK;
    const int dbg = g_debug_mode;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full + i, 1);
            mbar_init(q_empty + i, 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(s_empty + i, 4);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(k_full + i, 1);
            mbar_init(k_empty + i, 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_ptr);  // S[grp][buf] fp32, then Q (kQT)
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_ptr;

    if (warp < 4) {
        set_maxnreg_dec56();
        if (warp == 0) {
            // ------------------------------------------------------------------- producer
            // (whole warp in the loop, one elected lane issues -- see the MMA issuer below)
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_k = policy_evict_last();
            uint32_t ld = 0;
            int32_t local = 0;
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                const int32_t h = item / g.NB, r = item % g.NB;
                const int qb = 0;  // single Q buffer
                mbar_wait(q_empty + qb, (local & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(q_full + qb, C::kBoxes * BK * 128);
                    tma_tile<D>(smem + L::kQOff + qb * C::kQBytes, C::kQBox, &tq, q_full + qb, h,
                                r * BK, 0, pol_q);
                }
                __syncwarp();
                for (int32_t j = 0; j < tiles_per_item; ++j) {
                    const int32_t c = j % g.NBK;
                    const uint32_t slot = ld % S, ph = (ld / S) & 1;
                    ++ld;
                    if (local == 0 && lane == 0) CSA_TRACE(3, j, 0);
                    mbar_wait(k_empty + slot, ph ^ 1);
                    if (local == 0 && lane == 0) CSA_TRACE(3, j, 1);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(k_full + slot, L::kKVB);
                        tma_tile<D>(smem + L::kKOff + slot * L::kKVB, L::kKBoxV, &tk,
                                    k_full + slot, h, c * BKV, 0, pol_k);
                    }
                    __syncwarp();
                }
            }
        } else if (warp == 1) {
            // ---------------------------------------------------------------- MMA issuer
            // The whole warp runs the loop (warp-uniform values stay in uniform registers);
            // one elected lane issues.  A single-lane branch makes ptxas wrap every
            // tcgen05.mma in an ELECT / R2UR.BROADCAST / BRA.U.ANY loop (~16 instructions of
            // dependent latency each), which capped the issue rate below the tensor pipe's.
            uint32_t cons = 0;
            uint32_t sused0 = 0, sused1 = 0;
            int32_t local = 0;
            const uint32_t q_base = smem_u32(smem + L::kQOff);
            const uint32_t k_base = smem_u32(smem + L::kKOff);
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                const int qb = 0;
                mbar_wait(q_full + qb, local & 1);
                if constexpr (L::kQT) {
                    // Q tile -> TMEM columns [kQCol, kQCol + D/2): one 128x256b copy per K = 16
                    // slice.  In-order with the MMAs: the previous item's MMAs have read the old
                    // Q before this copy lands; the smem buffer is free once the copy is done.
                    tc_fence_after();
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            tmem_cp_128x256b(tmem + L::kQCol + kk * 8,
                                             umma_desc_sw128(q_base + qb * C::kQBytes +
                                                                 (kk >> 2) * C::kQBox + (kk & 3) * 32,
                                                             16, 1024));
                        mma_commit(q_empty + qb);
                    }
                    __syncwarp();
                }
                for (int32_t j = 0; j < tiles_per_item; ++j) {
                    // tile j -> group j & 1 (S single- or double-buffered per group)
                    const int grp = j & 1;
                    uint32_t& sused = grp ? sused1 : sused0;
                    const uint32_t sb = grp * L::kSBufs + (sused % L::kSBufs);
                    if (local == 0 && lane == 0) CSA_TRACE(2, j, 0);
                    mbar_wait(s_empty + sb, ((sused / L::kSBufs) & 1) ^ 1);
                    if (local == 0 && lane == 0) CSA_TRACE(2, j, 1);
                    ++sused;
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    mbar_wait(k_full + slot, ph);
                    if (local == 0 && lane == 0) CSA_TRACE(2, j, 2);
                    tc_fence_after();
                    if (elect_one()) {
                        if constexpr (L::kQT) {
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk) {
                                const uint64_t b = umma_desc_sw128(
                                    k_base + slot * L::kKVB + (kk >> 2) * L::kKBoxV +
                                        (kk & 3) * 32, 16, 1024);
                                mma_ts(tmem + sb * L::kSB, tmem + L::kQCol + kk * 8, b,
                                       L::kIdescQKV, kk > 0 ? 1u : 0u);
                            }
                        } else {
                            issue_qk<BK, D>(tmem + sb * L::kSB, q_base + qb * C::kQBytes,
                                            k_base + slot * L::kKVB);
                        }
                        mma_commit(s_full + sb);
                        mma_commit(k_empty + slot);
                        if (!L::kQT && j == tiles_per_item - 1) mma_commit(q_empty + qb);
                    }
                    __syncwarp();
                }
            }
        }
        __syncwarp();
    } else {
        set_maxnreg_inc224();
        // ----------------------------------------------------------------- row groups
        const int grp = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int gtid = threadIdx.x - 128;  // 0..255
        const uint32_t s_lane = tmem + ((uint32_t)(quarter * 32) << 16);
        const float sl2 = a.scale_log2;
        const int32_t tail_valid = g.N - (g.NBK - 1) * BKV;
        // scratch: one float per (row, key block) -- the tile's log2-sum-exp u = m + log2(t)
        float* scr = use_scratch ? reinterpret_cast<float*>(a.scratch) +
                                       (int64_t)blockIdx.x * g.NBK * 128
                                 : nullptr;
        // scratch kept in L2 (evict_last) and its lines discarded once read: no DRAM write-back
        const uint64_t pol_scr = policy_evict_last();
        const bool discard_ok = (reinterpret_cast<uintptr_t>(scr) & 127u) == 0u;  // 128-B lines
        uint32_t scount = 0;
        int32_t local = 0;
        for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
            const int32_t h = item / g.NB, r = item % g.NB;
            const int32_t rows_valid = min(BK, g.N - r * BK);
            const bool row_ok = row < rows_valid;
            float* erow = e_row;
            float m_run = -INFINITY, l_run = 0.0f, lse2 = 0.0f;
            int32_t mine = 0;
            // S row of this group's next tile into registers; frees S[grp] for the next MMA
            auto load_s = [&](uint32_t (&s)[BKV], int32_t c) {
                const uint32_t sb = grp * L::kSBufs + (scount % L::kSBufs);
                const bool tr = local == 0 && (warp & 3) == 0 && lane == 0;
                if (tr) CSA_TRACE(grp, c, 0);
                mbar_wait(s_full + sb, (scount / L::kSBufs) & 1);
                if (tr) CSA_TRACE(grp, c, 1);
                ++scount;
                tc_fence_after();
                const uint32_t s_addr = s_lane + sb * L::kSB;
#pragma unroll
                for (int cc = 0; cc + 32 <= BKV; cc += 32) {
                    uint32_t(&rr)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[cc]);
                    tmem_ld32(s_addr + cc, rr);
                }
                if constexpr (BKV % 32 == 16)
                    tmem_ld16(s_addr + BKV - 16,
                              *reinterpret_cast<uint32_t(*)[16]>(&s[BKV - 16]));
                tmem_ld_wait();
#pragma unroll
                for (int x = 0; x < BKV; ++x) asm volatile("" : "+r"(s[x]));  // no use above
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty + sb);
                if (tr) CSA_TRACE(grp, c, 2);
                if (c == g.NBK - 1 && tail_valid < BKV) {  // keys >= N do not exist (Q2)
#pragma unroll
                    for (int x = 0; x < BKV; ++x)
                        if (x >= tail_valid) s[x] = 0xff800000u;
                }
            };
            // ---------------- LSE (a2): two-pass pass A, or the scratch single pass
            if (!have_lse) {
                for (int32_t c = grp; c < g.NBK; c += 2, ++mine) {
                    uint32_t s[BKV];
                    load_s(s, c);
                    if (dbg >= 11) continue;  // debug: pipeline without the softmax math
                    const float mt = max_half<BKV>(s) * sl2;
                    float m_use = m_run;
                    if (mine == 0 || mt > m_run + kRescaleThreshold) {  // lazy running max
                        const float m_new = fmaxf(m_run, mt);
                        if (mine > 0) l_run *= ex2_approx(m_run - m_new);
                        m_run = m_new;
                        m_use = m_new;
                    }
                    const float t = exp_sum<BKV>(s, sl2, m_use);
                    l_run += t;
                    if (use_scratch)
                        st_global_hint(scr + (int64_t)c * 128 + row,
                                       t > 0.0f ? m_use + __log2f(t) : -INFINITY, pol_scr);
                    if (local == 0 && (warp & 3) == 0 && lane == 0) CSA_TRACE(grp, c, 3);
                }
                row_m[grp * 128 + row] = m_run;
                row_l[grp * 128 + row] = l_run;
            }
            named_bar_sync(1, 256);
            if (!have_lse) {
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
            if (use_scratch) {
                // ---------------- E from the stored partials: column c of the [NB][128] matrix
                // weighted by 2^(m_ic - lse2_i) and summed over the valid rows.  Warp w (of 8)
                // takes columns c = w mod 8, four at a time; lane l holds rows l, l+32, l+64,
                // l+96 (coalesced 256 B loads, 16 in flight), then a fixed butterfly.
                if (grp == 0) row_lse2[row] = lse2;
                named_bar_sync(1, 256);
                const int w8 = gtid >> 5;
                float lr[4];
                bool okr[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    okr[q4] = lane + 32 * q4 < rows_valid;
                    lr[q4] = okr[q4] ? row_lse2[lane + 32 * q4] : 0.0f;  // no NaN from dead rows
                }
                for (int32_t c0 = w8; c0 < g.NBK; c0 += 32) {
                    float v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t c = c0 + 8 * u;
                        float uu[4];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4)
                            uu[q4] = (c < g.NBK && okr[q4]) ? scr[(int64_t)c * 128 + lane + 32 * q4]
                                                           : -INFINITY;
                        float acc = 0.0f;
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) acc += ex2_approx(uu[q4] - lr[q4]);
                        v[u] = acc;
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[u] += __shfl_xor_sync(0xffffffffu, v[u], off);
                    if (lane == 0) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (c0 + 8 * u < g.NBK) erow[c0 + 8 * u] = v[u] / (float)rows_valid;
                    }
                    if (discard_ok && lane < 16) {  // the 4 columns' 512-B scratch rows are dead
                        const int32_t c = c0 + 8 * (lane >> 2);
                        if (c < g.NBK) discard_l2_line(scr + (int64_t)c * 128 + 32 * (lane & 3));
                    }
                }
            } else {
                // ---------------- E tile by tile against the known lse (a3)
                const int32_t first_b = passes == 2 ? g.NBK : 0;
                int32_t nb_mine = 0;
                for (int32_t j = first_b + (((first_b & 1) != grp) ? 1 : 0); j < tiles_per_item;
                     j += 2, ++nb_mine) {
                    const int32_t c = j - first_b;
                    uint32_t s[BKV];
                    load_s(s, c);
                    float acc = row_ok ? exp_sum<BKV>(s, sl2, lse2) : 0.0f;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
                        acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    float* pp = part + (grp * 2 + (nb_mine & 1)) * 4;
                    if (lane == 0) pp[quarter] = acc;
                    named_bar_sync(2 + grp, 128);
                    if (quarter == 0 && lane == 0)
                        erow[c] = (((pp[0] + pp[1]) + pp[2]) + pp[3]) / (float)rows_valid;
                }
            }
            // ---------------------------------------------------- selection (group 0)
            named_bar_sync(1, 256);  // E row complete
            if (grp == 0) {
                const int t = row;  // 0..127
                float* eout = a.energy_out ? a.energy_out + ((int64_t)h * g.NB + r) * g.NBK : nullptr;
                int32_t p2 = 1;
                while (p2 < g.NBK) p2 <<= 1;
                for (int32_t x = t; x < p2; x += 128) {
                    uint64_t key = ~0ull;
                    if (x < g.NBK) {
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
                if (t == 0) {
                    double acc = 0.0;
                    int32_t cnt = 0;
                    for (int32_t x = 0; x < g.NBK; ++x) {
                        const uint32_t c = (uint32_t)(keys[x] & 0xFFFFFFFFu);
                        ++cnt;
                        acc = __dadd_rn(acc, (double)erow[c]);
                        if (acc >= a.eps) break;
                    }
                    *s_cnt = cnt;
                }
                named_bar_sync(3, 128);
                const int32_t cnt = *s_cnt;
                uint16_t* kc = a.keep_count + ((int64_t)h * g.NB + r) * g.NBK;
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
        tmem_dealloc<512>(tmem);
    }
}

template <int BK, int D, int BKV = BK>
cudaError_t launch_t(const CalibArgs& a, const CUtensorMap& tq, const CUtensorMap& tk, int grid,
                     cudaStream_t s) {
    auto kern = calib_kernel<BK, D, BKV>;
    const int smem = CalibSmem<BK, D, BKV>::kAlloc;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(a, tq, tk);
    return cudaGetLastError();
}

}  // namespace

static int calib_grid(const Geo& g, int32_t n_heads, int num_sms) {
    const int64_t items = (int64_t)n_heads * g.NB;
    return (int)(items < num_sms ? items : num_sms);
}

size_t calib_scratch_bytes(const Geo& g, int32_t n_heads, int num_sms) {
    return (size_t)calib_grid(g, n_heads, num_sms) * g.NBK * 128 * sizeof(float);
}

cudaError_t set_calib_trace(void* buf, int mode) {
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    cudaError_t e = cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(g_debug_mode, &mode, sizeof(mode));
}

cudaError_t launch_calib(const CalibArgs& a, int head_dim, const CUtensorMap& tq,
                         const CUtensorMap& tk, int num_sms, cudaStream_t s) {
    const int grid = calib_grid(a.g, a.n_heads, num_sms);
    if (a.g.BK != a.g.B) {  // non-square B_q = 128 x B_kv, head_dim 128
        if (a.g.B != 128 || head_dim != 128) return cudaErrorInvalidValue;
        switch (a.g.BK) {
            case 64: return launch_t<128, 128, 64>(a, tq, tk, grid, s);
            case 80: return launch_t<128, 128, 80>(a, tq, tk, grid, s);
            case 96: return launch_t<128, 128, 96>(a, tq, tk, grid, s);
            case 112: return launch_t<128, 128, 112>(a, tq, tk, grid, s);
            case 144: return launch_t<128, 128, 144>(a, tq, tk, grid, s);
            case 160: return launch_t<128, 128, 160>(a, tq, tk, grid, s);
            case 176: return launch_t<128, 128, 176>(a, tq, tk, grid, s);
            case 192: return launch_t<128, 128, 192>(a, tq, tk, grid, s);
            default: return cudaErrorInvalidValue;
        }
    }
    if (a.g.B == 128 && head_dim == 128) return launch_t<128, 128>(a, tq, tk, grid, s);
    if (a.g.B == 128 && head_dim == 64) return launch_t<128, 64>(a, tq, tk, grid, s);
    if (a.g.B == 64 && head_dim == 128) return launch_t<64, 128>(a, tq, tk, grid, s);
    if (a.g.B == 64 && head_dim == 64) return launch_t<64, 64>(a, tq, tk, grid, s);
    return cudaErrorInvalidValue;
}

}  // namespace csa
