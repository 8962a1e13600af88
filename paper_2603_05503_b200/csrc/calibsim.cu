// calibsim.cu -- a2..a5 and f1 of one calibration prompt at one (t, l), all heads, in ONE pass
// over the key tiles per (head, query block) (block 128 x 128, head_dim 128 or 64).
//
// PAPER.md P:486-571 + P:643 (block energies E at block granularity, P never materialised) and
// P:624-626 (the spatial-similarity statistic of the repetitive-head decision; computed together
// with the calibration statistics, as P:1224 names the lever of the calibration cost):
//   a2  lse_i = log sum_j exp(scale q_i.k_j)
//   a3  E_{r,c} = (1/|I_r|) sum_{i in I_r} sum_{j in J_c} exp(s_ij - lse_i)      (reading Q2)
//   a4  shortest prefix of (E desc, c asc) reaching eps(t), fp64 sequential     (Q4, Q5)
//   a5  keep_count[h][r][c] += kept
//   f1  per query token t and its anchor token t_a = (f, a(i), j) (Q9, Q23-Q25):
//       dot_t = sum_j p_tj p_{t_a j},  nn_t = sum_j p_tj^2,  na_t = sum_j p_{t_a j}^2
//       -> the [h][t][3] partials that sim.cu's reduce kernel turns into cos(f, i) and sim_sum.
// Same results as csa_calib_accumulate (single pass) followed by csa_spatial_similarity, up to
// fp32 rounding order.  One work item = one (head, query block): the CTA owns the row (no atomics,
// fixed reduction order, bit-reproducible).
//
// Per key tile c the MMA warp computes S = Q K_c^T and S_a = Q_a K_c^T (Q_a: the anchor tokens'
// queries, gathered row by row), both SS-MMAs into TMEM.  Each softmax thread owns one query row:
// in chunks of 32 keys it takes p = 2^(s l2e - m) and p_a = 2^(s_a l2e - m_a) against lazily
// updated running maxes of the row and of its anchor row (rescale only when a chunk max exceeds
// the reference by > 8 in log2 units: every accumulator stays below 2^8 per element), and
// accumulates l, the tile partial, sum p^2, l_a, sum p_a^2 and sum p p_a.  The per-(row, key block)
// partial of a3 goes to scratch as ONE float u_ic = m + log2(sum_{j in J_c} 2^(s l2e - m)) -- the
// tile's log2-sum-exp, independent of the reference -- so E_{r,c} = sum_i 2^(u_ic - lse2_i) / |I_r|
// once the row LSE is known (4 bytes per entry).  The anchor row's own normaliser l_a comes from
// the same S_a pass, so dot / (l l_a), nn / l^2, na / l_a^2 need no other item's result.
// Roles (persistent, 12 warps): warp 0 producer (Q by TMA, Q_a gathered, K ring), warp 1 MMA
// issuer, warp 2 TMEM allocator, warps 4-7 / 8-11 two row groups taking alternate key tiles
// (TMEM: S_0 | S_a0 | S_1 | S_a1, 128 columns each), merged at the end of the item.
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kThreadsCS = 384;
#ifndef CSA_CS_EMU
#define CSA_CS_EMU 0
#endif
constexpr int kCSEmu = CSA_CS_EMU;  // pairs p with (p & 7) >= 8 - kCSEmu -> exp2_poly5 (FMA pipe)

static __device__ unsigned long long* g_trace_cs;
#ifdef CSA_ENABLE_TRACE
#define TRACE_CS(slot, k, e)                                                                 \
    do {                                                                                     \
        if (g_trace_cs != nullptr && blockIdx.x == 0 && (k) < 1024)                          \
            g_trace_cs[((slot) * 1024 + (k)) * 8 + (e)] = clock64();                         \
    } while (0)
#else
#define TRACE_CS(slot, k, e) \
    do {                     \
    } while (0)
#endif

template <int D>
struct CalibSimSmem {
    using C = TileCfg<128, D>;
    static constexpr int kQOff = 0;                  // own Q tile (TMA)
    static constexpr int kQAOff = C::kQBytes;        // anchor Q tile (gathered)
    static constexpr int kKOff = 2 * C::kQBytes;
    static constexpr int kFixed = 2 * C::kQBytes + 2048 * 4 + 2048 * 8 + 6144;
    static constexpr int kBudget = 232448 - kFixed;
    static constexpr int kSlots = kBudget / C::kKVBytes > 8 ? 8 : kBudget / C::kKVBytes;
    static constexpr int kERowOff = kKOff + kSlots * C::kKVBytes;  // float [2048]
    static constexpr int kSortOff = kERowOff + 2048 * 4;           // u64 [2048] (a4 sort)
    static constexpr int kBarOff = kSortOff + 2048 * 8;
    // q_full q_empty | k_full[S] k_empty[S] | s_full[2] s_empty[2]
    static constexpr int kNumBars = 2 + 2 * kSlots + 4;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;  // group-1 state [7][128] + lse2 [128]
    static constexpr int kMiscOff = kRowOff + 8 * 128 * 4;  // int32 s_cnt
    static constexpr int kTmemPtrOff = kMiscOff + 16;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(kSlots >= 3, "K ring");
    static_assert(kBytes <= 232448, "smem");
};

__device__ __forceinline__ int64_t anchor_token_cs(const Geo& g, int32_t kA, int64_t t) {
    const int64_t hw = (int64_t)g.H * g.W;
    const int64_t f = t / hw;
    const int32_t i = (int32_t)((t / g.W) % g.H);
    const int64_t j = t % g.W;
    int32_t best = 0, bestd = 0x7fffffff;  // nearest anchor row (Q9), tie -> lower m
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

__device__ __forceinline__ float max32cs(const uint32_t (&r)[32]) {
    float mc[8];
#pragma unroll
    for (int q8 = 0; q8 < 8; ++q8)
        mc[q8] = fmax3(__uint_as_float(r[q8]), __uint_as_float(r[q8 + 8]),
                       fmaxf(__uint_as_float(r[q8 + 16]), __uint_as_float(r[q8 + 24])));
    return fmaxf(fmax3(mc[0], mc[1], mc[2]), fmaxf(fmax3(mc[3], mc[4], mc[5]), fmaxf(mc[6], mc[7])));
}

__device__ __forceinline__ float hsum(uint64_t v) { return lo_f(v) + hi_f(v); }

template <int D>
__global__ void __launch_bounds__(kThreadsCS, 1)
    calib_sim_kernel(const CalibArgs a, const SimArgs sa, const __grid_constant__ CUtensorMap tq,
                     const __grid_constant__ CUtensorMap tk) {
    using C = TileCfg<128, D>;
    using L = CalibSimSmem<D>;
    constexpr int BK = 128, S = L::kSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;
    uint64_t* k_empty = k_full + S;
    uint64_t* s_full = k_empty + S;  // [grp]
    uint64_t* s_empty = s_full + 2;  // [grp]
    float* e_row = reinterpret_cast<float*>(smem + L::kERowOff);       // [2048]
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + L::kSortOff);  // [2048]
    float* st1 = reinterpret_cast<float*>(smem + L::kRowOff);          // [7][128] group 1 state
    float* row_lse2 = st1 + 7 * 128;                                   // [128]
    volatile int32_t* s_cnt = reinterpret_cast<int32_t*>(smem + L::kMiscOff);
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
    if (warp == 2) tmem_alloc<512>(tmem_ptr);  // [grp][S | S_a] x 128 fp32 columns
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
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_k = policy_evict_last();
            uint32_t ld = 0;
            int32_t local = 0;
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                const int32_t h = item / g.NB, r = item % g.NB;
                mbar_wait(q_empty, (local & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(q_full, C::kQBytes);
                    tma_tile<D>(smem + L::kQOff, C::kQBox, &tq, q_full, h, r * BK, 0, pol_q);
                }
                __syncwarp();
                constexpr int kChunks = D / 8;  // 16-byte chunks per row
                const __nv_bfloat16* qb = sa.q + (int64_t)h * sa.q_sh;
                for (int x = lane; x < BK * kChunks; x += 32) {
                    const int row = x / kChunks, ch = x % kChunks;
                    const int64_t t = (int64_t)r * BK + row;
                    uint4 val = make_uint4(0u, 0u, 0u, 0u);
                    if (t < g.N)
                        val = *reinterpret_cast<const uint4*>(
                            qb + anchor_token_cs(g, sa.anchor_k, t) * sa.q_sn + ch * 8);
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
            uint32_t cons = 0, sused0 = 0, sused1 = 0;
            int32_t local = 0;
            const uint32_t q_base = smem_u32(smem + L::kQOff);
            const uint32_t qa_base = smem_u32(smem + L::kQAOff);
            const uint32_t k_base = smem_u32(smem + L::kKOff);
            for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
                mbar_wait(q_full, local & 1);
                for (int32_t c = 0; c < g.NB; ++c) {
                    const int grp = c & 1;
                    const uint32_t use = grp ? sused1++ : sused0++;
                    if (lane == 0) TRACE_CS(2, cons, 0);
                    mbar_wait(s_empty + grp, (use & 1) ^ 1);
                    if (lane == 0) TRACE_CS(2, cons, 1);
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    mbar_wait(k_full + slot, ph);
                    if (lane == 0) TRACE_CS(2, cons - 1, 2);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t kb = k_base + slot * C::kKVBytes;
                        issue_qk<BK, D>(tmem + grp * 256, q_base, kb);
                        issue_qk<BK, D>(tmem + grp * 256 + 128, qa_base, kb);
                        mma_commit(s_full + grp);
                        mma_commit(k_empty + slot);
                        if (c == g.NB - 1) mma_commit(q_empty);
                    }
                    __syncwarp();
                    if (lane == 0) TRACE_CS(2, cons - 1, 3);
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
        const uint32_t s_lane = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)grp * 256u;
        const float sl2 = a.scale_log2;
        const uint64_t sl2x2 = f2(sl2, sl2);
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;
        float* scr = reinterpret_cast<float*>(a.scratch) + (int64_t)blockIdx.x * g.NB * 128;
        // scratch kept in L2 (evict_last) and its lines discarded once read: no DRAM write-back
        const uint64_t pol_scr = policy_evict_last();
        const bool discard_ok = (reinterpret_cast<uintptr_t>(scr) & 127u) == 0u;  // 128-B lines
        uint32_t scount = 0;
        for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
            const int32_t h = item / g.NB, r = item % g.NB;
            const int32_t rows_valid = min(BK, g.N - r * BK);
            const bool row_ok = row < rows_valid;
            // running references (log2 units) and accumulators of the row and of its anchor row
            float m = -INFINITY, ma = -INFINITY;
            float l = 0.0f;
            uint64_t nn2 = 0, la2 = 0, na2 = 0, dd2 = 0;  // packed (even, odd column) partials
            const bool tr = quarter == 0 && lane == 0;
            (void)tr;
            for (int32_t c = grp; c < g.NB; c += 2) {
                if (tr) TRACE_CS(grp, scount, 0);
                mbar_wait(s_full + grp, scount & 1);
                if (tr) TRACE_CS(grp, scount, 1);
                ++scount;
                tc_fence_after();
                const bool ragged = c == g.NB - 1 && tail_valid < BK;
                uint64_t tt2 = 0;  // this tile's partial sum against m
                // chunks software-pipelined: chunk ch+1's TMEM loads are in flight while chunk
                // ch is computed (tcgen05.wait::ld waits for all of a thread's loads, so the
                // next load is issued after the wait and waited for after the math)
                uint32_t so[2][32], sx[2][32];
                tmem_ld32(s_lane, so[0]);
                tmem_ld32(s_lane + 128, sx[0]);
                tmem_ld_wait(so[0]);
                tmem_ld_wait(sx[0]);
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t(&co)[32] = so[ch & 1];
                    uint32_t(&cx)[32] = sx[ch & 1];
                    if (ch < 3) {
                        tmem_ld32(s_lane + (ch + 1) * 32, so[(ch + 1) & 1]);
                        tmem_ld32(s_lane + 128 + (ch + 1) * 32, sx[(ch + 1) & 1]);
                    }
                    if (ragged) {
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if (ch * 32 + x >= tail_valid) {  // keys >= N do not exist (Q2)
                                co[x] = 0xff800000u;
                                cx[x] = 0xff800000u;
                            }
                    }
                    const float mt = max32cs(co) * sl2;
                    const float mat = max32cs(cx) * sl2;
                    if (mt > m + kRescaleThreshold) {  // lazy reference of the row
                        const float f = ex2_approx(m - mt);  // 0 on the first chunk (m = -inf)
                        const uint64_t f1 = f2(f, f), fq = f2(f * f, f * f);
                        l *= f;
                        tt2 = fmul2(tt2, f1);
                        nn2 = fmul2(nn2, fq);
                        dd2 = fmul2(dd2, f1);
                        m = mt;
                    }
                    if (mat > ma + kRescaleThreshold) {  // lazy reference of the anchor row
                        const float f = ex2_approx(ma - mat);
                        const uint64_t f1 = f2(f, f), fq = f2(f * f, f * f);
                        la2 = fmul2(la2, f1);
                        na2 = fmul2(na2, fq);
                        dd2 = fmul2(dd2, f1);
                        ma = mat;
                    }
                    const uint64_t negm = f2(-m, -m), negma = f2(-ma, -ma);
#pragma unroll
                    for (int x = 0; x < 32; x += 2) {
                        const uint64_t to = ffma2(pk2(co[x], co[x + 1]), sl2x2, negm);
                        const uint64_t ta = ffma2(pk2(cx[x], cx[x + 1]), sl2x2, negma);
                        uint64_t p, pa;
                        if (((x / 2) & 7) >= 8 - kCSEmu) {  // FMA-pipe exponentials (A/B knob)
                            p = exp2_poly5(to);
                            pa = exp2_poly5(ta);
                        } else {
                            p = f2(ex2_approx(lo_f(to)), ex2_approx(hi_f(to)));
                            pa = f2(ex2_approx(lo_f(ta)), ex2_approx(hi_f(ta)));
                        }
                        tt2 = fadd2(tt2, p);
                        nn2 = ffma2(p, p, nn2);
                        la2 = fadd2(la2, pa);
                        na2 = ffma2(pa, pa, na2);
                        dd2 = ffma2(p, pa, dd2);
                    }
                    if (ch < 3) {
                        tmem_ld_wait(so[(ch + 1) & 1]);
                        tmem_ld_wait(sx[(ch + 1) & 1]);
                        if (ch == 2) {  // S / S_a of this group free for its next tile
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(s_empty + grp);
                            if (tr) TRACE_CS(grp, scount - 1, 2);
                        }
                    }
                }
                const float tt = hsum(tt2);
                l += tt;
                st_global_hint(scr + (int64_t)c * 128 + row, tt > 0.0f ? m + __log2f(tt) : -INFINITY,
                               pol_scr);
                if (tr) TRACE_CS(grp, scount - 1, 3);
            }
            // ------------------------------------------- merge the two groups (fixed order)
            float nn = hsum(nn2), la = hsum(la2), na = hsum(na2), dd = hsum(dd2);
            if (grp == 1) {
                st1[row] = m;
                st1[128 + row] = l;
                st1[256 + row] = ma;
                st1[384 + row] = la;
                st1[512 + row] = nn;
                st1[640 + row] = na;
                st1[768 + row] = dd;
            }
            named_bar_sync(1, 256);
            if (grp == 0) {
                const float m1 = st1[row], l1 = st1[128 + row], ma1 = st1[256 + row];
                const float M = fmaxf(m, m1), MA = fmaxf(ma, ma1);
                // a group without tiles (N_B = 1) has m = -inf and zero sums: factor 0
                const float f0 = l > 0.0f ? ex2_approx(m - M) : 0.0f;
                const float f1 = l1 > 0.0f ? ex2_approx(m1 - M) : 0.0f;
                const float g0 = la > 0.0f ? ex2_approx(ma - MA) : 0.0f;
                const float g1 = st1[384 + row] > 0.0f ? ex2_approx(ma1 - MA) : 0.0f;
                const float Lr = l * f0 + l1 * f1;
                const float La = la * g0 + st1[384 + row] * g1;
                const float NN = nn * (f0 * f0) + st1[512 + row] * (f1 * f1);
                const float NA = na * (g0 * g0) + st1[640 + row] * (g1 * g1);
                const float DD = dd * (f0 * g0) + st1[768 + row] * (f1 * g1);
                const float lse2 = M + __log2f(Lr);
                row_lse2[row] = lse2;
                if (row_ok) {
                    const int64_t t = (int64_t)r * BK + row;
                    if (a.lse_out != nullptr)
                        a.lse_out[(int64_t)h * g.N + t] = lse2 * 0.69314718055994531f;
                    float* w = sa.partials + ((int64_t)h * g.N + t) * 3;
                    w[0] = DD / (Lr * La);
                    w[1] = NN / (Lr * Lr);
                    w[2] = NA / (La * La);
                }
            }
            named_bar_sync(1, 256);
            // ---------------- E from the stored tile log-sum-exps: column c of the [NB][128]
            // matrix, 2^(u_ic - lse2_i) summed over the valid rows.  Warp w (of 8) takes columns
            // c = w mod 8, four at a time; lane l holds rows l, l+32, l+64, l+96 (coalesced 128 B
            // loads), then a fixed butterfly.
            {
                float* erow = e_row;
                const int w8 = gtid >> 5;
                float lr[4];
                bool okr[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    okr[q4] = lane + 32 * q4 < rows_valid;
                    lr[q4] = okr[q4] ? row_lse2[lane + 32 * q4] : 0.0f;
                }
                for (int32_t c0 = w8; c0 < g.NB; c0 += 32) {
                    float v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t c = c0 + 8 * u;
                        float uu[4];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4)
                            uu[q4] = (c < g.NB && okr[q4]) ? scr[(int64_t)c * 128 + lane + 32 * q4]
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
                            if (c0 + 8 * u < g.NB) erow[c0 + 8 * u] = v[u] / (float)rows_valid;
                    }
                    if (discard_ok && lane < 16) {  // the 4 columns' 512-B scratch rows are dead
                        const int32_t c = c0 + 8 * (lane >> 2);
                        if (c < g.NB) discard_l2_line(scr + (int64_t)c * 128 + 32 * (lane & 3));
                    }
                }
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
                        const float e = e_row[x];
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
                                if ((ka > kb) == up) {
                                    keys[x] = kb;
                                    keys[y] = ka;
                                }
                            }
                        }
                        named_bar_sync(3, 128);
                    }
                }
                if (t == 0) {
                    double acc = 0.0;
                    int32_t cnt = 0;
                    for (int32_t x = 0; x < g.NB; ++x) {
                        const uint32_t c = (uint32_t)(keys[x] & 0xFFFFFFFFu);
                        ++cnt;
                        acc = __dadd_rn(acc, (double)e_row[c]);
                        if (acc >= a.eps) break;
                    }
                    *s_cnt = cnt;
                }
                named_bar_sync(3, 128);
                const int32_t cnt = *s_cnt;
                uint16_t* kc = a.keep_count + ((int64_t)h * g.NB + r) * g.NB;
                for (int32_t x = t; x < cnt; x += 128) {
                    const uint32_t c = (uint32_t)(keys[x] & 0xFFFFFFFFu);
                    const uint16_t v = kc[c];
                    if (v != 0xFFFFu) kc[c] = (uint16_t)(v + 1);
                }
                named_bar_sync(3, 128);  // keys / s_cnt reused by the next item
            }
            named_bar_sync(1, 256);  // st1 / row_lse2 / scratch reused by the next item
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int D>
cudaError_t launch_cs(const CalibArgs& a, const SimArgs& s, const CUtensorMap& tq,
                      const CUtensorMap& tk, int grid, cudaStream_t st) {
    auto kern = calib_sim_kernel<D>;
    const int smem = CalibSimSmem<D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreadsCS, smem, st>>>(a, s, tq, tk);
    return cudaGetLastError();
}

}  // namespace

cudaError_t set_calib_sim_trace(void* buf, int mode) {
    (void)mode;
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    return cudaMemcpyToSymbol(g_trace_cs, &p, sizeof(p));
}

size_t calib_sim_scratch_bytes(const Geo& g, int32_t n_heads, int num_sms) {
    const int64_t items = (int64_t)n_heads * g.NB;
    const int64_t grid = items < num_sms ? items : num_sms;
    return (size_t)grid * g.NB * 128 * sizeof(float);
}

cudaError_t launch_calib_sim(const CalibArgs& a, const SimArgs& s, int head_dim,
                             const CUtensorMap& tq, const CUtensorMap& tk, int num_sms,
                             cudaStream_t st) {
    if (a.g.B != 128 || a.g.BK != 128 || a.scratch == nullptr) return cudaErrorInvalidValue;
    const int64_t items = (int64_t)a.n_heads * a.g.NB;
    const int grid = (int)(items < num_sms ? items : num_sms);
    cudaError_t e = head_dim == 128 ? launch_cs<128>(a, s, tq, tk, grid, st)
                    : head_dim == 64 ? launch_cs<64>(a, s, tq, tk, grid, st)
                                     : cudaErrorInvalidValue;
    if (e != cudaSuccess) return e;
    return launch_similarity_reduce(s, st);
}

}  // namespace csa
