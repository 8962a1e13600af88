// attn3.cu -- a7 + a8 for block 128, head_dim 128 (the production shape): one CTA per query
// block, Q resident in tensor memory, column-split softmax.
//
// Same mathematics as attn.cu (readings Q1, Q2, Q9, Q10).
//
// Why this layout (measured): with Q in shared memory the S = Q K^T MMA
// reads 64 KB of operands per 128x128x128 tile (107 cycles per K = 16 dispatch, vs 74 with A in
// TMEM), and when P aliases S the next S of a softmax group cannot start before that group's
// P.V has run.  Here:
//   TMEM (512 columns): S0 [0,128) S1 [128,256) | O [256,384) | Q [384,448) | P [448,512)
//   Q is copied smem -> TMEM once per item (tcgen05.cp, in order with the S-MMAs), so every
//   S-MMA is a TS-MMA reading only K from shared memory; S is double-buffered and freed as soon
//   as the softmax warps have loaded it; P has its own single buffer.
// All eight softmax warps work on every tile: warps 4-7 take key columns 0-63, warps 8-11
// columns 64-127 of the same 128 rows (one row per thread per half); the two halves agree on the
// running max through shared memory once per tile, and each half owns 64 of the head-dim
// columns of O for the lazy rescale and the epilogue.
// Roles: warp 0 scheduler + producer (Q by TMA or anchor-row gather; K and V through separate
// rings), warp 1 S-issuer (Q copy + S = Q K^T), warp 3 PV-issuer (O += P V), warp 2 TMEM
// allocator.  Issuers and producer run warp-uniform loops; one elected lane issues.
#include <cstdint>
#include <cstdlib>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kItemSlots3 = 4;
// P placement: true -> own 64-column TMEM buffer (S[b] is released as soon as the softmax has
// loaded it, so S-MMAs never wait for a P.V; the softmax waits for the previous tile's P.V
// before overwriting P); false -> P over S[b]'s first 64 columns (S[b] released by the P.V).
constexpr bool kSeparateP = false;
constexpr int kEmu3 = 1;  // element pairs p with (p & 7) >= 8 - kEmu3 -> polynomial exp2 (A/B: 1 >= 2 > 0 > 3)
static __device__ unsigned long long* g_trace;
static __device__ int g_debug_mode;

// CG = softmax column groups (4 warps each): every tile is split over CG x 4 warps, group g
// taking key columns g*128/CG ...; more groups = more warps per SM sub-partition to hide the
// TMEM-load / exchange / P-store latencies of the per-tile softmax.
template <int CG>
struct Smem3 {
    static constexpr int kThreads = 128 + 128 * CG;
    static constexpr int kBox = 128 * 128;      // [128 rows][64 cols] bf16, SWIZZLE_128B
    static constexpr int kTile = 2 * kBox;      // 128 x 128 bf16 (Q, K or V tile)
    static constexpr int kQOff = 0;             // single Q buffer (freed once copied to TMEM)
    static constexpr int kKOff = kTile;
    static constexpr int kKSlots = CG == 2 ? 4 : 3, kVSlots = 2;  // A/B: K4V2 >= K3V3 >= K2V4
    static constexpr int kVOff = kKOff + kKSlots * kTile;
    static constexpr int kBarOff = kVOff + kVSlots * kTile;
    // q_full q_empty | k_full[KS] k_empty[KS] | v_full[VS] v_empty[VS] | s_full[2] s_free[2] |
    // p_full p_empty | o_full o_empty | item_full[4] item_empty[4]
    static constexpr int kNumBars =
        2 + 2 * kKSlots + 2 * kVSlots + 4 + 2 + 2 + 2 * kItemSlots3 + 2 * CG;
    static constexpr int kHmaxOff = kBarOff + kNumBars * 8;     // float [2 parity][CG][128]
    static constexpr int kItemOff = kHmaxOff + 2 * CG * 128 * 4;  // int32 [kItemSlots3]
    static constexpr int kTmemPtrOff = kItemOff + kItemSlots3 * 4;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(kBytes <= 232448, "smem");
    static constexpr uint32_t kS = 0, kO = 256, kQ = 384, kP = 448;  // kP unused if P aliases S
    static constexpr uint32_t kIdescQK = umma_idesc_bf16(128, 128, 0, 0);
    static constexpr uint32_t kIdescPV = umma_idesc_bf16(128, 128, 0, 1);
};

#ifdef CSA_ENABLE_TRACE  // trace builds only (see attn_common.cuh)
#define TRACE3(slot, k, e)                                                                  \
    do {                                                                                    \
        if (g_trace != nullptr && blockIdx.x == 0 && local == 0 && (k) < 1024)              \
            g_trace[((slot) * 1024 + (k)) * 8 + (e)] = clock64();                           \
    } while (0)
#else
#define TRACE3(slot, k, e) \
    do {                   \
    } while (0)
#endif

template <int CG>
__global__ void __launch_bounds__(Smem3<CG>::kThreads, 1)
    sparse_attn_q_tmem_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                              const __grid_constant__ CUtensorMap tk,
                              const __grid_constant__ CUtensorMap tv) {
    using L = Smem3<CG>;
    constexpr int BK = 128, D = 128, HC = 128 / CG;
    constexpr int KS = L::kKSlots, VS = L::kVSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;
    uint64_t* k_empty = k_full + KS;
    uint64_t* v_full = k_empty + KS;
    uint64_t* v_empty = v_full + VS;
    uint64_t* s_full = v_empty + VS;
    uint64_t* pv_done = s_full + 2;  // [b]: S[b] free (softmax loaded it / its P.V completed)
    uint64_t* p_full = pv_done + 2;
    uint64_t* p_empty = p_full + 1;
    uint64_t* o_full = p_empty + 1;
    uint64_t* o_empty = o_full + 1;
    uint64_t* item_full = o_empty + 1;
    uint64_t* item_empty = item_full + kItemSlots3;
    uint64_t* hx_full = item_empty + kItemSlots3;  // [group][parity]: group posted its tile max
    float* hmax = reinterpret_cast<float*>(smem + L::kHmaxOff);
    volatile int32_t* item_slot = reinterpret_cast<int32_t*>(smem + L::kItemOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < KS; ++i) {
            mbar_init(k_full + i, 1);
            mbar_init(k_empty + i, 1);
        }
        for (int i = 0; i < VS; ++i) {
            mbar_init(v_full + i, 1);
            mbar_init(v_empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(pv_done + i, kSeparateP ? 4 * CG : 1);
        }
        mbar_init(p_full, 4 * CG);
        mbar_init(p_empty, 1);
        mbar_init(o_full, 1);
        mbar_init(o_empty, 4 * CG);
        for (int i = 0; i < kItemSlots3; ++i) {
            mbar_init(item_full + i, 1);
            mbar_init(item_empty + i, 2 + 4 * CG);  // S-issuer, PV-issuer, softmax warps
        }
        for (int i = 0; i < 2 * CG; ++i) mbar_init(hx_full + i, 4);  // 4 warps per group
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_ptr);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk);
        tma_prefetch(&tv);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_ptr;
    const int32_t n_items = (*a.n_work) * a.batch;
    const Geo& g = a.g;

    auto next_item = [&](int32_t local) -> int32_t {
        const int s = local % kItemSlots3;
        mbar_wait(item_full + s, (local / kItemSlots3) & 1);
        const int32_t idx = item_slot[s];
        __syncwarp();
        if (lane == 0) mbar_arrive(item_empty + s);
        return idx;
    };

    if (warp < 4) {
        if constexpr (CG == 2) set_maxnreg_dec56();
        if (warp == 0) {
            // ------------------------------------------------------------ scheduler + producer
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_kv = policy_evict_last();
            uint32_t ldk = 0, ldv = 0;
            for (int32_t local = 0;; ++local) {
                const int s = local % kItemSlots3;
                mbar_wait(item_empty + s, ((local / kItemSlots3) & 1) ^ 1);
                int32_t item = 0;
                if (lane == 0) {
                    item = a.sched ? (int32_t)atomicAdd(a.sched, 1u)
                                   : (int32_t)blockIdx.x + local * (int32_t)gridDim.x;
                    if (item >= n_items) item = -1;
                    item_slot[s] = item;
                    mbar_arrive(item_full + s);
                }
                item = __shfl_sync(0xffffffffu, item, 0);
                if (item < 0) break;
                const Item it = decode_item(a, item);
                const TileList tl = tile_list(a, it);
                uint8_t* qdst = smem + L::kQOff;
                mbar_wait(q_empty, (local & 1) ^ 1);
                if (it.kind == 0) {
                    if (elect_one()) {
                        mbar_arrive_expect_tx(q_full, L::kTile);
                        tma_tile<D>(qdst, L::kBox, &tq, q_full, it.h, it.idx * BK, it.b, pol_q);
                    }
                    __syncwarp();
                } else {
                    // anchor query rows of tile u = it.idx: g = u*128 + row -> (f, m, j)
                    const int32_t kA = a.plan.anchor_k[it.cell];
                    const int32_t per_frame = kA * g.W;
                    const int32_t n_anchor = g.F * per_frame;
                    const __nv_bfloat16* qb_ptr =
                        a.q + (int64_t)it.b * a.q_sb + (int64_t)it.h * a.q_sh;
                    constexpr int kChunks = D / 8;
                    for (int x = lane; x < 128 * kChunks; x += 32) {
                        const int row = x / kChunks, ch = x % kChunks;
                        const int32_t gi = it.idx * 128 + row;
                        uint4 val = make_uint4(0u, 0u, 0u, 0u);
                        if (gi < n_anchor) {
                            const int32_t f = gi / per_frame;
                            const int32_t m = (gi / g.W) % kA;
                            const int32_t j = gi % g.W;
                            const int64_t tok = (int64_t)f * g.H * g.W +
                                                (int64_t)anchor_row(g.H, kA, m) * g.W + j;
                            val = *reinterpret_cast<const uint4*>(qb_ptr + tok * a.q_sn + ch * 8);
                        }
                        *reinterpret_cast<uint4*>(qdst + (ch >> 3) * L::kBox +
                                                  sw128_offset(row, ch & 7)) = val;
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(q_full);
                }
                // K tiles and V tiles through their own rings, interleaved in consumption order
                // (K0, K1, V0, K2, V1, ...) so neither ring starves the issuer waiting on it.
                for (int32_t step = 0; step <= tl.n; ++step) {
                    for (int kv = 0; kv < 2; ++kv) {
                        int32_t j;
                        if (kv == 0) {
                            if (step >= tl.n) continue;
                            j = step;
                        } else {
                            if (step == 0) continue;
                            j = step - 1;
                        }
                        const int32_t c = tl.at(j);
                        uint32_t slot, ph;
                        uint8_t* dst;
                        uint64_t* fb;
                        if (kv == 0) {
                            slot = ldk % KS;
                            ph = (ldk / KS) & 1;
                            ++ldk;
                            mbar_wait(k_empty + slot, ph ^ 1);
                            dst = smem + L::kKOff + slot * L::kTile;
                            fb = k_full + slot;
                        } else {
                            slot = ldv % VS;
                            ph = (ldv / VS) & 1;
                            ++ldv;
                            mbar_wait(v_empty + slot, ph ^ 1);
                            dst = smem + L::kVOff + slot * L::kTile;
                            fb = v_full + slot;
                        }
                        if (elect_one()) {
                            mbar_arrive_expect_tx(fb, L::kTile);
                            tma_tile<D>(dst, L::kBox, kv == 0 ? &tk : &tv, fb, it.h, c * BK,
                                        it.b, pol_kv);
                        }
                        __syncwarp();
                    }
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------- S-issuer: Q -> TMEM, S_j = Q K_j^T
            uint32_t cons = 0, tcount = 0;
            const uint32_t q_base = smem_u32(smem + L::kQOff);
            const uint32_t k_base = smem_u32(smem + L::kKOff);
            for (int32_t local = 0;; ++local) {
                const int32_t item = next_item(local);
                if (item < 0) break;
                const Item it = decode_item(a, item);
                const TileList tl = tile_list(a, it);
                mbar_wait(q_full, local & 1);
                tc_fence_after();
                if (elect_one()) {
                    // in order behind the previous item's S-MMAs, ahead of this item's
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        tmem_cp_128x256b(tmem + L::kQ + kk * 8,
                                         umma_desc_sw128(q_base + (kk >> 2) * L::kBox +
                                                             (kk & 3) * 32, 16, 1024));
                    mma_commit(q_empty);
                }
                __syncwarp();
                for (int32_t j = 0; j < tl.n; ++j, ++tcount) {
                    const uint32_t b = tcount & 1, use = tcount >> 1;
                    if (lane == 0) TRACE3(2, j, 0);
                    // S[b] still holds tile t-2 (its S until loaded, or its P until its P.V ran)
                    mbar_wait(pv_done + b, (use & 1) ^ 1);
                    const uint32_t slot = cons % KS, ph = (cons / KS) & 1;
                    ++cons;
                    mbar_wait(k_full + slot, ph);
                    if (lane == 0) TRACE3(2, j, 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t kb = k_base + slot * L::kTile;
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            mma_ts(tmem + L::kS + b * BK, tmem + L::kQ + kk * 8,
                                   umma_desc_sw128(kb + (kk >> 2) * L::kBox + (kk & 3) * 32, 16,
                                                   1024),
                                   L::kIdescQK, kk > 0 ? 1u : 0u);
                        mma_commit(s_full + b);
                        mma_commit(k_empty + slot);
                    }
                    __syncwarp();
                }
            }
        } else if (warp == 3) {
            // ------------------------------------------------------- PV-issuer: O += P_j V_j
            uint32_t cons = 0, tcount = 0;
            const uint32_t v_base = smem_u32(smem + L::kVOff);
            for (int32_t local = 0;; ++local) {
                const int32_t item = next_item(local);
                if (item < 0) break;
                const Item it = decode_item(a, item);
                const TileList tl = tile_list(a, it);
                for (int32_t j = 0; j < tl.n; ++j, ++tcount) {
                    if (lane == 0) TRACE3(3, j, 0);
                    mbar_wait(p_full, tcount & 1);
                    if (lane == 0) TRACE3(3, j, 1);
                    if (j == 0) mbar_wait(o_empty, (local & 1) ^ 1);  // last item's epilogue
                    const uint32_t slot = cons % VS, ph = (cons / VS) & 1;
                    ++cons;
                    mbar_wait(v_full + slot, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t vb = v_base + slot * L::kTile;
                        const uint32_t pcol = kSeparateP ? L::kP : L::kS + (tcount & 1) * BK;
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            mma_ts(tmem + L::kO, tmem + pcol + kk * 8,
                                   umma_desc_sw128(vb + kk * 16 * 128, L::kBox, 1024),
                                   L::kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(p_empty);
                        if (!kSeparateP) mma_commit(pv_done + (tcount & 1));
                        mma_commit(v_empty + slot);
                    }
                    __syncwarp();
                }
                if (elect_one()) mma_commit(o_full);
                __syncwarp();
            }
        }
        __syncwarp();
    } else {
        if constexpr (CG == 2) set_maxnreg_inc224();
        // ------------------------------------------------------------------------ softmax
        const int half = (warp - 4) >> 2;   // column group: key columns half*HC .. +HC-1 of
                                            // every tile, O columns half*D/CG .. likewise
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const float sl2 = a.scale_log2;
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;
        const bool dbg = g_debug_mode != 0;
        uint32_t tcount = 0;
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local);
            if (item < 0) break;
            const Item it = decode_item(a, item);
            const TileList tl = tile_list(a, it);
            const bool last_ragged = tail_valid < BK && tl.n > 0 && tl.at(tl.n - 1) == g.NB - 1;
            float m_run = -INFINITY, l_run = 0.0f;
            for (int32_t j = 0; j < tl.n; ++j, ++tcount) {
                const uint32_t b = tcount & 1;
                const bool tr = quarter == 0 && lane == 0 && half < 2;
                if (tr) TRACE3(half, j, 0);
                mbar_wait(s_full + b, (tcount >> 1) & 1);
                if (tr) TRACE3(half, j, 1);
                tc_fence_after();
                uint32_t r[HC];
                tmem_load_half<HC>(lane_addr + L::kS + b * BK + half * HC, r);
                if constexpr (kSeparateP) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(pv_done + b);  // S[b] may be overwritten
                }
                if (tr) TRACE3(half, j, 3);
                if (last_ragged && j == tl.n - 1) {
#pragma unroll
                    for (int x = 0; x < HC; ++x)
                        if (half * HC + x >= tail_valid) r[x] = 0xff800000u;  // keys >= N (Q2)
                }
                uint32_t pk[HC / 2];
                float lsum;
                bool redo = false;
                // Max exchange between the halves without a full rendezvous: each half posts its
                // tile max and signals (bar.arrive on its own id), does the exponentials against
                // the running max, then waits for the other half's post (bar.sync on the other
                // id).  Having passed that wait also proves the other half has loaded its S
                // columns, so P may then overwrite S[b] (P aliases the first 64 columns).
                float* hm = hmax + (tcount & 1) * (CG * 128);
                hm[half * 128 + row] = dbg ? 0.0f : max_half<HC>(r);
                __syncwarp();
                if (lane == 0) mbar_arrive(hx_full + half * 2 + (tcount & 1));
                // wait for every other group's post of this tile; returns the row's tile max
                auto exchange = [&]() -> float {
#pragma unroll
                    for (int g2 = 0; g2 < CG; ++g2)
                        if (g2 != half)
                            mbar_wait(hx_full + g2 * 2 + (tcount & 1), (tcount >> 1) & 1);
                    float mx = hm[row];
#pragma unroll
                    for (int g2 = 1; g2 < CG; ++g2) mx = fmaxf(mx, hm[g2 * 128 + row]);
                    return mx;
                };
                if (dbg) {
#pragma unroll
                    for (int x = 0; x < HC / 2; ++x) pk[x] = 0u;
                    lsum = 0.0f;
                    exchange();
                } else if (j == 0) {
                    m_run = exchange() * sl2;
                    lsum = exp_half<HC, kEmu3>(r, sl2, m_run, pk);
                } else {
                    // exponentials against the running max first (the common case); redo only
                    // when the tile max jumps by more than 2^8
                    lsum = exp_half<HC, kEmu3>(r, sl2, m_run, pk);
                    if (tr) TRACE3(half, j, 4);
                    const float m_tile = exchange() * sl2;
                    if (tr) TRACE3(half, j, 5);
                    // warp-uniform decision: the O rescale uses warp-collective tcgen05.ld/st
                    const bool need = m_tile > m_run + kRescaleThreshold;
                    redo = __any_sync(0xffffffffu, need);
                    if (redo) {
                        const float m_new = need ? m_tile : m_run;
                        const float alpha = ex2_approx(m_run - m_new);  // 1 where !need
                        l_run *= alpha;
                        m_run = m_new;
                        lsum = exp_half<HC, kEmu3>(r, sl2, m_run, pk);
                        // every earlier P.V must be complete before O is rescaled
                        mbar_wait(p_empty, (tcount - 1) & 1);
                        tc_fence_after();
                        const uint64_t al2 = f2(alpha, alpha);
#pragma unroll
                        for (int cc = 0; cc < D / CG; cc += 32) {
                            uint32_t o[32];
                            const uint32_t oa = lane_addr + L::kO + half * (D / CG) + cc;
                            tmem_ld32(oa, o);
                            tmem_ld_wait(o);
#pragma unroll
                            for (int x = 0; x < 32; x += 2) {
                                const uint64_t v = fmul2(pk2(o[x], o[x + 1]), al2);
                                o[x] = (uint32_t)v;
                                o[x + 1] = (uint32_t)(v >> 32);
                            }
                            tmem_st32(oa, o);
                        }
                    }
                }
                l_run += lsum;
                // one P buffer: the previous tile's P.V must have read it (redo already waited)
                if (kSeparateP && tcount > 0 && !redo) mbar_wait(p_empty, (tcount - 1) & 1);
                if (tr) TRACE3(half, j, 6);
                tmem_store_p<HC>(lane_addr + (kSeparateP ? L::kP : L::kS + b * BK) +
                                     half * (HC / 2), pk);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full);
                if (tr) TRACE3(half, j, 2);
            }
            // ------------------------------------------------------------------ epilogue
            mbar_wait(o_full, local & 1);
            tc_fence_after();
            // the last tile's buffer: o_full implies both halves are past their reads of it,
            // and the next item's first tile uses the other one
            float* row_l = hmax + ((tcount - 1) & 1) * (CG * 128);
            row_l[half * 128 + row] = l_run;
            named_bar_sync(3, 128 * CG);
            float Lsum = row_l[row];
#pragma unroll
            for (int g2 = 1; g2 < CG; ++g2) Lsum += row_l[g2 * 128 + row];
            const float inv = Lsum > 0.0f ? 1.0f / Lsum : 0.0f;
            int64_t tok0 = -1;
            int32_t n_dst = 0, dst_stride_rows = 0;
            if (it.kind == 0) {
                const int64_t t = (int64_t)it.idx * BK + row;
                if (t < g.N) {
                    tok0 = t;
                    n_dst = 1;
                }
            } else {
                const int32_t kA = a.plan.anchor_k[it.cell];
                const int32_t per_frame = kA * g.W;
                const int32_t gi = it.idx * 128 + row;
                if (gi < g.F * per_frame) {
                    const int32_t f = gi / per_frame, m = (gi / g.W) % kA, jj = gi % g.W;
                    const int32_t am = anchor_row(g.H, kA, m);
                    const int32_t lo = m == 0 ? 0 : (anchor_row(g.H, kA, m - 1) + am) / 2 + 1;
                    const int32_t hi =
                        m == kA - 1 ? g.H : (am + anchor_row(g.H, kA, m + 1)) / 2 + 1;
                    tok0 = (int64_t)f * g.H * g.W + (int64_t)lo * g.W + jj;
                    n_dst = hi - lo;
                    dst_stride_rows = g.W;
                }
            }
            __nv_bfloat16* obase = a.o + (int64_t)it.b * a.o_sb + (int64_t)it.h * a.o_sh;
            const uint64_t inv2 = f2(inv, inv);
#pragma unroll
            for (int cc = 0; cc < D / CG; cc += 32) {
                const int col = half * (D / CG) + cc;
                uint32_t r0[32];
                tmem_ld32(lane_addr + L::kO + col, r0);
                tmem_ld_wait(r0);
                uint32_t packed[16];
#pragma unroll
                for (int x = 0; x < 32; x += 2) {
                    const uint64_t v = fmul2(pk2(r0[x], r0[x + 1]), inv2);
                    packed[x / 2] = pack_bf16(lo_f(v), hi_f(v));
                }
                for (int32_t dI = 0; dI < n_dst; ++dI) {
                    uint4* dst = reinterpret_cast<uint4*>(
                        obase + (tok0 + (int64_t)dI * dst_stride_rows) * a.o_sn + col);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2],
                                            packed[4 * v + 3]);
                }
            }
            if (half == 0 && a.lse_out != nullptr) {
                const float lse = (m_run + __log2f(Lsum)) * 0.69314718055994531f;
                float* lb = a.lse_out + ((int64_t)it.b * a.n_heads + it.h) * (int64_t)g.N;
                for (int32_t dI = 0; dI < n_dst; ++dI)
                    lb[tok0 + (int64_t)dI * dst_stride_rows] = lse;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    // self-resetting dynamic scheduler: the last CTA to finish zeroes the counters
    if (threadIdx.x == 0 && a.sched != nullptr) {
        __threadfence();
        if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
            atomicExch(a.sched, 0u);
            atomicExch(a.sched + 1, 0u);
        }
    }
}

}  // namespace

cudaError_t set_attn3_trace(void* buf, int mode) {
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    cudaError_t e = cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(g_debug_mode, &mode, sizeof(mode));
}

namespace {
template <int CG>
cudaError_t launch_cg(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                      const CUtensorMap& tv, int grid, cudaStream_t s) {
    auto kern = sparse_attn_q_tmem_kernel<CG>;
    const int smem = Smem3<CG>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, Smem3<CG>::kThreads, smem, s>>>(a, tq, tk, tv);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_attn_q_tmem(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                               const CUtensorMap& tv, int grid, cudaStream_t s) {
    if (a.g.B != 128) return cudaErrorInvalidValue;
    const char* cg = std::getenv("CSA_ATTN_CG");  // A/B: softmax column groups (2 or 4)
    if (cg && std::atoi(cg) == 4) return launch_cg<4>(a, tq, tk, tv, grid, s);
    return launch_cg<2>(a, tq, tk, tv, grid, s);
}

}  // namespace csa
