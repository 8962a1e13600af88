// attn4.cu -- a7 + a8 for block 128, head_dim 128 with a fixed per-row reference max.
//
// Same mathematics as attn.cu / attn3.cu (readings Q1, Q2, Q9,
// Q10).  Softmax is shift-invariant: o_i = sum_j 2^(s_ij - m) v_j / sum_j 2^(s_ij - m) for any m.
// Here m = m_ref is fixed per row for the whole item: the max of the row's FIRST kept tile.  Later
// tiles then need no max, no exchange and no rescale of O or l; the two softmax groups take
// alternate tiles (two tiles in flight) and accumulate into ONE O (every P.V relative to the same
// m_ref), which leaves TMEM room for Q:
//   TMEM (512 columns): S0 [0,128) S1 [128,256) | O [256,384) | Q [384,448)
// P (bf16) overwrites the first 64 columns of its S buffer; S-MMAs are TS (Q from TMEM).
// Overflow guard: scores beyond m_ref + 56 (log2) would make P > 2^56; a tile whose row sum
// exceeds 2^56 (or is not finite) flags the item, which is appended to a fallback list that the
// API recomputes with the running-max kernel (attn3.cu) on the same stream.  Real attention rows
// never come near it; the test suite forces it.
// Roles: warp 0 scheduler + producer (Q by TMA / anchor gather, then K0, K1, V0, K2, V1, ...
// through one ring), warp 1 MMA issuer (Q -> TMEM copy, S_j into S[j&1], O += P_{j-1} V_{j-1}),
// warp 2 TMEM allocator, warps 4-7 / 8-11 softmax groups on even / odd tiles.
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kItemSlots4 = 4;
// CH4: column split of each softmax group: a group is 4 * CH4 warps, warp (quarter, ch) taking
// rows 32 * quarter ... and key columns ch * 128 / CH4 ... of the group's tiles.
#ifndef CSA_ATTN4_CH
#define CSA_ATTN4_CH 2
#endif
#ifndef CSA_ATTN4_NG
#define CSA_ATTN4_NG 2
#endif
constexpr int kCH4 = CSA_ATTN4_CH;
// NG: softmax groups = tiles in softmax at once (2: groups on alternate tiles, S buffer = group;
// 1: one group of 4 CH warps takes every tile, the two S buffers alternate under it)
constexpr int kNG4 = CSA_ATTN4_NG;
// kSplit4: the S-MMA of a tile is issued as two N = 64 halves (one per column part) with their
// own completion barriers, and the P.V as two K = 64 halves waiting for their own part's P: a
// column part's softmax starts when its half of S is done, and its half of P.V when its own P
// is stored (the chain QK -> softmax -> PV no longer waits for the whole tile).  CH 2 only.
// Measured slower (same box, Wan 720p: 1049 vs 1150 TF/s): off by default.
#ifndef CSA_ATTN4_SPLIT
#define CSA_ATTN4_SPLIT 0
#endif
constexpr bool kSplit4 = CSA_ATTN4_SPLIT != 0;
// CSA_ATTN4_PHASED: the softmax computes all exp2 arguments, then issues the exponentials back
// to back, then sums / packs (A/B against the interleaved loop).
#ifndef CSA_ATTN4_PHASED
#define CSA_ATTN4_PHASED 0
#endif
constexpr float kGuard = 72057594037927936.0f;  // 2^56: a tile row sum above it flags the item
static __device__ unsigned long long* g_trace4;
static __device__ int g_debug_mode4;
#ifdef CSA_ENABLE_TRACE  // trace builds only (see attn_common.cuh): CTA 0's first 1024 tiles
#define TRACE4(slot, k, e)                                                                   \
    do {                                                                                     \
        if (g_trace4 != nullptr && blockIdx.x == 0 && (k) < 1024)                            \
            g_trace4[((slot) * 1024 + (k)) * 8 + (e)] = clock64();                           \
    } while (0)
#define DEBUG4 (g_debug_mode4)
#else
#define TRACE4(slot, k, e) \
    do {                   \
    } while (0)
#define DEBUG4 0
#endif
constexpr int kEmu4 = 1;  // element pairs p with (p & 7) >= 8 - kEmu4 -> polynomial exp2

template <int CH, int NG>
struct Smem4 {
    static constexpr int kThreads = 128 + 128 * NG * CH;
    static constexpr int kBox = 128 * 128;      // [128 rows][64 cols] bf16, SWIZZLE_128B
    static constexpr int kTile = 2 * kBox;      // 128 x 128 bf16
    static constexpr int kQOff = 0;             // single Q buffer (freed once copied to TMEM)
    static constexpr int kKVOff = kTile;
    static constexpr int kSlots = CH == 1 ? 6 : 5;  // K/V ring, consumption order
    static constexpr int kBarOff = kKVOff + kSlots * kTile;
    // q_full q_empty | kv_full[S] kv_empty[S] | s_full[2][2] p_full[2][2] | o_full o_empty |
    // mref_full | item_full[4] item_empty[4]   ([grp][half]; only [grp][0] without kSplit4)
    static constexpr int kNumBars = 2 + 2 * kSlots + 8 + 2 + 1 + 2 * kItemSlots4;
    // m_ref[128] | l[2 * CH][128] | tile-0 max of each column part [CH][128]
    static constexpr int kRowOff = kBarOff + kNumBars * 8;
    static constexpr int kItemOff = kRowOff + (1 + NG * CH + CH) * 128 * 4;
    static constexpr int kFlagOff = kItemOff + kItemSlots4 * 4;
    static constexpr int kTmemPtrOff = kFlagOff + 16;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(kBytes <= 232448, "smem");
    static constexpr uint32_t kS = 0, kO = 256, kQ = 384;
    static constexpr uint32_t kIdescQK = umma_idesc_bf16(128, 128, 0, 0);
    static constexpr uint32_t kIdescQK64 = umma_idesc_bf16(128, 64, 0, 0);
    static constexpr uint32_t kIdescPV = umma_idesc_bf16(128, 128, 0, 1);
};

template <int CH, int NG>
__global__ void __launch_bounds__(Smem4<CH, NG>::kThreads, 1)
    sparse_attn_fixed_ref_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                                 const __grid_constant__ CUtensorMap tk,
                                 const __grid_constant__ CUtensorMap tv, const Fallback fb) {
    using L = Smem4<CH, NG>;
    constexpr int BK = 128, D = 128, S = L::kSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* kv_full = bars + 2;
    uint64_t* kv_empty = kv_full + S;
    constexpr bool kSplit = kSplit4 && CH == 2 && NG == 2;
    uint64_t* s_full = kv_empty + S;  // [grp][half]
    uint64_t* p_full = s_full + 4;    // [grp][half]
    uint64_t* o_full = p_full + 4;
    uint64_t* o_empty = o_full + 1;
    uint64_t* mref_full = o_empty + 1;
    uint64_t* item_full = mref_full + 1;
    uint64_t* item_empty = item_full + kItemSlots4;
    float* mref_s = reinterpret_cast<float*>(smem + L::kRowOff);  // [128] (log2 domain)
    float* row_l = mref_s + 128;                                   // [NG * CH][128]
    float* mx_s = row_l + NG * CH * 128;                           // [CH][128]
    volatile int32_t* item_slot = reinterpret_cast<int32_t*>(smem + L::kItemOff);
    volatile int32_t* flag_s = reinterpret_cast<int32_t*>(smem + L::kFlagOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < S; ++i) {
            mbar_init(kv_full + i, 1);
            mbar_init(kv_empty + i, 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, kSplit ? 4 : 4 * CH);
        }
        mbar_init(o_full, 1);
        mbar_init(o_empty, 4 * NG * CH);
        mbar_init(mref_full, 4 * CH);
        for (int i = 0; i < kItemSlots4; ++i) {
            mbar_init(item_full + i, 1);
            mbar_init(item_empty + i, 1 + 4 * NG * CH);  // MMA warp + the softmax warps
        }
        *flag_s = 0;
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
        const int s = local % kItemSlots4;
        mbar_wait(item_full + s, (local / kItemSlots4) & 1);
        const int32_t idx = item_slot[s];
        __syncwarp();
        if (lane == 0) mbar_arrive(item_empty + s);
        return idx;
    };

    if (warp < 4) {
        // registers: launch 65536 / kThreads each; what the producer warps give back must cover
        // what the softmax warps take (CH 2: 640 x 96 -> 4 warps at 56, 16 warps at 104)
        set_maxnreg_dec56();
        if (warp == 0) {
            // ------------------------------------------------------------ scheduler + producer
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_kv = policy_evict_last();
            uint32_t ld = 0;
            for (int32_t local = 0;; ++local) {
                const int s = local % kItemSlots4;
                mbar_wait(item_empty + s, ((local / kItemSlots4) & 1) ^ 1);
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
                        const uint32_t slot = ld % S, ph = (ld / S) & 1;
                        ++ld;
                        const int32_t c = tl.at(j);
                        mbar_wait(kv_empty + slot, ph ^ 1);
                        if (elect_one()) {
                            uint8_t* dst = smem + L::kKVOff + slot * L::kTile;
                            mbar_arrive_expect_tx(kv_full + slot, L::kTile);
                            tma_tile<D>(dst, L::kBox, kv == 0 ? &tk : &tv, kv_full + slot, it.h,
                                        c * BK, it.b, pol_kv);
                        }
                        __syncwarp();
                    }
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------------------------ MMA issuer
            uint32_t cons = 0, pcount[2] = {0, 0}, qk_tiles = 0, pv_tiles = 0;
            const uint32_t q_base = smem_u32(smem + L::kQOff);
            const uint32_t kv_base = smem_u32(smem + L::kKVOff);
            for (int32_t local = 0;; ++local) {
                const int32_t item = next_item(local);
                if (item < 0) break;
                const Item it = decode_item(a, item);
                const TileList tl = tile_list(a, it);
                mbar_wait(q_full, local & 1);
                tc_fence_after();
                if (elect_one()) {  // Q -> TMEM, in order with this thread's MMAs
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        tmem_cp_128x256b(tmem + L::kQ + kk * 8,
                                         umma_desc_sw128(q_base + (kk >> 2) * L::kBox +
                                                             (kk & 3) * 32, 16, 1024));
                    mma_commit(q_empty);
                    if (tl.n == 0) mma_commit(o_full);  // corrupt plan (empty row): no tiles
                }
                __syncwarp();
                if (tl.n == 0) continue;
                auto do_pv = [&](int32_t t) {
                    const int grp = t & 1;
                    TRACE4(3, pv_tiles, 0);
                    if constexpr (kSplit) {
                        const uint32_t slot = cons % S, ph = (cons / S) & 1;
                        ++cons;
                        const uint32_t vb = kv_base + slot * L::kTile;
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            mbar_wait(p_full + grp * 2 + half, pcount[grp] & 1);
                            if (half == 0) {
                                if (t == 0) mbar_wait(o_empty, (local & 1) ^ 1);
                                mbar_wait(kv_full + slot, ph);
                            }
                            tc_fence_after();
                            if (elect_one()) {
#pragma unroll
                                for (int k4 = 0; k4 < 4; ++k4) {
                                    const int kk = half * 4 + k4;  // P of part `half`
                                    mma_ts(tmem + L::kO, tmem + L::kS + grp * BK + half * 64 + k4 * 8,
                                           umma_desc_sw128(vb + kk * 16 * 128, L::kBox, 1024),
                                           L::kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
                                }
                                if (half == 1) mma_commit(kv_empty + slot);
                            }
                            __syncwarp();
                        }
                        ++pcount[grp];
                        TRACE4(3, pv_tiles, 2);
                        ++pv_tiles;
                        return;
                    }
                    mbar_wait(p_full + grp * 2, pcount[grp] & 1);
                    ++pcount[grp];
                    TRACE4(3, pv_tiles, 1);
                    if (t == 0) mbar_wait(o_empty, (local & 1) ^ 1);  // last item's epilogue
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    mbar_wait(kv_full + slot, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t vb = kv_base + slot * L::kTile;
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            // P of column part q sits over the first half of S's part q
                            mma_ts(tmem + L::kO,
                                   tmem + L::kS + grp * BK + (kk * 16 / (BK / CH)) * (BK / CH) +
                                       (kk * 16 % (BK / CH)) / 2,
                                   umma_desc_sw128(vb + kk * 16 * 128, L::kBox, 1024),
                                   L::kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(kv_empty + slot);
                    }
                    __syncwarp();
                    TRACE4(3, pv_tiles, 2);
                    ++pv_tiles;
                };
                for (int32_t j = 0; j < tl.n; ++j) {
                    const int grp = j & 1;
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    TRACE4(2, qk_tiles, 0);
                    mbar_wait(kv_full + slot, ph);
                    TRACE4(2, qk_tiles, 1);
                    ++qk_tiles;
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t kb = kv_base + slot * L::kTile;
                        if constexpr (kSplit) {
                            // two N = 64 halves: keys [64 half, 64 half + 64) of the tile are
                            // rows 64 half.. of the K-major tile (8 KB in, atom-aligned)
#pragma unroll
                            for (int half = 0; half < 2; ++half) {
#pragma unroll
                                for (int kk = 0; kk < D / 16; ++kk)
                                    mma_ts(tmem + L::kS + grp * BK + half * 64,
                                           tmem + L::kQ + kk * 8,
                                           umma_desc_sw128(kb + (kk >> 2) * L::kBox +
                                                               (kk & 3) * 32 + half * 64 * 128,
                                                           16, 1024),
                                           L::kIdescQK64, kk > 0 ? 1u : 0u);
                                mma_commit(s_full + grp * 2 + half);
                            }
                        } else {
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk)
                                mma_ts(tmem + L::kS + grp * BK, tmem + L::kQ + kk * 8,
                                       umma_desc_sw128(kb + (kk >> 2) * L::kBox + (kk & 3) * 32,
                                                       16, 1024),
                                       L::kIdescQK, kk > 0 ? 1u : 0u);
                            mma_commit(s_full + grp * 2);
                        }
                        mma_commit(kv_empty + slot);
                    }
                    __syncwarp();
                    if (j >= 1) do_pv(j - 1);
                }
                do_pv(tl.n - 1);
                if (elect_one()) mma_commit(o_full);
                __syncwarp();
            }
        }
        __syncwarp();
    } else {
        if constexpr (CH == 1) {
            set_maxnreg_inc224();
        } else {
            asm volatile("setmaxnreg.inc.sync.aligned.u32 104;" ::: "memory");
        }
        // ------------------------------------------------------------------ softmax groups
        constexpr int NC = BK / CH;  // key columns per thread
        const int grp = (int)(warp - 4) / (4 * CH);
        const int ch = (int)((warp - 4) >> 2) % CH;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        uint32_t sc1 = 0;  // uses of S buffer 1 (NG 1; scount counts buffer 0 / the own one)
        const float sl2 = a.scale_log2;
        const uint64_t sl2x2 = f2(sl2, sl2);
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;
        uint32_t scount = 0, tbase = 0;
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local);
            if (item < 0) break;
            const Item it = decode_item(a, item);
            const TileList tl = tile_list(a, it);
            const bool last_ragged = tail_valid < BK && tl.n > 0 && tl.at(tl.n - 1) == g.NB - 1;
            float m_ref = 0.0f, l_run = 0.0f;
            bool have_ref = false, bad = false;
            auto get_ref = [&]() {  // group 1: the reference group 0 posted for this item
                mbar_wait(mref_full, local & 1);
                m_ref = mref_s[row];
                have_ref = true;
            };
            for (int32_t j = grp; j < tl.n; j += NG) {
                const uint32_t tk = tbase + (uint32_t)j;
                (void)tk;
                const uint32_t sb = (uint32_t)j & 1u;  // S buffer of tile j (= grp for NG 2)
                const uint32_t s_col = L::kS + sb * BK + ch * NC;
                const uint32_t p_col = s_col;  // P over the first half of this part's S columns
                if (quarter == 0 && ch == 0 && lane == 0) TRACE4(grp, tk, 0);
                uint32_t sph;
                if (NG == 1 && sb) {
                    sph = sc1++;
                } else {
                    sph = scount++;
                }
                mbar_wait(s_full + sb * 2 + (kSplit ? ch : 0), sph & 1);
                if (quarter == 0 && ch == 0 && lane == 0) TRACE4(grp, tk, 1);
                tc_fence_after();
                uint32_t r[NC / 32][32];
#pragma unroll
                for (int c = 0; c < NC / 32; ++c) tmem_ld32(lane_addr + s_col + c * 32, r[c]);
#pragma unroll
                for (int c = 0; c < NC / 32; ++c) tmem_ld_wait(r[c]);
                if (quarter == 0 && ch == 0 && lane == 0) TRACE4(grp, tk, 2);
                if (last_ragged && j == tl.n - 1) {
#pragma unroll
                    for (int c = 0; c < NC / 32; ++c)
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if (ch * NC + c * 32 + x >= tail_valid)
                                r[c][x] = 0xff800000u;  // keys >= N
                }
                if (j == 0) {
                    // the row's reference: the max of its first kept tile (8 FMNMX3 chains)
                    constexpr int kPer = NC / 8;
                    float mc[8];
#pragma unroll
                    for (int q8 = 0; q8 < 8; ++q8) {
#define SV(e) __uint_as_float(r[(e) >> 5][(e) & 31])
                        mc[q8] = SV(q8);
#pragma unroll
                        for (int t = 1; t + 1 < kPer; t += 2)
                            mc[q8] = fmax3(mc[q8], SV(q8 + 8 * t), SV(q8 + 8 * (t + 1)));
                        mc[q8] = fmaxf(mc[q8], SV(q8 + 8 * (kPer - 1)));
#undef SV
                    }
                    m_ref = fmaxf(fmax3(mc[0], mc[1], mc[2]),
                                  fmaxf(fmax3(mc[3], mc[4], mc[5]), fmaxf(mc[6], mc[7]))) * sl2;
                    if constexpr (CH > 1) {  // the row's max over the column parts (group 0)
                        mx_s[ch * 128 + row] = m_ref;
                        named_bar_sync(2, 128 * CH);
#pragma unroll
                        for (int o = 0; o < CH; ++o) m_ref = fmaxf(m_ref, mx_s[o * 128 + row]);
                    }
                    if (ch == 0) mref_s[row] = m_ref;
                    have_ref = true;
                    if constexpr (NG > 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(mref_full);
                    }
                } else if (!have_ref) {
                    get_ref();
                }
                const uint64_t negm = f2(-m_ref, -m_ref);
                uint64_t acc[4] = {0, 0, 0, 0};
#if CSA_ATTN4_PHASED
                // phased: all arguments first, then the exponentials back to back (one MUFU
                // stream per warp), then sums and packing
                uint64_t tt[NC / 2];
#pragma unroll
                for (int c = 0; c < NC / 32; ++c)
#pragma unroll
                    for (int x = 0; x < 32; x += 2)
                        tt[c * 16 + x / 2] = ffma2(pk2(r[c][x], r[c][x + 1]), sl2x2, negm);
#pragma unroll
                for (int i = 0; i < NC / 2; ++i) {
                    if ((i & 7) >= 8 - kEmu4) {
                        tt[i] = exp2_poly2(tt[i]);
                    } else {
                        float e0, e1;
                        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(lo_f(tt[i])));
                        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(hi_f(tt[i])));
                        tt[i] = f2(e0, e1);
                    }
                }
#pragma unroll
                for (int c = 0; c < NC / 32; ++c) {
                    uint32_t pk[16];
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        const uint64_t p = tt[c * 16 + x];
                        acc[x & 3] = fadd2(acc[x & 3], p);
                        pk[x] = pack_bf16(lo_f(p), hi_f(p));
                    }
                    tmem_st16(lane_addr + p_col + c * 16, pk);
                }
#else
#pragma unroll
                for (int c = 0; c < NC / 32; ++c) {  // P overwrites the first BK/2 columns of S
                    uint32_t pk[16];
#pragma unroll
                    for (int x = 0; x < 32; x += 2) {
                        const uint64_t t = ffma2(pk2(r[c][x], r[c][x + 1]), sl2x2, negm);
                        uint64_t p;
                        if (DEBUG4 == 1) {
                            p = t;
                        } else if (((c * 16 + x / 2) & 7) >= 8 - kEmu4) {
                            p = exp2_poly2(t);
                        } else {
                            p = f2(ex2_approx(lo_f(t)), ex2_approx(hi_f(t)));
                        }
                        acc[(x / 2) & 3] = fadd2(acc[(x / 2) & 3], p);
                        pk[x / 2] = pack_bf16(lo_f(p), hi_f(p));
                    }
                    if (DEBUG4 == 2) {  // debug: no P store (timeline of the rest)
                        uint32_t sink = 0;
#pragma unroll
                        for (int x = 0; x < 16; ++x) sink ^= pk[x];
                        if (sink == 0x12345678u) mref_s[0] = 0.0f;
                        continue;
                    }
                    tmem_st16(lane_addr + p_col + c * 16, pk);
                }
#endif
                const uint64_t acc2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
                const float lsum = lo_f(acc2) + hi_f(acc2);
                bad |= !(lsum <= kGuard);  // also catches inf / NaN
                l_run += lsum;
                if (quarter == 0 && ch == 0 && lane == 0) TRACE4(grp, tk, 3);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + sb * 2 + (kSplit ? ch : 0));
                if (quarter == 0 && ch == 0 && lane == 0) TRACE4(grp, tk, 4);
            }
            tbase += (uint32_t)tl.n;
            if (NG == 1 && !have_ref) {  // corrupt plan (empty row): no reference needed
                m_ref = 0.0f;
                have_ref = true;
            }
            if (NG > 1 && grp == 0 && tl.n == 0) {  // corrupt plan: keep mref_full's phase
                if (ch == 0) mref_s[row] = 0.0f;
                __syncwarp();
                if (lane == 0) mbar_arrive(mref_full);
            }
            if (!have_ref) get_ref();  // group 1 without tiles (n <= 1)
            // -------------------------------------------------------------- epilogue
            if (__any_sync(0xffffffffu, bad) && lane == 0) *flag_s = 1;
            mbar_wait(o_full, local & 1);
            tc_fence_after();
            row_l[(grp * CH + ch) * 128 + row] = l_run;
            named_bar_sync(1, 128 * NG * CH);
            float Lsum = 0.0f;
#pragma unroll
            for (int o = 0; o < NG * CH; ++o) Lsum += row_l[o * 128 + row];
            const float inv = Lsum > 0.0f ? 1.0f / Lsum : 0.0f;
            const bool flagged = *flag_s != 0;
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
            for (int cc = 0; cc < D / (NG * CH); cc += 32) {
                const int col = (grp * CH + ch) * (D / (NG * CH)) + cc;
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
            if (grp == 0 && ch == 0 && a.lse_out != nullptr) {
                const float lse = (m_ref + __log2f(Lsum)) * 0.69314718055994531f;
                float* lb = a.lse_out + ((int64_t)it.b * a.n_heads + it.h) * (int64_t)g.N;
                for (int32_t dI = 0; dI < n_dst; ++dI)
                    lb[tok0 + (int64_t)dI * dst_stride_rows] = lse;
            }
            tc_fence_before();
            named_bar_sync(1, 128 * NG * CH);  // every thread has read flag_s / row_l
            if (threadIdx.x == 128) {
                if (flagged) {  // recomputed by the running-max kernel after this launch
                    // one entry per work-list item (the fallback launch redoes every batch of it)
                    const uint32_t w = (uint32_t)(item / a.batch), bit = 1u << (w & 31u);
                    if ((atomicOr(fb.flags + (w >> 5), bit) & bit) == 0u)
                        fb.list[atomicAdd(fb.count, 1u)] = a.work_list[w];
                }
                *flag_s = 0;
            }
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
    if (threadIdx.x == 0 && a.sched != nullptr) {
        __threadfence();
        if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
            atomicExch(a.sched, 0u);
            atomicExch(a.sched + 1, 0u);
        }
    }
}

}  // namespace

cudaError_t set_attn4_trace(void* buf, int mode) {
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    cudaError_t e = cudaMemcpyToSymbol(g_trace4, &p, sizeof(p));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(g_debug_mode4, &mode, sizeof(mode));
}

cudaError_t launch_attn_fixed_ref(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                                  const CUtensorMap& tv, int grid, const Fallback& fb,
                                  cudaStream_t s) {
    if (a.g.B != 128) return cudaErrorInvalidValue;
    auto kern = sparse_attn_fixed_ref_kernel<kCH4, kNG4>;
    const int smem = Smem4<kCH4, kNG4>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, Smem4<kCH4, kNG4>::kThreads, smem, s>>>(a, tq, tk, tv, fb);
    return cudaGetLastError();
}

}  // namespace csa
