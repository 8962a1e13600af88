// attn_rect.cu -- a7 + a8 with non-square blocks B_q x B_kv = 128 x B_kv (f3).
//
// PAPER.md P:1294-1328 (Table tab:block_size_ablation): FlashAttention tiles the problem into
// B_q x B_kv blocks (128 x 176 natively for d = 128 on H100) and the calibrated mask is built on
// that grid; the method is otherwise unchanged.  What is computed is exactly attn.cu's (P:647-656,
// P:616-622; readings Q1, Q2, Q9, Q10): for query block r (B_q = 128 rows) the keys are the
// union of the kept key blocks J_c = [c B_kv, (c+1) B_kv) clipped to N; REPETITIVE items attend
// to every key block.
//
// Design: the fixed-reference-max pipeline of attn4.cu (softmax is shift-invariant, so each row's
// shift is the max of its first kept tile, reading Q29) with the key-tile width B_kv a template
// parameter:
//   TMEM (512 columns): S0 [0,SB) S1 [SB,2SB) | O [2SB,2SB+128) | Q [2SB+128, +64) when it fits
//   (SB = B_kv rounded up to 32; B_kv <= 160 keeps Q in TMEM and runs TS S-MMAs, B_kv 176/192
//   read Q from shared memory (SS)).
//   Warp 0 scheduler + producer (Q tile by TMA or anchor gather; K0, K1, V0, K2, V1, ... through
//   one ring of [B_kv][128] bf16 slots), warp 1 MMA issuer (S_j = Q K_j^T, N = B_kv, into
//   S[j&1]; O += P_{j-1} V_{j-1}, K = B_kv), warp 2 TMEM allocator, warps 4-7 / 8-11 softmax
//   groups on even / odd tiles, one query row per thread, the row's B_kv scores processed in
//   parts of <= 64 columns (load, exp2, P store over the first half of the part's S columns).
// Overflow guard and its fallback (modes): mode 0 flags an item whose tile row sum exceeds 2^56
// (a later score > m_ref + 56 in log2) and appends it to the fallback list; mode 1 runs the list
// and computes each row's exact max over its kept keys (no output; the max is parked in the
// first 4 bytes of the row's first output row); mode 2 recomputes the list against that max
// (P <= 1, no overflow possible) and writes the outputs.  Real attention never trips the guard.
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kItemSlotsR = 4;
constexpr float kGuardR = 72057594037927936.0f;  // 2^56
// element pairs p with (p & 7) >= 8 - kEmu -> polynomial exp2 (FMA pipe) instead of MUFU
#ifndef CSA_RECT_EMU64
#define CSA_RECT_EMU64 1
#endif
template <int D>
constexpr int kEmuR = D == 64 ? CSA_RECT_EMU64 : 1;

template <int BKV, int D = 128>
struct SmemR {
    static constexpr int kThreads = 384;
    static constexpr int kBoxes = D / 64;          // 128-byte-wide boxes per row
    static constexpr int kQBox = 128 * 128;        // [128 rows][64] bf16, SWIZZLE_128B
    static constexpr int kQTile = kBoxes * kQBox;  // 128 x D
    static constexpr int kKVBox = BKV * 128;       // [B_kv rows][64]
    static constexpr int kTile = kBoxes * kKVBox;  // B_kv x D
    static constexpr uint32_t kSB = (BKV + 31) / 32 * 32;
    static constexpr bool kQT = 2 * kSB + D + D / 2 <= 512;
    static constexpr uint32_t kS = 0, kO = 2 * kSB, kQ = 2 * kSB + D;
    static constexpr int kQOff = 0;
    static constexpr int kKVOff = kQTile;
    static constexpr int kSlotsFit = (232448 - kQTile - 2048) / kTile;
    static constexpr int kSlots = kSlotsFit > 8 ? 8 : kSlotsFit;
    static constexpr int kBarOff = kKVOff + kSlots * kTile;
    // q_full q_empty | kv_full[S] kv_empty[S] | s_full[2] p_full[2] | o_full o_empty | mref_full
    // | item_full[4] item_empty[4]
    static constexpr int kNumBars = 2 + 2 * kSlots + 4 + 2 + 1 + 2 * kItemSlotsR;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;  // m_ref[128] | per-group [2][128]
    static constexpr int kItemOff = kRowOff + 3 * 128 * 4;
    static constexpr int kFlagOff = kItemOff + kItemSlotsR * 4;
    static constexpr int kTmemPtrOff = kFlagOff + 16;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(kBytes <= 232448, "smem");
    static_assert(kSlots >= 3, "K/V ring");
    static_assert(BKV % 16 == 0 && BKV >= 64 && BKV <= 192, "B_kv");
    static_assert(2 * kSB + D <= 512 && (!kQT || kQ + D / 2 <= 512), "TMEM");
    static_assert(D == 64 || D == 128, "head_dim");
    static constexpr uint32_t kIdescQK = umma_idesc_bf16(128, BKV, 0, 0);
    static constexpr uint32_t kIdescPV = umma_idesc_bf16(128, D, 0, 1);
};

// Load W (multiple of 16, <= 64) consecutive TMEM columns of this thread's lane into r[0, W).
template <int W>
__device__ __forceinline__ void ld_part(uint32_t addr, uint32_t (&r)[64]) {
    static_assert(W % 16 == 0 && W >= 16 && W <= 64, "part");
    if constexpr (W >= 32) tmem_ld32(addr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
    if constexpr (W == 64) tmem_ld32(addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
    if constexpr (W == 48) tmem_ld16(addr + 32, *reinterpret_cast<uint32_t(*)[16]>(&r[32]));
    if constexpr (W == 16) tmem_ld16(addr, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
    tmem_ld_wait();
#pragma unroll
    for (int x = 0; x < W; ++x) asm volatile("" : "+r"(r[x]));  // no use above the wait
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
        : "memory");
}

// Store W/2 packed bf16 pairs (W multiple of 16) at addr.
template <int W>
__device__ __forceinline__ void st_part(uint32_t addr, const uint32_t (&pk)[32]) {
    if constexpr (W == 64) {
        tmem_st32(addr, pk);
    } else {
        if constexpr (W >= 32) tmem_st16(addr, *reinterpret_cast<const uint32_t(*)[16]>(&pk[0]));
        if constexpr (W == 48 || W == 16) tmem_st8(addr + (W == 48 ? 16 : 0), &pk[W == 48 ? 16 : 0]);
    }
}

template <int W>
__device__ __forceinline__ void mask_part(uint32_t (&r)[64], int32_t col0, int32_t valid) {
#pragma unroll
    for (int x = 0; x < W; ++x)
        if (col0 + x >= valid) r[x] = 0xff800000u;  // keys >= N do not exist (Q2)
}

template <int W>
__device__ __forceinline__ float max_part(const uint32_t (&r)[64]) {
    float m[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = __uint_as_float(r[i]);
#pragma unroll
    for (int x = 4; x < W; x += 8)
#pragma unroll
        for (int i = 0; i < 4; ++i)
            m[i] = x + 4 + i < W ? fmax3(m[i], __uint_as_float(r[x + i]),
                                         __uint_as_float(r[x + 4 + i]))
                                 : fmaxf(m[i], __uint_as_float(r[x + i]));
    return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}

// exp2(s * sl2 - m) of W scores -> packed bf16 pk[W/2]; returns their fp32 sum.
template <int W, int kEmu>
__device__ __forceinline__ float exp_part(const uint32_t (&r)[64], uint64_t sl2x2, uint64_t negm,
                                          uint32_t (&pk)[32]) {
    uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int x = 0; x < W; x += 2) {
        const uint64_t t = ffma2(pk2(r[x], r[x + 1]), sl2x2, negm);
        uint64_t p;
        if (((x / 2) & 7) >= 8 - kEmu) {
            p = exp2_poly2(t);
        } else {
            p = f2(ex2_approx(lo_f(t)), ex2_approx(hi_f(t)));
        }
        acc[(x / 2) & 3] = fadd2(acc[(x / 2) & 3], p);
        pk[x / 2] = pack_bf16(lo_f(p), hi_f(p));
    }
    const uint64_t s2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    return lo_f(s2) + hi_f(s2);
}

// Part p of a B_kv-wide row: columns [64 p, 64 p + width).
template <int BKV, int P>
struct Part {
    static constexpr int kCol = 64 * P;
    static constexpr int kW = BKV - kCol < 64 ? BKV - kCol : 64;
};

template <int BKV, int D>
__global__ void __launch_bounds__(SmemR<BKV, D>::kThreads, 1)
    sparse_attn_rect_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                            const __grid_constant__ CUtensorMap tk,
                            const __grid_constant__ CUtensorMap tv, const Fallback fb,
                            const int mode) {
    using L = SmemR<BKV, D>;
    constexpr int S = L::kSlots;
    constexpr int kParts = (BKV + 63) / 64;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* kv_full = bars + 2;
    uint64_t* kv_empty = kv_full + S;
    uint64_t* s_full = kv_empty + S;  // [grp]
    uint64_t* p_full = s_full + 2;    // [grp]
    uint64_t* o_full = p_full + 2;
    uint64_t* o_empty = o_full + 1;
    uint64_t* mref_full = o_empty + 1;
    uint64_t* item_full = mref_full + 1;
    uint64_t* item_empty = item_full + kItemSlotsR;
    float* mref_s = reinterpret_cast<float*>(smem + L::kRowOff);  // [128] (log2 domain)
    float* row_x = mref_s + 128;                                   // [2][128]
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
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, 4);
        }
        mbar_init(o_full, 1);
        mbar_init(o_empty, 8);
        mbar_init(mref_full, 4);
        for (int i = 0; i < kItemSlotsR; ++i) {
            mbar_init(item_full + i, 1);
            mbar_init(item_empty + i, 9);  // MMA warp + 8 softmax warps
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
        const int s = local % kItemSlotsR;
        mbar_wait(item_full + s, (local / kItemSlotsR) & 1);
        const int32_t idx = item_slot[s];
        __syncwarp();
        if (lane == 0) mbar_arrive(item_empty + s);
        return idx;
    };

    if (warp < 4) {
        set_maxnreg_dec56();
        if (warp == 0) {
            // ------------------------------------------------------------ scheduler + producer
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_kv = policy_evict_last();
            uint32_t ld = 0;
            for (int32_t local = 0;; ++local) {
                const int s = local % kItemSlotsR;
                mbar_wait(item_empty + s, ((local / kItemSlotsR) & 1) ^ 1);
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
                        mbar_arrive_expect_tx(q_full, L::kQTile);
                        tma_tile<D>(qdst, L::kQBox, &tq, q_full, it.h, it.idx * 128, it.b, pol_q);
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
                        *reinterpret_cast<uint4*>(qdst + (ch >> 3) * L::kQBox +
                                                  sw128_offset(row, ch & 7)) = val;
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(q_full);
                }
                TileCursor kcur(tl), vcur(tl);
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
                        const int32_t c = kv == 0 ? kcur.next() : vcur.next();
                        (void)j;
                        mbar_wait(kv_empty + slot, ph ^ 1);
                        if (elect_one()) {
                            uint8_t* dst = smem + L::kKVOff + slot * L::kTile;
                            mbar_arrive_expect_tx(kv_full + slot, L::kTile);
                            tma_tile<D>(dst, L::kKVBox, kv == 0 ? &tk : &tv, kv_full + slot, it.h,
                                        c * BKV, it.b, pol_kv);
                        }
                        __syncwarp();
                    }
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------------------------ MMA issuer
            uint32_t cons = 0, pcount[2] = {0, 0};
            const uint32_t q_base = smem_u32(smem + L::kQOff);
            const uint32_t kv_base = smem_u32(smem + L::kKVOff);
            for (int32_t local = 0;; ++local) {
                const int32_t item = next_item(local);
                if (item < 0) break;
                const Item it = decode_item(a, item);
                const TileList tl = tile_list(a, it);
                mbar_wait(q_full, local & 1);
                tc_fence_after();
                if (elect_one()) {
                    if constexpr (L::kQT) {  // Q -> TMEM, in order with this thread's MMAs
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            tmem_cp_128x256b(tmem + L::kQ + kk * 8,
                                             umma_desc_sw128(q_base + (kk >> 2) * L::kQBox +
                                                                 (kk & 3) * 32, 16, 1024));
                        mma_commit(q_empty);
                    } else if (tl.n == 0) {
                        mma_commit(q_empty);
                    }
                    if (tl.n == 0) mma_commit(o_full);  // corrupt plan (empty row): no tiles
                }
                __syncwarp();
                if (tl.n == 0) continue;
                auto do_pv = [&](int32_t t) {
                    const int grp = t & 1;
                    mbar_wait(p_full + grp, pcount[grp] & 1);
                    ++pcount[grp];
                    if (t == 0) mbar_wait(o_empty, (local & 1) ^ 1);  // last item's epilogue
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    mbar_wait(kv_full + slot, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t vb = kv_base + slot * L::kTile;
#pragma unroll
                        for (int kk = 0; kk < BKV / 16; ++kk)  // P over S's first B_kv/2 columns
                            mma_ts(tmem + L::kO, tmem + L::kS + grp * L::kSB + kk * 8,
                                   umma_desc_sw128(vb + kk * 16 * 128, L::kKVBox, 1024),
                                   L::kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(kv_empty + slot);
                    }
                    __syncwarp();
                };
                for (int32_t j = 0; j < tl.n; ++j) {
                    const int grp = j & 1;
                    const uint32_t slot = cons % S, ph = (cons / S) & 1;
                    ++cons;
                    mbar_wait(kv_full + slot, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t kb = kv_base + slot * L::kTile;
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint64_t bdesc = umma_desc_sw128(
                                kb + (kk >> 2) * L::kKVBox + (kk & 3) * 32, 16, 1024);
                            if constexpr (L::kQT) {
                                mma_ts(tmem + L::kS + grp * L::kSB, tmem + L::kQ + kk * 8, bdesc,
                                       L::kIdescQK, kk > 0 ? 1u : 0u);
                            } else {
                                mma_ss(tmem + L::kS + grp * L::kSB,
                                       umma_desc_sw128(q_base + (kk >> 2) * L::kQBox +
                                                           (kk & 3) * 32, 16, 1024),
                                       bdesc, L::kIdescQK, kk > 0 ? 1u : 0u);
                            }
                        }
                        mma_commit(s_full + grp);
                        mma_commit(kv_empty + slot);
                        if (!L::kQT && j == tl.n - 1) mma_commit(q_empty);  // Q read for good
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
        set_maxnreg_inc224();
        // ------------------------------------------------------------------ softmax groups
        const int grp = (int)(warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t s_col = L::kS + grp * L::kSB;
        const float sl2 = a.scale_log2;
        const uint64_t sl2x2 = f2(sl2, sl2);
        const int32_t tail_valid = g.N - (g.NBK - 1) * BKV;
        uint32_t scount = 0;
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local);
            if (item < 0) break;
            const Item it = decode_item(a, item);
            const TileList tl = tile_list(a, it);
            const bool last_ragged = tail_valid < BKV && tl.n > 0 && tl.last() == g.NBK - 1;
            // output rows of this thread's query row (MASK: the row itself; REPETITIVE: the
            // nearest-anchor group of spatial rows of the anchor query, Q10)
            int64_t tok0 = -1;
            int32_t n_dst = 0, dst_stride_rows = 0;
            if (it.kind == 0) {
                const int64_t t = (int64_t)it.idx * 128 + row;
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
            uint32_t* park =
                tok0 >= 0 ? reinterpret_cast<uint32_t*>(out_row(a, it.b, it.h, tok0)) : nullptr;
            float m_ref = 0.0f, l_run = 0.0f, m_run = -INFINITY;
            bool have_ref = mode != 0, bad = false;
            if (mode == 2 && park != nullptr) m_ref = __uint_as_float(*park);
            auto get_ref = [&]() {  // group 1: the reference group 0 posted for this item
                mbar_wait(mref_full, local & 1);
                m_ref = mref_s[row];
                have_ref = true;
            };
            for (int32_t j = grp; j < tl.n; j += 2) {
                mbar_wait(s_full + grp, scount & 1);
                ++scount;
                tc_fence_after();
                const bool ragged = last_ragged && j == tl.n - 1;
                uint32_t r[64];
                if (mode == 1 || (mode == 0 && j == 0)) {
                    float mx = -INFINITY;
                    auto part_max = [&](auto pc) {
                        using PT = decltype(pc);
                        ld_part<PT::kW>(lane_addr + s_col + PT::kCol, r);
                        if (ragged) mask_part<PT::kW>(r, PT::kCol, tail_valid);
                        mx = fmaxf(mx, max_part<PT::kW>(r));
                    };
                    part_max(Part<BKV, 0>{});
                    if constexpr (kParts > 1) part_max(Part<BKV, 1>{});
                    if constexpr (kParts > 2) part_max(Part<BKV, 2>{});
                    if (mode == 1) {
                        m_run = fmaxf(m_run, mx * sl2);
                    } else {
                        m_ref = mx * sl2;
                        mref_s[row] = m_ref;
                        have_ref = true;
                        __syncwarp();
                        if (lane == 0) mbar_arrive(mref_full);
                    }
                } else if (!have_ref) {
                    get_ref();
                }
                if (mode != 1) {
                    const uint64_t negm = f2(-m_ref, -m_ref);
                    float lsum = 0.0f;
                    auto part_exp = [&](auto pc) {
                        using PT = decltype(pc);
                        ld_part<PT::kW>(lane_addr + s_col + PT::kCol, r);
                        if (ragged) mask_part<PT::kW>(r, PT::kCol, tail_valid);
                        uint32_t pk[32];
                        lsum += exp_part<PT::kW, kEmuR<D>>(r, sl2x2, negm, pk);
                        // P of columns [c, c + w) -> packed columns [c/2, c/2 + w/2): below
                        // every column this thread still has to load
                        st_part<PT::kW>(lane_addr + s_col + PT::kCol / 2, pk);
                    };
                    part_exp(Part<BKV, 0>{});
                    if constexpr (kParts > 1) part_exp(Part<BKV, 1>{});
                    if constexpr (kParts > 2) part_exp(Part<BKV, 2>{});
                    bad |= !(lsum <= kGuardR);  // also catches inf / NaN
                    l_run += lsum;
                    tmem_st_wait();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + grp);
            }
            if (mode == 0 && grp == 0 && tl.n == 0) {  // corrupt plan: keep mref_full's phase
                mref_s[row] = 0.0f;
                __syncwarp();
                if (lane == 0) mbar_arrive(mref_full);
            }
            if (!have_ref) get_ref();  // group 1 without tiles (n <= 1)
            // -------------------------------------------------------------- epilogue
            if (mode == 0 && __any_sync(0xffffffffu, bad) && lane == 0) *flag_s = 1;
            mbar_wait(o_full, local & 1);
            tc_fence_after();
            if (mode == 1) {
                row_x[grp * 128 + row] = m_run;
                named_bar_sync(1, 256);
                const float mx = fmaxf(row_x[row], row_x[128 + row]);
                if (grp == 0 && park != nullptr) *park = __float_as_uint(mx);
                tc_fence_before();
                named_bar_sync(1, 256);  // row_x read before the next item's writes
            } else {
                row_x[grp * 128 + row] = l_run;
                named_bar_sync(1, 256);
                const float Lsum = row_x[row] + row_x[128 + row];
                const float inv = Lsum > 0.0f ? 1.0f / Lsum : 0.0f;
                const bool flagged = mode == 0 && *flag_s != 0;
                const uint64_t inv2 = f2(inv, inv);
#pragma unroll
                for (int cc = 0; cc < D / 2; cc += 32) {
                    const int col = grp * (D / 2) + cc;
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
                            out_row(a, it.b, it.h, tok0 + (int64_t)dI * dst_stride_rows) + col);
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1],
                                                packed[4 * v + 2], packed[4 * v + 3]);
                    }
                }
                if (grp == 0 && a.lse_out != nullptr) {
                    const float lse = (m_ref + __log2f(Lsum)) * 0.69314718055994531f;
                    float* lb = a.lse_out + ((int64_t)it.b * a.n_heads + it.h) * (int64_t)g.N;
                    for (int32_t dI = 0; dI < n_dst; ++dI)
                        lb[tok0 + (int64_t)dI * dst_stride_rows] = lse;
                }
                tc_fence_before();
                named_bar_sync(1, 256);  // every thread has read flag_s / row_x
                if (threadIdx.x == 128 && mode == 0) {
                    if (flagged) {  // recomputed by modes 1 + 2 after this launch
                        const uint32_t w = (uint32_t)(item / a.batch), bit = 1u << (w & 31u);
                        if ((atomicOr(fb.flags + (w >> 5), bit) & bit) == 0u)
                            fb.list[atomicAdd(fb.count, 1u)] = a.work_list[w];
                    }
                    *flag_s = 0;
                }
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

template <int BKV, int D>
cudaError_t launch_rect_d(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                          const CUtensorMap& tv, int grid, const Fallback& fb, int mode,
                          cudaStream_t s) {
    auto kern = sparse_attn_rect_kernel<BKV, D>;
    const int smem = SmemR<BKV, D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, SmemR<BKV, D>::kThreads, smem, s>>>(a, tq, tk, tv, fb, mode);
    return cudaGetLastError();
}

template <int BKV>
cudaError_t launch_rect(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                        const CUtensorMap& tv, int grid, const Fallback& fb, int mode,
                        cudaStream_t s) {
    return a.head_dim == 64 ? launch_rect_d<BKV, 64>(a, tq, tk, tv, grid, fb, mode, s)
                            : launch_rect_d<BKV, 128>(a, tq, tk, tv, grid, fb, mode, s);
}

}  // namespace

cudaError_t launch_attn_rect(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, int grid, const Fallback& fb, int mode,
                             cudaStream_t s) {
    if (a.g.B != 128) return cudaErrorInvalidValue;
    switch (a.g.BK) {
        case 64: return launch_rect<64>(a, tq, tk, tv, grid, fb, mode, s);
        case 80: return launch_rect<80>(a, tq, tk, tv, grid, fb, mode, s);
        case 96: return launch_rect<96>(a, tq, tk, tv, grid, fb, mode, s);
        case 112: return launch_rect<112>(a, tq, tk, tv, grid, fb, mode, s);
        case 128: return launch_rect<128>(a, tq, tk, tv, grid, fb, mode, s);
        case 144: return launch_rect<144>(a, tq, tk, tv, grid, fb, mode, s);
        case 160: return launch_rect<160>(a, tq, tk, tv, grid, fb, mode, s);
        case 176: return launch_rect<176>(a, tq, tk, tv, grid, fb, mode, s);
        case 192: return launch_rect<192>(a, tq, tk, tv, grid, fb, mode, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace csa
