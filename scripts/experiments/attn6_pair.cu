// attn6_pair.cu -- EXPERIMENT, not built into libcsa.so ("Pair items").
// Measured slower than the production attn5.cu on the same box (Wan 720p d 128: 1064 vs 1282
// TF/s; Wan 480p d 64: 704 vs 929), parity green; built and tested as csrc/attn6.cu at commit
// 8f52c9f (scripts/experiments/ab_pair2.sh, scripts/experiments/trace_attn6.py, tests test_pair_items_*).
//
// a7 + a8 for block 128 (head_dim 128 and 64) on PAIR items: two query blocks per
// CTA share one K/V stream over the union of their kept-block lists.
//
// PAPER.md P:647-656 (block-sparse attention over the kept key blocks of each query block),
// P:616-622 (anchor rows of REPETITIVE heads); readings Q1, Q2, Q9, Q10, Q29 (DESIGN.md section
// 2): each row's softmax shift is the max of its first kept tile; an overshoot beyond 2^56 flags
// the row's unit, which the exact-max passes of attn_rect.cu recompute after this launch.
//
// A pair item (h, p) (csa_build_work_list order 3) stands for units 2p and 2p+1 of head h (query
// blocks of a MASK head, anchor-query tiles of a REPETITIVE head).  Unit g belongs to softmax
// group g; the groups run independently on their own lists, so their S-load / P-store / barrier
// phases fall on each other's exponentials and the MUFU (16 ex2 / clk / SM = the tensor pipe's
// rate at d = 128) stays fed, which one 16-warp group on every tile (attn5.cu) cannot do.
//   TMEM (512 columns): S0 [0,128) S1 [128,256) | O0 [256,256+D) O1 [256+D, 256+2D)
//     P_g aliases S_g: column half c of the softmax writes its 64 keys' bf16 pairs over the
//     first 32 columns of its own half of S_g, so no thread overwrites columns another reads.
//   smem: Q0 | Q1 (SS S-MMA A operands) | K/V ring in union order K_u0 V_u0 K_u1 V_u1 ...
//   warps: 0 scheduler + producer, 1 / 3 MMA issuers of group 0 / 1, 2 TMEM allocator,
//          4-11 softmax group 0, 12-19 softmax group 1 (lane quarter = warp & 3, column half =
//          (warp - 4) >> 2 & 1).
// Per group g and kept tile j: S_g = Q_g K_j^T -> softmax (P_g over S_g) -> O_g += P_g V_j ->
// S_g = Q_g K_{j+1}^T (issued after the P.V by the same thread: the tensor pipe executes one
// thread's MMAs in order, so the P.V has read P_g before the next S-MMA overwrites it).
// A ring slot is released by every group that uses its tile (kv_empty counts 2 arrivals: a
// tile kept by one unit only is released by that group's MMA commit plus a plain arrive).
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kItemSlots6 = 4;
constexpr float kGuard6 = 72057594037927936.0f;  // 2^56
#ifndef CSA_ATTN6_EMU
#define CSA_ATTN6_EMU 0
#endif
constexpr int kEmu6 = CSA_ATTN6_EMU;  // element pairs p with (p & 7) >= 8 - kEmu6 -> FMA exp2

static __device__ unsigned long long* g_trace6;
#ifdef CSA_ENABLE_TRACE
#define TRACE6(slot, k, e)                                                                   \
    do {                                                                                     \
        if (g_trace6 != nullptr && blockIdx.x == 0 && (k) < 1024)                            \
            g_trace6[((slot) * 1024 + (k)) * 8 + (e)] = clock64();                           \
    } while (0)
#else
#define TRACE6(slot, k, e) \
    do {                   \
    } while (0)
#endif

template <int D>
struct Smem6 {
    static constexpr int kThreads = 640;
    static constexpr int kBox = 128 * 128;          // [128 rows][64 cols] bf16, SWIZZLE_128B
    static constexpr int kTile = (D / 64) * kBox;   // 128 x D bf16 (Q, K and V tiles alike)
    static constexpr int kQOff = 0;                 // Q[2]: one per group
    static constexpr int kKVOff = 2 * kTile;
    static constexpr int kSlotsFit = (232448 - 2 * kTile - 2560) / kTile;
    static constexpr int kSlots = kSlotsFit > 8 ? 8 : kSlotsFit;
    static constexpr int kBarOff = kKVOff + kSlots * kTile;
    // q_full[2] q_empty[2] | kv_full[S] kv_empty[S] | s_full[2] p_full[2] | o_full[2]
    // o_empty[2] | item_full[4] item_empty[4]
    static constexpr int kNumBars = 4 + 2 * kSlots + 4 + 4 + 2 * kItemSlots6;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;  // xchg [group][half][128] floats
    static constexpr int kItemOff = kRowOff + 2 * 2 * 128 * 4;
    static constexpr int kPosOff = kItemOff + kItemSlots6 * 4;  // ring position of each slot
    static constexpr int kFlagOff = kPosOff + 8 * 4;
    static constexpr int kTmemPtrOff = kFlagOff + 16;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(kBytes <= 232448, "smem");
    static_assert(kSlots >= 4, "ring");
    static constexpr uint32_t kS = 0, kO = 256;
    static_assert(kO + 2 * D <= 512 && (D == 64 || D == 128), "TMEM / head_dim");
    static constexpr uint32_t kIdescQK = umma_idesc_bf16(128, 128, 0, 0);
    static constexpr uint32_t kIdescPV = umma_idesc_bf16(128, D, 0, 1);
};

struct PairItem {
    uint32_t kind;
    int32_t h, b;
    int32_t unit0;   // units 2p (group 0) and 2p + 1 (group 1)
    int32_t units;   // units of the head (query blocks or anchor tiles)
    int64_t cell;
};

__device__ __forceinline__ PairItem decode_pair(const AttnArgs& a, int32_t item) {
    const uint32_t code = a.work_list[item / a.batch];
    PairItem it;
    it.kind = code >> 31;
    it.h = (int32_t)((code >> 20) & 0x7FFu);
    it.unit0 = 2 * (int32_t)(code & 0xFFFFFu);
    it.b = item % a.batch;
    it.cell = a.cell_base + it.h;
    it.units = it.kind ? (int32_t)(((int64_t)a.g.F * a.plan.anchor_k[it.cell] * a.g.W +
                                    kAnchorTile - 1) / kAnchorTile)
                       : a.g.NB;
    return it;
}

// Kept tiles of unit u (empty when the unit does not exist: the odd last unit of a head).
__device__ __forceinline__ TileList unit_list(const AttnArgs& a, const PairItem& it, int32_t u) {
    if (u >= it.units) return TileList{nullptr, 0};
    Item one;
    one.kind = it.kind;
    one.h = it.h;
    one.idx = u;
    one.b = it.b;
    one.cell = it.cell;
    return tile_list(a, one);
}

__device__ __forceinline__ uint32_t mbar_test6(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok;
}

// Issue lock of the two MMA warps: a group's P.V + next S-MMA batch enters the tensor pipe
// whole, never interleaved with the other group's, so the batches queue FIFO and the groups
// settle half a period apart (softmax of one group under the other group's MMAs) instead of
// locking in phase.  Taken only after every wait of the batch: never held while blocking.
#ifndef CSA_ATTN6_LOCK
#define CSA_ATTN6_LOCK 1
#endif
__device__ __forceinline__ void issue_lock(int32_t* lk) {
    if (CSA_ATTN6_LOCK && lane_id() == 0) {
        for (;;) {
            while (*reinterpret_cast<volatile int32_t*>(lk) != 0) {
            }
            if (atomicCAS(lk, 0, 1) == 0) break;
        }
    }
    __syncwarp();
    tc_fence_after();
}
__device__ __forceinline__ void issue_unlock(int32_t* lk) {
    tc_fence_before();
    __syncwarp();
    if (CSA_ATTN6_LOCK && lane_id() == 0) atomicExch(lk, 0);
}

// exp2(s * sl2 - m) of 32 scores -> 16 packed bf16 pairs; returns the fp32 sum.
__device__ __forceinline__ float exp_chunk32(const uint32_t (&r)[32], uint64_t sl2x2, uint64_t negm,
                                             uint32_t (&pk)[16]) {
    uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int x = 0; x < 32; x += 2) {
        const uint64_t t = ffma2(pk2(r[x], r[x + 1]), sl2x2, negm);
        uint64_t p;
        if (((x / 2) & 7) >= 8 - kEmu6) {
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

__device__ __forceinline__ float max32(const uint32_t (&r)[32]) {
    float mc[8];
#pragma unroll
    for (int q8 = 0; q8 < 8; ++q8)
        mc[q8] = fmax3(__uint_as_float(r[q8]), __uint_as_float(r[q8 + 8]),
                       fmaxf(__uint_as_float(r[q8 + 16]), __uint_as_float(r[q8 + 24])));
    return fmaxf(fmax3(mc[0], mc[1], mc[2]), fmaxf(fmax3(mc[3], mc[4], mc[5]), fmaxf(mc[6], mc[7])));
}

template <int D>
__global__ void __launch_bounds__(Smem6<D>::kThreads, 1)
    sparse_attn_pair_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                            const __grid_constant__ CUtensorMap tk,
                            const __grid_constant__ CUtensorMap tv, const Fallback fb) {
    using L = Smem6<D>;
    constexpr int BK = 128, S = L::kSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;        // [group]
    uint64_t* q_empty = bars + 2;   // [group]
    uint64_t* kv_full = bars + 4;
    uint64_t* kv_empty = kv_full + S;
    uint64_t* s_full = kv_empty + S;  // [group]
    uint64_t* p_full = s_full + 2;    // [group]
    uint64_t* o_full = p_full + 2;    // [group]
    uint64_t* o_empty = o_full + 2;   // [group]
    uint64_t* item_full = o_empty + 2;
    uint64_t* item_empty = item_full + kItemSlots6;
    float* xchg = reinterpret_cast<float*>(smem + L::kRowOff);  // [group][half][128]
    volatile int32_t* item_slot = reinterpret_cast<int32_t*>(smem + L::kItemOff);
    volatile int32_t* flag_s = reinterpret_cast<int32_t*>(smem + L::kFlagOff);  // [group]
    // slot_pos[s]: ring position of the fill last issued into slot s.  An issuer skips the
    // other group's solo tiles, so it may reach a slot whose previous fill (a tile it does not
    // use) has not even been issued; an mbarrier parity wait would then pass one phase early.
    // Waiting for slot_pos == pos first guarantees the previous fill completed (the producer
    // issues fill k only after every user released fill k - 1, which they waited for).
    volatile uint32_t* slot_pos = reinterpret_cast<uint32_t*>(smem + L::kPosOff);
    int32_t* mma_lock = reinterpret_cast<int32_t*>(smem + L::kFlagOff + 8);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full + i, 1);
            mbar_init(q_empty + i, 1);
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, 8);
            mbar_init(o_full + i, 1);
            mbar_init(o_empty + i, 8);
            flag_s[i] = 0;
        }
        *mma_lock = 0;
        for (int i = 0; i < S; ++i) {
            mbar_init(kv_full + i, 1);
            mbar_init(kv_empty + i, 2);
            slot_pos[i] = 0xffffffffu;
        }
        for (int i = 0; i < kItemSlots6; ++i) {
            mbar_init(item_full + i, 1);
            mbar_init(item_empty + i, 2 + 16);  // two issuers + 16 softmax warps
        }
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
        const int s = local % kItemSlots6;
        mbar_wait(item_full + s, (local / kItemSlots6) & 1);
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
            uint32_t ld = 0, qn0 = 0, qn1 = 0;
            for (int32_t local = 0;; ++local) {
                const int s = local % kItemSlots6;
                mbar_wait(item_empty + s, ((local / kItemSlots6) & 1) ^ 1);
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
                const PairItem it = decode_pair(a, item);
                const TileList t0 = unit_list(a, it, it.unit0);
                const TileList t1 = unit_list(a, it, it.unit0 + 1);
                for (int grp = 0; grp < 2; ++grp) {
                    const int32_t unit = it.unit0 + grp;
                    if (unit >= it.units) continue;
                    const uint32_t qn = grp ? qn1++ : qn0++;
                    uint8_t* qdst = smem + L::kQOff + grp * L::kTile;
                    mbar_wait(q_empty + grp, (qn & 1) ^ 1);
                    if (it.kind == 0) {
                        if (elect_one()) {
                            mbar_arrive_expect_tx(q_full + grp, L::kTile);
                            tma_tile<D>(qdst, L::kBox, &tq, q_full + grp, it.h, unit * BK, it.b,
                                        pol_q);
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
                            const int row = x / kChunks, chk = x % kChunks;
                            const int32_t gi = unit * 128 + row;
                            uint4 val = make_uint4(0u, 0u, 0u, 0u);
                            if (gi < n_anchor) {
                                const int32_t f = gi / per_frame;
                                const int32_t m = (gi / g.W) % kA;
                                const int32_t j = gi % g.W;
                                const int64_t tok = (int64_t)f * g.H * g.W +
                                                    (int64_t)anchor_row(g.H, kA, m) * g.W + j;
                                val = *reinterpret_cast<const uint4*>(qb_ptr + tok * a.q_sn +
                                                                      chk * 8);
                            }
                            *reinterpret_cast<uint4*>(qdst + (chk >> 3) * L::kBox +
                                                      sw128_offset(row, chk & 7)) = val;
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(q_full + grp);
                    }
                }
                // K/V of the union of both lists, ascending: K_c then V_c per union tile
                auto load = [&](int kv, int32_t c) {
                    const uint32_t slot = ld % S, ph = (ld / S) & 1;
                    ++ld;
                    mbar_wait(kv_empty + slot, ph ^ 1);
                    if (elect_one()) {
                        slot_pos[slot] = ld - 1;
                        uint8_t* dst = smem + L::kKVOff + slot * L::kTile;
                        mbar_arrive_expect_tx(kv_full + slot, L::kTile);
                        tma_tile<D>(dst, L::kBox, kv == 0 ? &tk : &tv, kv_full + slot, it.h,
                                    c * BK, it.b, pol_kv);
                    }
                    __syncwarp();
                };
                int32_t i0 = 0, i1 = 0;
                while (i0 < t0.n || i1 < t1.n) {
                    const int32_t c0 = i0 < t0.n ? t0.at(i0) : 0x7fffffff;
                    const int32_t c1 = i1 < t1.n ? t1.at(i1) : 0x7fffffff;
                    const int32_t c = c0 < c1 ? c0 : c1;
                    i0 += c0 == c;
                    i1 += c1 == c;
                    load(0, c);
                    load(1, c);
                }
            }
        } else if (warp == 1 || warp == 3) {
            // ------------------------------------------- MMA issuer of group grp (S-MMA, P.V)
            const int grp = warp == 3 ? 1 : 0;
            const uint32_t kv_base = smem_u32(smem + L::kKVOff);
            const uint32_t q_base = smem_u32(smem + L::kQOff + grp * L::kTile);
            const uint32_t s_tm = tmem + L::kS + (uint32_t)grp * 128u;
            const uint32_t o_tm = tmem + L::kO + (uint32_t)grp * D;
            uint32_t base = 0, qn = 0, pn = 0;
            auto wait_fill = [&](uint32_t pos) -> uint32_t {
                const uint32_t slot = pos % S;
                while (slot_pos[slot] != pos) __nanosleep(32);
                mbar_wait(kv_full + slot, (pos / S) & 1);
                return slot;
            };
            for (int32_t local = 0;; ++local) {
                const int32_t item = next_item(local);
                if (item < 0) break;
                const PairItem it = decode_pair(a, item);
                const TileList own = unit_list(a, it, it.unit0 + grp);
                const TileList oth = unit_list(a, it, it.unit0 + 1 - grp);
                const bool has = it.unit0 + grp < it.units;
                if (!has) {  // union = the other unit's list
                    base += 2u * (uint32_t)oth.n;
                    continue;
                }
                const uint32_t item_n = qn++;
                mbar_wait(q_full + grp, item_n & 1);
                // other-only tiles below own tile c = (other tiles < c) - (shared tiles < c)
                int32_t io = 0, shared = 0;
                auto locate = [&](int32_t c, bool& solo) -> uint32_t {
                    while (io < oth.n && oth.at(io) < c) ++io;
                    const bool sh = io < oth.n && oth.at(io) == c;
                    const int32_t before = io - shared;  // other-only tiles below c
                    if (sh) {
                        ++shared;
                        ++io;
                    }
                    solo = !sh;
                    return (uint32_t)before;
                };
                // S-MMA of own tile j from K in `slot` (all waits done by the caller)
                auto issue_qk = [&](int32_t j, uint32_t slot, bool solo) {
                    const uint32_t kb = kv_base + slot * L::kTile;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * L::kBox + (kk & 3) * 32;
                        mma_ss(s_tm, umma_desc_sw128(q_base + off, 16, 1024),
                               umma_desc_sw128(kb + off, 16, 1024), L::kIdescQK,
                               kk > 0 ? 1u : 0u);
                    }
                    mma_commit(s_full + grp);
                    mma_commit(kv_empty + slot);
                    if (solo) mbar_arrive(kv_empty + slot);
                    if (j == own.n - 1) mma_commit(q_empty + grp);  // last read of Q_g
                };
                if (own.n == 0) {  // corrupt plan (empty row): no tiles; zero output
                    mbar_wait(o_empty + grp, (item_n & 1) ^ 1);
                    if (elect_one()) {
                        mma_commit(q_empty + grp);
                        mma_commit(o_full + grp);
                    }
                    __syncwarp();
                    base += 2u * (uint32_t)oth.n;
                    continue;
                }
                // union position of own tile j = j + ob (ob: other-only tiles below it); ring
                // positions K = base + 2 (j + ob), V = K + 1
                bool solo = false;
                uint32_t ob = locate(own.at(0), solo);
                {
                    const uint32_t kslot = wait_fill(base + 2u * ob);
                    issue_lock(mma_lock);
                    if (elect_one()) issue_qk(0, kslot, solo);
                    issue_unlock(mma_lock);
                }
                for (int32_t j = 0; j < own.n; ++j) {
                    const uint32_t vpos = base + 2u * (ob + (uint32_t)j) + 1u;
                    const bool vsolo = solo;
                    bool nsolo = false;
                    if (j + 1 < own.n) {
                        ob = locate(own.at(j + 1), nsolo);
                        solo = nsolo;
                    }
                    // V_j and a probe of K_{j+1} before waiting for P_j (they do not depend on
                    // it); K_{j+1} is only probed: its slot may be freed by this very P.V (two
                    // other-only tiles between)
                    const uint32_t vslot = wait_fill(vpos);
                    const bool more = j + 1 < own.n;
                    const uint32_t kpos = base + 2u * (ob + (uint32_t)(j + 1));
                    const uint32_t kslot = kpos % S;
                    auto probe_k = [&]() -> uint32_t {
                        uint32_t r = 0;
                        if (more && lane == 0)
                            r = slot_pos[kslot] == kpos ? mbar_test6(kv_full + kslot, (kpos / S) & 1)
                                                        : 0u;
                        return __shfl_sync(0xffffffffu, r, 0);
                    };
                    uint32_t k_ready = probe_k();
                    if (lane == 0) TRACE6(2 + grp, pn, 0);
                    mbar_wait(p_full + grp, pn & 1);
                    if (lane == 0) TRACE6(2 + grp, pn, 1);
                    ++pn;
                    if (j == 0) mbar_wait(o_empty + grp, (item_n & 1) ^ 1);  // last epilogue
                    if (lane == 0) TRACE6(2 + grp, pn - 1, 2);
                    issue_lock(mma_lock);
                    if (lane == 0) TRACE6(2 + grp, pn - 1, 3);
                    if (elect_one()) {
                        const uint32_t vb = kv_base + vslot * L::kTile;
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            mma_ts(o_tm, s_tm + (uint32_t)((kk >> 2) * 64 + (kk & 3) * 8),
                                   umma_desc_sw128(vb + kk * 16 * 128, L::kBox, 1024),
                                   L::kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(kv_empty + vslot);
                        if (vsolo) mbar_arrive(kv_empty + vslot);
                        if (k_ready) issue_qk(j + 1, kslot, nsolo);
                    }
                    issue_unlock(mma_lock);
                    if (more && !k_ready) {
                        wait_fill(kpos);
                        issue_lock(mma_lock);
                        if (elect_one()) issue_qk(j + 1, kslot, nsolo);
                        issue_unlock(mma_lock);
                    }
                    if (lane == 0) TRACE6(2 + grp, pn - 1, 4);
                }
                if (elect_one()) mma_commit(o_full + grp);
                __syncwarp();
                base += 2u * (uint32_t)(own.n + oth.n - shared);  // 2 x union size
            }
        }
        __syncwarp();
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 104;" ::: "memory");
        // ------------------------------------------------------- softmax (2 groups x 8 warps)
        const int grp = (int)(warp - 4) >> 3;
        const int half = ((int)(warp - 4) >> 2) & 1;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t s_addr = lane_addr + L::kS + (uint32_t)grp * 128u + (uint32_t)half * 64u;
        const uint32_t o_addr = lane_addr + L::kO + (uint32_t)grp * D + (uint32_t)half * (D / 2);
        float* xg = xchg + grp * 256;  // [half][128]
        const uint32_t bar_id = 1 + (uint32_t)grp;
        const float sl2 = a.scale_log2;
        const uint64_t sl2x2 = f2(sl2, sl2);
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;
        uint32_t sn = 0, on = 0;
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local);
            if (item < 0) break;
            const PairItem it = decode_pair(a, item);
            const int32_t unit = it.unit0 + grp;
            if (unit >= it.units) continue;
            const TileList tl = unit_list(a, it, unit);
            const bool last_ragged = tail_valid < BK && tl.n > 0 && tl.at(tl.n - 1) == g.NB - 1;
            float m_ref = 0.0f, l_run = 0.0f;
            bool bad = false;
            const bool tr = half == 0 && quarter == 0 && lane == 0;
            (void)tr;
            for (int32_t j = 0; j < tl.n; ++j) {
                if (tr) TRACE6(grp, sn, 0);
                mbar_wait(s_full + grp, sn & 1);
                if (tr) TRACE6(grp, sn, 1);
                ++sn;
                tc_fence_after();
                uint32_t ra[32], rb[32];
                tmem_ld32(s_addr, ra);
                tmem_ld32(s_addr + 32, rb);
                tmem_ld_wait(ra);
                tmem_ld_wait(rb);
                if (tr) TRACE6(grp, sn - 1, 2);
                if (last_ragged && j == tl.n - 1) {
#pragma unroll
                    for (int x = 0; x < 32; ++x) {
                        if (half * 64 + x >= tail_valid) ra[x] = 0xff800000u;  // keys >= N
                        if (half * 64 + 32 + x >= tail_valid) rb[x] = 0xff800000u;
                    }
                }
                if (j == 0) {  // the row's reference: the max of its first kept tile
                    const float mh = fmaxf(max32(ra), max32(rb)) * sl2;
                    xg[half * 128 + row] = mh;
                    named_bar_sync(bar_id, 256);
                    m_ref = fmaxf(mh, xg[(half ^ 1) * 128 + row]);
                }
                const uint64_t negm = f2(-m_ref, -m_ref);
                uint32_t pk[16];
                float lsum = exp_chunk32(ra, sl2x2, negm, pk);
                tmem_st16(s_addr, pk);
                lsum += exp_chunk32(rb, sl2x2, negm, pk);
                tmem_st16(s_addr + 16, pk);
                bad |= !(lsum <= kGuard6);  // also catches inf / NaN
                l_run += lsum;
                if (tr) TRACE6(grp, sn - 1, 3);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + grp);
                if (tr) TRACE6(grp, sn - 1, 4);
            }
            // -------------------------------------------------------------- epilogue
            if (__any_sync(0xffffffffu, bad) && lane == 0) flag_s[grp] = 1;
            mbar_wait(o_full + grp, on & 1);
            ++on;
            tc_fence_after();
            xg[half * 128 + row] = l_run;
            named_bar_sync(bar_id, 256);
            const float Lsum = xg[row] + xg[128 + row];
            const float inv = Lsum > 0.0f ? 1.0f / Lsum : 0.0f;
            const bool flagged = flag_s[grp] != 0;
            int64_t tok0 = -1;
            int32_t n_dst = 0, dst_stride_rows = 0;
            if (it.kind == 0) {
                const int64_t t = (int64_t)unit * BK + row;
                if (t < g.N) {
                    tok0 = t;
                    n_dst = 1;
                }
            } else {
                const int32_t kA = a.plan.anchor_k[it.cell];
                const int32_t per_frame = kA * g.W;
                const int32_t gi = unit * 128 + row;
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
            constexpr int NO = D / 2;  // output columns of this thread's half (64 or 32)
            const int col = half * NO;
#pragma unroll
            for (int part = 0; part < NO / 32; ++part) {
                uint32_t r0[32];
                tmem_ld32(o_addr + part * 32, r0);
                tmem_ld_wait(r0);
                uint32_t packed[16];
#pragma unroll
                for (int x = 0; x < 32; x += 2) {
                    const uint64_t v = fmul2(pk2(r0[x], r0[x + 1]), inv2);
                    packed[x / 2] = pack_bf16(lo_f(v), hi_f(v));
                }
                for (int32_t dI = 0; dI < n_dst; ++dI) {
                    uint4* dst = reinterpret_cast<uint4*>(
                        obase + (tok0 + (int64_t)dI * dst_stride_rows) * a.o_sn + col + part * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2],
                                            packed[4 * v + 3]);
                }
            }
            if (half == 0 && a.lse_out != nullptr) {
                const float lse = (m_ref + __log2f(Lsum)) * 0.69314718055994531f;
                float* lb = a.lse_out + ((int64_t)it.b * a.n_heads + it.h) * (int64_t)g.N;
                for (int32_t dI = 0; dI < n_dst; ++dI)
                    lb[tok0 + (int64_t)dI * dst_stride_rows] = lse;
            }
            tc_fence_before();
            named_bar_sync(bar_id, 256);  // every thread has read flag_s / xchg
            if (half == 0 && quarter == 0 && lane == 0) {
                if (flagged) {  // recomputed by the exact-max passes after this launch
                    const uint32_t w = (uint32_t)(it.h * g.NB + unit), bit = 1u << (w & 31u);
                    if ((atomicOr(fb.flags + (w >> 5), bit) & bit) == 0u)
                        fb.list[atomicAdd(fb.count, 1u)] =
                            (it.kind << 31) | ((uint32_t)it.h << 20) | (uint32_t)unit;
                }
                flag_s[grp] = 0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty + grp);
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

cudaError_t set_attn6_trace(void* buf, int mode) {
    (void)mode;
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    return cudaMemcpyToSymbol(g_trace6, &p, sizeof(p));
}

namespace {
template <int D>
cudaError_t launch_pair_d(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                          const CUtensorMap& tv, int grid, const Fallback& fb, cudaStream_t s) {
    const int smem = Smem6<D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(sparse_attn_pair_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    sparse_attn_pair_kernel<D><<<grid, Smem6<D>::kThreads, smem, s>>>(a, tq, tk, tv, fb);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_pair(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, int grid, const Fallback& fb,
                             cudaStream_t s) {
    if (a.g.B != 128 || a.g.BK != 128) return cudaErrorInvalidValue;
    if (a.head_dim == 128) return launch_pair_d<128>(a, tq, tk, tv, grid, fb, s);
    if (a.head_dim == 64) return launch_pair_d<64>(a, tq, tk, tv, grid, fb, s);
    return cudaErrorInvalidValue;
}

}  // namespace csa
