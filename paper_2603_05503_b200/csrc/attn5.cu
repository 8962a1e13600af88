// attn5.cu -- a7 + a8 for block 128 (head_dim 128 and 64): fixed reference max, one softmax
// group on every tile, Q read by the S-MMA from shared memory, P double-buffered in TMEM.
//
// PAPER.md P:647-656 (block-sparse attention over the kept key blocks of each query block),
// P:616-622 (anchor rows of REPETITIVE heads); readings Q1, Q2, Q9, Q10, Q29 (DESIGN.md section
// 2): each row's softmax shift is the max of its first kept tile; an overshoot beyond 2^56 flags
// the item, which the exact-max passes of attn_rect.cu recompute after this launch.
//   TMEM (512 columns): S0 [0,128) S1 [128,256) | O [256,256+D) | P0, P1 (64 columns each)
//   smem: Q[2] (double-buffered, SS S-MMA A operand) | K/V ring in consumption order
//   * all 16 softmax warps take every tile (4 column parts of 32 keys: 4 warps per SMSP keep the
//     MUFU fed);
//   * S_j is released as soon as it is loaded (s_empty); P_j goes to P[j&1], so the P store of
//     tile j waits only for P.V_{j-2}; QK_{j+2} is issued while the softmax works on tile j;
//   * S_j = Q K_j^T runs as SS-MMAs (Q never copied to TMEM): interleaved with the TS P.V MMAs the
//     tensor pipe sustains 66.7 cycles per 128x128x16 dispatch against 72.6 for TS + TS
//     (scripts/mma_bench.cu, profiles/r02_mma_bench.txt; floor 64);
//   * warp 1 issues the S-MMAs, warp 3 the P.V MMAs (each blocks ~600 cycles per 8-MMA batch);
//     the producer loads the ring in issue order (K0, K1, K2, V0, K3, V1, ...).
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kItemSlots5 = 4;
constexpr int kCH5 = 4;                          // column parts (32 keys each)
constexpr float kGuard5 = 72057594037927936.0f;  // 2^56
constexpr int kEmu5 = 0;  // pairs p with (p & 7) >= 8 - kEmu5 -> polynomial exp2 (A/B: 0 1172, 1/8 1164, 1/4 1121)

// Ring positions (per item, n kept tiles) of the producer order K0, K1, then per step s >= 2:
// K_s (s < n), V_{s-2}: K_j after j K's and max(0, j-2) V's; V_j after min(j+2, n-1)+1 K's and
// j V's.
__device__ __forceinline__ uint32_t kpos5(int32_t j) { return (uint32_t)(j + (j > 2 ? j - 2 : 0)); }
__device__ __forceinline__ uint32_t vpos5(int32_t j, int32_t n) {
    return (uint32_t)((j + 2 < n - 1 ? j + 2 : n - 1) + 1 + j);
}
// Non-blocking barrier probe: issued as soon as the next wait's phase is known, its ~140-cycle
// round trip overlaps the exponentials, and the blocking wait is skipped when the phase had
// already completed (an mbarrier wait costs ~140 cycles even then, scripts/mbar_micro.cu).
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
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
static __device__ unsigned long long* g_trace5;
#ifdef CSA_ENABLE_TRACE
#define TRACE5(slot, k, e)                                                                   \
    do {                                                                                     \
        if (g_trace5 != nullptr && blockIdx.x == 0 && (k) < 1024)                            \
            g_trace5[((slot) * 1024 + (k)) * 8 + (e)] = clock64();                           \
    } while (0)
#else
#define TRACE5(slot, k, e) \
    do {                   \
    } while (0)
#endif

template <int D>
struct Smem5 {
    static constexpr int kThreads = 128 + 128 * kCH5;
    static constexpr int kBox = 128 * 128;          // [128 rows][64 cols] bf16, SWIZZLE_128B
    static constexpr int kTile = (D / 64) * kBox;   // 128 x D bf16 (Q, K and V tiles alike)
    static constexpr int kQOff = 0;                 // Q[2]: double-buffered (SS S-MMA operand)
    static constexpr int kKVOff = 2 * kTile;
    static constexpr int kSlotsFit = (232448 - 2 * kTile - 6144) / kTile;
    static constexpr int kSlots = kSlotsFit > 8 ? 8 : kSlotsFit;
    static constexpr int kBarOff = kKVOff + kSlots * kTile;
    // q_full[2] q_empty[2] | kv_full[S] kv_empty[S] | s_full[2] s_empty[2] | p_full[2]
    // p_empty[2] | o_full o_empty | item_full[4] item_empty[4]
    static constexpr int kNumBars = 4 + 2 * kSlots + 4 + 4 + 2 + 2 * kItemSlots5;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;  // l[CH][128] | tile-0 max [CH][128]
    static constexpr int kItemOff = kRowOff + 2 * kCH5 * 128 * 4;
    static constexpr int kFlagOff = kItemOff + kItemSlots5 * 4;
    static constexpr int kTmemPtrOff = kFlagOff + 16;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(kBytes <= 232448, "smem");
    static_assert(kSlots >= 3, "ring");
    // TMEM: S0 [0,128) S1 [128,256) | O [256, 256+D) | P0, P1 (64 columns each)
    static constexpr uint32_t kS = 0, kO = 256, kP = 256 + D;
    static_assert(kP + 128 <= 512 && (D == 64 || D == 128), "TMEM / head_dim");
    static constexpr uint32_t kIdescQK = umma_idesc_bf16(128, 128, 0, 0);
    static constexpr uint32_t kIdescPV = umma_idesc_bf16(128, D, 0, 1);
};

template <int D>
__global__ void __launch_bounds__(Smem5<D>::kThreads, 1)
    sparse_attn_sepp_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                            const __grid_constant__ CUtensorMap tk,
                            const __grid_constant__ CUtensorMap tv, const Fallback fb) {
    using L = Smem5<D>;
    constexpr int BK = 128, S = L::kSlots, CH = kCH5;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;          // [Q buffer]
    uint64_t* q_empty = bars + 2;     // [Q buffer]
    uint64_t* kv_full = bars + 4;
    uint64_t* kv_empty = kv_full + S;
    uint64_t* s_full = kv_empty + S;  // [S buffer]
    uint64_t* s_empty = s_full + 2;   // [S buffer]
    uint64_t* p_full = s_empty + 2;   // [P buffer]
    uint64_t* p_empty = p_full + 2;   // [P buffer]
    uint64_t* o_full = p_empty + 2;
    uint64_t* o_empty = o_full + 1;
    uint64_t* item_full = o_empty + 1;
    uint64_t* item_empty = item_full + kItemSlots5;
    float* row_l = reinterpret_cast<float*>(smem + L::kRowOff);  // [CH][128]
    float* mx_s = row_l + CH * 128;                               // [CH][128]
    volatile int32_t* item_slot = reinterpret_cast<int32_t*>(smem + L::kItemOff);
    volatile int32_t* flag_s = reinterpret_cast<int32_t*>(smem + L::kFlagOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full + i, 1);
            mbar_init(q_empty + i, 1);
            mbar_init(s_full + i, 1);
            mbar_init(s_empty + i, 4 * CH);
            mbar_init(p_full + i, 4 * CH);
            mbar_init(p_empty + i, 1);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(kv_full + i, 1);
            mbar_init(kv_empty + i, 1);
        }
        mbar_init(o_full, 1);
        mbar_init(o_empty, 4 * CH);
        for (int i = 0; i < kItemSlots5; ++i) {
            mbar_init(item_full + i, 1);
            mbar_init(item_empty + i, 2 + 4 * CH);  // two issuers + softmax warps
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
        const int s = local % kItemSlots5;
        mbar_wait(item_full + s, (local / kItemSlots5) & 1);
        const int32_t idx = item_slot[s];
        __syncwarp();
        if (lane == 0) mbar_arrive(item_empty + s);
        return idx;
    };

    if (warp < 4) {
        set_maxnreg_dec56();  // 4 x 56 + 16 x 104 fits the 640 x 96 launch allocation
        if (warp == 0) {
            // ------------------------------------------------------------ scheduler + producer
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_kv = policy_evict_last();
            uint32_t ld = 0;
            for (int32_t local = 0;; ++local) {
                const int s = local % kItemSlots5;
                mbar_wait(item_empty + s, ((local / kItemSlots5) & 1) ^ 1);
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
                const uint32_t qb = (uint32_t)local & 1u;
                uint8_t* qdst = smem + L::kQOff + qb * L::kTile;
                mbar_wait(q_empty + qb, ((local >> 1) & 1) ^ 1);
                if (it.kind == 0) {
                    if (elect_one()) {
                        mbar_arrive_expect_tx(q_full + qb, L::kTile);
                        tma_tile<D>(qdst, L::kBox, &tq, q_full + qb, it.h, it.idx * BK, it.b,
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
                        const int32_t gi = it.idx * 128 + row;
                        uint4 val = make_uint4(0u, 0u, 0u, 0u);
                        if (gi < n_anchor) {
                            const int32_t f = gi / per_frame;
                            const int32_t m = (gi / g.W) % kA;
                            const int32_t j = gi % g.W;
                            const int64_t tok = (int64_t)f * g.H * g.W +
                                                (int64_t)anchor_row(g.H, kA, m) * g.W + j;
                            val = *reinterpret_cast<const uint4*>(qb_ptr + tok * a.q_sn + chk * 8);
                        }
                        *reinterpret_cast<uint4*>(qdst + (chk >> 3) * L::kBox +
                                                  sw128_offset(row, chk & 7)) = val;
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(q_full + qb);
                }
                // ring order = issue order: K0, K1, then per step s >= 2: K_s, V_{s-2}; V tail
                TileCursor kcur(tl), vcur(tl);
                auto load = [&](int kv, int32_t c) {
                    const uint32_t slot = ld % S, ph = (ld / S) & 1;
                    ++ld;
                    mbar_wait(kv_empty + slot, ph ^ 1);
                    if (elect_one()) {
                        uint8_t* dst = smem + L::kKVOff + slot * L::kTile;
                        mbar_arrive_expect_tx(kv_full + slot, L::kTile);
                        tma_tile<D>(dst, L::kBox, kv == 0 ? &tk : &tv, kv_full + slot, it.h,
                                    c * BK, it.b, pol_kv);
                    }
                    __syncwarp();
                };
                for (int32_t step = 0; step < tl.n + 2; ++step) {
                    if (step < tl.n) load(0, kcur.next());
                    if (step >= 2) load(1, vcur.next());
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------ QK issuer: S_j = Q K_j^T (SS)
            uint32_t base = 0, sis0 = 0, sis1 = 0, tiles = 0;
            const uint32_t kv_base = smem_u32(smem + L::kKVOff);
            for (int32_t local = 0;; ++local) {
                const int32_t item = next_item(local);
                if (item < 0) break;
                const Item it = decode_item(a, item);
                const TileList tl = tile_list(a, it);
                const uint32_t qb = (uint32_t)local & 1u;
                const uint32_t q_base = smem_u32(smem + L::kQOff + qb * L::kTile);
                mbar_wait(q_full + qb, (local >> 1) & 1);
                for (int32_t j = 0; j < tl.n; ++j) {
                    const uint32_t b = (uint32_t)j & 1u;
                    const uint32_t use = b ? sis1++ : sis0++;
                    TRACE5(2, tiles + (uint32_t)j, 0);
                    mbar_wait(s_empty + b, (use & 1) ^ 1);  // softmax loaded S_{j-2}
                    const uint32_t pos = base + kpos5(j), slot = pos % S, ph = (pos / S) & 1;
                    mbar_wait(kv_full + slot, ph);
                    TRACE5(2, tiles + (uint32_t)j, 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t kb = kv_base + slot * L::kTile;
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t off = (kk >> 2) * L::kBox + (kk & 3) * 32;
                            mma_ss(tmem + L::kS + b * BK, umma_desc_sw128(q_base + off, 16, 1024),
                                   umma_desc_sw128(kb + off, 16, 1024), L::kIdescQK,
                                   kk > 0 ? 1u : 0u);
                        }
                        mma_commit(s_full + b);
                        mma_commit(kv_empty + slot);
                        if (j == tl.n - 1) mma_commit(q_empty + qb);  // last read of this Q
                    }
                    __syncwarp();
                }
                if (tl.n == 0) {  // corrupt plan (empty row): no tiles, release Q at once
                    if (elect_one()) mma_commit(q_empty + qb);
                    __syncwarp();
                }
                base += 2u * (uint32_t)tl.n;
                tiles += (uint32_t)tl.n;
            }
        } else if (warp == 3) {
            // ------------------------------------------------------------- P.V issuer (O)
            uint32_t base = 0, pc0 = 0, pc1 = 0, tiles = 0;
            const uint32_t kv_base = smem_u32(smem + L::kKVOff);
            for (int32_t local = 0;; ++local) {
                const int32_t item = next_item(local);
                if (item < 0) break;
                const Item it = decode_item(a, item);
                const TileList tl = tile_list(a, it);
                if (tl.n == 0) {  // corrupt plan (empty row): no tiles
                    if (elect_one()) mma_commit(o_full);
                    __syncwarp();
                    continue;
                }
                for (int32_t j = 0; j < tl.n; ++j) {
                    const uint32_t pb = (tiles + (uint32_t)j) & 1u;
                    const uint32_t use = pb ? pc1++ : pc0++;
                    TRACE5(3, tiles + (uint32_t)j, 0);
                    mbar_wait(p_full + pb, use & 1);
                    TRACE5(3, tiles + (uint32_t)j, 1);
                    if (j == 0) mbar_wait(o_empty, (local & 1) ^ 1);  // last item's epilogue
                    const uint32_t pos = base + vpos5(j, tl.n), slot = pos % S, ph = (pos / S) & 1;
                    mbar_wait(kv_full + slot, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t vb = kv_base + slot * L::kTile;
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            mma_ts(tmem + L::kO, tmem + L::kP + pb * 64 + kk * 8,
                                   umma_desc_sw128(vb + kk * 16 * 128, L::kBox, 1024),
                                   L::kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(p_empty + pb);
                        mma_commit(kv_empty + slot);
                    }
                    __syncwarp();
                    TRACE5(3, tiles + (uint32_t)j, 2);
                }
                base += 2u * (uint32_t)tl.n;
                tiles += (uint32_t)tl.n;
                if (elect_one()) mma_commit(o_full);
                __syncwarp();
            }
        }
        __syncwarp();
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 104;" ::: "memory");
        // ------------------------------------------------------------------ softmax (16 warps)
        constexpr int NC = BK / CH;  // 32 key columns per thread
        const int ch = (int)(warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const float sl2 = a.scale_log2;
        const uint64_t sl2x2 = f2(sl2, sl2);
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;
        uint32_t sc0 = 0, sc1 = 0, ps0 = 0, ps1 = 0, tbase = 0;
        const bool tr = quarter == 0 && ch == 0 && lane == 0;
        (void)tr;
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local);
            if (item < 0) break;
            const Item it = decode_item(a, item);
            const TileList tl = tile_list(a, it);
            const bool last_ragged = tail_valid < BK && tl.n > 0 && tl.last() == g.NB - 1;
            float m_ref = 0.0f, l_run = 0.0f;
            bool bad = false;
            uint32_t s_ready = 0;  // probe result for the next tile's S
            uint32_t r[NC];
            for (int32_t j = 0; j < tl.n; ++j) {
                const uint32_t b = (uint32_t)j & 1u;
                const uint32_t use = b ? sc1++ : sc0++;
                const uint32_t pb = (tbase + (uint32_t)j) & 1u;
                const uint32_t puse = pb ? ps1++ : ps0++;
                if (tr) TRACE5(0, tbase + (uint32_t)j, 0);
                if (!s_ready) mbar_wait(s_full + b, use & 1);
                tc_fence_after();
                tmem_ld32(lane_addr + L::kS + b * BK + ch * NC, r);
                if (tr) TRACE5(0, tbase + (uint32_t)j, 1);
                tmem_ld_wait(r);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty + b);  // S_j may be overwritten (QK_{j+2})
                // probe of the P buffer (P.V_{j-2} done), resolved before the P store
                const uint32_t p_ready = mbar_test(p_empty + pb, (puse & 1) ^ 1);
                if (tr) TRACE5(0, tbase + (uint32_t)j, 2);
                if (last_ragged && j == tl.n - 1) {
#pragma unroll
                    for (int x = 0; x < NC; ++x)
                        if (ch * NC + x >= tail_valid) r[x] = 0xff800000u;  // keys >= N
                }
                if (j == 0) {  // the row's reference: the max of its first kept tile
                    float mc[8];
#pragma unroll
                    for (int q8 = 0; q8 < 8; ++q8)
                        mc[q8] = fmax3(__uint_as_float(r[q8]), __uint_as_float(r[q8 + 8]),
                                       fmaxf(__uint_as_float(r[q8 + 16]),
                                             __uint_as_float(r[q8 + 24])));
                    m_ref = fmaxf(fmax3(mc[0], mc[1], mc[2]),
                                  fmaxf(fmax3(mc[3], mc[4], mc[5]), fmaxf(mc[6], mc[7]))) * sl2;
                    mx_s[ch * 128 + row] = m_ref;
                    named_bar_sync(2, 128 * CH);
                    m_ref = fmaxf(fmaxf(mx_s[row], mx_s[128 + row]),
                                  fmaxf(mx_s[256 + row], mx_s[384 + row]));
                }
                const uint64_t negm = f2(-m_ref, -m_ref);
                uint64_t acc[4] = {0, 0, 0, 0};
                uint32_t pk[16];
#pragma unroll
                for (int x = 0; x < NC; x += 2) {
                    const uint64_t t = ffma2(pk2(r[x], r[x + 1]), sl2x2, negm);
                    uint64_t p;
                    if (((x / 2) & 7) >= 8 - kEmu5) {
                        p = exp2_poly2(t);
                    } else {
                        p = f2(ex2_approx(lo_f(t)), ex2_approx(hi_f(t)));
                    }
                    acc[(x / 2) & 3] = fadd2(acc[(x / 2) & 3], p);
                    pk[x / 2] = pack_bf16(lo_f(p), hi_f(p));
                }
                const uint64_t acc2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
                const float lsum = lo_f(acc2) + hi_f(acc2);
                bad |= !(lsum <= kGuard5);  // also catches inf / NaN
                l_run += lsum;
                if (tr) TRACE5(0, tbase + (uint32_t)j, 3);
                // probe the next S after the exponentials: its round trip hides under the store
                s_ready = j + 1 < tl.n ? mbar_test(s_full + (b ^ 1u), (b ? sc0 : sc1) & 1) : 0u;
                if (!p_ready) mbar_wait(p_empty + pb, (puse & 1) ^ 1);  // P.V_{j-2} read P[pb]
                tc_fence_after();
                tmem_st16(lane_addr + L::kP + pb * 64 + ch * (NC / 2), pk);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + pb);
                if (tr) TRACE5(0, tbase + (uint32_t)j, 4);
            }
            tbase += (uint32_t)tl.n;
            // -------------------------------------------------------------- epilogue
            if (__any_sync(0xffffffffu, bad) && lane == 0) *flag_s = 1;
            mbar_wait(o_full, local & 1);
            tc_fence_after();
            row_l[ch * 128 + row] = l_run;
            named_bar_sync(1, 128 * CH);
            const float Lsum = (row_l[row] + row_l[128 + row]) + (row_l[256 + row] + row_l[384 + row]);
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
            const uint64_t inv2 = f2(inv, inv);
            {
                constexpr int NO = D / CH;  // output columns of this thread's part (32 or 16)
                const int col = ch * NO;
                uint32_t r0[32];
                if constexpr (NO == 32) {
                    tmem_ld32(lane_addr + L::kO + col, r0);
                    tmem_ld_wait(r0);
                } else {
                    tmem_ld16(lane_addr + L::kO + col, *reinterpret_cast<uint32_t(*)[16]>(&r0[0]));
                    tmem_ld_wait();
#pragma unroll
                    for (int x = 0; x < 16; ++x) asm volatile("" : "+r"(r0[x]));
                }
                uint32_t packed[16];
#pragma unroll
                for (int x = 0; x < NO; x += 2) {
                    const uint64_t v = fmul2(pk2(r0[x], r0[x + 1]), inv2);
                    packed[x / 2] = pack_bf16(lo_f(v), hi_f(v));
                }
                // local output: one base pointer per item; output scatter: out_row per row
                __nv_bfloat16* obase = a.o_peer == nullptr
                                           ? a.o + (int64_t)it.b * a.o_sb + (int64_t)it.h * a.o_sh
                                           : nullptr;
                for (int32_t dI = 0; dI < n_dst; ++dI) {
                    const int64_t tok = tok0 + (int64_t)dI * dst_stride_rows;
                    uint4* dst = reinterpret_cast<uint4*>(
                        (obase != nullptr ? obase + tok * a.o_sn : out_row(a, it.b, it.h, tok)) +
                        col);
#pragma unroll
                    for (int v = 0; v < NO / 8; ++v)
                        dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2],
                                            packed[4 * v + 3]);
                }
            }
            if (ch == 0 && a.lse_out != nullptr) {
                const float lse = (m_ref + __log2f(Lsum)) * 0.69314718055994531f;
                float* lb = a.lse_out + ((int64_t)it.b * a.n_heads + it.h) * (int64_t)g.N;
                for (int32_t dI = 0; dI < n_dst; ++dI)
                    lb[tok0 + (int64_t)dI * dst_stride_rows] = lse;
            }
            tc_fence_before();
            named_bar_sync(1, 128 * CH);  // every thread has read flag_s / row_l
            if (threadIdx.x == 128) {
                if (flagged) {  // recomputed by the running-max kernel after this launch
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

cudaError_t set_attn5_trace(void* buf, int mode) {
    (void)mode;
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    return cudaMemcpyToSymbol(g_trace5, &p, sizeof(p));
}

namespace {
template <int D>
cudaError_t launch_sepp_d(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                          const CUtensorMap& tv, int grid, const Fallback& fb, cudaStream_t s) {
    const int smem = Smem5<D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(sparse_attn_sepp_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    sparse_attn_sepp_kernel<D><<<grid, Smem5<D>::kThreads, smem, s>>>(a, tq, tk, tv, fb);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_attn_sepp(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, int grid, const Fallback& fb,
                             cudaStream_t s) {
    if (a.g.B != 128 || a.g.BK != 128) return cudaErrorInvalidValue;
    if (a.head_dim == 128) return launch_sepp_d<128>(a, tq, tk, tv, grid, fb, s);
    if (a.head_dim == 64) return launch_sepp_d<64>(a, tq, tk, tv, grid, fb, s);
    return cudaErrorInvalidValue;
}

}  // namespace csa
