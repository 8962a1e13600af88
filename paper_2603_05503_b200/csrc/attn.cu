// attn.cu -- a7 + a8: calibrated block-sparse attention forward on sm_100a, BLOCK 64 layouts
// (BASELINE configs[0], the tiny / ragged twins; block 128 runs attn5.cu / attn_rect.cu).
//
// What it computes:
//   MASK cells: for query block r, softmax(scale Q_r K^T) V restricted to the keys of
//     the kept key blocks c of row r (Eq. eq:p / eq:pv) -- skipped blocks excluded
//     from numerator and normaliser (reading Q1) and never loaded.  Online softmax over the kept
//     tiles in ascending c.
//   REPETITIVE cells: only the k anchor spatial rows of every frame are
//     computed, densely against all N keys; row (f,i,j) receives row (f, a(i), j) (Q9, Q10).
//
// Design: persistent, one CTA per SM, 12 warps.
//   warp 0      scheduler + producer: claims items (dynamic, head-major work list) and publishes
//               them through a 4-deep shared-memory ring; loads the Q tile (TMA, or an in-warp
//               gather of anchor rows), then the kept K/V tiles of the item's block list through
//               a FIFO ring of smem slots in MMA consumption order K0, K1, V0, K2, V1, ...
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into S[j&1] (TMEM), then
//               O[(j-1)&1] += P_{j-1} V_{j-1} with P read from TMEM (TS-MMA).
//   warp 2      TMEM allocator (512 columns: S0 S1 O0 O1).
//   warps 4-7   softmax group 0: even tiles of the item's list   } each keeps its own (m, l, O);
//   warps 8-11  softmax group 1: odd tiles                          } merged in the epilogue.
// One thread owns one query row (= one TMEM lane).  Lazy rescale: O is rescaled only when the
// running max grows by more than 2^8.  Packed f32x2 FMA/ADD; all exp2 on the MUFU (kEmuEvery 0).
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kThreads = 384;
static __device__ unsigned long long* g_trace;  // csa_debug_trace: CTA 0's first item timeline
#ifdef CSA_ENABLE_TRACE  // trace builds only (see attn_common.cuh)
#define ATRACE(slot, k, e)                                                                  \
    do {                                                                                    \
        if (g_trace != nullptr && blockIdx.x == 0 && local == 0 && (k) < 1024)              \
            g_trace[((slot) * 1024 + (k)) * 8 + (e)] = clock64();                           \
    } while (0)
#else
#define ATRACE(slot, k, e) \
    do {                   \
    } while (0)
#endif
constexpr float kRedoSum = 32768.0f;        // lazy max: a tile's P row sum above 2^15 -> redo
constexpr bool kLazyMax = false;            // A/B switch
constexpr int kItemSlots = 4;
constexpr int kEmuEvery = 0;  // every kEmuEvery-th element pair uses the polynomial exp2 (0:
                               // none -- measured fastest: the softmax is issue-bound, not MUFU-bound)

template <int BK, int D>
struct AttnSmem {
    using C = TileCfg<BK, D>;
    static constexpr int kSlots = (BK == 128 && D == 128) ? 5 : 8;
    static constexpr int kQOff = 0;
    static constexpr int kKVOff = 2 * C::kQBytes;
    static constexpr int kBarOff = kKVOff + kSlots * C::kKVBytes;
    // q_full[2] q_empty[2] kv_full[S] kv_empty[S] s_full[2] p_full[2] o_full o_empty
    // item_full[4] item_empty[4]
    static constexpr int kNumBars = 4 + 2 * kSlots + 4 + 2 + 2 * kItemSlots;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;           // m[2][128], l[2][128]
    static constexpr int kItemOff = kRowOff + 4 * 128 * 4;           // int32 [kItemSlots]
    static constexpr int kTmemPtrOff = kItemOff + kItemSlots * 4;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static constexpr int kAlloc = kBytes;  // base is 1 KiB aligned (__align__ on the extern)
    static_assert(kAlloc <= 232448, "smem");
};

// Item decoding, kept-tile lists, anchor rows, packed fp32 math, exp2_poly2 and setmaxnreg:
// attn_common.cuh (shared with attn2.cu / attn3.cu).

template <int BK, int D, int kEmuE = kEmuEvery>
__global__ void __launch_bounds__(kThreads, 1)
    sparse_attn_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                       const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv) {
    using C = TileCfg<BK, D>;
    using L = AttnSmem<BK, D>;
    constexpr int S = L::kSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();  // SWIZZLE_128B atoms need 1 KiB alignment
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 2;
    uint64_t* kv_full = bars + 4;
    uint64_t* kv_empty = bars + 4 + S;
    uint64_t* s_full = bars + 4 + 2 * S;
    uint64_t* p_full = bars + 6 + 2 * S;
    uint64_t* o_full = bars + 8 + 2 * S;
    uint64_t* o_empty = bars + 9 + 2 * S;
    uint64_t* item_full = bars + 10 + 2 * S;
    uint64_t* item_empty = item_full + kItemSlots;
    float* row_m = reinterpret_cast<float*>(smem + L::kRowOff);  // [2][128]
    float* row_l = row_m + 256;                                   // [2][128]
    volatile int32_t* item_slot = reinterpret_cast<int32_t*>(smem + L::kItemOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full + i, 1);
            mbar_init(q_empty + i, 1);
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, 4);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(kv_full + i, 1);
            mbar_init(kv_empty + i, 1);
        }
        mbar_init(o_full, 1);
        mbar_init(o_empty, 8);
        for (int i = 0; i < kItemSlots; ++i) {
            mbar_init(item_full + i, 1);
            mbar_init(item_empty + i, 9);  // MMA thread + 8 softmax warps
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

    // consumer side of the item ring
    auto next_item = [&](int32_t local, bool is_warp_consumer) -> int32_t {
        const int s = local % kItemSlots;
        mbar_wait(item_full + s, (local / kItemSlots) & 1);
        const int32_t idx = item_slot[s];
        if (is_warp_consumer) {
            __syncwarp();
            if (lane == 0) mbar_arrive(item_empty + s);
        } else {
            mbar_arrive(item_empty + s);
        }
        return idx;
    };

    if (warp < 4) {
    set_maxnreg_dec56();  // producer / MMA / allocator warpgroup hands registers to softmax
    if (warp == 0) {
        // ------------------------------------------------------------ scheduler + producer
        const uint64_t pol_q = policy_evict_first();
        const uint64_t pol_kv = policy_evict_last();
        uint32_t ld = 0;  // K/V loads issued (ring position)
        for (int32_t local = 0;; ++local) {
            const int s = local % kItemSlots;
            mbar_wait(item_empty + s, ((local / kItemSlots) & 1) ^ 1);
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
            const int qb = local & 1;
            uint8_t* qdst = smem + L::kQOff + qb * C::kQBytes;
            mbar_wait(q_empty + qb, ((local >> 1) & 1) ^ 1);
            if (it.kind == 0) {
                if (lane == 0) {
                    mbar_arrive_expect_tx(q_full + qb, C::kBoxes * BK * 128);
                    tma_tile<D>(qdst, C::kQBox, &tq, q_full + qb, it.h, it.idx * BK, it.b, pol_q);
                }
            } else {
                // gather the anchor query rows of tile u: g = u*128 + row -> (f, m, j)
                const int32_t kA = a.plan.anchor_k[it.cell];
                const int32_t per_frame = kA * g.W;
                const int32_t n_anchor = g.F * per_frame;
                const __nv_bfloat16* qb_ptr =
                    a.q + (int64_t)it.b * a.q_sb + (int64_t)it.h * a.q_sh;
                constexpr int kChunks = D / 8;  // 16-byte chunks per row
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
                    *reinterpret_cast<uint4*>(qdst + (ch >> 3) * C::kQBox +
                                              sw128_offset(row, ch & 7)) = val;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(q_full + qb);
            }
            // K/V tiles in MMA consumption order: K0, (K1, V0), (K2, V1), ..., V_{n-1}.  The
            // whole warp walks the list (warp-uniform values live in uniform registers); one
            // elected lane issues -- a lane-0-only loop makes ptxas wrap each TMA in an
            // ELECT / R2UR / BRA.U.ANY loop.
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
                        uint8_t* dst = smem + L::kKVOff + slot * C::kKVBytes;
                        mbar_arrive_expect_tx(kv_full + slot, C::kKVBytes);
                        tma_tile<D>(dst, C::kKBox, kv == 0 ? &tk : &tv, kv_full + slot, it.h,
                                    c * BK, it.b, pol_kv);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        // Whole warp in the loop, one elected lane issues (see the producer above): the
        // lane-0-only form cost ~16 dependent instructions per tcgen05.mma.
        uint32_t cons = 0;            // K/V ring position consumed
        uint32_t pcount[2] = {0, 0};  // p_full completions waited, per group
        const uint32_t q_base = smem_u32(smem + L::kQOff);
        const uint32_t kv_base = smem_u32(smem + L::kKVOff);
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local, true);
            if (item < 0) break;
            const Item it = decode_item(a, item);
            const TileList tl = tile_list(a, it);
            const int qb = local & 1;
            mbar_wait(q_full + qb, (local >> 1) & 1);
            const uint32_t q_smem = q_base + qb * C::kQBytes;
            if (tl.n == 0) {  // corrupt plan (empty MASK row): release Q, no tiles
                if (elect_one()) {
                    mma_commit(q_empty + qb);
                    mma_commit(o_full);
                }
                __syncwarp();
                continue;
            }
            auto do_pv = [&](int32_t t) {
                const int grp = t & 1;
                if (lane == 0) ATRACE(2, t, 2);
                mbar_wait(p_full + grp, pcount[grp] & 1);
                if (lane == 0) ATRACE(2, t, 3);
                ++pcount[grp];
                if (t == 0) mbar_wait(o_empty, (local & 1) ^ 1);  // epilogue of last item
                const uint32_t slot = cons % S, ph = (cons / S) & 1;
                ++cons;
                mbar_wait(kv_full + slot, ph);
                tc_fence_after();
                if (elect_one()) {
                    issue_pv<BK, D>(tmem + 2 * BK + grp * D, tmem + grp * BK,
                                    kv_base + slot * C::kKVBytes, t >= 2);
                    mma_commit(kv_empty + slot);
                }
                __syncwarp();
            };
            for (int32_t j = 0; j < tl.n; ++j) {
                const int grp = j & 1;
                const uint32_t slot = cons % S, ph = (cons / S) & 1;
                ++cons;
                if (lane == 0) ATRACE(2, j, 0);
                mbar_wait(kv_full + slot, ph);
                if (lane == 0) ATRACE(2, j, 1);
                tc_fence_after();
                if (elect_one()) {
                    issue_qk<BK, D>(tmem + grp * BK, q_smem, kv_base + slot * C::kKVBytes);
                    mma_commit(s_full + grp);
                    mma_commit(kv_empty + slot);
                    if (j == tl.n - 1) mma_commit(q_empty + qb);
                }
                __syncwarp();
                if (j >= 1) do_pv(j - 1);
            }
            do_pv(tl.n - 1);
            if (elect_one()) mma_commit(o_full);
            __syncwarp();
        }
    }
    } else {
        set_maxnreg_inc224();
        // ------------------------------------------------------------------ softmax groups
        const int grp = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t s_col = grp * BK;
        const uint32_t o_col = 2 * BK + grp * D;
        const float sl2 = a.scale_log2;
        const uint64_t sl2x2 = f2(sl2, sl2);
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;  // keys in the last (ragged) block
        uint32_t scount = 0;
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local, true);
            if (item < 0) break;
            const Item it = decode_item(a, item);
            const TileList tl = tile_list(a, it);
            // only the last listed tile can be the ragged block N_B - 1
            const bool last_ragged = tail_valid < BK && tl.n > 0 && tl.last() == g.NB - 1;
            float m_run = -INFINITY, l_run = 0.0f;
            int32_t mine = 0;
            for (int32_t j = grp; j < tl.n; j += 2, ++mine) {
                const bool tr = quarter == 0 && lane == 0;
                if (tr) ATRACE(grp, j, 0);
                mbar_wait(s_full + grp, scount & 1);
                if (tr) ATRACE(grp, j, 1);
                ++scount;
                tc_fence_after();
                uint32_t r[BK / 32][32];
#pragma unroll
                for (int c = 0; c < BK / 32; ++c) tmem_ld32(lane_addr + s_col + c * 32, r[c]);
#pragma unroll
                for (int c = 0; c < BK / 32; ++c) tmem_ld_wait(r[c]);
                if (last_ragged && j == tl.n - 1) {
#pragma unroll
                    for (int c = 0; c < BK / 32; ++c)
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if (c * 32 + x >= tail_valid) r[c][x] = 0xff800000u;  // -inf
                }
                // row max: 8 independent FMNMX3 chains (short dependency depth), then combine
                auto row_max = [&]() -> float {
                    constexpr int kPer = BK / 8;  // elements per chain (even)
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
                    return fmaxf(fmax3(mc[0], mc[1], mc[2]),
                                 fmaxf(fmax3(mc[3], mc[4], mc[5]), fmaxf(mc[6], mc[7])));
                };
                // P = 2^(s*scale*log2e - m) -> bf16 over the first BK/2 columns of S; returns the
                // fp32 row sum (4 packed partial sums, 8 independent chains)
                auto exp_tile = [&](float m) -> float {
                    const uint64_t negm = f2(-m, -m);
                    uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
                    for (int c = 0; c < BK / 32; ++c) {
                        uint32_t pk[16];
#pragma unroll
                        for (int x = 0; x < 32; x += 2) {
                            const uint64_t sx = pk2(r[c][x], r[c][x + 1]);
                            const uint64_t t = ffma2(sx, sl2x2, negm);
                            uint64_t p;
                            if (kEmuE > 0 &&
                                ((c * 16 + x / 2) % (kEmuE > 0 ? kEmuE : 1)) == kEmuE - 1) {
                                p = exp2_poly2(t);
                            } else {
                                p = f2(ex2_approx(lo_f(t)), ex2_approx(hi_f(t)));
                            }
                            acc[(x / 2) & 3] = fadd2(acc[(x / 2) & 3], p);
                            pk[x / 2] = pack_bf16(lo_f(p), hi_f(p));
                        }
                        tmem_st16(lane_addr + s_col + c * 16, pk);
                    }
                    const uint64_t acc2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
                    return lo_f(acc2) + hi_f(acc2);
                };
                float alpha = 1.0f;
                bool rescale = false;
                float lsum;
                if constexpr (kLazyMax) {
                    // No max on the common tile: exponentials against the running max; only when
                    // the tile's row sum passes 2^15 (an element may exceed 2^8, non-finite
                    // included) is the max taken, l and O rescaled and the tile redone.
                    if (mine == 0) m_run = row_max() * sl2;
                    lsum = exp_tile(m_run);
                    const bool need = mine > 0 && !(lsum <= kRedoSum);
                    // tcgen05.ld/st are warp-collective: the whole warp redoes (alpha = 1 rows)
                    if (__any_sync(0xffffffffu, need)) {
                        const float m_new = need ? fmaxf(m_run, row_max() * sl2) : m_run;
                        alpha = ex2_approx(m_run - m_new);
                        l_run *= alpha;
                        m_run = m_new;
                        tmem_st_wait();
                        lsum = exp_tile(m_run);
                        rescale = true;
                    }
                } else {
                    const float m_new = fmaxf(m_run, row_max() * sl2);
                    bool need = false;
                    if (mine == 0) {
                        m_run = m_new;
                    } else if (m_new > m_run + kRescaleThreshold) {
                        alpha = ex2_approx(m_run - m_new);
                        l_run *= alpha;
                        m_run = m_new;
                        need = true;
                    }
                    // tcgen05.ld/st are warp-collective (.sync.aligned): the O rescale below runs
                    // for the whole warp when any of its rows needs it (alpha = 1 for the others)
                    rescale = __any_sync(0xffffffffu, need);
                    lsum = exp_tile(m_run);
                }
                l_run += lsum;
                if (rescale) {
                    // O_grp holds only this group's earlier tiles; their P.V completed before
                    // this tile's S (issued after it on the in-order tensor pipe) was ready
                    const uint64_t al2 = f2(alpha, alpha);
#pragma unroll
                    for (int c = 0; c < D; c += 32) {
                        uint32_t o[32];
                        tmem_ld32(lane_addr + o_col + c, o);
                        tmem_ld_wait(o);
#pragma unroll
                        for (int x = 0; x < 32; x += 2) {
                            const uint64_t v = fmul2(pk2(o[x], o[x + 1]), al2);
                            o[x] = (uint32_t)v;
                            o[x + 1] = (uint32_t)(v >> 32);
                        }
                        tmem_st32(lane_addr + o_col + c, o);
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + grp);
                if (tr) ATRACE(grp, j, 2);
            }
            // -------------------------------------------------------------- epilogue
            mbar_wait(o_full, local & 1);
            tc_fence_after();
            row_m[grp * 128 + row] = m_run;
            row_l[grp * 128 + row] = l_run;
            named_bar_sync(1, 256);
            const bool has0 = tl.n >= 1, has1 = tl.n >= 2;
            const float m0 = row_m[row], m1 = row_m[128 + row];
            const float l0 = row_l[row], l1 = row_l[128 + row];
            const float M = has1 ? fmaxf(m0, m1) : m0;
            const float a0 = has0 ? ex2_approx(m0 - M) : 0.0f;
            const float a1 = has1 ? ex2_approx(m1 - M) : 0.0f;
            const float Lsum = l0 * a0 + l1 * a1;
            const float inv = 1.0f / Lsum;
            const float f0 = a0 * inv, f1 = a1 * inv;
            // output rows of this thread
            int64_t tok0 = -1;
            int32_t n_dst = 0, dst_stride_rows = 0;
            if (it.kind == 0) {
                const int64_t t = (int64_t)it.idx * BK + row;
                if (row < BK && t < g.N) {
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
            const uint64_t f0x2 = f2(f0, f0), f1x2 = f2(f1, f1);
#pragma unroll
            for (int c = 0; c < D / 2; c += 32) {
                const int col = grp * (D / 2) + c;
                uint32_t r0[32], r1[32];
                tmem_ld32(lane_addr + 2 * BK + col, r0);
                if (has1) tmem_ld32(lane_addr + 2 * BK + D + col, r1);
                tmem_ld_wait(r0);
                if (has1) tmem_ld_wait(r1);
                uint32_t packed[16];
#pragma unroll
                for (int x = 0; x < 32; x += 2) {
                    uint64_t v = fmul2(pk2(r0[x], r0[x + 1]), f0x2);
                    if (has1) v = ffma2(pk2(r1[x], r1[x + 1]), f1x2, v);
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
            if (grp == 0 && a.lse_out != nullptr) {
                const float lse = (M + __log2f(Lsum)) * 0.69314718055994531f;
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

template <int BK, int D, int kEmuE = kEmuEvery>
cudaError_t launch_t(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                     const CUtensorMap& tv, int grid, cudaStream_t s) {
    auto kern = sparse_attn_kernel<BK, D, kEmuE>;
    const int smem = AttnSmem<BK, D>::kAlloc;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(a, tq, tk, tv);
    return cudaGetLastError();
}

}  // namespace

cudaError_t set_attn_trace(void* buf, int mode) {
    (void)mode;
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    return cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
}

cudaError_t launch_attn(const AttnArgs& a, int head_dim, const CUtensorMap& tq,
                        const CUtensorMap& tk, const CUtensorMap& tv, int grid, cudaStream_t s) {
    // block 64 only: block 128 layouts run attn5.cu / attn_rect.cu (csa_sparse_attn_fwd)
    if (a.g.B == 64 && head_dim == 128) return launch_t<64, 128>(a, tq, tk, tv, grid, s);
    if (a.g.B == 64 && head_dim == 64) return launch_t<64, 64>(a, tq, tk, tv, grid, s);
    return cudaErrorInvalidValue;
}

}  // namespace csa
