// attn.cu -- a7 + a8: calibrated block-sparse attention forward on sm_100a.
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
//   warp 0      scheduler + producer: claims items (dynamic, head-major work list) through a
//               4-deep shared-memory item ring; loads the Q tile (TMA, or an in-warp gather of
//               anchor rows), then the kept K/V tiles of the item's block list through a FIFO ring
//               of smem slots in MMA consumption order K0 K1 K2 V0 K3 V1 ... V_{n-1}.
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into TMEM S[j&1]; S_{j+2} is issued as
//               soon as the softmax warps have read S_j; O += P_j V_j with P_j read from TMEM
//               buffer P[j&1] (TS-MMA).  TMEM: S0 S1 | P0 P1 | O  (2BK + BK + D <= 512 columns).
//   warp 2      TMEM allocator.
//   warps 4-11  softmax: one query row (TMEM lane) per thread; warps 4-7 take the first half of
//               the tile's key columns, warps 8-11 the second half.  exp2 is taken against the
//               running max speculatively; the two halves agree on the tile max through shared
//               memory once per tile and, in the rare case it exceeds the running max by more
//               than 2^8, redo the tile with the new max and rescale O (lazy rescale).
// Packed f32x2 FMA/ADD; a fixed fraction of the exp2 are evaluated by a degree-3 polynomial on
// the FMA pipe to offload the MUFU unit.
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

constexpr int kThreads = 384;
constexpr int kItemSlots = 4;

template <int BK, int D>
struct AttnSmem {
    using C = TileCfg<BK, D>;
    static constexpr int kQOff = 0;
    static constexpr int kKVOff = 2 * C::kQBytes;
    static constexpr int kBudget = 224 * 1024 - kKVOff;
    static constexpr int kSlots = kBudget / C::kKVBytes > 8 ? 8 : kBudget / C::kKVBytes;
    static constexpr int kBarOff = kKVOff + kSlots * C::kKVBytes;
    // q_full[2] q_empty[2] kv_full[S] kv_empty[S] s_full[2] s_free[2] p_full[2] p_empty[2]
    // o_full o_empty item_full[4] item_empty[4]
    static constexpr int kNumBars = 4 + 2 * kSlots + 8 + 2 + 2 * kItemSlots;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;  // hmax[parity][half][128]
    static constexpr int kItemOff = kRowOff + 4 * 128 * 4;  // int32 [kItemSlots]
    static constexpr int kTmemPtrOff = kItemOff + kItemSlots * 4;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static constexpr int kAlloc = kBytes;  // base is 1 KiB aligned (__align__ on the extern)
    static_assert(kSlots >= 4, "K/V ring too shallow");
    static_assert(kAlloc <= 232448, "smem");
    // TMEM columns
    static constexpr uint32_t kS = 0;           // S0 at 0, S1 at BK
    static constexpr uint32_t kP = 2 * BK;      // P0 at 2BK, P1 at 2BK + BK/2
    static constexpr uint32_t kO = 3 * BK;      // O: D columns
    static_assert(3 * BK + D <= 512, "TMEM");
};

using namespace attn;

// Debug timeline (csa_debug_trace): clock64 stamps of CTA 0's pipeline events; nullptr = off.
static __device__ unsigned long long* g_trace;
static __device__ int g_debug_mode;  // 0 normal; != 0 pipeline measurements (no softmax work)

template <int BK, int D>
__global__ void __launch_bounds__(kThreads, 1)
    sparse_attn_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                       const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv) {
    using C = TileCfg<BK, D>;
    using L = AttnSmem<BK, D>;
    constexpr int S = L::kSlots;
    constexpr int HC = BK / 2;  // columns per softmax thread
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();  // SWIZZLE_128B atoms need 1 KiB alignment
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 2;
    uint64_t* kv_full = bars + 4;
    uint64_t* kv_empty = bars + 4 + S;
    uint64_t* s_full = bars + 4 + 2 * S;
    uint64_t* s_free = s_full + 2;
    uint64_t* p_full = s_full + 4;
    uint64_t* p_empty = s_full + 6;
    uint64_t* o_full = s_full + 8;
    uint64_t* o_empty = s_full + 9;
    uint64_t* item_full = s_full + 10;
    uint64_t* item_empty = item_full + kItemSlots;
    float* hmax = reinterpret_cast<float*>(smem + L::kRowOff);  // [parity][half][128]
    volatile int32_t* item_slot = reinterpret_cast<int32_t*>(smem + L::kItemOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full + i, 1);
            mbar_init(q_empty + i, 1);
            mbar_init(s_full + i, 1);
            mbar_init(s_free + i, 8);
            mbar_init(p_full + i, 8);
            mbar_init(p_empty + i, 1);
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
            // -------------------------------------------------------- scheduler + producer
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
                        tma_tile<D>(qdst, C::kQBox, &tq, q_full + qb, it.h, it.idx * BK, it.b,
                                    pol_q);
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
                // K/V tiles in MMA consumption order: K0 K1, then per j: K_{j+2} (if any), V_j
                if (lane == 0) {
                    auto load = [&](const CUtensorMap* map, int32_t j) {
                        const uint32_t slot = ld % S, ph = (ld / S) & 1;
                        ++ld;
                        mbar_wait(kv_empty + slot, ph ^ 1);
                        mbar_arrive_expect_tx(kv_full + slot, C::kKVBytes);
                        tma_tile<D>(smem + L::kKVOff + slot * C::kKVBytes, C::kKBox, map,
                                    kv_full + slot, it.h, tl.at(j) * BK, it.b, pol_kv);
                    };
                    for (int32_t j = 0; j < tl.n && j < 2; ++j) load(&tk, j);
                    for (int32_t j = 0; j < tl.n; ++j) {
                        if (j + 2 < tl.n) load(&tk, j + 2);
                        load(&tv, j);
                    }
                }
                __syncwarp();
            }
        } else if (warp == 1) {
            // ---------------------------------------------------------------- MMA issuer
            if (lane == 0) {
                uint32_t cons = 0;   // K/V ring position consumed
                uint32_t gbase = 0;  // tiles of earlier items: tile j of this item is global
                                     // tile gbase + j, buffer (gbase + j) & 1, use (..) >> 1
                int32_t ntr_s = 0, ntr_pv = 0;  // trace counters (debug timeline only)
                const uint32_t q_base = smem_u32(smem + L::kQOff);
                const uint32_t kv_base = smem_u32(smem + L::kKVOff);
                for (int32_t local = 0;; ++local) {
                    const int32_t item = next_item(local, false);
                    if (item < 0) break;
                    const Item it = decode_item(a, item);
                    const TileList tl = tile_list(a, it);
                    const int32_t n = tl.n;
                    const int qb = local & 1;
                    mbar_wait(q_full + qb, (local >> 1) & 1);
                    const uint32_t q_smem = q_base + qb * C::kQBytes;
                    if (n == 0) {  // corrupt plan (empty MASK row): release Q, no tiles
                        mma_commit(q_empty + qb);
                        mma_commit(o_full);
                        continue;
                    }
                    auto do_s = [&](int32_t j) {
                        const uint32_t gj = gbase + (uint32_t)j;
                        const int b = gj & 1;
                        const uint32_t use = gj >> 1;
                        if (use > 0) mbar_wait(s_free + b, (use - 1) & 1);
                        const uint32_t slot = cons % S, ph = (cons / S) & 1;
                        ++cons;
                        mbar_wait(kv_full + slot, ph);
                        tc_fence_after();
                        CSA_TRACE(2, ntr_s, 0);
                        ++ntr_s;
                        issue_qk<BK, D>(tmem + L::kS + b * BK, q_smem,
                                        kv_base + slot * C::kKVBytes,
                                        (g_debug_mode == 7 || g_debug_mode == 8) ? 1 : D / 16);
                        mma_commit(s_full + b);
                        mma_commit(kv_empty + slot);
                        if (j == n - 1) mma_commit(q_empty + qb);
                    };
                    auto do_pv = [&](int32_t j) {
                        const uint32_t gj = gbase + (uint32_t)j;
                        const int b = gj & 1;
                        CSA_TRACE(3, ntr_pv, 0);
                        mbar_wait(p_full + b, (gj >> 1) & 1);
                        CSA_TRACE(3, ntr_pv, 1);
                        ++ntr_pv;
                        if (j == 0) mbar_wait(o_empty, (local & 1) ^ 1);  // epilogue of last item
                        const uint32_t slot = cons % S, ph = (cons / S) & 1;
                        ++cons;
                        mbar_wait(kv_full + slot, ph);
                        tc_fence_after();
                        issue_pv<BK, D>(tmem + L::kO, tmem + L::kP + b * (BK / 2),
                                        kv_base + slot * C::kKVBytes, j > 0,
                                        (g_debug_mode == 6 || g_debug_mode == 8) ? 1 : BK / 16);
                        mma_commit(kv_empty + slot);
                        mma_commit(p_empty + b);
                    };
                    for (int32_t j = 0; j < n && j < 2; ++j) do_s(j);
                    for (int32_t j = 0; j < n; ++j) {
                        if (j + 2 < n) do_s(j + 2);
                        do_pv(j);
                    }
                    mma_commit(o_full);
                    gbase += (uint32_t)n;
                }
            }
            __syncwarp();
        }
    } else {
        set_maxnreg_inc224();
        // ------------------------------------------------------------------ softmax warps
        const int half = (warp - 4) >> 2;  // key-column half of every tile
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const float sl2 = a.scale_log2;
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;  // keys in the last (ragged) block
        uint32_t tcount = 0;  // tiles processed (s_full / p phases, hmax parity)
        for (int32_t local = 0;; ++local) {
            const int32_t item = next_item(local, true);
            if (item < 0) break;
            const Item it = decode_item(a, item);
            const TileList tl = tile_list(a, it);
            // only the last listed tile can be the ragged block N_B - 1
            const bool last_ragged = tail_valid < BK && tl.n > 0 && tl.at(tl.n - 1) == g.NB - 1;
            float m_run = -INFINITY, l_run = 0.0f;
            for (int32_t j = 0; j < tl.n; ++j, ++tcount) {
                const int b = tcount & 1;          // S / P buffer of this (global) tile
                const uint32_t use = tcount >> 1;  // earlier uses of buffer b
                mbar_wait(s_full + b, use & 1);
                const bool tr = (quarter == 0 && lane == 0);
                if (tr) CSA_TRACE(half, tcount, 0);
                if (g_debug_mode != 0) {  // debug: pipeline without softmax work
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(s_free + b);
                    if (use > 0) mbar_wait(p_empty + b, (use - 1) & 1);  // no phase overrun
                    if (lane == 0) mbar_arrive(p_full + b);
                    continue;
                }
                tc_fence_after();
                uint32_t r[HC];
                tmem_load_half<HC>(lane_addr + L::kS + b * BK + half * HC, r);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_free + b);  // S[b] may be overwritten now
                if (tr) CSA_TRACE(half, tcount, 1);
                if (last_ragged && j == tl.n - 1) {
#pragma unroll
                    for (int x = 0; x < HC; ++x)
                        if (half * HC + x >= tail_valid) r[x] = 0xff800000u;  // -inf
                }
                float* hm = hmax + (tcount & 1) * 256;
                uint32_t pk[HC / 2];
                float lsum;
                bool redo = false;
                float m_tile;
                if (j == 0) {
                    // first tile: agree on the tile max before exponentiating
                    hm[half * 128 + row] = max_half<HC>(r);
                    named_bar_sync(1, 256);
                    m_tile = fmaxf(hm[row], hm[128 + row]) * sl2;
                    m_run = m_tile;
                    lsum = exp_half<HC>(r, sl2, m_run, pk);
                } else {
                    // speculative: exponentiate against the running max, then agree on the max
                    lsum = exp_half<HC>(r, sl2, m_run, pk);
                    hm[half * 128 + row] = max_half<HC>(r);
                    named_bar_sync(1, 256);
                    m_tile = fmaxf(hm[row], hm[128 + row]) * sl2;
                    redo = m_tile > m_run + kRescaleThreshold;  // same decision in both halves
                }
                if (tr) CSA_TRACE(half, tcount, 2);
                // P[b] and O may be written once the P.V that last read P[b] has completed
                if (use > 0) mbar_wait(p_empty + b, (use - 1) & 1);
                if (redo) {  // rare: new max -> rescale O (after every earlier P.V) and redo P
                    mbar_wait(p_empty + (b ^ 1), ((tcount - 1) >> 1) & 1);  // P.V of tile j-1
                    tc_fence_after();
                    const float alpha = ex2_approx(m_run - m_tile);
                    l_run *= alpha;
                    m_run = m_tile;
                    lsum = exp_half<HC>(r, sl2, m_run, pk);
                    const uint64_t al2 = f2(alpha, alpha);
#pragma unroll
                    for (int c = 0; c < D / 2; c += 32) {
                        uint32_t o[32];
                        const uint32_t oa = lane_addr + L::kO + half * (D / 2) + c;
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
                l_run += lsum;
                tmem_store_p<HC>(lane_addr + L::kP + b * (BK / 2) + half * (HC / 2), pk);
                tmem_st_wait();
                if (tr) CSA_TRACE(half, tcount, 3);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + b);
                if (tr) CSA_TRACE(half, tcount, 4);
            }
            // -------------------------------------------------------------- epilogue
            mbar_wait(o_full, local & 1);
            tc_fence_after();
            // row sums of the two halves; uses the hmax slot the last tile did not use
            float* row_l = hmax + (tcount & 1) * 256;
            row_l[half * 128 + row] = l_run;
            named_bar_sync(1, 256);
            const float inv = 1.0f / (row_l[row] + row_l[128 + row]);
            const float Lsum = row_l[row] + row_l[128 + row];
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
            const uint64_t inv2 = f2(inv, inv);
#pragma unroll
            for (int c = 0; c < D / 2; c += 32) {
                const int col = half * (D / 2) + c;
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
            named_bar_sync(1, 256);  // row_l reused by the next item's epilogue
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

template <int BK, int D>
cudaError_t launch_t(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                     const CUtensorMap& tv, int grid, cudaStream_t s) {
    auto kern = sparse_attn_kernel<BK, D>;
    const int smem = AttnSmem<BK, D>::kAlloc;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(a, tq, tk, tv);
    return cudaGetLastError();
}

}  // namespace

cudaError_t set_attn_trace(void* buf, int mode) {
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    cudaError_t e = cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(g_debug_mode, &mode, sizeof(mode));
}

cudaError_t launch_attn(const AttnArgs& a, int head_dim, const CUtensorMap& tq,
                        const CUtensorMap& tk, const CUtensorMap& tv, int grid, cudaStream_t s) {
    if (a.g.B == 128 && head_dim == 128) return launch_t<128, 128>(a, tq, tk, tv, grid, s);
    if (a.g.B == 128 && head_dim == 64) return launch_t<128, 64>(a, tq, tk, tv, grid, s);
    if (a.g.B == 64 && head_dim == 128) return launch_t<64, 128>(a, tq, tk, tv, grid, s);
    if (a.g.B == 64 && head_dim == 64) return launch_t<64, 64>(a, tq, tk, tv, grid, s);
    return cudaErrorInvalidValue;
}

}  // namespace csa
