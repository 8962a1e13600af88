// attn2.cu -- a7 + a8 on CTA pairs (cta_group::2): the B = 128, head_dim = 128 production path.
//
// Same mathematics as attn.cu (readings Q1, Q2, Q9, Q10): every
// query row attends, with an online softmax, to exactly the keys of its own kept blocks.
//
// Why pairs: one CTA per 128-row query block streams 64 KB of K/V through TMA and reads 96 KB of
// operands from shared memory per 128x128 tile, which bounds the tensor pipe well below peak
// (measured).  Here a cluster of two CTAs on one TPC processes two adjacent
// query blocks r0 = 2p, r1 = 2p + 1 of the same head with M = 256 tcgen05 MMAs: CTA rank q holds
// the Q rows of block 2p + q and HALF of every K tile (keys 64q..64q+63) and V tile (head-dim
// columns 64q..64q+63), so each SM moves half the K/V bytes.  The pair walks the union of the two
// rows' kept-block lists (ascending); a row whose own list lacks a union tile contributes P = 0
// for it (exactly nothing), so each row's result is its own masked softmax.
//
// Roles per CTA (12 warps): warp 0 producer (own Q, own K/V halves; completion counted on the
// leader's barriers), warp 1 MMA issuer (leader CTA only), warp 2 TMEM allocator (both CTAs),
// warps 4-11 softmax on the CTA's own 128 rows (column halves, as in attn.cu).  The follower's
// softmax warps arrive on the leader's barriers remotely; the leader's commits are multicast.
#include <cstdint>

#include "attn_common.cuh"

namespace csa {
namespace {

using namespace attn;

constexpr int kThreads2 = 384;
static __device__ unsigned long long* g_trace;
static __device__ int g_debug_mode;

template <int D>
struct PairSmem {
    static constexpr int BK = 128;
    static constexpr int kQBox = 128 * 128;                  // [128 rows][64 cols] bf16
    static constexpr int kQBytes = (D / 64) * kQBox;         // own 128 query rows
    static constexpr int kKHalfBox = 64 * 128;               // [64 keys][64 cols]
    static constexpr int kSlotBytes = 16384;                 // K half (64 keys x 128) or V half
    static constexpr int kQOff = 0;
    static constexpr int kKVOff = 2 * kQBytes;
    static constexpr int kSlots = (224 * 1024 - kKVOff) / kSlotBytes > 12
                                      ? 12 : (224 * 1024 - kKVOff) / kSlotBytes;
    static constexpr int kBarOff = kKVOff + kSlots * kSlotBytes;
    // q_full[2] q_empty[2] kv_full[S] kv_empty[S] s_full[2] s_free[2] p_full[2] p_empty[2]
    // o_full o_empty
    static constexpr int kNumBars = 4 + 2 * kSlots + 8 + 2;
    static constexpr int kRowOff = kBarOff + kNumBars * 8;  // hmax[parity][half][128]
    static constexpr int kTmemPtrOff = kRowOff + 4 * 128 * 4;
    static constexpr int kBytes = kTmemPtrOff + 16;
    static_assert(D == 128, "pair kernel: head_dim 128 (V halves are full 128-byte rows)");
    static_assert(kBytes <= 232448, "smem");
    // TMEM columns (per CTA, own 128 rows): S0 S1 | P0 P1 | O
    static constexpr uint32_t kS = 0, kP = 2 * BK, kO = 3 * BK;
    // M = 256 (pair), N = 128 keys (QK) / N = D (PV)
    static constexpr uint32_t kIdescQK = umma_idesc_bf16(256, 128, 0, 0);
    static constexpr uint32_t kIdescPV = umma_idesc_bf16(256, D, 0, 1);
};

struct PairItem {
    uint32_t kind;
    int32_t h, p, b;
    int64_t cell;
};

__device__ __forceinline__ PairItem decode_pair(const AttnArgs& a, int32_t item) {
    const uint32_t code = a.work_list[item / a.batch];
    PairItem it;
    it.kind = code >> 31;
    it.h = (int32_t)((code >> 20) & 0x7FFu);
    it.p = (int32_t)(code & 0xFFFFFu);
    it.b = item % a.batch;
    it.cell = a.cell_base + it.h;
    return it;
}

// Kept-tile list of one member of the pair (row 2p + q); empty when that row does not exist.
__device__ __forceinline__ TileList member_list(const AttnArgs& a, const PairItem& it, int q) {
    TileList t;
    if (it.kind) {  // REPETITIVE: anchor tiles u = 2p + q, dense over all key blocks
        const int32_t kA = a.plan.anchor_k[it.cell];
        const int32_t n_tiles = (int32_t)(((int64_t)a.g.F * kA * a.g.W + 127) / 128);
        t.idx = nullptr;
        t.n = (2 * it.p + q < n_tiles) ? a.g.NB : 0;
        return t;
    }
    const int32_t r = 2 * it.p + q;
    if (r >= a.g.NB) {
        t.idx = nullptr;
        t.n = 0;
        return t;
    }
    const int32_t* rp = a.plan.blk_row_ptr + it.cell * (a.g.NB + 1);
    const int32_t r0 = rp[r], r1 = rp[r + 1];
    t.idx = a.plan.blk_idx + a.plan.blk_base[it.cell] + r0;
    t.n = r1 - r0;
    return t;
}

// Sequential walk over the ascending union of two kept-tile lists.
struct UnionIter {
    TileList l0, l1;
    int32_t i0, i1;
    __device__ __forceinline__ void init(const TileList& a, const TileList& b) {
        l0 = a;
        l1 = b;
        i0 = 0;
        i1 = 0;
    }
    // next union element c, with membership flags
    __device__ __forceinline__ int32_t next(bool& in0, bool& in1) {
        const int32_t c0 = i0 < l0.n ? l0.at(i0) : 0x7fffffff;
        const int32_t c1 = i1 < l1.n ? l1.at(i1) : 0x7fffffff;
        const int32_t c = c0 < c1 ? c0 : c1;
        in0 = (c0 == c);
        in1 = (c1 == c);
        i0 += in0;
        i1 += in1;
        return c;
    }
};

__device__ __forceinline__ int32_t union_size(const TileList& a, const TileList& b) {
    if (a.idx == nullptr || b.idx == nullptr) return a.n > b.n ? a.n : b.n;  // dense or empty
    int32_t i = 0, j = 0, n = 0;
    while (i < a.n && j < b.n) {
        const int32_t x = a.idx[i], y = b.idx[j];
        i += (x <= y);
        j += (y <= x);
        ++n;
    }
    return n + (a.n - i) + (b.n - j);
}

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    sparse_attn_pair_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tq,
                            const __grid_constant__ CUtensorMap tk_half,
                            const __grid_constant__ CUtensorMap tv) {
    using L = PairSmem<D>;
    constexpr int BK = 128;
    constexpr int S = L::kSlots;
    constexpr int SK = S / 2, SV = S - SK;  // K-half ring slots, V-half ring slots
    constexpr int HC = BK / 2;
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
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
    float* hmax = reinterpret_cast<float*>(smem + L::kRowOff);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);

    const uint32_t warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the pair's MMAs)
    // leader-CTA (shared::cluster) addresses of the barriers both CTAs arrive on
    auto lead = [&](uint64_t* bar) { return mapa_shared(smem_u32(bar), 0); };

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full + i, 2);   // one arrive (+tx) per CTA
            mbar_init(q_empty + i, 1);
            mbar_init(s_full + i, 1);
            mbar_init(s_free + i, 16);  // 8 softmax warps x 2 CTAs
            mbar_init(p_full + i, 16);
            mbar_init(p_empty + i, 1);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(kv_full + i, 2);
            mbar_init(kv_empty + i, 1);
        }
        mbar_init(o_full, 1);
        mbar_init(o_empty, 16);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair<512>(tmem_ptr);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tq);
        tma_prefetch(&tk_half);
        tma_prefetch(&tv);
    }
    tc_fence_before();
    cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
    tc_fence_after();
    const uint32_t tmem = *tmem_ptr;

    const int32_t n_items = (*a.n_work) * a.batch;
    const int32_t cl = (int32_t)(blockIdx.x >> 1), ncl = (int32_t)(gridDim.x >> 1);
    const Geo& g = a.g;

    if (warp < 4) {
        set_maxnreg_dec56();
        if (warp == 0) {
            // ------------------------------------------------------------------- producer
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_kv = policy_evict_last();
            uint32_t ldk = 0, ldv = 0;  // loads issued into the K ring / the V ring
            int32_t local = 0;
            for (int32_t item = cl; item < n_items; item += ncl, ++local) {
                const PairItem it = decode_pair(a, item);
                const TileList l0 = member_list(a, it, 0), l1 = member_list(a, it, 1);
                const TileList mine = rank ? l1 : l0;
                const int qb = local & 1;
                uint8_t* qdst = smem + L::kQOff + qb * L::kQBytes;
                mbar_wait(q_empty + qb, ((local >> 1) & 1) ^ 1);
                if (it.kind == 0) {
                    if (lane == 0) {
                        if (mine.n > 0) {
                            mbar_arrive_expect_tx_cluster(lead(q_full + qb), L::kQBytes);
#pragma unroll
                            for (int x = 0; x < D / 64; ++x)
                                tma_load_4d_pair(qdst + x * L::kQBox, &tq, lead(q_full + qb),
                                                 x * 64, it.h, (2 * it.p + (int)rank) * BK, it.b,
                                                 pol_q);
                        } else {
                            mbar_arrive_cluster(lead(q_full + qb));  // no rows: Q unused
                        }
                    }
                } else {
                    const int32_t kA = a.plan.anchor_k[it.cell];
                    const int32_t per_frame = kA * g.W;
                    const int32_t n_anchor = g.F * per_frame;
                    const int32_t u = 2 * it.p + (int32_t)rank;
                    const __nv_bfloat16* qb_ptr =
                        a.q + (int64_t)it.b * a.q_sb + (int64_t)it.h * a.q_sh;
                    constexpr int kChunks = D / 8;
                    for (int x = lane; x < 128 * kChunks; x += 32) {
                        const int row = x / kChunks, ch = x % kChunks;
                        const int32_t gi = u * 128 + row;
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
                    fence_cluster();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(lead(q_full + qb));
                }
                {  // whole warp walks the union (uniform values); one elected lane issues
                    const int32_t n = union_size(l0, l1);
                    UnionIter ik, iv;
                    ik.init(l0, l1);
                    iv.init(l0, l1);
                    auto load = [&](bool is_k) {
                        bool in0, in1;
                        const int32_t c = is_k ? ik.next(in0, in1) : iv.next(in0, in1);
                        uint32_t slot, ph;
                        if (is_k) {
                            slot = ldk % SK;
                            ph = (ldk / SK) & 1;
                            ++ldk;
                        } else {
                            slot = SK + ldv % SV;
                            ph = (ldv / SV) & 1;
                            ++ldv;
                        }
                        mbar_wait(kv_empty + slot, ph ^ 1);
                        if (elect_one()) {
                            uint8_t* dst = smem + L::kKVOff + slot * L::kSlotBytes;
                            const uint32_t fb = lead(kv_full + slot);
                            mbar_arrive_expect_tx_cluster(fb, L::kSlotBytes);
                            if (is_k) {  // keys 64*rank .. +63 of block c, all D columns
#pragma unroll
                                for (int x = 0; x < D / 64; ++x)
                                    tma_load_4d_pair(dst + x * L::kKHalfBox, &tk_half, fb, x * 64,
                                                     it.h, c * BK + 64 * (int)rank, it.b, pol_kv);
                            } else {     // all 128 keys of block c, columns 64*rank .. +63
                                tma_load_4d_pair(dst, &tv, fb, 64 * (int)rank, it.h, c * BK,
                                                 it.b, pol_kv);
                            }
                        }
                        __syncwarp();
                    };
                    for (int32_t j = 0; j < n && j < 2; ++j) load(true);
                    for (int32_t j = 0; j < n; ++j) {
                        if (j + 2 < n) load(true);
                        load(false);
                    }
                }
                __syncwarp();
            }
        } else if ((warp == 1 || warp == 3) && rank == 0) {
            // ------------------------------------------- MMA issuers (leader CTA): warp 1 issues
            // every S = Q K^T, warp 3 every O += P V, each in order from its own ring of K or V
            // halves, so neither stream's waits stall the other (tcgen05.commit tracks the
            // issuing thread's own MMAs).
            const bool s_issuer = (warp == 1);
            {  // whole warp in the loop, one elected lane issues
                uint32_t cons = 0, gbase = 0;
                int32_t local = 0;
                const uint32_t q_base = smem_u32(smem + L::kQOff);
                const uint32_t kv_base = smem_u32(smem + L::kKVOff);
                for (int32_t item = cl; item < n_items; item += ncl, ++local) {
                    const PairItem it = decode_pair(a, item);
                    const int32_t n = union_size(member_list(a, it, 0), member_list(a, it, 1));
                    const int qb = local & 1;
                    if (s_issuer) {
                        mbar_wait(q_full + qb, (local >> 1) & 1);
                        const uint32_t q_smem = q_base + qb * L::kQBytes;
                        if (n == 0) {
                            if (elect_one()) mma_commit_pair(q_empty + qb);
                            __syncwarp();
                        }
                        for (int32_t j = 0; j < n; ++j) {
                            const uint32_t gj = gbase + (uint32_t)j;
                            const int b = gj & 1;
                            const uint32_t use = gj >> 1;
                            if (lane == 0) CSA_TRACE(2, gj, 0);
                            if (use > 0) mbar_wait(s_free + b, (use - 1) & 1);
                            if (lane == 0) CSA_TRACE(2, gj, 1);
                            const uint32_t slot = cons % SK, ph = (cons / SK) & 1;
                            ++cons;
                            mbar_wait(kv_full + slot, ph);
                            if (lane == 0) CSA_TRACE(2, gj, 2);
                            tc_fence_after();
                            const uint32_t k_smem = kv_base + slot * L::kSlotBytes;
                            if (elect_one()) {
#pragma unroll
                                for (int kk = 0; kk < D / 16; ++kk) {
                                    const uint32_t off = (kk & 3) * 32;
                                    const uint64_t ad = umma_desc_sw128(
                                        q_smem + (kk >> 2) * L::kQBox + off, 16, 1024);
                                    const uint64_t bd = umma_desc_sw128(
                                        k_smem + (kk >> 2) * L::kKHalfBox + off, 16, 1024);
                                    mma_ss_pair(tmem + L::kS + b * BK, ad, bd, L::kIdescQK,
                                                kk > 0);
                                }
                                mma_commit_pair(s_full + b);
                                mma_commit_pair(kv_empty + slot);
                                if (j == n - 1) mma_commit_pair(q_empty + qb);
                            }
                            __syncwarp();
                            if (lane == 0) CSA_TRACE(2, gj, 3);
                        }
                    } else {
                        for (int32_t j = 0; j < n; ++j) {
                            const uint32_t gj = gbase + (uint32_t)j;
                            const int b = gj & 1;
                            if (lane == 0) CSA_TRACE(3, gj, 0);
                            mbar_wait(p_full + b, (gj >> 1) & 1);
                            if (lane == 0) CSA_TRACE(3, gj, 1);
                            if (j == 0) mbar_wait(o_empty, (local & 1) ^ 1);
                            const uint32_t slot = SK + cons % SV, ph = (cons / SV) & 1;
                            ++cons;
                            mbar_wait(kv_full + slot, ph);
                            if (lane == 0) CSA_TRACE(3, gj, 2);
                            tc_fence_after();
                            const uint32_t v_smem = kv_base + slot * L::kSlotBytes;
                            if (elect_one()) {
#pragma unroll
                                for (int kk = 0; kk < BK / 16; ++kk) {
                                    const uint64_t bd =
                                        umma_desc_sw128(v_smem + kk * 16 * 128, 16384, 1024);
                                    mma_ts_pair(tmem + L::kO, tmem + L::kP + b * (BK / 2) + kk * 8,
                                                bd, L::kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
                                }
                                mma_commit_pair(kv_empty + slot);
                                mma_commit_pair(p_empty + b);
                            }
                            __syncwarp();
                            if (lane == 0) CSA_TRACE(3, gj, 3);
                        }
                        if (elect_one()) mma_commit_pair(o_full);
                        __syncwarp();
                    }
                    gbase += (uint32_t)n;
                }
            }
            __syncwarp();
        }
    } else {
        set_maxnreg_inc224();
        // ------------------------------------------------------------- softmax (own rows)
        const int half = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const float sl2 = a.scale_log2;
        const int32_t tail_valid = g.N - (g.NB - 1) * BK;
        const uint32_t lf_free[2] = {lead(s_free), lead(s_free + 1)};
        const uint32_t lf_pful[2] = {lead(p_full), lead(p_full + 1)};
        const uint32_t l_oempty = lead(o_empty);
        uint32_t tcount = 0;
        int32_t local = 0;
        for (int32_t item = cl; item < n_items; item += ncl, ++local) {
            const PairItem it = decode_pair(a, item);
            const TileList l0 = member_list(a, it, 0), l1 = member_list(a, it, 1);
            const int32_t n = union_size(l0, l1);
            UnionIter iu;
            iu.init(l0, l1);
            float m_run = -INFINITY, l_run = 0.0f;
            int32_t mine = 0;
            for (int32_t j = 0; j < n; ++j, ++tcount) {
                bool in0, in1;
                const int32_t c = iu.next(in0, in1);
                const bool in_me = rank ? in1 : in0;
                const int b = tcount & 1;
                const uint32_t use = tcount >> 1;
                mbar_wait(s_full + b, use & 1);
                const bool tr = (quarter == 0 && lane == 0);
                if (tr) CSA_TRACE(half, tcount, 0);
                tc_fence_after();
                uint32_t pk[HC / 2];
                float lsum = 0.0f;
                bool redo = false;
                float m_tile = 0.0f;
                if (!in_me || g_debug_mode != 0) {
                    // this row does not keep block c: P = 0 for it (S is not even read)
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(lf_free[b]);
#pragma unroll
                    for (int x = 0; x < HC / 2; ++x) pk[x] = 0u;
                } else {
                    uint32_t r[HC];
                    tmem_load_half<HC>(lane_addr + L::kS + b * BK + half * HC, r);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(lf_free[b]);
                    if (c == g.NB - 1 && tail_valid < BK) {
#pragma unroll
                        for (int x = 0; x < HC; ++x)
                            if (half * HC + x >= tail_valid) r[x] = 0xff800000u;  // -inf
                    }
                    float* hm = hmax + (tcount & 1) * 256;
                    if (mine == 0) {
                        hm[half * 128 + row] = max_half<HC>(r);
                        named_bar_sync(1, 256);
                        m_tile = fmaxf(hm[row], hm[128 + row]) * sl2;
                        m_run = m_tile;
                        lsum = exp_half<HC>(r, sl2, m_run, pk);
                    } else {
                        lsum = exp_half<HC>(r, sl2, m_run, pk);
                        hm[half * 128 + row] = max_half<HC>(r);
                        named_bar_sync(1, 256);
                        m_tile = fmaxf(hm[row], hm[128 + row]) * sl2;
                        // warp-uniform decision: the O rescale uses warp-collective tcgen05 ops
                        const bool need = m_tile > m_run + kRescaleThreshold;
                        redo = __any_sync(0xffffffffu, need);
                        if (!need) m_tile = m_run;  // alpha = 1 for rows that need no rescale
                    }
                    ++mine;
                    if (redo) {
                        // every earlier P.V (the previous union tile's) must have completed
                        mbar_wait(p_empty + (b ^ 1), ((tcount - 1) >> 1) & 1);
                        tc_fence_after();
                        const float alpha = ex2_approx(m_run - m_tile);
                        l_run *= alpha;
                        m_run = m_tile;
                        lsum = exp_half<HC>(r, sl2, m_run, pk);
                        const uint64_t al2 = f2(alpha, alpha);
#pragma unroll
                        for (int cc = 0; cc < D / 2; cc += 32) {
                            uint32_t o[32];
                            const uint32_t oa = lane_addr + L::kO + half * (D / 2) + cc;
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
                if (use > 0) mbar_wait(p_empty + b, (use - 1) & 1);
                tmem_store_p<HC>(lane_addr + L::kP + b * (BK / 2) + half * (HC / 2), pk);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(lf_pful[b]);
                if (tr) CSA_TRACE(half, tcount, 4);
            }
            // -------------------------------------------------------------- epilogue
            mbar_wait(o_full, local & 1);
            tc_fence_after();
            float* row_l = hmax + (tcount & 1) * 256;
            row_l[half * 128 + row] = l_run;
            named_bar_sync(1, 256);
            const float Lsum = row_l[row] + row_l[128 + row];
            const float inv = 1.0f / Lsum;
            int64_t tok0 = -1;
            int32_t n_dst = 0, dst_stride_rows = 0;
            if (it.kind == 0) {
                const int32_t r = 2 * it.p + (int32_t)rank;
                const int64_t t = (int64_t)r * BK + row;
                if (r < g.NB && t < g.N) {
                    tok0 = t;
                    n_dst = 1;
                }
            } else {
                const int32_t kA = a.plan.anchor_k[it.cell];
                const int32_t per_frame = kA * g.W;
                const int32_t gi = (2 * it.p + (int32_t)rank) * 128 + row;
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
            for (int cc = 0; cc < D / 2; cc += 32) {
                const int col = half * (D / 2) + cc;
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
            named_bar_sync(1, 256);
            if (lane == 0) mbar_arrive_cluster(l_oempty);
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the leader's last MMAs into this CTA's TMEM are complete
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem);
    }
}

}  // namespace

cudaError_t set_attn2_trace(void* buf, int mode) {
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    cudaError_t e = cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(g_debug_mode, &mode, sizeof(mode));
}

cudaError_t launch_attn_pair(const AttnArgs& a, int head_dim, const CUtensorMap& tq,
                             const CUtensorMap& tk_half, const CUtensorMap& tv, int grid,
                             cudaStream_t s) {
    if (a.g.B != 128 || head_dim != 128) return cudaErrorInvalidValue;
    auto kern = sparse_attn_pair_kernel<128>;
    const int smem = PairSmem<128>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    grid &= ~1;
    if (grid < 2) grid = 2;
    kern<<<grid, kThreads2, smem, s>>>(a, tq, tk_half, tv);
    return cudaGetLastError();
}

}  // namespace csa
