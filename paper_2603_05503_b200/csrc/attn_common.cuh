// attn_common.cuh -- device helpers shared by the attention kernels (attn.cu: one CTA per query
// block; attn2.cu: CTA pairs, cta_group::2): work-item decoding, kept-tile lists, packed fp32
// arithmetic, the polynomial exp2, the per-thread softmax pieces and the debug timeline hooks.
#pragma once
#include <cstdint>

#include "csa_internal.cuh"
#include "tiles.cuh"

namespace csa {
namespace attn {

constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kEmuPerOctet = 3;            // element pairs p with (p & 7) >= 8 - this -> poly exp2

struct Item {
    uint32_t kind;  // 0 MASK, 1 REPETITIVE
    int32_t h, idx, b;
    int64_t cell;
};

__device__ __forceinline__ Item decode_item(const AttnArgs& a, int32_t item) {
    const uint32_t code = a.work_list[item / a.batch];
    Item it;
    it.kind = code >> 31;
    it.h = (int32_t)((code >> 20) & 0x7FFu);
    it.idx = (int32_t)(code & 0xFFFFFu);
    it.b = item % a.batch;
    it.cell = a.cell_base + it.h;
    return it;
}

// Kept key-block list of a MASK item, or all N_Bkv key blocks for a REPETITIVE item.  A MASK row
// is read from the CSR index list when the plan has one, else from its 1-D interval list
// ((start, end) pairs: the form the paper leaves its kernel for as future work) --
// an intervals-only plan drops the CSR index array (2 bytes per kept block).  The kernels walk
// a list sequentially with TileCursor; last() is the row's last kept block.
struct TileList {
    const uint16_t* idx;  // CSR indices; nullptr -> intervals (ivl) or dense 0..n-1 (ivl null)
    const uint16_t* ivl;  // (start, end) pairs when idx == nullptr
    int32_t n;            // kept tiles
    int32_t n_ivl;
    __device__ __forceinline__ int32_t last() const {
        return idx ? (int32_t)idx[n - 1] : ivl ? (int32_t)ivl[2 * n_ivl - 1] - 1 : n - 1;
    }
};

struct TileCursor {
    const uint16_t* idx;
    const uint16_t* ivl;
    int32_t k, c, e;
    __device__ __forceinline__ explicit TileCursor(const TileList& t)
        : idx(t.idx), ivl(t.ivl), k(0), c(0), e(0) {}
    __device__ __forceinline__ int32_t next() {
        if (idx) return (int32_t)idx[k++];
        if (!ivl) return k++;
        if (c == e) {
            c = ivl[2 * k];
            e = ivl[2 * k + 1];
            ++k;
        }
        return c++;
    }
};

__device__ __forceinline__ TileList tile_list(const AttnArgs& a, const Item& it) {
    TileList t;
    t.idx = nullptr;
    t.ivl = nullptr;
    t.n_ivl = 0;
    if (it.kind) {
        t.n = a.g.NBK;
    } else {
        const int32_t* rp = a.plan.blk_row_ptr + it.cell * (a.g.NB + 1);
        const int32_t r0 = rp[it.idx], r1 = rp[it.idx + 1];
        t.n = r1 - r0;
        if (a.plan.blk_idx != nullptr) {
            t.idx = a.plan.blk_idx + a.plan.blk_base[it.cell] + r0;
        } else {
            const int32_t* irp = a.plan.ivl_row_ptr + it.cell * (a.g.NB + 1);
            const int32_t i0 = irp[it.idx];
            t.ivl = a.plan.ivl + 2 * (a.plan.ivl_base[it.cell] + i0);
            t.n_ivl = irp[it.idx + 1] - i0;
        }
    }
    return t;
}

// Address of the output row of token tok (batch b, head h): the local O tensor, or -- output
// scatter -- the receive buffer of the rank that owns tok's sequence shard.
__device__ __forceinline__ __nv_bfloat16* out_row(const AttnArgs& a, int32_t b, int32_t h,
                                                  int64_t tok) {
    __nv_bfloat16* base = a.o;
    if (a.o_peer != nullptr) {
        const int64_t p = tok / a.o_peer_tokens;
        base = a.o_peer[p];
        tok -= p * a.o_peer_tokens;
    }
    return base + (int64_t)b * a.o_sb + (int64_t)h * a.o_sh + tok * a.o_sn;
}

__device__ __forceinline__ int32_t anchor_row(int32_t H, int32_t k, int32_t m) {
    return (int32_t)(((int64_t)(2 * m + 1) * H) / (2 * k));
}

// ------------------------------------------------------------------------ packed fp32 helpers
__device__ __forceinline__ uint64_t pk2(uint32_t lo, uint32_t hi) {
    return (uint64_t)lo | ((uint64_t)hi << 32);
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fadd2_rm(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rm.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
    return pk2(__float_as_uint(lo), __float_as_uint(hi));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// 2^x for a pair of x <= 127 on the FMA pipe: x = n + f, 2^f by a degree-3 minimax polynomial
// (max rel. error 8.6e-5, far below the bf16 rounding of P), exponent added as integer.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
    // clamp to [-127, 128]: above 128 the exponent add overflows to inf / NaN, which the
    // kernels' overflow guard (!(sum <= 2^56)) catches instead of wrapping into the sign bit
    const float x0 = fminf(fmaxf(lo_f(x), -127.0f), 128.0f);
    const float x1 = fminf(fmaxf(hi_f(x), -127.0f), 128.0f);
    const uint64_t xc = f2(x0, x1);
    const uint64_t kRound = f2(12582912.0f, 12582912.0f);  // 2^23 + 2^22
    const uint64_t rnd = fadd2_rm(xc, kRound);               // floor(x) in the low mantissa bits
    const uint64_t frac = fsub2(xc, fsub2(rnd, kRound));     // in [0, 1)
    uint64_t p = f2(0.077066176f, 0.077066176f);
    p = ffma2(p, frac, f2(0.22764593f, 0.22764593f));
    p = ffma2(p, frac, f2(0.6951166f, 0.6951166f));
    p = ffma2(p, frac, f2(1.0f, 1.0f));
    const uint32_t e0 = (uint32_t)rnd << 23, e1 = (uint32_t)(rnd >> 32) << 23;
    return pk2((uint32_t)p + e0, (uint32_t)(p >> 32) + e1);
}

// 2^x for a pair of x on the FMA pipe with a degree-5 polynomial for 2^frac (relative
// minimax fit on [0,1), max rel. error 1.7e-7 -- as accurate as ex2.approx, which the energies
// need: unlike P in the attention kernel they are not rounded to bf16 afterwards).
__device__ __forceinline__ uint64_t exp2_poly5(uint64_t x) {
    // clamp at -126: the fit's p(0) = 0.99999994 < 1, so floor(x) = -127 would borrow out of
    // the exponent field (0x3F7FFFFF - 0x3F800000 = NaN bits); at -126 the result is a
    // denormal that the .ftz arithmetic downstream reads as 0 (masked keys hold -inf).
    const float x0 = fmaxf(lo_f(x), -126.0f), x1 = fmaxf(hi_f(x), -126.0f);
    const uint64_t xc = f2(x0, x1);
    const uint64_t kRound = f2(12582912.0f, 12582912.0f);  // 2^23 + 2^22
    const uint64_t rnd = fadd2_rm(xc, kRound);               // floor(x) in the low mantissa bits
    const uint64_t frac = fsub2(xc, fsub2(rnd, kRound));     // in [0, 1)
    uint64_t p = f2(0.0018775767f, 0.0018775767f);
    p = ffma2(p, frac, f2(0.0089893406f, 0.0089893406f));
    p = ffma2(p, frac, f2(0.055826318f, 0.055826318f));
    p = ffma2(p, frac, f2(0.24015361f, 0.24015361f));
    p = ffma2(p, frac, f2(0.69315308f, 0.69315308f));
    p = ffma2(p, frac, f2(0.99999994f, 0.99999994f));
    const uint32_t e0 = (uint32_t)rnd << 23, e1 = (uint32_t)(rnd >> 32) << 23;
    return pk2((uint32_t)p + e0, (uint32_t)(p >> 32) + e1);
}

// Debug timeline (csa_debug_trace): clock64 stamps of CTA 0's pipeline events; nullptr = off.
// Each translation unit defines its own `static __device__` g_trace / g_debug_mode (debug only).
// Compiled in only for trace builds (CSA_TRACE_BUILD=1 python -m paper_2603_05503_b200._build
// --force): the global load of g_trace in the hot loops costs several percent otherwise.
#ifdef CSA_ENABLE_TRACE
#define CSA_TRACE(slot, k, e)                                                             \
    do {                                                                                  \
        if (g_trace != nullptr && blockIdx.x == 0 && (k) < 1024)                          \
            g_trace[((slot) * 1024 + (k)) * 8 + (e)] = clock64();                         \
    } while (0)
#else
#define CSA_TRACE(slot, k, e) \
    do {                      \
    } while (0)
#endif

__device__ __forceinline__ void set_maxnreg_dec56() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
}
__device__ __forceinline__ void set_maxnreg_inc224() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
}

// Half-row tile: HC = BK/2 columns per thread.  exp2(s*sl2 - m) -> packed bf16 pk[HC/2], returns
// the sum of the fp32 values.
template <int HC, int kEmu = kEmuPerOctet>
__device__ __forceinline__ float exp_half(const uint32_t (&r)[HC], float sl2, float m,
                                          uint32_t (&pk)[HC / 2]) {
    const uint64_t sl2x2 = f2(sl2, sl2);
    const uint64_t negm = f2(-m, -m);
    uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int x = 0; x < HC; x += 2) {
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

template <int HC>
__device__ __forceinline__ float max_half(const uint32_t (&r)[HC]) {
    constexpr int kPer = HC / 8;  // elements per chain (even)
    float mc[8];
#pragma unroll
    for (int q8 = 0; q8 < 8; ++q8) {
        mc[q8] = __uint_as_float(r[q8]);
#pragma unroll
        for (int t = 1; t + 1 < kPer; t += 2)
            mc[q8] = fmax3(mc[q8], __uint_as_float(r[q8 + 8 * t]), __uint_as_float(r[q8 + 8 * (t + 1)]));
        if (kPer % 2 == 0) mc[q8] = fmaxf(mc[q8], __uint_as_float(r[q8 + 8 * (kPer - 1)]));
    }
    return fmaxf(fmax3(mc[0], mc[1], mc[2]), fmaxf(fmax3(mc[3], mc[4], mc[5]), fmaxf(mc[6], mc[7])));
}

template <int HC>
__device__ __forceinline__ void tmem_load_half(uint32_t addr, uint32_t (&r)[HC]) {
    static_assert(HC == 32 || HC == 64, "half tile");
    if constexpr (HC == 64) {
        uint32_t(&a0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
        uint32_t(&a1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
        tmem_ld32(addr, a0);
        tmem_ld32(addr + 32, a1);
        tmem_ld_wait(a0);
        tmem_ld_wait(a1);
    } else {
        uint32_t(&a0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
        tmem_ld32(addr, a0);
        tmem_ld_wait(a0);
    }
}

template <int HC>
__device__ __forceinline__ void tmem_store_p(uint32_t addr, const uint32_t (&pk)[HC / 2]) {
    if constexpr (HC == 64) {
        tmem_st32(addr, pk);
    } else {
        tmem_st16(addr, pk);
    }
}


}  // namespace attn
}  // namespace csa
