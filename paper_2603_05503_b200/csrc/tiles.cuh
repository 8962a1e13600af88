// tiles.cuh -- shared-memory tile geometry and the two tcgen05 contractions of the CSA kernels.
//
// Tiles are staged by TMA with SWIZZLE_128B in boxes of [rows][64 bf16] (128 B per row,
// 1 KiB per 8-row atom); a head_dim of D occupies D/64 boxes laid out back to back.
//   Q tile   : 128 query rows  -> A operand of S = Q K^T   (K-major, SBO 1 KiB)
//   K tile   : BK key rows     -> B operand of S = Q K^T   (K-major)
//   V tile   : BK key rows     -> B operand of O += P V    (MN-major: N = head_dim is the
//              contiguous axis; LBO = one box, SBO = 1 KiB per 8 keys)
//   P        : bf16 in tensor memory (A operand of the TS-MMA), 2 elements per 32-bit column.
#pragma once
#include "sm100.cuh"

namespace csa {

template <int BK, int D>
struct TileCfg {
    static constexpr int kQRows = 128;                    // UMMA M
    static constexpr int kBoxes = D / 64;                 // 128-byte-wide boxes per row
    static constexpr int kQBox = kQRows * 128;            // bytes of one Q box
    static constexpr int kKBox = BK * 128;                // bytes of one K/V box
    static constexpr int kQBytes = kBoxes * kQBox;        // Q tile
    static constexpr int kKVBytes = kBoxes * kKBox;       // one K or V tile (one ring slot)
    static constexpr uint32_t kIdescQK = umma_idesc_bf16(128, BK, 0, 0);
    static constexpr uint32_t kIdescPV = umma_idesc_bf16(128, D, 0, 1);
    static_assert(D == 64 || D == 128, "head_dim");
    static_assert(BK == 64 || BK == 128, "block");
};

// S[tmem] = Q . K^T over head_dim (D/16 MMAs of K = 16).
template <int BK, int D>
__device__ __forceinline__ void issue_qk(uint32_t s_tmem, uint32_t q_smem, uint32_t k_smem,
                                         int nsteps = D / 16) {
    using C = TileCfg<BK, D>;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
        if (kk >= nsteps) break;  // debug measurements only (truncated contraction)
        const uint32_t off = (kk & 3) * 32;  // 16 bf16 = 32 B inside a 128-B box row
        const uint64_t a = umma_desc_sw128(q_smem + (kk >> 2) * C::kQBox + off, 16, 1024);
        const uint64_t b = umma_desc_sw128(k_smem + (kk >> 2) * C::kKBox + off, 16, 1024);
        mma_ss(s_tmem, a, b, C::kIdescQK, kk > 0 ? 1u : 0u);
    }
}

// O[tmem] (+)= P[tmem] . V over the BK keys of the tile (BK/16 MMAs of K = 16).
template <int BK, int D>
__device__ __forceinline__ void issue_pv(uint32_t o_tmem, uint32_t p_tmem, uint32_t v_smem,
                                         bool accumulate, int nsteps = BK / 16) {
    using C = TileCfg<BK, D>;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
        if (kk >= nsteps) break;  // debug measurements only (truncated contraction)
        const uint64_t b = umma_desc_sw128(v_smem + kk * 16 * 128, C::kKBox, 1024);
        mma_ts(o_tmem, p_tmem + kk * 8, b, C::kIdescPV, (accumulate || kk > 0) ? 1u : 0u);
    }
}

// O[tmem] (+)= P[smem] . V with P a 128 x BK bf16 tile staged K-major in SW128 boxes of
// [128 rows][64 keys] (written by the softmax threads), V MN-major (BK/16 MMAs of K = 16).
template <int BK, int D>
__device__ __forceinline__ void issue_pv_ss(uint32_t o_tmem, uint32_t p_smem, uint32_t v_smem,
                                            bool accumulate) {
    using C = TileCfg<BK, D>;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
        const uint64_t a = umma_desc_sw128(p_smem + (kk >> 2) * C::kQBox + (kk & 3) * 32, 16, 1024);
        const uint64_t b = umma_desc_sw128(v_smem + kk * 16 * 128, C::kKBox, 1024);
        mma_ss(o_tmem, a, b, C::kIdescPV, (accumulate || kk > 0) ? 1u : 0u);
    }
}

// TMA-load one [rows][D] tile of a [batch, N, heads, D] tensor (4-D map: d, h, n, b).
template <int D>
__device__ __forceinline__ void tma_tile(uint8_t* dst, int box_bytes, const CUtensorMap* map,
                                         uint64_t* bar, int32_t h, int32_t n0, int32_t b,
                                         uint64_t policy) {
#pragma unroll
    for (int x = 0; x < D / 64; ++x)
        tma_load_4d(dst + x * box_bytes, map, bar, x * 64, h, n0, b, policy);
}

// Byte offset of 16-byte chunk `cj` (0..7) of row `row` inside a SWIZZLE_128B box.
__device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t cj) {
    return row * 128u + ((cj ^ (row & 7u)) << 4);
}

}  // namespace csa
