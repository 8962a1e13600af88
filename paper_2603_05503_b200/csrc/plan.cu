// plan.cu -- a6: keep counts -> calibrated plan (integer-only, bit-exact with the oracle).
//
// P:557-571 Eq. (eq:mask_threshold): M[r,c] = [M_bar[r,c] >= rho], evaluated in count space as
// count >= min_count (min_count = ceil-ish(rho |D|) from the host).  An emptied row re-keeps its
// argmax-count block (tie -> lowest c), reading Q7.  P:625-626 + P:656: a cell whose
// similarity exceeds gamma is REPETITIVE *instead of* masked.  P:651-653 / P:947-950: per query
// block-row the kept key-block columns as a CSR list (what the attention producer walks) and as
// maximal half-open intervals (the paper's 1D skip list).  P:728: kept area per cell.
//
// Layout: one warp per (cell, row); the row's N_B counts are read coalesced, thresholded 32
// columns per ballot into the packed mask word.  HBM-bound: reads 2 B x N_B^2 per cell, writes
// N_B^2/8 B of bits + 2 B per kept block.
#include <cstdint>

#include "csa_internal.cuh"

namespace csa {
namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ int64_t blk_size(int64_t c, int32_t B, int32_t N) {
    const int64_t hi = (c + 1) * B;
    return (hi < N ? hi : N) - c * B;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    plan_count_kernel(Geo g, int64_t n_cells, const uint16_t* __restrict__ counts,
                      int32_t min_count, const double* __restrict__ sim, double gamma,
                      int32_t anchor_k, PlanDev p) {
    const int lane = threadIdx.x & 31;
    const int64_t total = n_cells * g.NB;
    for (int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); gw < total;
         gw += (int64_t)gridDim.x * kWarpsPerBlock) {
        const int64_t cell = gw / g.NB;
        const int32_t r = (int32_t)(gw % g.NB);
        const bool rep = sim != nullptr && sim[cell] > gamma;  // strict "exceeds" (Q8)
        uint32_t* words = p.mask_bits + (cell * g.NB + r) * g.W32;
        int32_t* brp = p.blk_row_ptr + cell * (g.NB + 1);
        int32_t* irp = p.ivl_row_ptr + cell * (g.NB + 1);
        if (r == 0 && lane == 0) {
            p.kind[cell] = rep ? 1 : 0;
            p.anchor_k[cell] = rep ? anchor_k : 0;
            brp[0] = 0;
            irp[0] = 0;
            if (rep) p.kept_area[cell] = (int64_t)g.F * anchor_k * g.W * (int64_t)g.N;
        }
        if (rep) {
            for (int w = lane; w < g.W32; w += 32) words[w] = 0u;
            if (lane == 0) { brp[r + 1] = 0; irp[r + 1] = 0; }
            continue;
        }
        const uint16_t* row = counts + (cell * g.NB + r) * (int64_t)g.NBK;
        int32_t nnz = 0;
        for (int w = 0; w < g.W32; ++w) {
            const int c = w * 32 + lane;
            const bool keep = c < g.NBK && (int32_t)row[c] >= min_count;
            const uint32_t word = __ballot_sync(0xffffffffu, keep);
            nnz += __popc(word);
        }
        int32_t repair = -1;
        if (nnz == 0) {  // argmax count, lowest c on ties (Q7)
            int32_t best_v = -1, best_c = 0x7fffffff;
            for (int c = lane; c < g.NBK; c += 32) {
                const int32_t v = row[c];
                if (v > best_v) { best_v = v; best_c = c; }
            }
            for (int off = 16; off > 0; off >>= 1) {
                const int32_t ov = __shfl_xor_sync(0xffffffffu, best_v, off);
                const int32_t oc = __shfl_xor_sync(0xffffffffu, best_c, off);
                if (ov > best_v || (ov == best_v && oc < best_c)) { best_v = ov; best_c = oc; }
            }
            repair = best_c;
            nnz = 1;
        }
        // second sweep: write words, count run starts, sum kept key extents
        int32_t nivl = 0;
        int64_t cols = 0;
        uint32_t carry = 0;  // kept bit of column w*32-1
        for (int w = 0; w < g.W32; ++w) {
            const int c = w * 32 + lane;
            const bool keep = c < g.NBK && ((int32_t)row[c] >= min_count || c == repair);
            const uint32_t word = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) words[w] = word;
            const uint32_t starts = word & ~((word << 1) | carry);
            nivl += __popc(starts);
            carry = word >> 31;
            if (keep) cols += blk_size(c, g.BK, g.N);
        }
        for (int off = 16; off > 0; off >>= 1) cols += __shfl_xor_sync(0xffffffffu, cols, off);
        if (lane == 0) {
            brp[r + 1] = nnz;
            irp[r + 1] = nivl;
            atomicAdd(reinterpret_cast<unsigned long long*>(p.kept_area + cell),
                      (unsigned long long)(cols * blk_size(r, g.B, g.N)));
        }
    }
}

// Per-cell inclusive scan of the row counts (in place) -> row pointers; cell totals go to
// base[cell + 1] for the cross-cell scan.
__global__ void __launch_bounds__(1024)
    plan_scan_rows_kernel(Geo g, int64_t n_cells, PlanDev p) {
    __shared__ int32_t warp_tot[2][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t cell = blockIdx.x; cell < n_cells; cell += gridDim.x) {
        for (int which = 0; which < 2; ++which) {
            int32_t* rp = (which == 0 ? p.blk_row_ptr : p.ivl_row_ptr) + cell * (g.NB + 1);
            int32_t carry = 0;
            for (int base = 0; base < g.NB; base += 1024) {
                const int r = base + threadIdx.x;
                int32_t v = r < g.NB ? rp[r + 1] : 0;
                for (int off = 1; off < 32; off <<= 1) {
                    const int32_t o = __shfl_up_sync(0xffffffffu, v, off);
                    if (lane >= off) v += o;
                }
                if (lane == 31) warp_tot[which][wid] = v;
                __syncthreads();
                if (wid == 0) {
                    int32_t t = warp_tot[which][lane];
                    for (int off = 1; off < 32; off <<= 1) {
                        const int32_t o = __shfl_up_sync(0xffffffffu, t, off);
                        if (lane >= off) t += o;
                    }
                    warp_tot[which][lane] = t;
                }
                __syncthreads();
                const int32_t prefix = (wid > 0 ? warp_tot[which][wid - 1] : 0) + carry;
                if (r < g.NB) rp[r + 1] = v + prefix;
                carry += warp_tot[which][31];
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                if (which == 0) p.blk_base[cell + 1] = carry;
                else p.ivl_base[cell + 1] = carry;
            }
        }
    }
}

// Single-CTA inclusive scan of base[1..n_cells] (cell totals) -> exclusive cell offsets.
__global__ void __launch_bounds__(1024) plan_scan_cells_kernel(int64_t n_cells, PlanDev p) {
    __shared__ int64_t warp_tot[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int which = 0; which < 2; ++which) {
        int64_t* base = which == 0 ? p.blk_base : p.ivl_base;
        if (threadIdx.x == 0) base[0] = 0;
        int64_t carry = 0;
        for (int64_t b0 = 0; b0 < n_cells; b0 += 1024) {
            const int64_t c = b0 + threadIdx.x;
            int64_t v = c < n_cells ? base[c + 1] : 0;
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t o = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += o;
            }
            if (lane == 31) warp_tot[wid] = v;
            __syncthreads();
            if (wid == 0) {
                int64_t t = warp_tot[lane];
                for (int off = 1; off < 32; off <<= 1) {
                    const int64_t o = __shfl_up_sync(0xffffffffu, t, off);
                    if (lane >= off) t += o;
                }
                warp_tot[lane] = t;
            }
            __syncthreads();
            const int64_t prefix = (wid > 0 ? warp_tot[wid - 1] : 0) + carry;
            if (c < n_cells) base[c + 1] = v + prefix;
            carry += warp_tot[31];
            __syncthreads();
        }
    }
}

// Phase 1: CSR indices and skip-list intervals from the packed mask words.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    plan_fill_kernel(Geo g, int64_t n_cells, PlanDev p) {
    const int lane = threadIdx.x & 31;
    const uint32_t lower = (1u << lane) - 1u;
    const int64_t total = n_cells * g.NB;
    for (int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); gw < total;
         gw += (int64_t)gridDim.x * kWarpsPerBlock) {
        const int64_t cell = gw / g.NB;
        const int32_t r = (int32_t)(gw % g.NB);
        if (p.kind[cell] != 0) continue;
        const uint32_t* words = p.mask_bits + (cell * g.NB + r) * g.W32;
        int64_t bpos = p.blk_base[cell] + p.blk_row_ptr[cell * (g.NB + 1) + r];
        int64_t spos = p.ivl_base[cell] + p.ivl_row_ptr[cell * (g.NB + 1) + r];
        int64_t epos = spos;
        uint32_t carry_prev = 0;  // kept bit of column w*32-1
        for (int w = 0; w < g.W32; ++w) {
            const uint32_t word = words[w];
            const uint32_t next_word = (w + 1 < g.W32) ? words[w + 1] : 0u;
            const uint32_t starts = word & ~((word << 1) | carry_prev);
            const uint32_t ends = word & ~((word >> 1) | (next_word << 31));  // last kept of a run
            const int c = w * 32 + lane;
            if ((word >> lane) & 1u) {
                const int64_t at = bpos + __popc(word & lower);
                if (at < p.blk_capacity) p.blk_idx[at] = (uint16_t)c;
            }
            if ((starts >> lane) & 1u) {
                const int64_t at = spos + __popc(starts & lower);
                if (at < p.ivl_capacity) p.ivl[2 * at] = (uint16_t)c;
            }
            if ((ends >> lane) & 1u) {
                const int64_t at = epos + __popc(ends & lower);
                if (at < p.ivl_capacity) p.ivl[2 * at + 1] = (uint16_t)(c + 1);
            }
            bpos += __popc(word);
            spos += __popc(starts);
            epos += __popc(ends);
            carry_prev = word >> 31;
        }
    }
}

// ------------------------------------------------------------------------------- work list
// One CTA sorts all items of one launch in shared memory (bitonic, 32-bit keys):
//   key = (2047 - cost) << 21 | p      (order 0, longest first; p = natural position)
//   key = p                            (order 1)
// p enumerates (h asc, index asc) -- each head has one kind, so this is (h, kind, index) order.
__global__ void __launch_bounds__(1024)
    work_list_kernel(Geo g, PlanDev p, int64_t cell_base, int32_t n_heads, int32_t order,
                     uint32_t* __restrict__ out, int32_t capacity, int32_t* __restrict__ n_work) {
    extern __shared__ uint32_t sm_keys[];
    __shared__ int32_t head_off[2049];
    __shared__ int32_t s_total;
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (int h = 0; h < n_heads; ++h) {
            head_off[h] = acc;
            const int64_t cell = cell_base + h;
            const int32_t cnt =
                p.kind[cell] ? (int32_t)(((int64_t)g.F * p.anchor_k[cell] * g.W + kAnchorTile - 1) /
                                         kAnchorTile)
                             : g.NB;
            acc += cnt;
        }
        head_off[n_heads] = acc;
        s_total = acc;
    }
    __syncthreads();
    const int32_t total = s_total;
    if (total > kMaxWorkItems || total > capacity) {
        if (threadIdx.x == 0) *n_work = -1;
        return;
    }
    int32_t pow2 = 1;
    while (pow2 < total) pow2 <<= 1;
    for (int32_t x = threadIdx.x; x < pow2; x += blockDim.x) {
        uint32_t key = 0xffffffffu;
        if (x < total) {
            int lo = 0, hi = n_heads - 1;  // head of position x: last h with head_off[h] <= x
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (head_off[mid] <= x) lo = mid; else hi = mid - 1;
            }
            const int h = lo;
            const int idx = x - head_off[h];
            const int64_t cell = cell_base + h;
            int32_t cost = g.NBK;
            if (!p.kind[cell]) {
                const int32_t* rp = p.blk_row_ptr + cell * (g.NB + 1);
                cost = rp[idx + 1] - rp[idx];
            }
            key = order == 0 ? ((uint32_t)(2047 - cost) << 21) | (uint32_t)x : (uint32_t)x;
        }
        sm_keys[x] = key;
    }
    __syncthreads();
    for (int32_t k = 2; k <= pow2; k <<= 1) {
        for (int32_t j = k >> 1; j > 0; j >>= 1) {
            for (int32_t x = threadIdx.x; x < pow2; x += blockDim.x) {
                const int32_t y = x ^ j;
                if (y > x) {
                    const uint32_t a = sm_keys[x], b = sm_keys[y];
                    const bool up = (x & k) == 0;
                    if ((a > b) == up) { sm_keys[x] = b; sm_keys[y] = a; }
                }
            }
            __syncthreads();
        }
    }
    for (int32_t x = threadIdx.x; x < total; x += blockDim.x) {
        const int32_t pos = (int32_t)(sm_keys[x] & 0x1FFFFFu);
        int lo = 0, hi = n_heads - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (head_off[mid] <= pos) lo = mid; else hi = mid - 1;
        }
        const uint32_t kind = p.kind[cell_base + lo] ? 1u : 0u;
        out[x] = (kind << 31) | ((uint32_t)lo << 20) | (uint32_t)(pos - head_off[lo]);
    }
    if (threadIdx.x == 0) *n_work = total;
}

// Order 2 (head-major, longest-first within a head): one CTA per head sorts its own segment.
//   key = (4095 - cost) << 11 | index     (cost <= 4094, index <= 2047)
// Order 3 (pairs): item p of a head stands for rows (2p, 2p+1) [or anchor tiles (2p, 2p+1)];
//   cost = sum of the members' costs (the pair kernel walks the union of their lists).
__global__ void __launch_bounds__(256)
    work_list_head_kernel(Geo g, PlanDev p, int64_t cell_base, int32_t n_heads, int32_t pairs,
                          uint32_t* __restrict__ out, int32_t capacity, int32_t* __restrict__ n_work) {
    __shared__ uint32_t keys[2048];
    __shared__ int32_t s_off, s_cnt, s_total;
    const int h = blockIdx.x;
    auto units_of = [&](int hh) -> int32_t {  // rows (MASK) or anchor tiles (REPETITIVE)
        const int64_t cell = cell_base + hh;
        return p.kind[cell] ? (int32_t)(((int64_t)g.F * p.anchor_k[cell] * g.W + kAnchorTile - 1) /
                                        kAnchorTile)
                            : g.NB;
    };
    auto items_of = [&](int hh) -> int32_t {
        const int32_t u = units_of(hh);
        return pairs ? (u + 1) / 2 : u;
    };
    if (threadIdx.x == 0) {
        int32_t off = 0, tot = 0;
        for (int hh = 0; hh < n_heads; ++hh) {
            const int32_t c = items_of(hh);
            if (hh < h) off += c;
            tot += c;
        }
        s_off = off;
        s_cnt = items_of(h);
        s_total = tot;
    }
    __syncthreads();
    const int32_t cnt = s_cnt, off = s_off, total = s_total;
    if (total > capacity || cnt > 2048) {
        if (h == 0 && threadIdx.x == 0) *n_work = -1;
        return;
    }
    const int64_t cell = cell_base + h;
    const bool rep = p.kind[cell] != 0;
    int32_t pow2 = 1;
    while (pow2 < cnt) pow2 <<= 1;
    for (int32_t x = threadIdx.x; x < pow2; x += blockDim.x) {
        uint32_t key = 0xffffffffu;
        if (x < cnt) {
            const int32_t units = units_of(h);
            auto unit_cost = [&](int32_t u) -> int32_t {
                if (u >= units) return 0;
                if (rep) return g.NBK;
                const int32_t* rp = p.blk_row_ptr + cell * (g.NB + 1);
                return rp[u + 1] - rp[u];
            };
            const int32_t cost = pairs ? unit_cost(2 * x) + unit_cost(2 * x + 1) : unit_cost(x);
            key = ((uint32_t)(4095 - cost) << 11) | (uint32_t)x;
        }
        keys[x] = key;
    }
    __syncthreads();
    for (int32_t k = 2; k <= pow2; k <<= 1) {
        for (int32_t j = k >> 1; j > 0; j >>= 1) {
            for (int32_t x = threadIdx.x; x < pow2; x += blockDim.x) {
                const int32_t y = x ^ j;
                if (y > x) {
                    const uint32_t a = keys[x], b = keys[y];
                    const bool up = (x & k) == 0;
                    if ((a > b) == up) { keys[x] = b; keys[y] = a; }
                }
            }
            __syncthreads();
        }
    }
    for (int32_t x = threadIdx.x; x < cnt; x += blockDim.x)
        out[off + x] = ((rep ? 1u : 0u) << 31) | ((uint32_t)h << 20) | (keys[x] & 0x7FFu);
    if (h == 0 && threadIdx.x == 0) *n_work = total;
}

// --------------------------------------------------------------------------------- validate
__global__ void plan_validate_kernel(Geo g, int64_t n_cells, PlanDev p, uint32_t* flag) {
    const int64_t total = n_cells * g.NB;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cell = x / g.NB;
        const int32_t r = (int32_t)(x % g.NB);
        const int32_t* brp = p.blk_row_ptr + cell * (g.NB + 1);
        const int32_t* irp = p.ivl_row_ptr + cell * (g.NB + 1);
        uint32_t bad = 0;
        const int64_t bb0 = p.blk_base[cell], bb1 = p.blk_base[cell + 1];
        const int64_t ib0 = p.ivl_base[cell], ib1 = p.ivl_base[cell + 1];
        if (bb1 < bb0 || ib1 < ib0 || bb0 < 0 || ib0 < 0) bad |= 1;
        if ((p.blk_idx != nullptr && p.blk_base[n_cells] > p.blk_capacity) ||
            p.ivl_base[n_cells] > p.ivl_capacity)
            bad |= 2;
        if (cell == 0 && r == 0 && (p.blk_base[0] != 0 || p.ivl_base[0] != 0)) bad |= 2048;
        if (r == 0 && (brp[0] != 0 || irp[0] != 0)) bad |= 2048;
        const int32_t b0 = brp[r], b1 = brp[r + 1], i0 = irp[r], i1 = irp[r + 1];
        // row pointers inside the cell's own list (no read below this check leaves it)
        if (b1 < b0 || i1 < i0 || b0 < 0 || i0 < 0 || (int64_t)b1 > bb1 - bb0 ||
            (int64_t)i1 > ib1 - ib0)
            bad |= 4;
        if (p.kind[cell] > 1) bad |= 512;
        if (p.kind[cell] == 1 && (p.anchor_k[cell] < 1 || p.anchor_k[cell] > g.H)) bad |= 1024;
        if (p.kind[cell] == 0 && !(bad & 4)) {
            if (b1 == b0) bad |= 8;  // empty MASK row
            if (brp[g.NB] != p.blk_base[cell + 1] - p.blk_base[cell]) bad |= 16;
            if (!bad) {
                // intervals-only plans (blk_idx == nullptr): the intervals alone
                // must cover exactly the row's count, in order, inside the mask bits
                const uint16_t* bi = p.blk_idx ? p.blk_idx + p.blk_base[cell] : nullptr;
                const uint16_t* iv = p.ivl + 2 * p.ivl_base[cell];
                const uint32_t* words = p.mask_bits + (cell * g.NB + r) * g.W32;
                int32_t prev = -1, cover = 0, bj = b0;
                for (int32_t t = i0; t < i1; ++t) {
                    const int32_t s = iv[2 * t], e = iv[2 * t + 1];
                    if (!(s < e) || e > g.NBK || s <= prev) bad |= 32;  // ordered, non-adjacent
                    prev = e;
                    for (int32_t c = s; c < e && !bad; ++c, ++bj) {
                        if (bi != nullptr && (bj >= b1 || bi[bj] != c)) bad |= 64;  // CSR == ivl
                        if (bi == nullptr && !((words[c >> 5] >> (c & 31)) & 1u)) bad |= 128;
                    }
                    cover += e - s;
                }
                if (cover != b1 - b0) bad |= 64;
                for (int32_t t = b0; bi != nullptr && t < b1 && !bad; ++t) {
                    const int32_t c = bi[t];
                    if (c >= g.NBK || (t > b0 && c <= bi[t - 1])) bad |= 128;
                    if (!((words[c >> 5] >> (c & 31)) & 1u)) bad |= 128;
                }
            }
        } else if (b1 != b0 || i1 != i0) {
            bad |= 256;
        }
        if (bad) atomicOr(flag, bad);
    }
}

int grid_for(int64_t warps) {
    int64_t blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks > 148 * 64) blocks = 148 * 64;
    return (int)(blocks < 1 ? 1 : blocks);
}

}  // namespace

cudaError_t launch_plan_count(const Geo& g, int64_t n_cells, const uint16_t* counts,
                              int32_t min_count, const double* sim, double gamma, int32_t anchor_k,
                              const PlanDev& p, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.kept_area, 0, sizeof(int64_t) * n_cells, s);
    if (e != cudaSuccess) return e;
    plan_count_kernel<<<grid_for(n_cells * g.NB), kWarpsPerBlock * 32, 0, s>>>(
        g, n_cells, counts, min_count, sim, gamma, anchor_k, p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int blocks = (int)(n_cells < 148 * 8 ? n_cells : 148 * 8);
    plan_scan_rows_kernel<<<blocks, 1024, 0, s>>>(g, n_cells, p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    plan_scan_cells_kernel<<<1, 1024, 0, s>>>(n_cells, p);
    return cudaGetLastError();
}

cudaError_t launch_plan_fill(const Geo& g, int64_t n_cells, const PlanDev& p, cudaStream_t s) {
    plan_fill_kernel<<<grid_for(n_cells * g.NB), kWarpsPerBlock * 32, 0, s>>>(g, n_cells, p);
    return cudaGetLastError();
}

cudaError_t launch_work_list(const Geo& g, const PlanDev& p, int64_t cell_base, int32_t n_heads,
                             int32_t order, uint32_t* out, int32_t capacity, int32_t* n_work,
                             cudaStream_t s) {
    if (order == 2 || order == 3) {
        work_list_head_kernel<<<n_heads, 256, 0, s>>>(g, p, cell_base, n_heads, order == 3 ? 1 : 0,
                                                     out, capacity, n_work);
        return cudaGetLastError();
    }
    const size_t smem = sizeof(uint32_t) * kMaxWorkItems;
    cudaError_t e =
        cudaFuncSetAttribute(work_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    work_list_kernel<<<1, 1024, smem, s>>>(g, p, cell_base, n_heads, order, out, capacity, n_work);
    return cudaGetLastError();
}

cudaError_t launch_validate(const Geo& g, int64_t n_cells, const PlanDev& p, uint32_t* flag,
                            cudaStream_t s) {
    int64_t threads = n_cells * g.NB;
    int blocks = (int)((threads + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks < 1) blocks = 1;
    plan_validate_kernel<<<blocks, 256, 0, s>>>(g, n_cells, p, flag);
    return cudaGetLastError();
}

}  // namespace csa
