// compact.cu -- f2: plan memory compaction on the GPU.
//
// Interval merging (Table tab:skip_list_memory "Merge %"): the target row width is the
// nearest-rank p-th percentile of the per-row interval counts over the rows of the given MASK
// cells (Q26); a row above it fills its (n - target) smallest gaps, ties -> leftmost (Q28) --
// exactly what repeated smallest-gap merging does, since merging two neighbours removes just the
// gap between them.  The filled blocks are written into keep_count as min_count, so recompiling
// (csa_compile_plan) yields the merged plan.
// Timestep sharing: per group g of cells (t, g) = t * n_groups + g, the IoU of the
// compiled masks' skipped sets for every timestep pair (Eq. eq:timestep_iou), greedy cliques in
// ascending t with IoU >= tau (Q27), and the OR of each clique's kept masks written back as
// keep_count = min_count * M_shared for every member (one identical mask per clique after the
// recompile).  REPETITIVE cells take part in neither (IoU reported as -1, singleton cliques).
// All integer / exact-ratio work: results are bit-exact against the oracle.
#include <cstdint>

#include "csa_internal.cuh"

namespace csa {
namespace {

// ---------------------------------------------------------------- percentile of row widths
__global__ void __launch_bounds__(1024)
    width_percentile_kernel(Geo g, int64_t n_cells, PlanDev p, double pct, int32_t* target,
                            int32_t* hist_ws) {
    __shared__ unsigned long long total;
    const int32_t nbins = g.NBK + 1;  // widths 0 .. N_Bkv
    for (int32_t i = threadIdx.x; i < nbins; i += blockDim.x) hist_ws[i] = 0;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    const int64_t rows = n_cells * g.NB;
    unsigned long long mine = 0;
    for (int64_t x = threadIdx.x; x < rows; x += blockDim.x) {
        const int64_t cell = x / g.NB, r = x % g.NB;
        if (p.kind[cell] != 0) continue;  // REPETITIVE cells carry no intervals
        const int32_t* rp = p.ivl_row_ptr + cell * (g.NB + 1);
        atomicAdd(hist_ws + (rp[r + 1] - rp[r]), 1);
        ++mine;
    }
    atomicAdd(&total, mine);
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t n = (int64_t)total;
        int32_t out = 0;
        if (n > 0) {
            int64_t rank = (int64_t)ceil(pct / 100.0 * (double)n);  // nearest rank, 1-based
            if (rank < 1) rank = 1;
            int64_t acc = 0;
            for (int32_t w = 0; w < nbins; ++w) {
                acc += hist_ws[w];
                if (acc >= rank) {
                    out = w;
                    break;
                }
            }
        }
        *target = out;
    }
}

// ---------------------------------------------------------------- merge: one warp per row
__global__ void __launch_bounds__(256)
    merge_rows_kernel(Geo g, int64_t n_cells, PlanDev p, const int32_t* target_ptr,
                      int32_t min_count, uint16_t* keep_count, unsigned long long* added) {
    const int32_t lane = threadIdx.x & 31;
    const int64_t x = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= n_cells * g.NB) return;
    const int64_t cell = x / g.NB, r = x % g.NB;
    if (p.kind[cell] != 0) return;
    const int32_t* rp = p.ivl_row_ptr + cell * (g.NB + 1);
    const int32_t n = rp[r + 1] - rp[r];
    const int32_t target = *target_ptr < 1 ? 1 : *target_ptr;
    if (n <= target) return;
    const uint16_t* iv = p.ivl + 2 * (p.ivl_base[cell] + rp[r]);
    const int32_t k = n - target;  // gaps to fill: the k smallest by (gap, index)
    uint16_t* cnt = keep_count + (cell * g.NB + r) * (int64_t)g.NBK;
    unsigned long long mine = 0;
    for (int32_t i = lane; i < n - 1; i += 32) {
        const int32_t gi = (int32_t)iv[2 * (i + 1)] - (int32_t)iv[2 * i + 1];
        int32_t rank = 0;
        for (int32_t j = 0; j < n - 1; ++j) {
            const int32_t gj = (int32_t)iv[2 * (j + 1)] - (int32_t)iv[2 * j + 1];
            rank += (gj < gi) || (gj == gi && j < i);
        }
        if (rank < k) {
            for (int32_t c = iv[2 * i + 1]; c < iv[2 * (i + 1)]; ++c) cnt[c] = (uint16_t)min_count;
            mine += (unsigned long long)gi;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
    if (lane == 0 && mine) atomicAdd(added, mine);
}

// ---------------------------------------------------------------- skipped-set IoU
// one warp per (group, t1, t2); words of the kept bits, tail bits beyond N_B masked off
__global__ void __launch_bounds__(256)
    iou_kernel(Geo g, int32_t n_groups, int32_t T, PlanDev p, double* iou) {
    const int32_t lane = threadIdx.x & 31;
    const int64_t x = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= (int64_t)n_groups * T * T) return;
    const int32_t grp = (int32_t)(x / ((int64_t)T * T));
    const int32_t t1 = (int32_t)((x / T) % T), t2 = (int32_t)(x % T);
    const int64_t c1 = (int64_t)t1 * n_groups + grp, c2 = (int64_t)t2 * n_groups + grp;
    double out;
    if (p.kind[c1] != 0 || p.kind[c2] != 0) {
        out = -1.0;
    } else {
        const uint32_t* a = p.mask_bits + c1 * (int64_t)g.NB * g.W32;
        const uint32_t* b = p.mask_bits + c2 * (int64_t)g.NB * g.W32;
        const int32_t tail = g.NBK - (g.W32 - 1) * 32;  // valid bits in a row's last word
        const uint32_t tail_mask = tail == 32 ? 0xffffffffu : ((1u << tail) - 1u);
        unsigned long long inter = 0, uni = 0;
        const int64_t words = (int64_t)g.NB * g.W32;
        for (int64_t w = lane; w < words; w += 32) {
            const uint32_t valid = (w % g.W32 == g.W32 - 1) ? tail_mask : 0xffffffffu;
            const uint32_t sa = ~a[w] & valid, sb = ~b[w] & valid;
            inter += __popc(sa & sb);
            uni += __popc(sa | sb);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            inter += __shfl_xor_sync(0xffffffffu, inter, off);
            uni += __shfl_xor_sync(0xffffffffu, uni, off);
        }
        out = uni == 0 ? 1.0 : (double)inter / (double)uni;
    }
    if (lane == 0) iou[x] = out;
}

// ---------------------------------------------------------------- greedy cliques
__global__ void cluster_kernel(int32_t n_groups, int32_t T, const double* iou, double tau,
                               int32_t* cluster) {
    const int32_t grp = blockIdx.x * blockDim.x + threadIdx.x;
    if (grp >= n_groups) return;
    const double* m = iou + (int64_t)grp * T * T;
    int32_t* cl = cluster + (int64_t)grp * T;
    int32_t n_clusters = 0;
    for (int32_t t = 0; t < T; ++t) {
        int32_t joined = -1;
        for (int32_t c = 0; c < n_clusters && joined < 0; ++c) {
            bool ok = true;
            for (int32_t u = 0; u < t && ok; ++u)
                if (cl[u] == c && !(m[(int64_t)t * T + u] >= tau)) ok = false;
            if (ok) joined = c;
        }
        cl[t] = joined >= 0 ? joined : n_clusters++;
    }
}

// ---------------------------------------------------------------- OR of a clique's masks
// one warp per (cell, row): keep_count = min_count where any clique member keeps, else 0
__global__ void __launch_bounds__(256)
    share_rows_kernel(Geo g, int32_t n_groups, int32_t T, PlanDev p, const int32_t* cluster,
                      int32_t min_count, uint16_t* keep_count) {
    const int32_t lane = threadIdx.x & 31;
    const int64_t x = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t n_cells = (int64_t)n_groups * T;
    if (x >= n_cells * g.NB) return;
    const int64_t cell = x / g.NB, r = x % g.NB;
    if (p.kind[cell] != 0) return;
    const int32_t t = (int32_t)(cell / n_groups), grp = (int32_t)(cell % n_groups);
    const int32_t* cl = cluster + (int64_t)grp * T;
    const int32_t mine = cl[t];
    uint16_t* cnt = keep_count + (cell * g.NB + r) * (int64_t)g.NBK;
    for (int32_t w = 0; w < g.W32; ++w) {
        uint32_t bits = 0;
        for (int32_t u = 0; u < T; ++u) {
            if (cl[u] != mine) continue;
            const int64_t cu = (int64_t)u * n_groups + grp;
            if (p.kind[cu] != 0) continue;
            bits |= p.mask_bits[(cu * g.NB + r) * g.W32 + w];
        }
        const int32_t c = w * 32 + lane;
        if (c < g.NBK) cnt[c] = ((bits >> lane) & 1u) ? (uint16_t)min_count : (uint16_t)0;
    }
}

}  // namespace

cudaError_t launch_merge_intervals(const Geo& g, int64_t n_cells, const PlanDev& p, double pct,
                                   int32_t min_count, uint16_t* keep_count, int32_t* target,
                                   unsigned long long* added, int32_t* hist_ws, cudaStream_t s) {
    width_percentile_kernel<<<1, 1024, 0, s>>>(g, n_cells, p, pct, target, hist_ws);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t warps = n_cells * g.NB;
    if (warps == 0) return cudaSuccess;
    merge_rows_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(g, n_cells, p, target, min_count,
                                                                 keep_count, added);
    return cudaGetLastError();
}

cudaError_t launch_share_timesteps(const Geo& g, int32_t n_groups, int32_t T, const PlanDev& p,
                                   double tau, int32_t min_count, uint16_t* keep_count,
                                   int32_t* cluster, double* iou, cudaStream_t s) {
    const int64_t pairs = (int64_t)n_groups * T * T;
    iou_kernel<<<(unsigned)((pairs + 7) / 8), 256, 0, s>>>(g, n_groups, T, p, iou);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cluster_kernel<<<(n_groups + 127) / 128, 128, 0, s>>>(n_groups, T, iou, tau, cluster);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int64_t warps = (int64_t)n_groups * T * g.NB;
    share_rows_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(g, n_groups, T, p, cluster,
                                                                 min_count, keep_count);
    return cudaGetLastError();
}

}  // namespace csa
