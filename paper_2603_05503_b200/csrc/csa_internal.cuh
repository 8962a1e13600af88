// csa_internal.cuh -- shared declarations of the CUDA side (kernels <-> C ABI layer).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/csa.h"

namespace csa {

constexpr int kMaxBlocks = 2047;     // N_B limit (11-bit cost field of the work-list sort key)
constexpr int kMaxWorkItems = 32768;  // single-CTA shared-memory sort of one launch's items
constexpr int kAnchorTile = 128;      // gathered anchor-query rows per REPETITIVE work item

struct Geo {
    int32_t F, H, W, B;
    int32_t N;   // F*H*W
    int32_t NB;  // ceil(N/B): query blocks (plan rows)
    int32_t BK;  // key block B_kv (= B for square blocks, P:1294-1328 for B_q x B_kv)
    int32_t NBK; // ceil(N/BK): key blocks (plan columns)
    int32_t W32; // ceil(NBK/32) mask words per row
};

inline Geo make_geo(const csa_layout_t& L) {
    Geo g;
    g.F = L.frames;
    g.H = L.rows;
    g.W = L.cols;
    g.B = L.block;
    g.N = L.frames * L.rows * L.cols;
    g.NB = (g.N + g.B - 1) / g.B;
    g.BK = L.block_kv > 0 ? L.block_kv : L.block;
    g.NBK = (g.N + g.BK - 1) / g.BK;
    g.W32 = (g.NBK + 31) / 32;
    return g;
}

// Plan pointers passed by value to kernels.
struct PlanDev {
    uint8_t* kind;
    int32_t* anchor_k;
    uint32_t* mask_bits;
    int64_t* blk_base;
    int32_t* blk_row_ptr;
    uint16_t* blk_idx;
    int64_t* ivl_base;
    int32_t* ivl_row_ptr;
    uint16_t* ivl;
    int64_t* kept_area;
    int64_t blk_capacity;
    int64_t ivl_capacity;
};

inline PlanDev to_dev(const csa_plan_t& p) {
    return PlanDev{p.kind,        p.anchor_k, p.mask_bits, p.blk_base,  p.blk_row_ptr, p.blk_idx,
                   p.ivl_base,    p.ivl_row_ptr, p.ivl,    p.kept_area, p.blk_capacity,
                   p.ivl_capacity};
}

// Launchers implemented in the .cu files; each returns a cudaError_t of the launch.
cudaError_t launch_plan_count(const Geo& g, int64_t n_cells, const uint16_t* counts,
                              int32_t min_count, const double* sim, double gamma, int32_t anchor_k,
                              const PlanDev& p, cudaStream_t s);
cudaError_t launch_plan_fill(const Geo& g, int64_t n_cells, const PlanDev& p, cudaStream_t s);
cudaError_t launch_work_list(const Geo& g, const PlanDev& p, int64_t cell_base, int32_t n_heads,
                             int32_t order, uint32_t* out, int32_t capacity, int32_t* n_work,
                             cudaStream_t s);
cudaError_t launch_validate(const Geo& g, int64_t n_cells, const PlanDev& p, uint32_t* flag,
                            cudaStream_t s);

struct CalibArgs {
    Geo g;
    int32_t n_heads;
    float scale_log2;  // softmax_scale * log2(e)
    const float* lse_in;
    double eps;
    uint16_t* keep_count;
    float* energy_out;
    float* lse_out;
    float2* scratch;  // [grid][N_B][128] float log2-sum-exp partials (typed float2 for 8-byte
                      // alignment); nullptr -> two passes (or lse_in)
};
size_t calib_scratch_bytes(const Geo& g, int32_t n_heads, int num_sms);
cudaError_t set_calib_trace(void* buf, int mode);
cudaError_t launch_calib(const CalibArgs& a, int head_dim, const CUtensorMap& tq,
                         const CUtensorMap& tk, int num_sms, cudaStream_t s);

// f2 plan compaction (compact.cu)
cudaError_t launch_merge_intervals(const Geo& g, int64_t n_cells, const PlanDev& p, double pct,
                                   int32_t min_count, uint16_t* keep_count, int32_t* target,
                                   unsigned long long* added, int32_t* hist_ws, cudaStream_t s);
cudaError_t launch_share_timesteps(const Geo& g, int32_t n_groups, int32_t T, const PlanDev& p,
                                   double tau, int32_t min_count, uint16_t* keep_count,
                                   int32_t* cluster, double* iou, cudaStream_t s);

// f1 spatial similarity (sim.cu)
struct SimArgs {
    Geo g;
    int32_t n_heads;
    float scale_log2;
    const __nv_bfloat16* q;  // batch 0, for the anchor-row gather
    int64_t q_sn, q_sh;
    const float* lse;        // [n_heads][N] natural log
    int32_t anchor_k;
    float* partials;         // workspace [n_heads][N][3]
    double* sim_sum;         // [n_heads] += sum over (f, i) of cos
    float* cos_out;          // optional [n_heads][F*H]
};
cudaError_t launch_similarity(const SimArgs& a, int head_dim, const CUtensorMap& tq,
                              const CUtensorMap& tk, int num_sms, cudaStream_t s);
// sim_reduce_kernel alone: partials -> cos(f, i) and sim_sum (one CTA per head).
cudaError_t launch_similarity_reduce(const SimArgs& a, cudaStream_t s);
// a2-a5 + f1 in one pass (calibsim.cu; block 128 x 128, head_dim 128 / 64): a.scratch holds
// calib_sim_scratch_bytes (one float per (row, key block) and CTA), s.partials the
// [n_heads][N][3] similarity partials; ends with the similarity reduce.
size_t calib_sim_scratch_bytes(const Geo& g, int32_t n_heads, int num_sms);
cudaError_t set_calib_sim_trace(void* buf, int mode);
cudaError_t launch_calib_sim(const CalibArgs& a, const SimArgs& s, int head_dim,
                             const CUtensorMap& tq, const CUtensorMap& tk, int num_sms,
                             cudaStream_t st);

struct AttnArgs {
    Geo g;
    int32_t batch;
    int32_t n_heads;
    int32_t head_dim;
    float scale_log2;
    // q (for anchor-row gathers) and o: raw pointers + element strides
    const __nv_bfloat16* q;
    __nv_bfloat16* o;
    int64_t q_sb, q_sn, q_sh;
    int64_t o_sb, o_sn, o_sh;
    float* lse_out;
    PlanDev plan;
    int64_t cell_base;
    const uint32_t* work_list;
    const int32_t* n_work;
    uint32_t* sched;  // [2] dynamic-scheduler counters (zero on entry and on exit) or nullptr
    // Output scatter (csa_sparse_attn_fwd_scatter): when o_peer != nullptr, token t's output row
    // goes to o_peer[t / o_peer_tokens] at local token t % o_peer_tokens (strides o_s*), i.e.
    // straight into the sequence-sharded receive buffers of the ranks (Ulysses return exchange
    // fused into the epilogue); o is unused then.
    __nv_bfloat16* const* o_peer;
    int64_t o_peer_tokens;
};
cudaError_t set_attn_trace(void* buf, int mode);
cudaError_t launch_attn(const AttnArgs& a, int head_dim, const CUtensorMap& tq,
                        const CUtensorMap& tk, const CUtensorMap& tv, int grid,
                        cudaStream_t s);
// Fallback list of the fixed-reference kernels: work-list codes of items whose scores overshot
// their reference max, recomputed by attn_rect.cu's exact-max passes (modes 1 and 2).  count and flags (one bit per
// work-list index) zero on entry; list has room for every work-list entry.
struct Fallback {
    uint32_t* count;
    uint32_t* flags;
    uint32_t* list;
};
// Block 128 x 128, head_dim 128 or 64: one softmax group on every tile, SS S-MMAs (attn5.cu).
cudaError_t set_attn5_trace(void* buf, int mode);
cudaError_t launch_attn_sepp(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, int grid, const Fallback& fb,
                             cudaStream_t s);
// Non-square blocks B_q = 128 x B_kv (attn_rect.cu), head_dim 128.  mode 0: fixed reference
// max (first kept tile), overshooting items appended to fb; mode 1: exact row max of every item
// of the (fallback) list, parked in the item's first output row; mode 2: recompute the list
// against that max.  Modes 1 and 2 run with static assignment over fb's list.
cudaError_t launch_attn_rect(const AttnArgs& a, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, int grid, const Fallback& fb, int mode,
                             cudaStream_t s);
}  // namespace csa
