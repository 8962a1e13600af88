/*
 * csa.h -- C ABI of the B200 (sm_100a) calibrated-sparse-attention hot path.
 *
 * Paper: "Accelerating Text-to-Video Generation with Calibrated Sparse Attention"
 * (arxiv 2603.05503), cited as P:<line> of PAPER.md (section / equation).
 *
 * Three operations, in the order the method runs them:
 *   csa_calib_accumulate  -- calibration statistics: row LSE, block energy E_{r,c}
 *                            (Eq. eq:block_energy), per-prompt energy selection at eps(t)
 *                            (Eq. eq:row_energy_constraint), keep-count accumulation
 *                            (numerator of Eq. eq:mask_mean).
 *   csa_compile_plan      -- rho threshold (Eq. eq:mask_threshold), repetitive-head override
 *                            (P:624-626), skip lists / block lists (1D form P:947-950),
 *                            kept area (sparsity metric P:728);  csa_build_work_list orders one
 *                            launch's (head, query-block) items.
 *   csa_sparse_attn_fwd   -- block-sparse attention forward over the kept blocks and
 *                            anchor-row attention + broadcast for repetitive heads.
 * Also: csa_calib_accumulate_sim (calibration statistics and the repetitive-head similarity
 * statistic, in one pass), csa_spatial_similarity (the statistic alone, from a given
 * LSE), csa_merge_intervals / csa_share_timesteps (plan compaction),
 * csa_sparse_attn_fwd_scatter (attention whose output rows go straight to the ranks' receive
 * buffers: the head-sharded layer's return exchange fused into the epilogue), csa_validate_plan,
 * csa_copy_heads, csa_workspace_size.  Plans may omit the CSR index (intervals-only: the kernels
 * walk the 1-D interval lists).
 *
 * Conventions (all entry points):
 *   - Ownership: the caller owns every buffer (e.g. torch.empty on the device); the library never
 *     allocates device memory, never frees, and keeps no pointer past the enqueued work.
 *   - Asynchrony: work is enqueued on `stream`; no host synchronisation, except
 *     csa_validate_plan (documented).  Pointers are DEVICE pointers unless stated otherwise.
 *   - Errors: host-side argument checks return a status; csa_last_error() gives a thread-local
 *     detail string.  Device-side corruption is detected only by csa_validate_plan.
 *     Non-finite inputs are not scanned; NaN propagates.
 *   - Geometry (Eq. eq:indices P:196-204): N = frames*rows*cols video tokens in
 *     row-major (f, i, j) order; N_B = ceil(N / block); the last block may be ragged.
 *   - Tensors: bf16, layout [batch, N, heads, head_dim] given by element strides; head_dim
 *     contiguous; base and strides 16-byte aligned (TMA).
 *   - Supported: sm_100 devices; head_dim in {64, 128}; block in {64, 128}; N_B <= 2047.
 *   - Non-square blocks (block_kv != 0 and != block): every entry point accepts block 128,
 *     block_kv a multiple of 16 in [64, 192], N_Bkv <= 2047 (head_dim 128 for calibration and
 *     attention; csa_sparse_attn_fwd then needs its workspace).  csa_spatial_similarity (and the
 *     similarity part of csa_calib_accumulate_sim) ignores block_kv (the statistic is defined
 *     over all N keys).
 *     Everywhere below, "N_B x N_B" of a plan or keep-count cell reads "N_B x N_Bkv" (rows are
 *     query blocks, columns key blocks), and mask rows hold ceil(N_Bkv/32) words.
 */
#ifndef CSA_H
#define CSA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CSA_API __attribute__((visibility("default")))
#else
#define CSA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* csa_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    CSA_OK = 0,
    CSA_ERR_INVALID_ARGUMENT = 1,   /* shape / stride / alignment / range error */
    CSA_ERR_UNSUPPORTED = 2,        /* head_dim, block, size limit or device not supported */
    CSA_ERR_CORRUPT_PLAN = 3,       /* csa_validate_plan found an inconsistent plan */
    CSA_ERR_CUDA = 4,               /* a CUDA runtime/driver call failed (see csa_last_error) */
    CSA_ERR_INSUFFICIENT_CAPACITY = 5
} csa_status_t;

/* Video token grid and block sizes (128x128 blocks).  Non-square blocks
 * B_q x B_kv (Table tab:block_size_ablation): block = B_q, block_kv = B_kv; a plan's
 * rows are the N_B = ceil(N/B_q) query blocks, its columns the N_Bkv = ceil(N/B_kv) key blocks
 * (J_c = {j | c B_kv <= j < (c+1) B_kv}, clipped to N).  block_kv = 0 (or = block): square. */
typedef struct {
    int32_t frames;   /* F */
    int32_t rows;     /* H, spatial rows per frame */
    int32_t cols;     /* W, tokens per spatial row */
    int32_t block;    /* B_q (query block size; = key block size when block_kv is 0) */
    int32_t block_kv; /* B_kv, 0 -> block */
} csa_layout_t;

/* bf16 tensor [batch, N, heads, head_dim]; strides in ELEMENTS; head_dim stride is 1. */
typedef struct {
    void* ptr;
    int64_t stride_b;
    int64_t stride_n;
    int64_t stride_h;
} csa_tensor_t;

/* Compiled plan for n_cells cells (a cell is one (t, l, h); cell id chosen by the
 * caller, e.g. (t*L + l)*H + h).  Every pointer is a caller-allocated device buffer.
 *   kind        [n_cells]                0 = MASK, 1 = REPETITIVE (anchor rows)
 *   anchor_k    [n_cells]                anchor rows per frame (REPETITIVE only)
 *   mask_bits   [n_cells][N_B][ceil(N_B/32)] kept bit (r,c) = word c/32 bit c%32 (LSB first)
 *   blk_base    [n_cells + 1]            cell offset into blk_idx; blk_base[n_cells] = total
 *   blk_row_ptr [n_cells][N_B + 1]       CSR row pointers relative to blk_base[cell]
 *   blk_idx     [blk_capacity]           kept key-block indices c, ascending per row; OPTIONAL:
 *                                        NULL with blk_capacity 0 makes an intervals-only plan --
 *                                        the attention kernels then walk ivl (the 1-D skip list,
 *                                        P:947-950) and blk_row_ptr keeps only the row counts
 *   ivl_base    [n_cells + 1]            cell offset (in intervals) into ivl
 *   ivl_row_ptr [n_cells][N_B + 1]       interval row pointers relative to ivl_base[cell]
 *   ivl         [2 * ivl_capacity]       skip-list intervals (start, end) half-open, maximal runs
 *   kept_area   [n_cells]                sum over kept (r,c) of |I_r||J_c|; REPETITIVE: F*k*W*N
 * REPETITIVE cells have empty rows (row_ptr all 0) and mask_bits all 0 ("instead"). */
typedef struct {
    int64_t n_cells;
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
    int64_t blk_capacity; /* elements of blk_idx */
    int64_t ivl_capacity; /* intervals (pairs) of ivl */
} csa_plan_t;

/* Which workspace a call needs (csa_workspace_size). */
enum { CSA_WS_CALIB = 0, CSA_WS_COMPILE = 1, CSA_WS_WORK_LIST = 2, CSA_WS_ATTN = 3,
       CSA_WS_SIMILARITY = 4, CSA_WS_MERGE = 5, CSA_WS_CALIB_SIM = 6 };

/* ------------------------------------------------------------------------------------------
 * csa_calib_accumulate -- one calibration prompt at one (t, l), all heads.
 * For each head h and query block r:
 *   lse_i   = log sum_{j<N} exp(softmax_scale * q_i.k_j)              (dense P, Eq. eq:p)
 *             -- taken from lse_in when given (the dense calibration run's own statistic);
 *   E_{r,c} = (1/|I_r|) sum_{i in I_r} sum_{j in J_c} exp(s_ij - lse_i)  (Eq. eq:block_energy;
 *             divides by the actual |I_r| of a ragged last block), P never materialised;
 *   M_p[r,.] = shortest prefix of (E desc, c asc) whose fp64 sequential sum of the fp32 E values
 *             reaches eps (keep all if never reached; >= 1 block);
 *   keep_count[h][r][c] += M_p[r][c]  (uint16, saturating at 65535).
 * Arguments:
 *   q, k        bf16 [1, N, n_heads, head_dim] (batch index 0 only: conditional branch)
 *   lse_in      optional fp32 [n_heads][N] natural-log row LSE; NULL -> computed in-kernel
 *   eps         eps(t) computed by the caller (Eq. eq:epsilon_schedule), 0 < eps
 *   keep_count  uint16 [n_heads][N_B][N_B], accumulated in place
 *   energy_out  optional fp32 [n_heads][N_B][N_B] (the exact values the selection consumed)
 *   lse_out     optional fp32 [n_heads][N] (natural log; the values pass B used)
 * Workspace (device, 16-byte aligned, contents irrelevant): with lse_in == NULL and a buffer of
 * at least csa_workspace_size(CSA_WS_CALIB, L, n_heads, head_dim) bytes, the kernel makes ONE
 * exponential pass (per-(row, key block) partial sums kept there until the row LSE is known);
 * NULL -> two passes (LSE, then E), same results up to fp32 rounding order.  Ignored when lse_in
 * is given (one pass).  A non-NULL buffer that is too small -> CSA_ERR_INVALID_ARGUMENT. */
CSA_API csa_status_t csa_calib_accumulate(csa_layout_t L, int32_t n_heads, int32_t head_dim,
                                  float softmax_scale, csa_tensor_t q, csa_tensor_t k,
                                  const float* lse_in, double eps, uint16_t* keep_count,
                                  float* energy_out, float* lse_out, void* workspace,
                                  size_t workspace_bytes, csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_spatial_similarity -- the repetitive-head statistic of one calibration prompt (f1),
 * for every frame f and spatial row i, the cosine between P^(f,i) and P^(f,a(i)),
 * where P^(f,i) are the rows of the dense map P = softmax(softmax_scale Q K^T) (all N keys,
 * Eq. eq:p) of the W query tokens (f,i,0..W-1) and a(i) the nearest of the anchor rows
 * floor((2m+1)H/(2k)) (tie -> lower).  Readings (Q23-Q25): Frobenius cosine of the two
 * W x N blocks, query (f,i,j) paired with (f,a(i),j); the average runs over all (f,i).
 *   q, k        bf16 [1, N, n_heads, head_dim] (batch index 0)
 *   lse         fp32 [n_heads][N] natural-log row LSE of the same prompt (csa_calib_accumulate's
 *               lse_out, or the dense forward's) -- required
 *   sim_sum     fp64 [n_heads], accumulated in place: += sum over (f,i) of cos; after |D| prompts
 *               s[h] = sim_sum[h] / (F * H * |D|) is the `similarity` of csa_compile_plan
 *   cos_out     optional fp32 [n_heads][F*H] (this prompt's cos per (f,i))
 * P is never materialised (one pass over the key tiles per (head, query block)); reductions run
 * in a fixed order (bit-reproducible).  Workspace (required): csa_workspace_size(
 * CSA_WS_SIMILARITY, L, n_heads, head_dim) bytes, 16-byte aligned, contents irrelevant. */
CSA_API csa_status_t csa_spatial_similarity(csa_layout_t L, int32_t n_heads, int32_t head_dim,
                                    float softmax_scale, csa_tensor_t q, csa_tensor_t k,
                                    const float* lse, int32_t anchor_k, double* sim_sum,
                                    float* cos_out, void* workspace, size_t workspace_bytes,
                                    csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_calib_accumulate_sim -- csa_calib_accumulate (lse computed in-kernel) AND
 * csa_spatial_similarity of the same prompt in ONE pass over the key tiles per (head, query
 * block) (the similarity statistic is computed alongside the
 * calibration statistics): per key tile both S = Q K^T and the anchor tokens' scores
 * S_a = Q_a K^T, each score's exponential taken once.  Outputs and their definitions are those
 * of the two calls: keep_count (+= the selection at eps), optional energy_out / lse_out, sim_sum
 * (+= sum over (f,i) of cos), optional cos_out; equal to the two-call sequence up to fp32
 * rounding order (the selection is taken on this pass's own E).
 * Block 128 x 128 (head_dim 128 or 64) runs the fused kernel; other layouts run the two calls'
 * kernels in sequence (same results).  anchor_k in [1, rows].
 * Workspace (required): csa_workspace_size(CSA_WS_CALIB_SIM, L, n_heads, head_dim) bytes,
 * 16-byte aligned, contents irrelevant. */
CSA_API csa_status_t csa_calib_accumulate_sim(csa_layout_t L, int32_t n_heads, int32_t head_dim,
                                      float softmax_scale, csa_tensor_t q, csa_tensor_t k,
                                      double eps, uint16_t* keep_count, float* energy_out,
                                      float* lse_out, int32_t anchor_k, double* sim_sum,
                                      float* cos_out, void* workspace, size_t workspace_bytes,
                                      csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_compile_plan -- keep counts -> plan, for cells [0, n_cells).
 *   M[r,c] = keep_count[cell][r][c] >= min_count (Eq. eq:mask_threshold in count space:
 *            min_count = smallest integer >= rho*|D|, computed by the caller);
 *   a row emptied by the threshold re-keeps argmax_c count (tie -> lowest c);
 *   similarity (optional fp64 [n_cells]): s[cell] > gamma -> REPETITIVE with anchor_k rows.
 * Two phases on the same plan struct:
 *   phase 0 (COUNT): writes kind, anchor_k, mask_bits, row pointers, kept_area, blk_base,
 *                    ivl_base (blk_idx / ivl may be NULL).  The caller reads blk_base[n_cells]
 *                    and ivl_base[n_cells] to size blk_idx / ivl.
 *   phase 1 (FILL):  writes blk_idx (if not NULL) and ivl (writes beyond the capacities are
 *                    dropped; a plan filled with too small a capacity fails csa_validate_plan).
 * keep_count: uint16 [n_cells][N_B][N_B]. */
CSA_API csa_status_t csa_compile_plan(csa_layout_t L, int64_t n_cells, const uint16_t* keep_count,
                              int32_t min_count, const double* similarity, double gamma,
                              int32_t anchor_k, int32_t phase, const csa_plan_t* plan,
                              void* workspace, size_t workspace_bytes, csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_merge_intervals -- interval merging of a compiled plan (f2, Table
 * tab:skip_list_memory "Merge %").  target = nearest-rank `percentile`-th percentile (0 < p <=
 * 100) of the per-row interval counts over every row of the MASK cells [0, n_cells) (DESIGN.md
 * Q26); every row with more intervals fills its (count - target) smallest gaps, ties -> leftmost
 * (= repeated smallest-gap merging, Q28): the gap blocks' keep_count entries are set to
 * min_count, so csa_compile_plan on the same counts yields the merged plan (kept set superset of
 * the original, at most max(target, 1) intervals per row).  REPETITIVE cells are skipped.
 *   plan        compiled from keep_count with this min_count (read only)
 *   keep_count  uint16 [n_cells][N_B][N_B], updated in place
 *   target_out  device int32 (the width reached);  added_out device uint64, += blocks added
 * Workspace: csa_workspace_size(CSA_WS_MERGE, ...) bytes (device, 4-byte aligned). */
CSA_API csa_status_t csa_merge_intervals(csa_layout_t L, int64_t n_cells, const csa_plan_t* plan,
                                 double percentile, int32_t min_count, uint16_t* keep_count,
                                 int32_t* target_out, unsigned long long* added_out,
                                 void* workspace, size_t workspace_bytes, csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_share_timesteps -- timestep mask sharing (f2, Eq. eq:timestep_iou).  Cells
 * are (t, g) = t * n_groups + g for t < n_steps (g e.g. = l * n_heads + h).  Per group: the IoU
 * of the compiled masks' skipped-block sets for every pair (t1, t2) (1 when both are empty),
 * greedy cliques over t ascending -- t joins the earliest-created clique whose every member has
 * IoU >= tau with it (Q27), else opens one -- and the OR of each clique's kept masks written to
 * every member's keep_count as min_count * M_shared, so csa_compile_plan gives all members one
 * identical mask.  REPETITIVE cells: IoU -1 with everything, singleton cliques, counts untouched.
 *   plan         compiled from keep_count with this min_count (read only)
 *   keep_count   uint16 [n_steps * n_groups][N_B][N_B], updated in place
 *   cluster_out  device int32 [n_groups][n_steps] clique index (creation order)
 *   iou_out      device fp64 [n_groups][n_steps][n_steps] (required; also the scratch) */
CSA_API csa_status_t csa_share_timesteps(csa_layout_t L, int32_t n_groups, int32_t n_steps,
                                 const csa_plan_t* plan, double tau, int32_t min_count,
                                 uint16_t* keep_count, int32_t* cluster_out, double* iou_out,
                                 csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_build_work_list -- items of one attention launch over heads [0, n_heads) whose cells are
 * cell_base + h.  MASK head: items (h, r), r < N_B, cost = kept blocks of row r; REPETITIVE
 * head: items (h, u), u < ceil(F*k*W/128) anchor-query tiles, cost = N_B.
 * order 0: longest-first, ties (h asc, kind asc, index asc) -- a total order (unique output);
 * order 1: natural (h asc, index asc);
 * order 2: head-major, longest-first within a head (h asc, cost desc, index asc) -- the L2-local
 *          order the dynamic scheduler of csa_sparse_attn_fwd is built for;
 * order 3: PAIR items: item (h, p) stands for rows (2p, 2p+1) of a MASK head or anchor tiles
 *          (2p, 2p+1) of a REPETITIVE head, p < ceil(units/2), cost = sum of the members' costs;
 *          head-major, cost desc, p asc.  No attention kernel of this build consumes them
 *          (the pair-item kernel measured slower and was removed: DESIGN.md section 5).
 * Encoding: kind<<31 | h<<20 | (r, u or p).  work_list: uint32 [capacity]; n_work: device int32.
 * Requires n_heads <= 2048 and at most 32768 items. */
CSA_API csa_status_t csa_build_work_list(csa_layout_t L, const csa_plan_t* plan, int64_t cell_base,
                                 int32_t n_heads, int32_t order, uint32_t* work_list,
                                 int32_t capacity, int32_t* n_work, void* workspace,
                                 size_t workspace_bytes, csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_sparse_attn_fwd -- calibrated sparse attention of one layer at one timestep.
 * For batch b, head h (cell = cell_base + h), query token i in block r:
 *   MASK:       o_i = sum_{j in K_r} softmax_{j in K_r}(softmax_scale q_i.k_j) v_j with
 *               K_r = U_{c: M[r,c]=1} J_c (skipped blocks excluded from numerator and
 *               normaliser; skipped K/V blocks are never loaded), P:647-653;
 *   REPETITIVE: o[f,i,j] = dense attention of q[f, a(i), j] over all N keys, a(i) the nearest
 *               of the anchor rows floor((2m+1)H/(2k)) (tie -> lower).
 * The batch shares the plan (CFG branches).
 *   q, k, v, o  bf16 [batch, N, n_heads, head_dim]
 *   lse_out     optional fp32 [batch][n_heads][N], natural log over the kept keys
 *   work_list   items from csa_build_work_list; n_work device int32 (count)
 *   max_work    host upper bound of *n_work (sizes the persistent grid)
 *   pair_items  must be 0 (single items, orders 0-2); 1 -> CSA_ERR_UNSUPPORTED in this build.
 * Workspace: csa_workspace_size(CSA_WS_ATTN, L, n_heads, ...) bytes of device memory (8-byte
 * aligned).  Bytes [0, 256) hold the dynamic scheduler's counters: zero-filled before the first
 * use, left zero-filled when the launch completes (one buffer serves every launch on one stream).
 * NULL -> static round-robin assignment of work items to CTAs (block 64 only).
 * Kernels: block 128 x 128 (head_dim 128 or 64) runs attn5.cu, block 128 x block_kv runs
 * attn_rect.cu -- both with each row's softmax shift fixed at the max of its first kept tile
 * (P:647-653 is shift-invariant); the workspace is REQUIRED for block 128.  An item whose later
 * scores exceed that shift by more than 2^56 in exp2 terms is listed in bytes [256, size)
 * (rewritten every launch, needs max_work <= n_heads * N_B) and recomputed on the same stream by
 * attn_rect.cu's exact-row-max pass (the row max is parked in the first 4 bytes of the row's
 * first output row) and a pass against that max.  Block 64 runs attn.cu (running max).  Every
 * path is deterministic (bitwise run to run, independent of the item order). */
CSA_API csa_status_t csa_sparse_attn_fwd(csa_layout_t L, int32_t batch, int32_t n_heads,
                                 int32_t head_dim, float softmax_scale, csa_tensor_t q,
                                 csa_tensor_t k, csa_tensor_t v, csa_tensor_t o, float* lse_out,
                                 const csa_plan_t* plan, int64_t cell_base,
                                 const uint32_t* work_list, const int32_t* n_work,
                                 int32_t max_work, int32_t pair_items, void* workspace,
                                 size_t workspace_bytes, csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_sparse_attn_fwd_scatter -- csa_sparse_attn_fwd (same arithmetic, bit for bit) whose output
 * rows are written straight into the sequence-sharded receive buffers of n_peers ranks: the
 * row of token t goes to o_peers[t / (N / n_peers)] at local token t % (N / n_peers).  This fuses
 * the return all-to-all of the head-sharded (Ulysses) layer into the attention epilogue (SURVEY
 * 8.6; heads are independent): with symmetric / peer-mapped buffers the stores travel over
 * NVLink as each tile row is finished, and the consumer only needs a cross-rank barrier after
 * the launch (stream-ordered; the caller's).
 *   o_peers     DEVICE array [n_peers] of bf16 pointers (peer-accessible from this device),
 *               each pointing at THIS rank's first head inside peer p's receive buffer (e.g.
 *               recv_p + h0 * head_dim for a [batch, N / n_peers, H_total, head_dim] buffer);
 *               16-byte aligned
 *   o_stride_*  element strides of every receive buffer (batch, token, head); multiples of 8
 *   n_peers     >= 1, must divide N; block 128 layouts only (square or B_kv) -- the fallback
 *               passes scatter the same way
 * Other arguments as csa_sparse_attn_fwd (lse_out stays local, [batch][n_heads][N]). */
CSA_API csa_status_t csa_sparse_attn_fwd_scatter(csa_layout_t L, int32_t batch, int32_t n_heads,
                                         int32_t head_dim, float softmax_scale, csa_tensor_t q,
                                         csa_tensor_t k, csa_tensor_t v, void* const* o_peers,
                                         int32_t n_peers, int64_t o_stride_b, int64_t o_stride_n,
                                         int64_t o_stride_h, float* lse_out,
                                         const csa_plan_t* plan, int64_t cell_base,
                                         const uint32_t* work_list, const int32_t* n_work,
                                         int32_t max_work, void* workspace,
                                         size_t workspace_bytes, csa_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * csa_copy_heads -- runtime helper for streaming a layer through the API from host memory:
 * copies heads [h0, h1) of a bf16 [1, N, n_heads, head_dim] tensor (head_dim contiguous, rows of
 * n_heads * head_dim) between pinned host memory and device memory of the same layout, as one
 * strided cudaMemcpy2DAsync on `stream` (height N, pitch n_heads * head_dim * 2 bytes).
 * direction 0: host -> device (src host, dst device); 1: device -> host. */
CSA_API csa_status_t csa_copy_heads(void* dst, const void* src, csa_layout_t L, int32_t n_heads,
                            int32_t head_dim, int32_t h0, int32_t h1, int32_t direction,
                            csa_stream_t stream);

/* Workspace bytes for `which` (CSA_WS_*). */
CSA_API size_t csa_workspace_size(int32_t which, csa_layout_t L, int32_t n_heads, int32_t head_dim);

/* Structural check of cells [0, n_cells) of a plan: kind in {0 MASK, 1 REPETITIVE}; REPETITIVE
 * anchor_k in [1, rows]; blk_base[0] = ivl_base[0] = 0, bases non-negative, monotone and within
 * the capacities; every cell's row pointers start at 0, are monotone and stay inside the cell's
 * list; MASK rows non-empty with indices ascending and < N_B (N_Bkv) and set in mask_bits;
 * intervals maximal/ordered and equal to the decoded blk_idx (intervals-only plans: the intervals
 * cover exactly the row count, inside mask_bits).  No read leaves the plan's buffers
 * once a bound is found broken.  Synchronises `stream`.  CSA_OK or CSA_ERR_CORRUPT_PLAN. */
CSA_API csa_status_t csa_validate_plan(const csa_plan_t* plan, csa_layout_t L, int64_t n_cells,
                               csa_stream_t stream);

/* Thread-local detail of the last error returned on this thread ("" if none). */
CSA_API const char* csa_last_error(void);

/* Debug only: device buffer of 4*1024*8 uint64 receiving clock64() stamps of CTA 0's attention
 * pipeline events (softmax groups, S and P.V issue); NULL switches tracing off. */
CSA_API csa_status_t csa_debug_trace(void* buf, int32_t mode);

/* Library version string. */
CSA_API const char* csa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CSA_H */
