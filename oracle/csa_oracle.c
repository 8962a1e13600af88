/*
 * csa_oracle.c -- plain, slow, fp64 CPU oracle for the calibrated-sparse-attention hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_2603_05503_b200/csrc); neither includes the other.
 *
 * Every function cites the PAPER.md passage it writes out (P:<line>, section / equation).
 * Built with  gcc -O2 -ffp-contract=off -fPIC -shared  (no FMA contraction, no BLAS, no threads).
 * Inputs are the same bf16 values the GPU sees, widened exactly to double by the caller.
 *
 * Readings of silent/ambiguous passages are the DESIGN.md register Q1..Q22:
 *   Q1 skipped keys are -inf logits (excluded from numerator and normaliser)
 *   Q2 ragged last block: I_r / J_c clipped to N, E divides by |I_r|, keys >= N do not exist
 *   Q4 selection order (E desc, c asc); Q5 fp64 sequential cumulative sum, stop at >= eps,
 *      keep all if never reached, always >= 1 block
 *   Q6 rho threshold in count space: count >= min_count
 *   Q7 emptied row re-keeps argmax count (tie -> lowest c)
 *   Q8 strict s > gamma;  Q9 anchors a_m = floor((2m+1)H/(2k)), nearest, tie -> lower
 *   Q10 per-position broadcast (f,i,j) <- (f,a(i),j);  Q11 anchor queries see all N keys
 *
 * Pins (tests/test_oracle_*.py) fix these functions against brute force, closed forms and the
 * paper's printed values; a function without a pin says "parity unpinned" below.  None does.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1

/* ------------------------------------------------------------------------------------------ */
/* Geometry.  P:196-204 Eq. (eq:indices): I_r = {i | r B <= i < (r+1) B}, clipped to N (Q2).     */
/* ------------------------------------------------------------------------------------------ */
int64_t csao_num_blocks(int64_t n, int64_t b) { return (n + b - 1) / b; }

static int64_t blk_lo(int64_t r, int64_t b) { return r * b; }
static int64_t blk_hi(int64_t r, int64_t b, int64_t n) {
    int64_t h = (r + 1) * b;
    return h < n ? h : n;
}

/* token index of (frame f, spatial row i, column j) in row-major order. */
int64_t csao_token_index(int64_t H, int64_t W, int64_t f, int64_t i, int64_t j) {
    return f * H * W + i * W + j;
}

/* ------------------------------------------------------------------------------------------ */
/* a1. eps(t) schedule.  P:518-526 Eq. (eq:epsilon_schedule): eps(t) = A + (C-A) exp(-k t / T),  */
/* t = 0 the highest-noise step.  P:888-894: A(N) = 0.796 + 1.41e-6 N, C = 0.99, k = 16.          */
/* ------------------------------------------------------------------------------------------ */
double csao_A_of_N(double n) { return 0.796 + 1.41e-6 * n; }

double csao_epsilon(int32_t t, int32_t T, double A, double C, double k) {
    return A + (C - A) * exp(-k * (double)t / (double)T);
}

/* P:1045-1052 is the IoU of skipped sets; not on the hot path (NEXT f2). */

/* ------------------------------------------------------------------------------------------ */
/* Shared helper: logits of one query row against a key range.  P:176-178 Eq. (eq:p):          */
/* s_j = scale * <q_i, k_j>, summed over t ascending.                                          */
/* ------------------------------------------------------------------------------------------ */
static double dot_scaled(const double* qi, const double* kj, int32_t d, double scale) {
    double acc = 0.0;
    for (int32_t t = 0; t < d; ++t) acc += qi[t] * kj[t];
    return scale * acc;
}

/* ------------------------------------------------------------------------------------------ */
/* a7. Block-sparse attention, plain definition.  P:176-187 (Eq. eq:p, eq:pv): for     */
/* query block r the kept keys are the union of J_c over c with M[r,c] = 1; all other keys are   */
/* skipped (Q1: -inf logits).  Rows [row_begin,row_end) of one head; q,k,v are [N,d] row-major.  */
/* mask is [N_B * N_B] bytes (row r, col c) or NULL for the all-ones (dense) mask.              */
/* out: [(row_end-row_begin) * d]; lse (natural log, may be NULL): [(row_end-row_begin)].        */
/* ------------------------------------------------------------------------------------------ */
/* Non-square blocks B_q x B_kv: I_r uses B_q = bq, J_c uses B_kv = bk; mask is     */
/* [N_Bq * N_Bkv] bytes.  bq == bk is the square case above (csao_masked_attention_rows).         */
int csao_masked_attention_rows_rect(int64_t n, int32_t d, int32_t bq, int32_t bk, const double* q,
                                    const double* k, const double* v, double scale,
                                    const uint8_t* mask, int64_t row_begin, int64_t row_end,
                                    double* out, double* lse);

int csao_masked_attention_rows(int64_t n, int32_t d, int32_t b, const double* q, const double* k,
                               const double* v, double scale, const uint8_t* mask,
                               int64_t row_begin, int64_t row_end, double* out, double* lse) {
    return csao_masked_attention_rows_rect(n, d, b, b, q, k, v, scale, mask, row_begin, row_end,
                                           out, lse);
}

int csao_masked_attention_rows_rect(int64_t n, int32_t d, int32_t bq, int32_t bk, const double* q,
                                    const double* k, const double* v, double scale,
                                    const uint8_t* mask, int64_t row_begin, int64_t row_end,
                                    double* out, double* lse) {
    if (n <= 0 || d <= 0 || bq <= 0 || bk <= 0 || row_begin < 0 || row_end > n ||
        row_begin > row_end)
        return ORC_EINVAL;
    const int64_t nb = csao_num_blocks(n, bk); /* key blocks = mask columns */
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    uint8_t* keep = (uint8_t*)malloc((size_t)n);
    if (!s || !keep) { free(s); free(keep); return ORC_EINVAL; }
    for (int64_t i = row_begin; i < row_end; ++i) {
        const int64_t r = i / bq;
        /* kept key set K_r = U_{c : M[r,c]=1} J_c, j < N (Q2) */
        for (int64_t c = 0; c < nb; ++c) {
            const uint8_t m = mask ? mask[r * nb + c] : 1;
            for (int64_t j = blk_lo(c, bk); j < blk_hi(c, bk, n); ++j) keep[j] = m;
        }
        double mx = -INFINITY;
        int64_t nkeep = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (!keep[j]) continue;
            s[j] = dot_scaled(q + i * d, k + j * d, d, scale);
            if (s[j] > mx) mx = s[j];
            ++nkeep;
        }
        double* o = out + (i - row_begin) * d;
        if (nkeep == 0) { /* a plan never produces an empty row (Q7); define output as NaN */
            for (int32_t t = 0; t < d; ++t) o[t] = NAN;
            if (lse) lse[i - row_begin] = NAN;
            continue;
        }
        double l = 0.0;
        for (int32_t t = 0; t < d; ++t) o[t] = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (!keep[j]) continue;
            const double p = exp(s[j] - mx); /* softmax numerator, row-max shifted */
            l += p;
            for (int32_t t = 0; t < d; ++t) o[t] += p * v[j * d + t];
        }
        for (int32_t t = 0; t < d; ++t) o[t] /= l; /* A = P V with P row-normalised (Eq. eq:pv) */
        if (lse) lse[i - row_begin] = mx + log(l);
    }
    free(s);
    free(keep);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* a8. Anchor rows.  P:616-622: "select k equispaced anchor spatial rows per frame, compute     */
/* their attention against all keys and values, and broadcast each result to its nearest       */
/* spatial rows".  Reading Q9: a_m = floor((2m+1) H / (2k)); nearest anchor, tie -> lower m.    */
/* ------------------------------------------------------------------------------------------ */
int csao_anchor_rows(int32_t H, int32_t kA, int32_t* rows) {
    if (kA < 1 || kA > H) return ORC_EINVAL;
    for (int32_t m = 0; m < kA; ++m) rows[m] = (int32_t)(((int64_t)(2 * m + 1) * H) / (2 * kA));
    return ORC_OK;
}

int32_t csao_nearest_anchor(int32_t H, int32_t kA, int32_t i) {
    int32_t best = 0;
    int64_t bestd = -1;
    for (int32_t m = 0; m < kA; ++m) {
        const int64_t a = ((int64_t)(2 * m + 1) * H) / (2 * kA);
        const int64_t dd = a > i ? a - i : i - a;
        if (bestd < 0 || dd < bestd) { best = m; bestd = dd; } /* strict: tie keeps lower m */
    }
    return best;
}

/* Output rows [row_begin,row_end) (token indices) of a REPETITIVE head: row (f,i,j) receives
 * dense attention of query token (f, a_near(i), j) over all N keys (Q10, Q11).  P:616-622,656. */
int csao_anchor_attention_rows(int32_t F, int32_t H, int32_t W, int32_t d, const double* q,
                               const double* k, const double* v, double scale, int32_t kA,
                               int64_t row_begin, int64_t row_end, double* out, double* lse) {
    const int64_t n = (int64_t)F * H * W;
    if (kA < 1 || kA > H || row_begin < 0 || row_end > n || row_begin > row_end) return ORC_EINVAL;
    for (int64_t i = row_begin; i < row_end; ++i) {
        const int64_t f = i / ((int64_t)H * W);
        const int32_t row = (int32_t)((i / W) % H);
        const int64_t j = i % W;
        const int32_t m = csao_nearest_anchor(H, kA, row);
        const int32_t a = (int32_t)(((int64_t)(2 * m + 1) * H) / (2 * kA));
        const int64_t src = csao_token_index(H, W, f, a, j);
        /* dense attention of one query row over all N keys ("against all keys") */
        double mx = -INFINITY, l = 0.0;
        double* o = out + (i - row_begin) * d;
        double* s = (double*)malloc(sizeof(double) * (size_t)n);
        if (!s) return ORC_EINVAL;
        for (int64_t jj = 0; jj < n; ++jj) {
            s[jj] = dot_scaled(q + src * d, k + jj * d, d, scale);
            if (s[jj] > mx) mx = s[jj];
        }
        for (int32_t t = 0; t < d; ++t) o[t] = 0.0;
        for (int64_t jj = 0; jj < n; ++jj) {
            const double p = exp(s[jj] - mx);
            l += p;
            for (int32_t t = 0; t < d; ++t) o[t] += p * v[jj * d + t];
        }
        for (int32_t t = 0; t < d; ++t) o[t] /= l;
        if (lse) lse[i - row_begin] = mx + log(l);
        free(s);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* f1. Spatial similarity.  P:624-626: "We compute the cosine similarity between each P^(f,i)   */
/* and its nearest anchor row, then average over f, i, and the input prompts to obtain s".      */
/* P^(f,i) is the block of the dense map P (Eq. eq:p, all N keys) whose query rows are the W     */
/* tokens (f,i,0..W-1) of spatial row i of frame f.  Readings (DESIGN.md */
/* Q23-Q25): the cosine is that of the two W x N blocks flattened, pairing query (f,i,j) with    */
/* (f,a(i),j); the average runs over every (f,i) including the anchor rows themselves (cos 1);   */
/* a(i) is the nearest anchor of Q9.  This function returns cos for one (f,i) of one prompt.     */
/* ------------------------------------------------------------------------------------------ */
static int dense_prob_row(int64_t n, int32_t d, const double* qi, const double* k, double scale,
                          double* p) {
    double mx = -INFINITY;
    for (int64_t j = 0; j < n; ++j) {
        p[j] = dot_scaled(qi, k + j * d, d, scale);
        if (p[j] > mx) mx = p[j];
    }
    double l = 0.0;
    for (int64_t j = 0; j < n; ++j) l += exp(p[j] - mx);
    const double lse = mx + log(l);
    for (int64_t j = 0; j < n; ++j) p[j] = exp(p[j] - lse);
    return ORC_OK;
}

int csao_spatial_cos(int32_t F, int32_t H, int32_t W, int32_t d, const double* q, const double* k,
                     double scale, int32_t kA, int32_t f, int32_t i, double* cos_out) {
    const int64_t n = (int64_t)F * H * W;
    if (kA < 1 || kA > H || f < 0 || f >= F || i < 0 || i >= H) return ORC_EINVAL;
    const int32_t m = csao_nearest_anchor(H, kA, i);
    const int32_t a = (int32_t)(((int64_t)(2 * m + 1) * H) / (2 * kA));
    double* pi = (double*)malloc(sizeof(double) * (size_t)n);
    double* pa = (double*)malloc(sizeof(double) * (size_t)n);
    if (!pi || !pa) {
        free(pi);
        free(pa);
        return ORC_EINVAL;
    }
    double dot = 0.0, ni = 0.0, na = 0.0;
    for (int32_t j = 0; j < W; ++j) {
        dense_prob_row(n, d, q + csao_token_index(H, W, f, i, j) * d, k, scale, pi);
        dense_prob_row(n, d, q + csao_token_index(H, W, f, a, j) * d, k, scale, pa);
        for (int64_t t = 0; t < n; ++t) {
            dot += pi[t] * pa[t];
            ni += pi[t] * pi[t];
            na += pa[t] * pa[t];
        }
    }
    *cos_out = dot / (sqrt(ni) * sqrt(na));
    free(pi);
    free(pa);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* a2. Row log-sum-exp over all N keys of the dense map P (Eq. eq:p), two-pass:       */
/* lse_i = m_i + log sum_j exp(s_ij - m_i).  Rows [row_begin,row_end).                           */
/* ------------------------------------------------------------------------------------------ */
int csao_row_lse(int64_t n, int32_t d, const double* q, const double* k, double scale,
                 int64_t row_begin, int64_t row_end, double* lse) {
    if (row_begin < 0 || row_end > n || row_begin > row_end) return ORC_EINVAL;
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    if (!s) return ORC_EINVAL;
    for (int64_t i = row_begin; i < row_end; ++i) {
        double mx = -INFINITY;
        for (int64_t j = 0; j < n; ++j) {
            s[j] = dot_scaled(q + i * d, k + j * d, d, scale);
            if (s[j] > mx) mx = s[j];
        }
        double l = 0.0;
        for (int64_t j = 0; j < n; ++j) l += exp(s[j] - mx);
        lse[i - row_begin] = mx + log(l);
    }
    free(s);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* a3. Block energy.  P:495-507 Eq. (eq:block_energy):                                          */
/*   E_{r,c} = (1/|I_r|) sum_{i in I_r} sum_{j in J_c} P_ij,  P_ij = exp(s_ij - lse_i).         */
/* The paper writes 1/B; Q2 divides by the actual |I_r| so every row sums to 1.          */
/* Block rows [r_begin,r_end); E_out is [(r_end-r_begin) * N_B].  lse may be NULL (computed).    */
/* ------------------------------------------------------------------------------------------ */
/* Non-square blocks B_q x B_kv: I_r from bq, J_c from bk; E_out is             */
/* [(r_end-r_begin) * N_Bkv].  bq == bk is csao_block_energy_rows.                              */
int csao_block_energy_rows_rect(int64_t n, int32_t d, int32_t bq, int32_t bk, const double* q,
                                const double* k, double scale, const double* lse_in,
                                int64_t r_begin, int64_t r_end, double* E_out);

int csao_block_energy_rows(int64_t n, int32_t d, int32_t b, const double* q, const double* k,
                           double scale, const double* lse_in, int64_t r_begin, int64_t r_end,
                           double* E_out) {
    return csao_block_energy_rows_rect(n, d, b, b, q, k, scale, lse_in, r_begin, r_end, E_out);
}

int csao_block_energy_rows_rect(int64_t n, int32_t d, int32_t bq, int32_t b, const double* q,
                                const double* k, double scale, const double* lse_in,
                                int64_t r_begin, int64_t r_end, double* E_out) {
    const int64_t nb = csao_num_blocks(n, b); /* key blocks (columns) of width b = B_kv */
    if (r_begin < 0 || r_end > csao_num_blocks(n, bq) || r_begin > r_end) return ORC_EINVAL;
    for (int64_t r = r_begin; r < r_end; ++r) {
        double* E = E_out + (r - r_begin) * nb;
        for (int64_t c = 0; c < nb; ++c) E[c] = 0.0;
        const int64_t i0 = blk_lo(r, bq), i1 = blk_hi(r, bq, n);
        for (int64_t i = i0; i < i1; ++i) {
            double li;
            if (lse_in) li = lse_in[i];
            else if (csao_row_lse(n, d, q, k, scale, i, i + 1, &li) != ORC_OK) return ORC_EINVAL;
            for (int64_t c = 0; c < nb; ++c) {
                double acc = 0.0;
                for (int64_t j = blk_lo(c, b); j < blk_hi(c, b, n); ++j)
                    acc += exp(dot_scaled(q + i * d, k + j * d, d, scale) - li);
                E[c] += acc;
            }
        }
        for (int64_t c = 0; c < nb; ++c) E[c] /= (double)(i1 - i0);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* a4. Per-prompt selection.  P:509-515 Eq. (eq:row_energy_constraint) and P:532-533: "sorting  */
/* {E_rc}_c in descending order and selecting the smallest prefix whose cumulative energy       */
/* reaches eps(t)".  Q4: order (E desc, c asc).  Q5: acc in fp64, sequential in that order,     */
/* stop once acc >= eps; keep all if never reached; always >= 1 block.  kept[c] in {0,1}.        */
/* Returns the number of kept blocks.                                                          */
/* ------------------------------------------------------------------------------------------ */
static const double* g_sel_E; /* qsort has no context argument in C; single-threaded use */
static int cmp_desc_then_idx(const void* a, const void* b) {
    const int32_t ia = *(const int32_t*)a, ib = *(const int32_t*)b;
    const double ea = g_sel_E[ia], eb = g_sel_E[ib];
    if (ea > eb) return -1;
    if (ea < eb) return 1;
    return (ia < ib) ? -1 : (ia > ib);
}

int32_t csao_select(int32_t nb, const double* E_row, double eps, uint8_t* kept) {
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)nb);
    if (!order) return -1;
    for (int32_t c = 0; c < nb; ++c) { order[c] = c; kept[c] = 0; }
    g_sel_E = E_row;
    qsort(order, (size_t)nb, sizeof(int32_t), cmp_desc_then_idx);
    double acc = 0.0;
    int32_t cnt = 0;
    for (int32_t t = 0; t < nb; ++t) {
        kept[order[t]] = 1;
        ++cnt;
        acc += E_row[order[t]];
        if (acc >= eps) break;
    }
    free(order);
    return cnt;
}

/* ------------------------------------------------------------------------------------------ */
/* a5. Cross-prompt accumulation, numerator of Eq. (eq:mask_mean) P:544-554:                    */
/* count[r,c] += M_p[r,c].  Saturates at 65535 (uint16 storage).                                 */
/* ------------------------------------------------------------------------------------------ */
void csao_accumulate(int64_t len, const uint8_t* kept, uint16_t* count) {
    for (int64_t x = 0; x < len; ++x)
        if (kept[x] && count[x] != 0xFFFF) count[x] = (uint16_t)(count[x] + 1);
}

/* Smallest integer c with c >= rho * |D| (Eq. eq:mask_threshold P:557-566 in count space, Q6):
 * mean = c/|D| >= rho  <=>  c >= rho |D|.                                                     */
int32_t csao_min_count(double rho, int32_t n_prompts) {
    const double target = rho * (double)n_prompts;
    int32_t c = (int32_t)ceil(target);
    while (c > 0 && (double)(c - 1) >= target) --c;
    while ((double)c < target) ++c;
    return c;
}

/* ------------------------------------------------------------------------------------------ */
/* a6. Plan compile for one cell (t,l,h).                                                       */
/*   - REPETITIVE iff similarity given and s > gamma ("exceeds", Q8); "instead":  */
/*     such a cell carries no block mask (all outputs below zero except kind/kept_area).        */
/*   - else M[r,c] = count[r,c] >= min_count (Eq. eq:mask_threshold, Q6); an emptied row        */
/*     re-keeps argmax_c count, tie -> lowest c (Q7).                                           */
/*   - CSR of kept c ascending (the "compacted per-query-block key-block list");                */
/*   - skip-list intervals = maximal runs [start,end) of kept columns (1D form       */
/*     P:947-950);                                                                               */
/*   - kept_area = sum over kept (r,c) of |I_r||J_c| (P:728 sparsity metric), REPETITIVE:        */
/*     F*k*W*N (query rows computed x all keys).                                     */
/* Outputs (caller-sized): mask[N_B*N_B] bytes, blk_row_ptr[N_B+1], blk_idx[<=N_B*N_B],          */
/* ivl_row_ptr[N_B+1], ivl[2*N_B*N_B] (start,end pairs).                                       */
/* ------------------------------------------------------------------------------------------ */
/* Non-square blocks B_q x B_kv: rows r < N_Bq (|I_r| from bq), columns          */
/* c < N_Bkv (|J_c| from bk); count and mask are [N_Bq * N_Bkv], blk_row_ptr / ivl_row_ptr       */
/* [N_Bq + 1].  bq == bk is csao_compile_cell.                                                  */
int csao_compile_cell_rect(int64_t n, int32_t bq, int32_t bk, int32_t F, int32_t H, int32_t W,
                           const uint16_t* count, int32_t min_count, int32_t has_sim, double sim,
                           double gamma, int32_t anchor_k, uint8_t* kind, uint8_t* mask,
                           int32_t* blk_row_ptr, uint16_t* blk_idx, int32_t* ivl_row_ptr,
                           uint16_t* ivl, int64_t* kept_area);

int csao_compile_cell(int64_t n, int32_t b, int32_t F, int32_t H, int32_t W,
                      const uint16_t* count, int32_t min_count, int32_t has_sim, double sim,
                      double gamma, int32_t anchor_k, uint8_t* kind, uint8_t* mask,
                      int32_t* blk_row_ptr, uint16_t* blk_idx, int32_t* ivl_row_ptr,
                      uint16_t* ivl, int64_t* kept_area) {
    return csao_compile_cell_rect(n, b, b, F, H, W, count, min_count, has_sim, sim, gamma,
                                  anchor_k, kind, mask, blk_row_ptr, blk_idx, ivl_row_ptr, ivl,
                                  kept_area);
}

int csao_compile_cell_rect(int64_t n, int32_t bq, int32_t bk, int32_t F, int32_t H, int32_t W,
                           const uint16_t* count, int32_t min_count, int32_t has_sim, double sim,
                           double gamma, int32_t anchor_k, uint8_t* kind, uint8_t* mask,
                           int32_t* blk_row_ptr, uint16_t* blk_idx, int32_t* ivl_row_ptr,
                           uint16_t* ivl, int64_t* kept_area) {
    const int64_t nbq = csao_num_blocks(n, bq); /* rows: query blocks */
    const int64_t nb = csao_num_blocks(n, bk);  /* columns: key blocks */
    (void)H; /* anchor geometry only enters through F*k*W*N */
    if (has_sim && sim > gamma) {
        *kind = 1;
        memset(mask, 0, (size_t)(nbq * nb));
        for (int64_t r = 0; r <= nbq; ++r) { blk_row_ptr[r] = 0; ivl_row_ptr[r] = 0; }
        *kept_area = (int64_t)F * anchor_k * W * n;
        return ORC_OK;
    }
    *kind = 0;
    int64_t area = 0;
    int32_t nblk = 0, nivl = 0;
    for (int64_t r = 0; r < nbq; ++r) {
        const uint16_t* cr = count + r * nb;
        uint8_t* mr = mask + r * nb;
        int32_t any = 0;
        for (int64_t c = 0; c < nb; ++c) {
            mr[c] = (int32_t)cr[c] >= min_count ? 1 : 0;
            any |= mr[c];
        }
        if (!any) {
            int64_t best = 0;
            for (int64_t c = 1; c < nb; ++c)
                if (cr[c] > cr[best]) best = c;
            mr[best] = 1;
        }
        blk_row_ptr[r] = nblk;
        ivl_row_ptr[r] = nivl;
        for (int64_t c = 0; c < nb; ++c) {
            if (!mr[c]) continue;
            blk_idx[nblk++] = (uint16_t)c;
            area += (blk_hi(r, bq, n) - blk_lo(r, bq)) * (blk_hi(c, bk, n) - blk_lo(c, bk));
            if (c == 0 || !mr[c - 1]) { ivl[2 * nivl] = (uint16_t)c; }
            if (c == nb - 1 || !mr[c + 1]) { ivl[2 * nivl + 1] = (uint16_t)(c + 1); ++nivl; }
        }
    }
    blk_row_ptr[nbq] = nblk;
    ivl_row_ptr[nbq] = nivl;
    *kept_area = area;
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* f2. Plan memory compaction (Table tab:skip_list_memory).             */
/* Interval merging: "progressively merging nearby intervals, which intentionally      */
/* marks a small number of additional blocks for computation"; the merge percentile p of the    */
/* table sets the target row width.  Readings (Q26-Q28): target = nearest-rank p-th    */
/* percentile of the per-row interval counts over all rows of the collection; a row above the   */
/* target repeatedly merges the adjacent pair with the smallest gap (leftmost on ties), the gap */
/* blocks becoming kept, until its count <= target.                                             */
/* ------------------------------------------------------------------------------------------ */
static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* nearest-rank percentile: sorted ascending, element ceil(p/100 * n) (1-based), p in (0,100] */
int32_t csao_percentile_nearest_rank(int64_t n, const int32_t* values, double p) {
    if (n <= 0 || !(p > 0.0) || p > 100.0) return -1;
    int32_t* v = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    if (!v) return -1;
    memcpy(v, values, sizeof(int32_t) * (size_t)n);
    qsort(v, (size_t)n, sizeof(int32_t), cmp_i32);
    int64_t rank = (int64_t)ceil(p / 100.0 * (double)n);
    if (rank < 1) rank = 1;
    const int32_t out = v[rank - 1];
    free(v);
    return out;
}

/* ivl: [n][2] half-open (start, end), ascending, disjoint, non-adjacent; merged in place.
 * Returns the new interval count; *added = blocks newly marked kept. */
int32_t csao_merge_row(int32_t n, uint16_t* ivl, int32_t target, int64_t* added) {
    *added = 0;
    while (n > target && n > 1) {
        int32_t best = 0;
        int32_t best_gap = (int32_t)ivl[2] - (int32_t)ivl[1];
        for (int32_t i = 1; i + 1 < n; ++i) {
            const int32_t gap = (int32_t)ivl[2 * (i + 1)] - (int32_t)ivl[2 * i + 1];
            if (gap < best_gap) { best = i; best_gap = gap; } /* strict: leftmost on ties */
        }
        *added += best_gap;
        ivl[2 * best + 1] = ivl[2 * (best + 1) + 1];
        for (int32_t i = best + 1; i + 1 < n; ++i) {
            ivl[2 * i] = ivl[2 * (i + 1)];
            ivl[2 * i + 1] = ivl[2 * (i + 1) + 1];
        }
        --n;
    }
    return n;
}

/* Timestep sharing: IoU of the skipped-block sets (Eq. eq:timestep_iou); greedy
 * cliques: timesteps in ascending order, each joins the earliest-created cluster whose every
 * member has IoU >= tau with it (Q27: the table caption's ">= tau"), else opens a new one; the
 * cluster's shared mask is the OR of the members' kept-block masks. */
double csao_skipped_iou(int64_t len, const uint8_t* kept1, const uint8_t* kept2) {
    int64_t inter = 0, uni = 0;
    for (int64_t x = 0; x < len; ++x) {
        const int s1 = !kept1[x], s2 = !kept2[x];
        inter += s1 & s2;
        uni += s1 | s2;
    }
    return uni == 0 ? 1.0 : (double)inter / (double)uni;
}

/* iou: [T][T]; cluster_out[t] = index of t's cluster (clusters numbered by creation order).
 * Returns the number of clusters. */
int32_t csao_cluster_timesteps(int32_t T, const double* iou, double tau, int32_t* cluster_out) {
    int32_t n_clusters = 0;
    for (int32_t t = 0; t < T; ++t) {
        int32_t joined = -1;
        for (int32_t c = 0; c < n_clusters && joined < 0; ++c) {
            int32_t ok = 1;
            for (int32_t u = 0; u < t && ok; ++u)
                if (cluster_out[u] == c && !(iou[t * T + u] >= tau)) ok = 0;
            if (ok) joined = c;
        }
        cluster_out[t] = joined >= 0 ? joined : n_clusters++;
    }
    return n_clusters;
}

/* ------------------------------------------------------------------------------------------ */
/* Work list for one launch over n_heads consecutive cells (not in the paper: the scheduling    */
/* artefact of DESIGN.md; its order is a total order so the output is unique).                 */
/*   MASK head h: items (h, r) for r < N_B, cost = nnz of row r;                                */
/*   REPETITIVE head h: items (h, u) for u < ceil(F*k*W/128), cost = N_B.                        */
/* order 0: (cost desc, h asc, kind asc, r-or-u asc); order 1: (h asc, r-or-u asc);             */
/* order 2: (h asc, cost desc, r-or-u asc).  Encoded kind<<31 | h<<20 | (r or u).               */
/* order 3: pair items p (members 2p, 2p+1), cost = members' sum, sorted as order 2.            */
/* row_nnz: [n_heads * N_B] (ignored for REPETITIVE heads).  Returns item count, -1 on error.   */
/* ------------------------------------------------------------------------------------------ */
typedef struct { int64_t cost; uint32_t code; } orc_item;
static int g_order; /* qsort has no context argument; single-threaded use */
static int cmp_item(const void* a, const void* b) {
    const orc_item* x = (const orc_item*)a;
    const orc_item* y = (const orc_item*)b;
    const uint32_t hx = (x->code >> 20) & 0x7FF, hy = (y->code >> 20) & 0x7FF;
    if (g_order != 0 && hx != hy) return hx < hy ? -1 : 1;
    if (g_order != 1 && x->cost != y->cost) return x->cost > y->cost ? -1 : 1;
    /* h, kind, index are laid out so that code order == (h asc, kind asc, idx asc) */
    const uint32_t kx = ((x->code >> 20) & 0x7FF) << 21 | (x->code >> 31) << 20 | (x->code & 0xFFFFF);
    const uint32_t ky = ((y->code >> 20) & 0x7FF) << 21 | (y->code >> 31) << 20 | (y->code & 0xFFFFF);
    return (kx < ky) ? -1 : (kx > ky);
}

int64_t csao_work_list(int32_t n_heads, int64_t n, int32_t b, int32_t F, int32_t W,
                       const uint8_t* kinds, const int32_t* anchor_k, const int32_t* row_nnz,
                       int32_t order, uint32_t* out, int64_t capacity) {
    const int64_t nb = csao_num_blocks(n, b);
    const int pairs = (order == 3);
    int64_t total = 0;
    for (int32_t h = 0; h < n_heads; ++h) {
        const int64_t units = kinds[h] ? ((int64_t)F * anchor_k[h] * W + 127) / 128 : nb;
        total += pairs ? (units + 1) / 2 : units;
    }
    if (total > capacity) return -1;
    orc_item* it = (orc_item*)malloc(sizeof(orc_item) * (size_t)(total ? total : 1));
    if (!it) return -1;
    int64_t x = 0;
    for (int32_t h = 0; h < n_heads && pairs; ++h) {
        /* order 3: item p = members 2p, 2p+1; cost = sum of the existing members' costs */
        const int64_t units = kinds[h] ? ((int64_t)F * anchor_k[h] * W + 127) / 128 : nb;
        for (int64_t p = 0; 2 * p < units; ++p) {
            int64_t cost = 0;
            for (int64_t u = 2 * p; u < 2 * p + 2 && u < units; ++u)
                cost += kinds[h] ? nb : row_nnz[(int64_t)h * nb + u];
            it[x].cost = cost;
            it[x].code = ((kinds[h] ? 1u : 0u) << 31) | ((uint32_t)h << 20) | (uint32_t)p;
            ++x;
        }
    }
    for (int32_t h = 0; h < n_heads && !pairs; ++h) {
        if (kinds[h]) {
            const int64_t nu = ((int64_t)F * anchor_k[h] * W + 127) / 128;
            for (int64_t u = 0; u < nu; ++u) {
                it[x].cost = nb;
                it[x].code = (1u << 31) | ((uint32_t)h << 20) | (uint32_t)u;
                ++x;
            }
        } else {
            for (int64_t r = 0; r < nb; ++r) {
                it[x].cost = row_nnz[(int64_t)h * nb + r];
                it[x].code = ((uint32_t)h << 20) | (uint32_t)r;
                ++x;
            }
        }
    }
    g_order = order;
    qsort(it, (size_t)total, sizeof(orc_item), cmp_item);
    for (int64_t y = 0; y < total; ++y) out[y] = it[y].code;
    free(it);
    return total;
}
