// api.cu -- the C ABI of include/csa.h: argument validation, TMA descriptor encoding, launches.
// No allocation, no host synchronisation (except csa_validate_plan), thread-local error text.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include <cudaTypedefs.h>

#include "csa_internal.cuh"

namespace {

thread_local std::string g_err;

csa_status_t fail(csa_status_t st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

csa_status_t ok() {
    g_err.clear();
    return CSA_OK;
}

csa_status_t cuda_fail(cudaError_t e, const char* what) {
    return fail(CSA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

struct DeviceInfo {
    int sms = 0;
    bool sm100 = false;
};

csa_status_t device_info(DeviceInfo* out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int major = 0, minor = 0, sms = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    out->sms = sms;
    out->sm100 = (major == 10 && minor == 0);
    if (!out->sm100)
        return fail(CSA_ERR_UNSUPPORTED, "device is sm_%d%d; this library is built for sm_100a",
                    major, minor);
    return CSA_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 4-D map over [batch, N, heads, D] bf16 (dims innermost first: d, h, n, b), box (64,1,rows,1),
// SWIZZLE_128B, out-of-bounds rows zero-filled (ragged last block).
csa_status_t make_map(CUtensorMap* map, const csa_tensor_t& t, int32_t batch, int32_t n,
                      int32_t heads, int32_t d, int32_t box_rows, const char* name) {
    auto enc = encode_fn();
    if (!enc) return fail(CSA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (!t.ptr) return fail(CSA_ERR_INVALID_ARGUMENT, "%s: null pointer", name);
    if (reinterpret_cast<uintptr_t>(t.ptr) % 16)
        return fail(CSA_ERR_INVALID_ARGUMENT, "%s: base not 16-byte aligned", name);
    int64_t sb = t.stride_b, sn = t.stride_n, sh = t.stride_h;
    if (batch == 1) sb = sn * n;  // unused dimension: any legal stride
    if (heads == 1) sh = d;
    if (sn <= 0 || sh <= 0 || sb <= 0 || (sn * 2) % 16 || (sh * 2) % 16 || (sb * 2) % 16)
        return fail(CSA_ERR_INVALID_ARGUMENT,
                    "%s: strides (b=%lld n=%lld h=%lld elements) must be positive and 16-byte "
                    "multiples", name, (long long)t.stride_b, (long long)t.stride_n,
                    (long long)t.stride_h);
    cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)heads, (cuuint64_t)n, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)(sh * 2), (cuuint64_t)(sn * 2), (cuuint64_t)(sb * 2)};
    cuuint32_t box[4] = {64, 1, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, t.ptr, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(CSA_ERR_INVALID_ARGUMENT, "%s: cuTensorMapEncodeTiled failed (%d)", name,
                    (int)r);
    return CSA_OK;
}

csa_status_t check_layout(const csa_layout_t& L, int32_t head_dim, int32_t n_heads) {
    if (L.frames <= 0 || L.rows <= 0 || L.cols <= 0)
        return fail(CSA_ERR_INVALID_ARGUMENT, "layout: frames/rows/cols must be positive");
    if (L.block != 64 && L.block != 128)
        return fail(CSA_ERR_UNSUPPORTED, "layout: block %d not in {64, 128}", L.block);
    const int64_t n = (int64_t)L.frames * L.rows * L.cols;
    if (n >= (1LL << 31)) return fail(CSA_ERR_UNSUPPORTED, "layout: N too large");
    if ((n + L.block - 1) / L.block > csa::kMaxBlocks)
        return fail(CSA_ERR_UNSUPPORTED, "layout: N_B > %d", csa::kMaxBlocks);
    if (L.block_kv != 0 && L.block_kv != L.block) {  // non-square B_q x B_kv
        if (L.block != 128 || L.block_kv < 64 || L.block_kv > 192 || L.block_kv % 16 != 0)
            return fail(CSA_ERR_UNSUPPORTED,
                        "layout: block %d x block_kv %d (non-square needs block 128, block_kv a "
                        "multiple of 16 in [64, 192])", L.block, L.block_kv);
        if ((n + L.block_kv - 1) / L.block_kv > csa::kMaxBlocks)
            return fail(CSA_ERR_UNSUPPORTED, "layout: N_Bkv > %d", csa::kMaxBlocks);
    } else if (L.block_kv < 0) {
        return fail(CSA_ERR_INVALID_ARGUMENT, "layout: block_kv < 0");
    }
    if (head_dim != 0 && head_dim != 64 && head_dim != 128)
        return fail(CSA_ERR_UNSUPPORTED, "head_dim %d not in {64, 128}", head_dim);
    if (n_heads < 0 || n_heads > 2048)
        return fail(CSA_ERR_UNSUPPORTED, "n_heads %d outside [0, 2048]", n_heads);
    return CSA_OK;
}

bool is_square(const csa_layout_t& L) { return L.block_kv == 0 || L.block_kv == L.block; }

bool plan_ptrs_ok(const csa_plan_t* p, bool need_lists) {
    if (!p || !p->kind || !p->anchor_k || !p->mask_bits || !p->blk_base || !p->blk_row_ptr ||
        !p->ivl_base || !p->ivl_row_ptr || !p->kept_area)
        return false;
    // blk_idx may be absent (intervals-only plan: blk_capacity 0); the intervals may not
    if (need_lists && (!p->ivl || (!p->blk_idx && p->blk_capacity != 0))) return false;
    return true;
}

__device__ uint32_t g_validate_flag;
std::mutex g_validate_mu;

}  // namespace

extern "C" {

const char* csa_last_error(void) { return g_err.c_str(); }

const char* csa_version(void) { return "csa-b200 0.1 (sm_100a)"; }

csa_status_t csa_debug_trace(void* buf, int32_t mode) {
    cudaError_t e = csa::set_attn_trace(buf, mode);
    if (e == cudaSuccess) e = csa::set_attn5_trace(buf, mode);
    if (e == cudaSuccess) e = csa::set_calib_trace(buf, mode);
    if (e == cudaSuccess) e = csa::set_calib_sim_trace(buf, mode);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyToSymbol");
    return ok();
}

size_t csa_workspace_size(int32_t which, csa_layout_t L, int32_t n_heads, int32_t head_dim) {
    (void)head_dim;
    if (which == CSA_WS_ATTN) {  // dynamic-scheduler counters + the fixed-reference kernel's
                                 // fallback list (count, item bitmap, codes; <= heads*N_B items)
        if (n_heads < 1 || check_layout(L, 0, 0) != CSA_OK) return 256;
        const size_t items = (size_t)n_heads * (size_t)csa::make_geo(L).NB;
        return 256 + 4 * (1 + (items + 31) / 32 + items);
    }
    if (which == CSA_WS_MERGE) {          // interval-width histogram
        if (check_layout(L, 0, 0) != CSA_OK) return 0;
        return (size_t)(csa::make_geo(L).NBK + 1) * sizeof(int32_t);
    }
    if (which == CSA_WS_SIMILARITY) {     // per-token (dot, |p|^2, |p_a|^2) partials
        if (check_layout(L, 0, 0) != CSA_OK || n_heads < 1) return 0;
        return (size_t)n_heads * (size_t)L.frames * L.rows * L.cols * 3 * sizeof(float);
    }
    if (which == CSA_WS_CALIB_SIM) {       // fused pass: row partials + similarity partials
        if (check_layout(L, 0, 0) != CSA_OK || n_heads < 1) return 0;
        DeviceInfo di;
        if (device_info(&di) != CSA_OK) return 0;
        const csa::Geo g = csa::make_geo(L);
        size_t scr = csa::calib_scratch_bytes(g, n_heads, di.sms);  // >= the fused kernel's
        scr = (scr + 255) / 256 * 256;
        csa_layout_t sq = L;
        sq.block_kv = 0;
        // + an LSE buffer for layouts that run the two calls' kernels in sequence
        return scr + csa_workspace_size(CSA_WS_SIMILARITY, sq, n_heads, head_dim) +
               (size_t)n_heads * g.N * sizeof(float);
    }
    if (which == CSA_WS_CALIB) {           // single-pass calibration: per-(row, key block) log2-sum-exp
        if (check_layout(L, 0, 0) != CSA_OK || n_heads < 1) return 0;
        DeviceInfo di;
        if (device_info(&di) != CSA_OK) return 0;
        return csa::calib_scratch_bytes(csa::make_geo(L), n_heads, di.sms);
    }
    return 0;
}

csa_status_t csa_calib_accumulate(csa_layout_t L, int32_t n_heads, int32_t head_dim,
                                  float softmax_scale, csa_tensor_t q, csa_tensor_t k,
                                  const float* lse_in, double eps, uint16_t* keep_count,
                                  float* energy_out, float* lse_out, void* workspace,
                                  size_t workspace_bytes, csa_stream_t stream) {
    csa_status_t st = check_layout(L, head_dim, n_heads);
    if (st != CSA_OK) return st;
    if (!is_square(L) && head_dim != 128)
        return fail(CSA_ERR_UNSUPPORTED, "non-square calibration needs head_dim 128");
    if (n_heads < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "n_heads must be >= 1");
    if (!(softmax_scale > 0.0f)) return fail(CSA_ERR_INVALID_ARGUMENT, "softmax_scale <= 0");
    if (!(eps > 0.0)) return fail(CSA_ERR_INVALID_ARGUMENT, "eps must be > 0");
    if (!keep_count) return fail(CSA_ERR_INVALID_ARGUMENT, "keep_count is null");
    DeviceInfo di;
    if ((st = device_info(&di)) != CSA_OK) return st;
    const csa::Geo g = csa::make_geo(L);
    CUtensorMap tq, tk;
    if ((st = make_map(&tq, q, 1, g.N, n_heads, head_dim, g.B, "q")) != CSA_OK) return st;
    if ((st = make_map(&tk, k, 1, g.N, n_heads, head_dim, g.BK, "k")) != CSA_OK) return st;
    csa::CalibArgs a;
    a.g = g;
    a.n_heads = n_heads;
    a.scale_log2 = softmax_scale * 1.4426950408889634f;
    a.lse_in = lse_in;
    a.eps = eps;
    a.keep_count = keep_count;
    a.energy_out = energy_out;
    a.lse_out = lse_out;
    a.scratch = nullptr;
    if (workspace != nullptr && lse_in == nullptr) {
        const size_t need = csa::calib_scratch_bytes(g, n_heads, di.sms);
        if (workspace_bytes < need)
            return fail(CSA_ERR_INVALID_ARGUMENT, "calibration workspace smaller than "
                                                  "csa_workspace_size(CSA_WS_CALIB)");
        if (reinterpret_cast<uintptr_t>(workspace) % 16 != 0)
            return fail(CSA_ERR_INVALID_ARGUMENT, "workspace must be 16-byte aligned");
        a.scratch = static_cast<float2*>(workspace);
    }
    cudaError_t e = csa::launch_calib(a, head_dim, tq, tk, di.sms, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "calib launch");
    return ok();
}

csa_status_t csa_calib_accumulate_sim(csa_layout_t L, int32_t n_heads, int32_t head_dim,
                                      float softmax_scale, csa_tensor_t q, csa_tensor_t k,
                                      double eps, uint16_t* keep_count, float* energy_out,
                                      float* lse_out, int32_t anchor_k, double* sim_sum,
                                      float* cos_out, void* workspace, size_t workspace_bytes,
                                      csa_stream_t stream) {
    csa_status_t st = check_layout(L, head_dim, n_heads);
    if (st != CSA_OK) return st;
    if (n_heads < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "n_heads must be >= 1");
    if (!(softmax_scale > 0.0f)) return fail(CSA_ERR_INVALID_ARGUMENT, "softmax_scale <= 0");
    if (!(eps > 0.0)) return fail(CSA_ERR_INVALID_ARGUMENT, "eps must be > 0");
    if (!keep_count || !sim_sum)
        return fail(CSA_ERR_INVALID_ARGUMENT, "keep_count and sim_sum are required");
    if (anchor_k < 1 || anchor_k > L.rows)
        return fail(CSA_ERR_INVALID_ARGUMENT, "anchor_k %d outside [1, rows=%d]", anchor_k, L.rows);
    const size_t need = csa_workspace_size(CSA_WS_CALIB_SIM, L, n_heads, head_dim);
    if (!workspace || workspace_bytes < need)
        return fail(CSA_ERR_INVALID_ARGUMENT,
                    "workspace smaller than csa_workspace_size(CSA_WS_CALIB_SIM) = %zu", need);
    if (reinterpret_cast<uintptr_t>(workspace) % 16 != 0)
        return fail(CSA_ERR_INVALID_ARGUMENT, "workspace must be 16-byte aligned");
    if (!q.ptr || (q.stride_n * 2) % 16 || (q.stride_h * 2) % 16)
        return fail(CSA_ERR_INVALID_ARGUMENT, "q: null or strides not 16-byte multiples");
    DeviceInfo di;
    if ((st = device_info(&di)) != CSA_OK) return st;
    const csa::Geo g = csa::make_geo(L);
    size_t scr = (csa::calib_scratch_bytes(g, n_heads, di.sms) + 255) / 256 * 256;
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    csa_layout_t sq = L;
    sq.block_kv = 0;
    const size_t part_bytes = csa_workspace_size(CSA_WS_SIMILARITY, sq, n_heads, head_dim);
    if (!(is_square(L) && L.block == 128 && (head_dim == 128 || head_dim == 64))) {
        // other layouts: the two calls' kernels in sequence on the same stream
        float* lse = lse_out ? lse_out : reinterpret_cast<float*>(ws + scr + part_bytes);
        st = csa_calib_accumulate(L, n_heads, head_dim, softmax_scale, q, k, nullptr, eps,
                                  keep_count, energy_out, lse, ws, scr, stream);
        if (st != CSA_OK) return st;
        return csa_spatial_similarity(sq, n_heads, head_dim, softmax_scale, q, k, lse, anchor_k,
                                      sim_sum, cos_out, ws + scr, part_bytes, stream);
    }
    CUtensorMap tq, tk;
    if ((st = make_map(&tq, q, 1, g.N, n_heads, head_dim, g.B, "q")) != CSA_OK) return st;
    if ((st = make_map(&tk, k, 1, g.N, n_heads, head_dim, g.B, "k")) != CSA_OK) return st;
    csa::CalibArgs a;
    a.g = g;
    a.n_heads = n_heads;
    a.scale_log2 = softmax_scale * 1.4426950408889634f;
    a.lse_in = nullptr;
    a.eps = eps;
    a.keep_count = keep_count;
    a.energy_out = energy_out;
    a.lse_out = lse_out;
    a.scratch = reinterpret_cast<float2*>(ws);
    csa::SimArgs s;
    s.g = g;
    s.n_heads = n_heads;
    s.scale_log2 = a.scale_log2;
    s.q = static_cast<const __nv_bfloat16*>(q.ptr);
    s.q_sn = q.stride_n;
    s.q_sh = q.stride_h;
    s.lse = nullptr;
    s.anchor_k = anchor_k;
    s.partials = reinterpret_cast<float*>(ws + scr);
    s.sim_sum = sim_sum;
    s.cos_out = cos_out;
    cudaError_t e = csa::launch_calib_sim(a, s, head_dim, tq, tk, di.sms, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "calibration + similarity launch");
    return ok();
}

csa_status_t csa_spatial_similarity(csa_layout_t L, int32_t n_heads, int32_t head_dim,
                                    float softmax_scale, csa_tensor_t q, csa_tensor_t k,
                                    const float* lse, int32_t anchor_k, double* sim_sum,
                                    float* cos_out, void* workspace, size_t workspace_bytes,
                                    csa_stream_t stream) {
    csa_status_t st = check_layout(L, head_dim, n_heads);
    if (st != CSA_OK) return st;
    L.block_kv = 0;  // s is defined over all N keys: independent of B_kv
    if (n_heads < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "n_heads must be >= 1");
    if (!(softmax_scale > 0.0f)) return fail(CSA_ERR_INVALID_ARGUMENT, "softmax_scale <= 0");
    if (anchor_k < 1 || anchor_k > L.rows)
        return fail(CSA_ERR_INVALID_ARGUMENT, "anchor_k %d outside [1, rows=%d]", anchor_k, L.rows);
    if (!lse || !sim_sum) return fail(CSA_ERR_INVALID_ARGUMENT, "lse and sim_sum are required");
    const size_t need = csa_workspace_size(CSA_WS_SIMILARITY, L, n_heads, head_dim);
    if (!workspace || workspace_bytes < need)
        return fail(CSA_ERR_INVALID_ARGUMENT,
                    "workspace smaller than csa_workspace_size(CSA_WS_SIMILARITY) = %zu", need);
    if (reinterpret_cast<uintptr_t>(workspace) % 16 != 0)
        return fail(CSA_ERR_INVALID_ARGUMENT, "workspace must be 16-byte aligned");
    if (!q.ptr || (q.stride_n * 2) % 16 || (q.stride_h * 2) % 16)
        return fail(CSA_ERR_INVALID_ARGUMENT, "q: null or strides not 16-byte multiples");
    DeviceInfo di;
    if ((st = device_info(&di)) != CSA_OK) return st;
    const csa::Geo g = csa::make_geo(L);
    CUtensorMap tq, tk;
    if ((st = make_map(&tq, q, 1, g.N, n_heads, head_dim, g.B, "q")) != CSA_OK) return st;
    if ((st = make_map(&tk, k, 1, g.N, n_heads, head_dim, g.B, "k")) != CSA_OK) return st;
    csa::SimArgs a;
    a.g = g;
    a.n_heads = n_heads;
    a.scale_log2 = softmax_scale * 1.4426950408889634f;
    a.q = static_cast<const __nv_bfloat16*>(q.ptr);
    a.q_sn = q.stride_n;
    a.q_sh = q.stride_h;
    a.lse = lse;
    a.anchor_k = anchor_k;
    a.partials = static_cast<float*>(workspace);
    a.sim_sum = sim_sum;
    a.cos_out = cos_out;
    cudaError_t e = csa::launch_similarity(a, head_dim, tq, tk, di.sms, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "similarity launch");
    return ok();
}

csa_status_t csa_merge_intervals(csa_layout_t L, int64_t n_cells, const csa_plan_t* plan,
                                 double percentile, int32_t min_count, uint16_t* keep_count,
                                 int32_t* target_out, unsigned long long* added_out,
                                 void* workspace, size_t workspace_bytes, csa_stream_t stream) {
    csa_status_t st = check_layout(L, 0, 0);
    if (st != CSA_OK) return st;
    if (n_cells < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "n_cells must be >= 1");
    if (!(percentile > 0.0) || percentile > 100.0)
        return fail(CSA_ERR_INVALID_ARGUMENT, "percentile must be in (0, 100]");
    if (min_count < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "min_count must be >= 1");
    if (!plan_ptrs_ok(plan, true) || plan->n_cells < n_cells)
        return fail(CSA_ERR_INVALID_ARGUMENT, "plan: missing buffers or fewer than n_cells cells");
    if (!keep_count || !target_out || !added_out)
        return fail(CSA_ERR_INVALID_ARGUMENT, "keep_count, target_out and added_out are required");
    const size_t need = csa_workspace_size(CSA_WS_MERGE, L, 0, 0);
    if (!workspace || workspace_bytes < need || reinterpret_cast<uintptr_t>(workspace) % 4)
        return fail(CSA_ERR_INVALID_ARGUMENT,
                    "workspace: need %zu bytes (csa_workspace_size(CSA_WS_MERGE)), 4-byte aligned",
                    need);
    DeviceInfo di;
    if ((st = device_info(&di)) != CSA_OK) return st;
    cudaError_t e = csa::launch_merge_intervals(
        csa::make_geo(L), n_cells, csa::to_dev(*plan), percentile, min_count, keep_count,
        target_out, added_out, static_cast<int32_t*>(workspace), (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "merge launch");
    return ok();
}

csa_status_t csa_share_timesteps(csa_layout_t L, int32_t n_groups, int32_t n_steps,
                                 const csa_plan_t* plan, double tau, int32_t min_count,
                                 uint16_t* keep_count, int32_t* cluster_out, double* iou_out,
                                 csa_stream_t stream) {
    csa_status_t st = check_layout(L, 0, 0);
    if (st != CSA_OK) return st;
    if (n_groups < 1 || n_steps < 1)
        return fail(CSA_ERR_INVALID_ARGUMENT, "n_groups and n_steps must be >= 1");
    if (!(tau >= 0.0) || tau > 1.0) return fail(CSA_ERR_INVALID_ARGUMENT, "tau must be in [0, 1]");
    if (min_count < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "min_count must be >= 1");
    if (!plan_ptrs_ok(plan, false) || plan->n_cells < (int64_t)n_groups * n_steps)
        return fail(CSA_ERR_INVALID_ARGUMENT,
                    "plan: missing buffers or fewer than n_groups * n_steps cells");
    if (!keep_count || !cluster_out || !iou_out)
        return fail(CSA_ERR_INVALID_ARGUMENT, "keep_count, cluster_out and iou_out are required");
    DeviceInfo di;
    if ((st = device_info(&di)) != CSA_OK) return st;
    cudaError_t e = csa::launch_share_timesteps(csa::make_geo(L), n_groups, n_steps,
                                                csa::to_dev(*plan), tau, min_count, keep_count,
                                                cluster_out, iou_out, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "timestep-sharing launch");
    return ok();
}

csa_status_t csa_copy_heads(void* dst, const void* src, csa_layout_t L, int32_t n_heads,
                            int32_t head_dim, int32_t h0, int32_t h1, int32_t direction,
                            csa_stream_t stream) {
    csa_status_t st = check_layout(L, head_dim, n_heads);
    if (st != CSA_OK) return st;
    if (!dst || !src) return fail(CSA_ERR_INVALID_ARGUMENT, "null pointer");
    if (n_heads < 1 || h0 < 0 || h1 > n_heads || h0 >= h1)
        return fail(CSA_ERR_INVALID_ARGUMENT, "head range [%d, %d) outside [0, %d)", h0, h1,
                    n_heads);
    if (direction != 0 && direction != 1)
        return fail(CSA_ERR_INVALID_ARGUMENT, "direction must be 0 (H2D) or 1 (D2H)");
    const size_t pitch = (size_t)n_heads * head_dim * 2, off = (size_t)h0 * head_dim * 2;
    const size_t width = (size_t)(h1 - h0) * head_dim * 2;
    const size_t rows = (size_t)L.frames * L.rows * L.cols;
    cudaError_t e = cudaMemcpy2DAsync(static_cast<char*>(dst) + off, pitch,
                                      static_cast<const char*>(src) + off, pitch, width, rows,
                                      direction == 0 ? cudaMemcpyHostToDevice
                                                     : cudaMemcpyDeviceToHost,
                                      (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync");
    return ok();
}

csa_status_t csa_compile_plan(csa_layout_t L, int64_t n_cells, const uint16_t* keep_count,
                              int32_t min_count, const double* similarity, double gamma,
                              int32_t anchor_k, int32_t phase, const csa_plan_t* plan,
                              void* workspace, size_t workspace_bytes, csa_stream_t stream) {
    (void)workspace;
    (void)workspace_bytes;
    csa_status_t st = check_layout(L, 0, 0);
    if (st != CSA_OK) return st;
    if (n_cells < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "n_cells must be >= 1");
    if (phase != 0 && phase != 1) return fail(CSA_ERR_INVALID_ARGUMENT, "phase must be 0 or 1");
    if (!plan_ptrs_ok(plan, phase == 1)) return fail(CSA_ERR_INVALID_ARGUMENT, "plan: null buffer");
    if (plan->n_cells < n_cells) return fail(CSA_ERR_INVALID_ARGUMENT, "plan holds fewer cells");
    if (phase == 0 && !keep_count) return fail(CSA_ERR_INVALID_ARGUMENT, "keep_count is null");
    if (similarity && (anchor_k < 1 || anchor_k > L.rows))
        return fail(CSA_ERR_INVALID_ARGUMENT, "anchor_k %d outside [1, rows=%d]", anchor_k, L.rows);
    const csa::Geo g = csa::make_geo(L);
    const csa::PlanDev p = csa::to_dev(*plan);
    cudaError_t e = phase == 0 ? csa::launch_plan_count(g, n_cells, keep_count, min_count,
                                                        similarity, gamma, anchor_k, p,
                                                        (cudaStream_t)stream)
                               : csa::launch_plan_fill(g, n_cells, p, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "compile launch");
    return ok();
}

csa_status_t csa_build_work_list(csa_layout_t L, const csa_plan_t* plan, int64_t cell_base,
                                 int32_t n_heads, int32_t order, uint32_t* work_list,
                                 int32_t capacity, int32_t* n_work, void* workspace,
                                 size_t workspace_bytes, csa_stream_t stream) {
    (void)workspace;
    (void)workspace_bytes;
    csa_status_t st = check_layout(L, 0, n_heads);
    if (st != CSA_OK) return st;
    if (n_heads < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "n_heads must be >= 1");
    if (order < 0 || order > 3) return fail(CSA_ERR_INVALID_ARGUMENT, "order must be 0..3");
    if (!plan_ptrs_ok(plan, false) || !work_list || !n_work)
        return fail(CSA_ERR_INVALID_ARGUMENT, "null buffer");
    if (cell_base < 0 || cell_base + n_heads > plan->n_cells)
        return fail(CSA_ERR_INVALID_ARGUMENT, "cells [%lld, %lld) outside the plan",
                    (long long)cell_base, (long long)(cell_base + n_heads));
    const csa::Geo g = csa::make_geo(L);
    cudaError_t e = csa::launch_work_list(g, csa::to_dev(*plan), cell_base, n_heads, order,
                                          work_list, capacity, n_work, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "work list launch");
    return ok();
}

}  // extern "C"

namespace {
// csa_sparse_attn_fwd and csa_sparse_attn_fwd_scatter: o_peer == nullptr -> output in o;
// otherwise token t's row goes to o_peer[t / (N / n_peers)] (device array of n_peers pointers)
// at local token t % (N / n_peers), with o's strides.
csa_status_t attn_fwd_impl(csa_layout_t L, int32_t batch, int32_t n_heads, int32_t head_dim,
                           float softmax_scale, csa_tensor_t q, csa_tensor_t k, csa_tensor_t v,
                           csa_tensor_t o, void* const* o_peer, int32_t n_peers, float* lse_out,
                           const csa_plan_t* plan, int64_t cell_base, const uint32_t* work_list,
                           const int32_t* n_work, int32_t max_work, int32_t pair_items,
                           void* workspace, size_t workspace_bytes, csa_stream_t stream) {
    csa_status_t st = check_layout(L, head_dim, n_heads);
    if (st != CSA_OK) return st;
    if (pair_items)
        return fail(CSA_ERR_UNSUPPORTED,
                    "pair work items: no kernel in this build (scripts/experiments/attn6_pair.cu)");
    // block 128 (square, or B_q = 128 x B_kv): fixed-reference kernels + exact-max fallback
    // passes, which keep their list in the workspace; block 64: attn.cu
    const bool b128 = L.block == 128;
    if (b128 && workspace == nullptr)
        return fail(CSA_ERR_INVALID_ARGUMENT, "block 128 needs the attention workspace");
    if (workspace != nullptr && (workspace_bytes < 8 || reinterpret_cast<uintptr_t>(workspace) % 8))
        return fail(CSA_ERR_INVALID_ARGUMENT, "attention workspace: >= 8 bytes, 8-byte aligned");
    if (batch < 1 || n_heads < 1) return fail(CSA_ERR_INVALID_ARGUMENT, "batch/n_heads < 1");
    if (!(softmax_scale > 0.0f)) return fail(CSA_ERR_INVALID_ARGUMENT, "softmax_scale <= 0");
    if (!plan_ptrs_ok(plan, true) || !work_list || !n_work)
        return fail(CSA_ERR_INVALID_ARGUMENT, "null plan / work list");
    if (cell_base < 0 || cell_base + n_heads > plan->n_cells)
        return fail(CSA_ERR_INVALID_ARGUMENT, "cells outside the plan");
    if (max_work < 0) return fail(CSA_ERR_INVALID_ARGUMENT, "max_work < 0");
    if ((o_peer == nullptr && (!o.ptr || reinterpret_cast<uintptr_t>(o.ptr) % 16)) ||
        o.stride_n % 8 || (n_heads > 1 && o.stride_h % 8) || (batch > 1 && o.stride_b % 8))
        return fail(CSA_ERR_INVALID_ARGUMENT, "o: null or not 16-byte aligned");
    if (o_peer != nullptr) {
        const int64_t n_tok = (int64_t)L.frames * L.rows * L.cols;
        if (!b128 || n_peers < 1 || n_tok % n_peers != 0)
            return fail(CSA_ERR_INVALID_ARGUMENT,
                        "output scatter: block 128 and N divisible by n_peers (%d)", n_peers);
    }
    if (!q.ptr || q.stride_n % 8 || (n_heads > 1 && q.stride_h % 8))
        return fail(CSA_ERR_INVALID_ARGUMENT, "q: null or strides not 16-byte multiples");
    DeviceInfo di;
    if ((st = device_info(&di)) != CSA_OK) return st;
    if (max_work == 0) return ok();
    const csa::Geo g = csa::make_geo(L);
    CUtensorMap tq, tk, tv;
    if ((st = make_map(&tq, q, batch, g.N, n_heads, head_dim, g.B, "q")) != CSA_OK) return st;
    if ((st = make_map(&tk, k, batch, g.N, n_heads, head_dim, g.BK, "k")) != CSA_OK) return st;
    if ((st = make_map(&tv, v, batch, g.N, n_heads, head_dim, g.BK, "v")) != CSA_OK) return st;
    csa::AttnArgs a;
    a.g = g;
    a.batch = batch;
    a.n_heads = n_heads;
    a.head_dim = head_dim;
    a.scale_log2 = softmax_scale * 1.4426950408889634f;
    a.q = static_cast<const __nv_bfloat16*>(q.ptr);
    a.o = static_cast<__nv_bfloat16*>(o.ptr);
    a.q_sb = q.stride_b;
    a.q_sn = q.stride_n;
    a.q_sh = q.stride_h;
    a.o_sb = o.stride_b;
    a.o_sn = o.stride_n;
    a.o_sh = o.stride_h;
    a.lse_out = lse_out;
    a.plan = csa::to_dev(*plan);
    a.cell_base = cell_base;
    a.work_list = work_list;
    a.n_work = n_work;
    a.sched = static_cast<uint32_t*>(workspace);
    a.o_peer = reinterpret_cast<__nv_bfloat16* const*>(o_peer);
    a.o_peer_tokens = o_peer ? (int64_t)g.N / n_peers : 0;
    const int64_t items = (int64_t)max_work * batch;
    const int grid = (int)(items < di.sms ? items : di.sms);
    cudaError_t e;
    if (b128) {
        // Mode 0: every row's softmax shift is the max of its first kept tile (reading Q29):
        // attn5.cu for square 128 x 128 blocks (head_dim 128 and 64), attn_rect.cu for B_kv !=
        // 128.  Items whose later scores overshoot that shift by more than 2^56 are listed in
        // the workspace (256 bytes past the counters) and recomputed on the same stream by
        // attn_rect.cu's exact-max passes (mode 1: each row's exact max over its kept keys,
        // mode 2: the softmax against it), statically assigned over the (normally empty) list.
        const size_t n_items = (size_t)n_heads * (size_t)g.NB;
        if (workspace_bytes < csa_workspace_size(CSA_WS_ATTN, L, n_heads, head_dim) ||
            (int64_t)max_work > (int64_t)n_items)
            return fail(CSA_ERR_INVALID_ARGUMENT, "attention workspace too small");
        uint32_t* base = static_cast<uint32_t*>(workspace) + 64;
        const size_t flag_words = (n_items + 31) / 32;
        csa::Fallback fb{base, base + 1, base + 1 + flag_words};
        e = cudaMemsetAsync(base, 0, 4 * (1 + flag_words), (cudaStream_t)stream);
        if (e == cudaSuccess)
            e = is_square(L) ? csa::launch_attn_sepp(a, tq, tk, tv, grid, fb, (cudaStream_t)stream)
                             : csa::launch_attn_rect(a, tq, tk, tv, grid, fb, 0,
                                                     (cudaStream_t)stream);
        csa::AttnArgs re = a;
        re.work_list = fb.list;
        re.n_work = reinterpret_cast<const int32_t*>(fb.count);
        re.sched = nullptr;
        for (int mode = 1; mode <= 2 && e == cudaSuccess; ++mode)
            e = csa::launch_attn_rect(re, tq, tk, tv, di.sms, fb, mode, (cudaStream_t)stream);
    } else {
        e = csa::launch_attn(a, head_dim, tq, tk, tv, grid, (cudaStream_t)stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "attention launch");
    return ok();
}
}  // namespace

extern "C" {

csa_status_t csa_sparse_attn_fwd(csa_layout_t L, int32_t batch, int32_t n_heads,
                                 int32_t head_dim, float softmax_scale, csa_tensor_t q,
                                 csa_tensor_t k, csa_tensor_t v, csa_tensor_t o, float* lse_out,
                                 const csa_plan_t* plan, int64_t cell_base,
                                 const uint32_t* work_list, const int32_t* n_work,
                                 int32_t max_work, int32_t pair_items, void* workspace,
                                 size_t workspace_bytes, csa_stream_t stream) {
    return attn_fwd_impl(L, batch, n_heads, head_dim, softmax_scale, q, k, v, o, nullptr, 0,
                         lse_out, plan, cell_base, work_list, n_work, max_work, pair_items,
                         workspace, workspace_bytes, stream);
}

csa_status_t csa_sparse_attn_fwd_scatter(csa_layout_t L, int32_t batch, int32_t n_heads,
                                         int32_t head_dim, float softmax_scale, csa_tensor_t q,
                                         csa_tensor_t k, csa_tensor_t v, void* const* o_peers,
                                         int32_t n_peers, int64_t o_stride_b, int64_t o_stride_n,
                                         int64_t o_stride_h, float* lse_out,
                                         const csa_plan_t* plan, int64_t cell_base,
                                         const uint32_t* work_list, const int32_t* n_work,
                                         int32_t max_work, void* workspace,
                                         size_t workspace_bytes, csa_stream_t stream) {
    if (o_peers == nullptr) return fail(CSA_ERR_INVALID_ARGUMENT, "o_peers is null");
    csa_tensor_t o;
    o.ptr = nullptr;
    o.stride_b = o_stride_b;
    o.stride_n = o_stride_n;
    o.stride_h = o_stride_h;
    return attn_fwd_impl(L, batch, n_heads, head_dim, softmax_scale, q, k, v, o, o_peers,
                         n_peers, lse_out, plan, cell_base, work_list, n_work, max_work, 0,
                         workspace, workspace_bytes, stream);
}

csa_status_t csa_validate_plan(const csa_plan_t* plan, csa_layout_t L, int64_t n_cells,
                               csa_stream_t stream) {
    csa_status_t st = check_layout(L, 0, 0);
    if (st != CSA_OK) return st;
    if (!plan_ptrs_ok(plan, true) || n_cells < 1 || n_cells > plan->n_cells)
        return fail(CSA_ERR_INVALID_ARGUMENT, "plan / n_cells");
    std::lock_guard<std::mutex> lk(g_validate_mu);
    uint32_t* flag = nullptr;
    cudaError_t e = cudaGetSymbolAddress(reinterpret_cast<void**>(&flag), g_validate_flag);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetSymbolAddress");
    cudaStream_t s = (cudaStream_t)stream;
    if ((e = cudaMemsetAsync(flag, 0, sizeof(uint32_t), s)) != cudaSuccess)
        return cuda_fail(e, "memset");
    if ((e = csa::launch_validate(csa::make_geo(L), n_cells, csa::to_dev(*plan), flag, s)) !=
        cudaSuccess)
        return cuda_fail(e, "validate launch");
    uint32_t h = 0;
    if ((e = cudaMemcpyAsync(&h, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
        return cuda_fail(e, "memcpy");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "sync");
    if (h) return fail(CSA_ERR_CORRUPT_PLAN, "plan check failed (flags 0x%x)", h);
    return ok();
}

}  // extern "C"
