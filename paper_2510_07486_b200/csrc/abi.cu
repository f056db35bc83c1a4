// abi.cu -- the extern "C" boundary (include/asyncspade.h): host-side
// validation, workspace sizing, and the launches.  Nothing is enqueued unless
// every check passes.
#include <stdint.h>

#include "common.cuh"

namespace {

bool aligned16(const void *ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }
// the tensor-core kernels (score.cu, decode.cu): head_dim 64 / 128, G <= 32
bool group_ok(int G) { return G == 1 || G == 2 || G == 4 || G == 8 || G == 16 || G == 32; }
bool dim_ok(int D) { return D == 64 || D == 128; }
bool tc_select_ok(const asp_select_params *p) {     // score.cu's instantiations
    const int G = p->n_q_heads / p->n_kv_heads, D = p->head_dim;
    if (dim_ok(D)) return group_ok(G) || G == 64;                 // G = 64: MQA
    if (D == 576) return G == 1 || G == 2 || G == 4 || G == 8 || G == 16;   // absorbed MLA
    if (D == 256) return G == 8 || G == 16;
    return false;
}
int v_dim_of(const asp_decode_params *p) { return p->v_head_dim ? p->v_head_dim : p->head_dim; }
bool tc_decode_ok(const asp_decode_params *p) {
    return dim_ok(p->head_dim) && group_ok(p->n_q_heads / p->n_kv_heads) && v_dim_of(p) == p->head_dim;
}
// MQA with 64 / 128 query heads on the tensor cores: the one KV head is taken as
// G / 32 "virtual" KV heads of 32 query heads each (decode.cu; dense caches only)
bool tc_decode_mqa_ok(const asp_decode_params *p) {
    const int G = p->n_q_heads / p->n_kv_heads;
    return dim_ok(p->head_dim) && p->n_kv_heads == 1 && (G == 64 || G == 128) &&
           v_dim_of(p) == p->head_dim;
}
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

asp_status from_cuda(cudaError_t e) { return e == cudaSuccess ? ASP_OK : ASP_ERR_CUDA; }

asp_status check_select(const asp_select_params *p) {
    if (!p) return ASP_ERR_INVALID_ARGUMENT;
    if (p->batch <= 0 || p->n_q_heads <= 0 || p->n_kv_heads <= 0 || p->head_dim <= 0 ||
        p->top_k <= 0 || p->max_seq_len <= 0)
        return ASP_ERR_SHAPE;
    if (p->n_q_heads % p->n_kv_heads) return ASP_ERR_SHAPE;
    // tensor-core stream, or the CUDA-core kernel for absorbed MLA / large groups
    if (!tc_select_ok(p) && !asp_score_cc_supported(p->head_dim, p->n_q_heads / p->n_kv_heads))
        return ASP_ERR_UNSUPPORTED;
    if (p->aggregation != ASP_AGG_MAX && p->aggregation != ASP_AGG_SUM) return ASP_ERR_INVALID_ARGUMENT;
    if (p->k_stride_t < p->head_dim || p->k_stride_b < 0 || p->k_stride_h < 0) return ASP_ERR_SHAPE;
    if ((p->k_stride_b | p->k_stride_h | p->k_stride_t) & 7) return ASP_ERR_INVALID_ARGUMENT;
    // TMA views the cache as [rows][head_dim] with row stride k_stride_t
    if (p->k_stride_b % p->k_stride_t || p->k_stride_h % p->k_stride_t) return ASP_ERR_UNSUPPORTED;
    return ASP_OK;
}

asp_status check_decode(const asp_decode_params *p) {
    if (!p) return ASP_ERR_INVALID_ARGUMENT;
    if (p->batch <= 0 || p->n_q_heads <= 0 || p->n_kv_heads <= 0 || p->head_dim <= 0 ||
        p->top_k <= 0 || p->n_fresh < 0 || p->max_seq_len <= 0)
        return ASP_ERR_SHAPE;
    if (p->n_q_heads % p->n_kv_heads) return ASP_ERR_SHAPE;
    if (p->v_head_dim < 0 || p->v_head_dim > p->head_dim) return ASP_ERR_SHAPE;
    if (!tc_decode_ok(p) &&
        !asp_decode_cc_supported(p->head_dim, v_dim_of(p), p->n_q_heads / p->n_kv_heads))
        return ASP_ERR_UNSUPPORTED;
    if (!(p->sm_scale == p->sm_scale)) return ASP_ERR_INVALID_ARGUMENT;
    // output strides: both 0 (dense [B][Hq][D]) or both set (e.g. head-major)
    if (p->out_stride_b < 0 || p->out_stride_h < 0 || ((p->out_stride_b == 0) != (p->out_stride_h == 0)))
        return ASP_ERR_SHAPE;
    if ((p->out_stride_b | p->out_stride_h) & 3) return ASP_ERR_INVALID_ARGUMENT;
    if (p->k_stride_t < p->head_dim || p->v_stride_t < v_dim_of(p) || p->k_stride_b < 0 ||
        p->k_stride_h < 0 || p->v_stride_b < 0 || p->v_stride_h < 0)
        return ASP_ERR_SHAPE;
    if ((p->k_stride_b | p->k_stride_h | p->k_stride_t | p->v_stride_b | p->v_stride_h |
         p->v_stride_t) & 7)
        return ASP_ERR_INVALID_ARGUMENT;
    // the gather views each cache as [rows][head_dim] with row stride stride_t
    if (p->k_stride_b % p->k_stride_t || p->k_stride_h % p->k_stride_t ||
        p->v_stride_b % p->v_stride_t || p->v_stride_h % p->v_stride_t)
        return ASP_ERR_UNSUPPORTED;
    return ASP_OK;
}

asp_status check_paged(const asp_paged_kv *pk, int n_kv_heads, int max_seq_len) {
    if (!pk) return ASP_ERR_INVALID_ARGUMENT;
    const int P = pk->page_size;
    if (P != 16 && P != 32 && P != 64 && P != 128) return ASP_ERR_UNSUPPORTED;
    if (pk->max_pages_per_seq <= 0 || pk->num_pages <= 0) return ASP_ERR_SHAPE;
    if ((int64_t)pk->max_pages_per_seq * P < max_seq_len) return ASP_ERR_SHAPE;
    if ((int64_t)pk->num_pages * n_kv_heads * P >= ((int64_t)1 << 31)) return ASP_ERR_SHAPE;
    return ASP_OK;
}

}  // namespace

int asp_sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

extern "C" {

asp_status asyncspade_append(const asp_append_params *p, const float *q_t, float *q_window,
                             asp_bf16 *q_cur, const asp_bf16 *k_new, const asp_bf16 *v_new,
                             asp_bf16 *k_cache, asp_bf16 *v_cache, const int32_t *pos,
                             asp_stream stream) {
    if (!p || !q_t || (!q_window && !q_cur)) return ASP_ERR_INVALID_ARGUMENT;
    if (p->batch <= 0 || p->n_q_heads <= 0 || p->n_kv_heads <= 0 || p->head_dim <= 0 ||
        p->window <= 0 || p->max_seq_len <= 0)
        return ASP_ERR_SHAPE;
    if (p->ring_slot < 0 || p->ring_slot >= p->window) return ASP_ERR_SHAPE;
    if (p->head_dim % 8) return ASP_ERR_UNSUPPORTED;
    if ((k_new && !k_cache) || (v_new && !v_cache) || ((k_new || v_new) && !pos))
        return ASP_ERR_INVALID_ARGUMENT;
    if ((p->k_stride_b | p->k_stride_h | p->k_stride_t | p->v_stride_b | p->v_stride_h |
         p->v_stride_t) & 7)
        return ASP_ERR_INVALID_ARGUMENT;
    const void *ptrs[] = {q_t, q_window, q_cur, k_new, v_new, k_cache, v_cache};
    for (const void *ptr : ptrs)
        if (ptr && !aligned16(ptr)) return ASP_ERR_INVALID_ARGUMENT;
    return from_cuda(asp_launch_append(*p, q_t, q_window, q_cur, k_new, v_new, k_cache, v_cache,
                                       pos, (cudaStream_t)stream));
}

asp_status asyncspade_predict_query(const asp_predict_params *p, const float *q_window,
                                    float *q_hat, uint32_t *dev_flags, asp_stream stream) {
    if (!p || !q_window || !q_hat) return ASP_ERR_INVALID_ARGUMENT;
    if (p->batch <= 0 || p->n_q_heads <= 0 || p->head_dim <= 0 || p->window <= 0)
        return ASP_ERR_SHAPE;
    if (p->ring_start < 0 || p->ring_start >= p->window) return ASP_ERR_SHAPE;
    if (!(dim_ok(p->head_dim) || p->head_dim == 256 || p->head_dim == 576) || p->window > 32)
        return ASP_ERR_UNSUPPORTED;
    const uint32_t mode = p->flags & 0xFu;
    const uint32_t known = 0xFu | ASP_SIGN_NEGATED | ASP_EPS_ABSOLUTE | ASP_NORM_NONE |
                           ASP_DOUBLE_SOFTMAX | ASP_WINDOW_BF16;
    if (mode > ASP_ASSEMBLY_PER_WINDOW || (p->flags & ~known)) return ASP_ERR_INVALID_ARGUMENT;
    if ((p->flags & ASP_WINDOW_BF16) &&
        (p->window < 2 || p->window > 16 || mode == ASP_ASSEMBLY_PER_WINDOW || !dim_ok(p->head_dim) ||
         (int64_t)p->batch * p->n_q_heads * p->window * p->head_dim >= ((int64_t)1 << 31)))
        return ASP_ERR_UNSUPPORTED;
    if ((p->flags & ASP_NORM_NONE) && mode != ASP_ASSEMBLY_SINGLE) return ASP_ERR_INVALID_ARGUMENT;
    if (!(p->eps == p->eps)) return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(q_window) || !aligned16(q_hat)) return ASP_ERR_INVALID_ARGUMENT;
    return from_cuda(asp_launch_predict(*p, q_window, q_hat, dev_flags, (cudaStream_t)stream));
}

size_t asyncspade_score_select_workspace(const asp_select_params *p) {
    if (check_select(p) != ASP_OK) return 0;
    return align256((size_t)p->batch * p->n_kv_heads * p->max_seq_len * sizeof(float));
}

asp_status asyncspade_score_select(const asp_select_params *p, const float *q_hat,
                                   const asp_bf16 *k_cache, const int32_t *seq_lens,
                                   int32_t *sel_idx, float *scores, void *workspace,
                                   size_t workspace_bytes, uint32_t *dev_flags,
                                   asp_stream stream) {
    asp_status st = check_select(p);
    if (st != ASP_OK) return st;
    if (!q_hat || !k_cache || !seq_lens || !sel_idx) return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(q_hat) || !aligned16(k_cache) || !aligned16(scores)) return ASP_ERR_INVALID_ARGUMENT;
    float *s_buf = scores;
    if (!s_buf) {
        if (!workspace || workspace_bytes < asyncspade_score_select_workspace(p))
            return ASP_ERR_WORKSPACE;
        if (reinterpret_cast<uintptr_t>(workspace) & 255u) return ASP_ERR_WORKSPACE;
        s_buf = static_cast<float *>(workspace);
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = tc_select_ok(p) ? asp_launch_score(*p, q_hat, k_cache, seq_lens, s_buf, dev_flags, s)
                                    : asp_launch_score_cc(*p, q_hat, k_cache, seq_lens, s_buf, dev_flags, s);
    if (e != cudaSuccess) return ASP_ERR_CUDA;
    return from_cuda(asp_launch_select(*p, s_buf, seq_lens, sel_idx, dev_flags, scores == nullptr, s));
}

asp_status asyncspade_score_select_paged(const asp_select_params *p, const asp_paged_kv *pk,
                                         const float *q_hat, const asp_bf16 *k_pages,
                                         const int32_t *block_table, const int32_t *seq_lens,
                                         int32_t *sel_idx, float *scores, void *workspace,
                                         size_t workspace_bytes, uint32_t *dev_flags,
                                         asp_stream stream) {
    if (!p) return ASP_ERR_INVALID_ARGUMENT;
    asp_select_params q = *p;                        // strides are the pool's (ignored)
    q.k_stride_t = q.head_dim;
    q.k_stride_h = q.k_stride_b = 0;
    asp_status st = check_select(&q);
    if (st != ASP_OK) return st;
    if (!tc_select_ok(&q) || !dim_ok(q.head_dim)) return ASP_ERR_UNSUPPORTED;   // paged: D 64 / 128
    st = check_paged(pk, q.n_kv_heads, q.max_seq_len);
    if (st != ASP_OK) return st;
    if (!q_hat || !k_pages || !block_table || !seq_lens || !sel_idx) return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(q_hat) || !aligned16(k_pages) || !aligned16(scores)) return ASP_ERR_INVALID_ARGUMENT;
    float *s_buf = scores;
    if (!s_buf) {
        if (!workspace || workspace_bytes < asyncspade_score_select_workspace(&q))
            return ASP_ERR_WORKSPACE;
        if (reinterpret_cast<uintptr_t>(workspace) & 255u) return ASP_ERR_WORKSPACE;
        s_buf = static_cast<float *>(workspace);
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = asp_launch_score(q, q_hat, k_pages, seq_lens, s_buf, dev_flags, s, pk, block_table);
    if (e != cudaSuccess) return ASP_ERR_CUDA;
    return from_cuda(asp_launch_select(q, s_buf, seq_lens, sel_idx, dev_flags, scores == nullptr, s));
}

size_t asyncspade_sparse_decode_workspace(const asp_decode_params *p) {
    if (check_decode(p) != ASP_OK) return 0;
    return tc_decode_ok(p) || tc_decode_mqa_ok(p) ? asp_decode_workspace_bytes(*p)
                                                  : asp_decode_cc_workspace_bytes(*p, v_dim_of(p));
}

asp_status asyncspade_sparse_decode(const asp_decode_params *p, const asp_bf16 *q,
                                    const asp_bf16 *k_cache, const asp_bf16 *v_cache,
                                    const int32_t *seq_lens, const int32_t *sel_idx, float *out,
                                    void *workspace, size_t workspace_bytes, asp_stream stream) {
    asp_status st = check_decode(p);
    if (st != ASP_OK) return st;
    if (!q || !k_cache || !v_cache || !seq_lens || !sel_idx || !out) return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out))
        return ASP_ERR_INVALID_ARGUMENT;
    if (!workspace || workspace_bytes < asyncspade_sparse_decode_workspace(p)) return ASP_ERR_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(workspace) & 255u) return ASP_ERR_WORKSPACE;
    if (!tc_decode_ok(p) && !tc_decode_mqa_ok(p))
        return from_cuda(asp_launch_decode_cc(*p, v_dim_of(p), q, k_cache, v_cache, seq_lens,
                                              sel_idx, out, workspace, (cudaStream_t)stream));
    return from_cuda(asp_launch_decode(*p, q, k_cache, v_cache, seq_lens, sel_idx, out, workspace,
                                       (cudaStream_t)stream));
}

asp_status asyncspade_sparse_decode_paged(const asp_decode_params *p, const asp_paged_kv *pk,
                                          const asp_bf16 *q, const asp_bf16 *k_pages,
                                          const asp_bf16 *v_pages, const int32_t *block_table,
                                          const int32_t *seq_lens, const int32_t *sel_idx,
                                          float *out, void *workspace, size_t workspace_bytes,
                                          asp_stream stream) {
    if (!p) return ASP_ERR_INVALID_ARGUMENT;
    asp_decode_params d = *p;                        // strides are the pool's (ignored)
    d.k_stride_t = d.v_stride_t = d.head_dim;
    d.k_stride_h = d.k_stride_b = d.v_stride_h = d.v_stride_b = 0;
    asp_status st = check_decode(&d);
    if (st != ASP_OK) return st;
    if (!tc_decode_ok(&d)) return ASP_ERR_UNSUPPORTED;           // paged: tensor-core shapes
    st = check_paged(pk, d.n_kv_heads, d.max_seq_len);
    if (st != ASP_OK) return st;
    if (!q || !k_pages || !v_pages || !block_table || !seq_lens || !sel_idx || !out)
        return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k_pages) || !aligned16(v_pages) || !aligned16(out))
        return ASP_ERR_INVALID_ARGUMENT;
    if (!workspace || workspace_bytes < asyncspade_sparse_decode_workspace(&d)) return ASP_ERR_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(workspace) & 255u) return ASP_ERR_WORKSPACE;
    return from_cuda(asp_launch_decode(d, q, k_pages, v_pages, seq_lens, sel_idx, out, workspace,
                                       (cudaStream_t)stream, pk, block_table));
}

size_t asyncspade_quest_meta_bytes(const asp_select_params *p, int32_t page_size) {
    if (check_select(p) != ASP_OK || !dim_ok(p->head_dim) || page_size < 1 || page_size > 128) return 0;
    return align256(asp_quest_meta_bytes(*p, page_size));
}

asp_status asyncspade_quest_summarize(const asp_select_params *p, int32_t page_size,
                                      const asp_bf16 *k_cache, const int32_t *seq_lens, void *meta,
                                      asp_stream stream) {
    asp_status st = check_select(p);
    if (st != ASP_OK) return st;
    if (page_size < 1 || page_size > 128 || !dim_ok(p->head_dim)) return ASP_ERR_UNSUPPORTED;
    if (!k_cache || !seq_lens || !meta) return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(k_cache) || !aligned16(meta)) return ASP_ERR_INVALID_ARGUMENT;
    return from_cuda(asp_launch_quest_summarize(*p, page_size, k_cache, seq_lens, meta,
                                                (cudaStream_t)stream));
}

// the Quest page-bound kernel is instantiated for G in {1, 2, 4, 8} only
static bool quest_group_ok(const asp_select_params *p) {
    const int G = p->n_q_heads / p->n_kv_heads;
    return (G == 1 || G == 2 || G == 4 || G == 8) && dim_ok(p->head_dim);
}

size_t asyncspade_quest_select_workspace(const asp_select_params *p, int32_t page_size) {
    if (check_select(p) != ASP_OK || !quest_group_ok(p) || page_size < 1 || page_size > 128 ||
        p->top_k % page_size)
        return 0;
    return align256(asp_quest_workspace_bytes(*p, page_size));
}

asp_status asyncspade_quest_select(const asp_select_params *p, int32_t page_size, const float *q,
                                   const void *meta, const int32_t *seq_lens, int32_t *sel_idx,
                                   void *workspace, size_t workspace_bytes, uint32_t *dev_flags,
                                   asp_stream stream) {
    asp_status st = check_select(p);
    if (st != ASP_OK) return st;
    if (page_size < 1 || page_size > 128 || !quest_group_ok(p)) return ASP_ERR_UNSUPPORTED;
    if (p->top_k % page_size) return ASP_ERR_SHAPE;
    if (!q || !meta || !seq_lens || !sel_idx) return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(meta)) return ASP_ERR_INVALID_ARGUMENT;
    if (!workspace || workspace_bytes < asyncspade_quest_select_workspace(p, page_size))
        return ASP_ERR_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(workspace) & 255u) return ASP_ERR_WORKSPACE;
    return from_cuda(asp_launch_quest_select(*p, page_size, q, meta, seq_lens, sel_idx, workspace,
                                             dev_flags, (cudaStream_t)stream));
}

asp_status asyncspade_gather_filtered(const asp_decode_params *p, const asp_bf16 *k_cache,
                                      const asp_bf16 *v_cache, const int32_t *seq_lens,
                                      const int32_t *sel_idx, asp_bf16 *k_out, asp_bf16 *v_out,
                                      int32_t *idx_out, asp_stream stream) {
    asp_status st = check_decode(p);
    if (st != ASP_OK) return st;
    if (!dim_ok(p->head_dim) || v_dim_of(p) != p->head_dim) return ASP_ERR_UNSUPPORTED;
    if (!k_cache || !v_cache || !seq_lens || !sel_idx || !k_out || !v_out)
        return ASP_ERR_INVALID_ARGUMENT;
    if (!aligned16(k_cache) || !aligned16(v_cache) || !aligned16(k_out) || !aligned16(v_out))
        return ASP_ERR_INVALID_ARGUMENT;
    return from_cuda(asp_launch_gather(*p, k_cache, v_cache, seq_lens, sel_idx, k_out, v_out,
                                       idx_out, (cudaStream_t)stream));
}

const char *asyncspade_status_string(asp_status s) {
    switch (s) {
        case ASP_OK: return "ASP_OK";
        case ASP_ERR_INVALID_ARGUMENT: return "ASP_ERR_INVALID_ARGUMENT";
        case ASP_ERR_SHAPE: return "ASP_ERR_SHAPE";
        case ASP_ERR_UNSUPPORTED: return "ASP_ERR_UNSUPPORTED";
        case ASP_ERR_WORKSPACE: return "ASP_ERR_WORKSPACE";
        case ASP_ERR_CUDA: return "ASP_ERR_CUDA";
        default: return "ASP_ERR_UNKNOWN";
    }
}

int32_t asyncspade_abi_version(void) { return ASYNCSPADE_ABI_VERSION; }

}  // extern "C"
