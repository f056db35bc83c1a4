/*
 * asyncspade.h -- C ABI of the B200 (sm_100a) AsyncSpade decode hot path.
 *
 * AsyncSpade (arXiv 2510.07486) hides query-aware KV selection behind the
 * decode step by PREDICTING the next query from a window of recent queries
 * and selecting tokens with the prediction.  The hot
 * path of one attention layer's decode step is four kernels, exposed as
 * three entry points:
 *
 *   asyncspade_append          a0  new query / K / V into the state
 *   asyncspade_predict_query   a1  q_hat from the query window     (Alg.1 Steps 1-6)
 *   asyncspade_score_select    a2  q_hat . K scores per KV head    (Alg.1 Step 7)
 *                              a3  per-row top-k token selection  (P:191, P:267 item (2))
 *   asyncspade_sparse_decode   a4  attention over the picked K/V
 *
 * ("P:<n>" = line n of the paper text, reference/PAPER.md.)
 *
 * Plain C types only: callers need neither CUDA nor torch headers.  Every
 * pointer argument named "device" must be CUDA device memory (or managed);
 * `asp_stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Ownership and lifetime
 *   The caller allocates every buffer, workspace included.  The library
 *   never allocates, frees or synchronizes; it only enqueues work on
 *   `stream`.  Pointers must stay valid until that work completes.  Calls
 *   are stateless and reentrant (the only internal state is a per-device
 *   cache of the SM count) and capturable into CUDA graphs.
 *
 * Errors
 *   Every call validates its arguments on the host and returns a non-zero
 *   asp_status BEFORE enqueuing anything if they are invalid: null
 *   pointers, non-positive sizes, n_q_heads % n_kv_heads != 0, unsupported
 *   head_dim / group size G = n_q_heads / n_kv_heads (score + select: head_dim
 *   64 / 128 with G in {1, 2, 4, ..., 64}, 576 with G <= 16 on the tensor
 *   cores, plus the CUDA-core shapes (head_dim 576 / 256 / 128 / 64, G up to
 *   128); decode: head_dim 64 / 128 with G <= 32, and one KV head with G =
 *   64 / 128 (MQA), on the tensor cores, plus absorbed MLA (576 / v_head_dim
 *   512, G <= 16) and G = 64 / 128 over several KV heads on the CUDA cores;
 *   predict: head_dim 64, 128, 256, 576) / window (1..32),
 *   misaligned pointers (16 B), strides not multiples of 8 elements,
 *   too-small workspace.  Launch failures return
 *   ASP_ERR_CUDA.  Numeric conditions never fail a call: they OR a bit into
 *   the optional device word `dev_flags` and produce the defined fallback
 *   output documented per call.
 *
 * Stream ordering (programmatic dependent launch)
 *   Every kernel is launched with programmatic stream serialization, so its
 *   prologue overlaps the previous kernel's tail.  Reads of inputs that only
 *   the CALLER (or asyncspade_append) writes may start before the previous
 *   kernel on the stream has finished: predict reads the window, the score
 *   stream reads K, and the score planning reads seq_lens early.  This is
 *   safe because asyncspade_append never lets its dependents start before it
 *   completes, and a kernel that does not trigger dependents early (any
 *   torch / cuBLAS / caller kernel) runs to completion before the next one
 *   starts; a caller kernel that issues griddepcontrol.launch_dependents
 *   before writing these buffers must not directly precede these calls.
 *   Everything else (q_hat, selections, outputs, workspaces) is touched only
 *   after the wait.
 *
 * Determinism
 *   Every output row is a function of that row's inputs and the call's
 *   sizes only -- never of the grid, the SM count, the batch size or how
 *   the heads are sharded over GPUs -- so a KV-head shard on rank r of P
 *   reproduces the matching slice of the P = 1 result bit for bit.
 */
#ifndef ASYNCSPADE_H
#define ASYNCSPADE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASYNCSPADE_ABI_VERSION 2

#if defined(__GNUC__)
#define ASP_API __attribute__((visibility("default")))
#else
#define ASP_API
#endif

typedef int32_t asp_status;
enum {
    ASP_OK = 0,
    ASP_ERR_INVALID_ARGUMENT = 1, /* null pointer, bad flag, misalignment     */
    ASP_ERR_SHAPE = 2,            /* inconsistent or out-of-range sizes        */
    ASP_ERR_UNSUPPORTED = 3,      /* valid but not built (head_dim, G, W)      */
    ASP_ERR_WORKSPACE = 4,        /* workspace missing or too small            */
    ASP_ERR_CUDA = 5              /* a CUDA launch/runtime error               */
};

/* Device-side condition bits, OR-ed into *dev_flags (a device uint32). */
enum {
    ASP_FLAG_NONFINITE = 1u, /* non-finite window value or score seen          */
    ASP_FLAG_NOT_PD = 2u,    /* ridge matrix not positive definite             */
    ASP_FLAG_SHORT_ROW = 4u  /* a row had fewer than top_k tokens (padded)     */
};

/* Predictor flags (asp_predict_params.flags).  The low nibble picks the
 * assembly; the rest are independent bits.  Defaults (0) are SURVEY §8(c)
 * readings R2-R8: masked-shared assembly, positive sign, relative eps,
 * single softmax. */
enum {
    ASP_ASSEMBLY_MASKED_SHARED = 0u, /* Alg.1 Steps 4-6, m = W    */
    ASP_ASSEMBLY_SINGLE = 1u,        /* Eq.4 single shifted window*/
    ASP_ASSEMBLY_PER_WINDOW = 2u,    /* Eq.5 literal, one solve per k, m = W-1 */
    ASP_SIGN_NEGATED = 1u << 4,      /* softmax(-omega) as Alg.1 Step 3 */
    ASP_EPS_ABSOLUTE = 1u << 5,      /* eps is absolute, not x mean diag(G0)  */
    ASP_NORM_NONE = 1u << 6,         /* raw ridge weights (SINGLE only; tests) */
    ASP_DOUBLE_SOFTMAX = 1u << 7,    /* literal Step 3 + Step 4 double softmax */
    ASP_WINDOW_BF16 = 1u << 8        /* q_window holds bf16 (asp_bf16) elements,
                                        widened exactly; 2 <= window <= 16 with the
                                        masked-shared or single assembly only */
};

enum { ASP_AGG_MAX = 0, ASP_AGG_SUM = 1 };

typedef uint16_t asp_bf16; /* raw bf16 bit pattern */
typedef void *asp_stream;  /* cudaStream_t */

/* ------------------------------------------------------------------------
 * a0  asyncspade_append
 *
 * The new token of every sequence enters the state the path reads (P:191:
 * the inference side "enqueues the query state to the sliding window"; the
 * new key / value join the cache):
 *   q_window[b][hq][ring_slot][:] = q_t[b][hq][:]             (fp32, or bf16_rn
 *                                                               with window_bf16)
 *   q_cur[b][hq][:]               = bf16_rn(q_t[b][hq][:])    (nullable)
 *   K[b][h][pos[b]][:] = k_new[b][h][:], V[b][h][pos[b]][:] = v_new[b][h][:]
 * One launch (programmatic-dependent after the previous step's kernels)
 * instead of four strided copies.  The caller then predicts with
 * ring_start = (ring_slot + 1) % window (the slot written is the newest).
 *
 * q_t       device fp32 [batch][n_q_heads][head_dim].
 * q_window  device fp32 [batch][n_q_heads][window][head_dim] (ring), or
 *           null (no predictor state here: the Inference Rank of the
 *           disaggregated form only needs q_cur and its fresh K / V row).
 * q_cur     nullable device bf16 [batch][n_q_heads][head_dim]; q_window and
 *           q_cur cannot both be null.
 * k_new, v_new  nullable device bf16 [batch][n_kv_heads][head_dim].
 * k_cache, v_cache  strided as asp_decode_params' caches (nullable iff the
 *           matching *_new is).  pos nullable device int32 [batch]: the
 *           cache position written; rows with pos outside [0, max_seq_len)
 *           are skipped.  Pure data movement: bit-exact.
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t batch, n_q_heads, n_kv_heads, head_dim, window, ring_slot, max_seq_len;
    int64_t k_stride_b, k_stride_h, k_stride_t, v_stride_b, v_stride_h, v_stride_t; /* elements */
    int32_t window_bf16; /* 1: q_window is a bf16 ring (ASP_WINDOW_BF16), q_t rounded into it */
} asp_append_params;

ASP_API asp_status asyncspade_append(const asp_append_params *p, const float *q_t, float *q_window,
                             asp_bf16 *q_cur, const asp_bf16 *k_new, const asp_bf16 *v_new,
                             asp_bf16 *k_cache, asp_bf16 *v_cache, const int32_t *pos,
                             asp_stream stream);

/* ------------------------------------------------------------------------
 * a1  asyncspade_predict_query
 *
 * Predicts q_hat_{t+1} for every (b, query head) from the window of the W
 * most recent query states (Eq. 2-5; Alg. 1 Steps
 * 1-6).  Default (masked-shared) computation per row, in fp64:
 *   H = window rows 0..W-2 (oldest..Q_{t-1}), y = row W-1 (= Q_t)
 *   G0 = H H^T, beta = H y, eps_eff = eps * mean(diag G0)   (R7)
 *   omega = (G0 + eps_eff I)^-1 beta   (Cholesky)
 *   for j = 1..W: n_j = min(j, W-1); r_j = softmax(omega[0..n_j-1]);
 *                 c_j = sum_i r_j[i] * window[W-n_j+i]       (R3-R6)
 *   q_hat = (1/W) sum_j c_j, rounded once to fp32.
 *
 * q_window  device fp32 (bf16 with ASP_WINDOW_BF16: pass the asp_bf16
 *           pointer cast) [batch][n_q_heads][window][head_dim]; logical slot
 *           j (0 = oldest, window-1 = newest) is physical slot
 *           (ring_start + j) % window.  Read only.
 * q_hat     device fp32 [batch][n_q_heads][head_dim], written.
 * dev_flags nullable device uint32.
 * Numeric fallback: a non-finite window or a non-PD ridge matrix gives
 * q_hat = the newest query (passthrough) and sets
 * ASP_FLAG_NONFINITE / ASP_FLAG_NOT_PD.  window == 1 is a passthrough.
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t batch, n_q_heads, window, head_dim, ring_start;
    float eps;      /* relative factor (default 1e-2) unless ASP_EPS_ABSOLUTE */
    uint32_t flags; /* ASP_ASSEMBLY_* | ASP_SIGN_NEGATED | ...                */
} asp_predict_params;

ASP_API asp_status asyncspade_predict_query(const asp_predict_params *p, const float *q_window,
                                    float *q_hat, uint32_t *dev_flags, asp_stream stream);

/* ------------------------------------------------------------------------
 * a2+a3  asyncspade_score_select
 *
 * Token criticality (Alg. 1 Step 7, in the GQA layout of P:260)
 * followed by per-row top-k (P:267 item (2)):
 *   s[b,h,n] = max_{g<G} sum_d q_hat[b,h*G+g,d] * K[b,h,n,d]   (R10, R11)
 *   for n < seq_lens[b]; no 1/sqrt(D), no softmax.  (ASP_AGG_SUM: sum_g.)
 *   sel_idx[b,h,:] = the top_k tokens of row (b,h), ties to the LOWER
 *   index (R9), written in ascending index order.
 * Precision: fp32 products/accumulation of the exact bf16 keys against the
 * fp32 q_hat (within ~1e-6 relative of the exact score).
 *
 * q_hat     device fp32 [batch][n_q_heads][head_dim].
 * k_cache   device bf16; element (b,h,n,d) at
 *           b*k_stride_b + h*k_stride_h + n*k_stride_t + d (d-stride 1);
 *           k_stride_b and k_stride_h must be multiples of k_stride_t (the
 *           kernel streams the cache as TMA tiles of a [rows][head_dim]
 *           view), else ASP_ERR_UNSUPPORTED.
 * seq_lens  device int32 [batch], 0 <= seq_lens[b] <= max_seq_len.  Read
 *           twice by the score kernel (once to balance valid tiles over the
 *           SMs before its programmatic-dependent-launch wait, once per
 *           tile), so it must be complete before the PRECEDING kernel on the
 *           stream was launched.  No asyncspade kernel writes seq_lens, and a
 *           kernel that does not trigger PDL (any torch/cuBLAS kernel) runs
 *           to completion before this call's kernels start, so ordinary
 *           stream order suffices; only a caller kernel that itself issues
 *           griddepcontrol.launch_dependents before writing seq_lens breaks
 *           the rule.
 * sel_idx   device int32 [batch][n_kv_heads][top_k], written.  A row with
 *           seq_lens[b] < top_k holds all its tokens then -1 padding and
 *           sets ASP_FLAG_SHORT_ROW (R13).
 * scores    nullable device fp32 [batch][n_kv_heads][max_seq_len]: if
 *           given, the scores are written there (debug/parity) instead of
 *           the workspace; positions >= seq_lens[b] are unspecified.
 * workspace device, >= asyncspade_score_select_workspace(p) bytes, any
 *           contents; 256-B aligned.
 * NaN scores rank below every number and set ASP_FLAG_NONFINITE (R14).
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t batch, n_q_heads, n_kv_heads, head_dim, top_k, max_seq_len, aggregation;
    int64_t k_stride_b, k_stride_h, k_stride_t; /* elements */
} asp_select_params;

ASP_API size_t asyncspade_score_select_workspace(const asp_select_params *p);
ASP_API asp_status asyncspade_score_select(const asp_select_params *p, const float *q_hat,
                                   const asp_bf16 *k_cache, const int32_t *seq_lens,
                                   int32_t *sel_idx, float *scores, void *workspace,
                                   size_t workspace_bytes, uint32_t *dev_flags,
                                   asp_stream stream);

/* ------------------------------------------------------------------------
 * a4  asyncspade_sparse_decode
 *
 * Decode attention of the current query over the selected tokens only
 * ("participate in the attention computation").  For query
 * head hq of KV head h = hq / G, the attended set is
 *     { sel_idx[b,h,j] : 0 <= sel_idx < seq_lens[b] - n_fresh }
 *   U [seq_lens[b] - n_fresh, seq_lens[b])                       (R12)
 * (each token once; -1 and out-of-range entries are ignored), and
 *     out = sum_j softmax_j(sm_scale * q . K_j) V_j
 * with fp32 logits (bf16 x bf16 products are exact), fp32 softmax and fp32
 * accumulation, split over 256-entry chunks of the selection (one chunk
 * when top_k + n_fresh <= 384 and G <= 16) merged in a fixed order (chunk 0
 * first); the split depends only on (top_k, n_fresh, G).  An empty set
 * gives out = 0.
 *
 * q         device bf16 [batch][n_q_heads][head_dim].
 * k_cache, v_cache  device bf16, strided like asp_select_params' K; rows
 *           are gathered by TMA, so stride_b and stride_h must be multiples
 *           of stride_t (ASP_ERR_UNSUPPORTED otherwise).  max_seq_len bounds
 *           every seq_lens[b] (the cache capacity).
 * seq_lens  device int32 [batch].   sel_idx device int32 [batch][n_kv_heads][top_k].
 * out       device fp32, written: element (b, hq, d) at
 *           b * out_stride_b + hq * out_stride_h + d.  out_stride_b ==
 *           out_stride_h == 0 means the dense [batch][n_q_heads][head_dim]
 *           layout; head-major [n_q_heads][batch][head_dim] (out_stride_b =
 *           head_dim, out_stride_h = batch * head_dim) makes the KV-head
 *           sharded outputs of several GPUs one contiguous concatenation
 *           (SURVEY §8(e)).  Strides are in elements, >= 0, multiples of 4.
 * workspace device, >= asyncspade_sparse_decode_workspace(p) bytes, 256-B
 *           aligned, any contents (the split-K partials).
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t batch, n_q_heads, n_kv_heads, head_dim, top_k, n_fresh, max_seq_len;
    float sm_scale; /* usually 1/sqrt(head_dim) */
    int64_t k_stride_b, k_stride_h, k_stride_t, v_stride_b, v_stride_h, v_stride_t;
    int64_t out_stride_b, out_stride_h; /* elements; both 0: dense [B][Hq][D] (ABI 2) */
    int32_t v_head_dim; /* value rows' width; 0: head_dim.  < head_dim: absorbed MLA (ABI 2) */
} asp_decode_params;

ASP_API size_t asyncspade_sparse_decode_workspace(const asp_decode_params *p);
ASP_API asp_status asyncspade_sparse_decode(const asp_decode_params *p, const asp_bf16 *q,
                                    const asp_bf16 *k_cache, const asp_bf16 *v_cache,
                                    const int32_t *seq_lens, const int32_t *sel_idx, float *out,
                                    void *workspace, size_t workspace_bytes, asp_stream stream);

/* ------------------------------------------------------------------------
 * asyncspade_gather_filtered -- the Cache Rank's transfer payload in the
 * paper's disaggregated design ("the
 * selected KV entries are then immediately transferred back"; SPEC
 * gather_filtered): the selected K and V rows packed
 * contiguously, bit-equal to the cache rows,
 *     k_out[b][h][j][:] = K[b][h][sel_idx[b][h][j]][:]   (V likewise)
 * entries that are -1 or >= seq_lens[b] give zero rows, and
 *     idx_out[b][h][j] = j if 0 <= sel_idx[b][h][j] < seq_lens[b] - n_fresh, else -1
 * is the selection over the packed rows: the Inference Rank attends with it
 * over the packed rows plus its own n_fresh newest tokens
 * (asyncspade_sparse_decode on a [B][Hkv][top_k + n_fresh][D] cache) and
 * gets exactly the attended set of the single-rank decode.
 * p         as asyncspade_sparse_decode (sm_scale unused).
 * k_out, v_out  device bf16, written: packed row (b, h, j) at
 *           b * out_stride_b + h * out_stride_h + j * head_dim (elements;
 *           both 0: dense [batch][n_kv_heads][top_k][head_dim]).  With
 *           out_stride_h = (top_k + 1) * head_dim the rows land in the
 *           Inference Rank's compact cache [batch][n_kv_heads][top_k + 1]
 *           [head_dim], whose last row per (b, h) is its own fresh token.
 * idx_out   nullable device int32 [batch][n_kv_heads][top_k], written.
 * ---------------------------------------------------------------------- */
ASP_API asp_status asyncspade_gather_filtered(const asp_decode_params *p, const asp_bf16 *k_cache,
                                      const asp_bf16 *v_cache, const int32_t *seq_lens,
                                      const int32_t *sel_idx, asp_bf16 *k_out, asp_bf16 *v_out,
                                      int32_t *idx_out, asp_stream stream);

/* ------------------------------------------------------------------------
 * Paged KV caches: the block-table layout of paged
 * serving engines, which the paper's baselines run on (P:45, P:78,
 * P:461-465).  The selection itself is unchanged -- token granularity over
 * the LOGICAL token positions of each sequence -- only where a token's K/V
 * row lives differs.
 *
 * A pool holds `num_pages` pages; a page holds `page_size` consecutive
 * tokens of every KV head, head-major inside the page (HND):
 *     element (page, h, t, d) at ((page * n_kv_heads + h) * page_size + t) * head_dim + d
 * Logical token n of sequence b lives in page
 *     block_table[b * max_pages_per_seq + n / page_size], slot n % page_size.
 * page_size is 16, 32, 64 or 128; num_pages * n_kv_heads * page_size < 2^31.
 * Only the block-table entries of pages a sequence uses (n < seq_lens[b])
 * are read; an id outside [0, num_pages) is clamped (the result is then
 * unspecified, but nothing outside the pool is touched).  max_seq_len of the
 * params must be <= max_pages_per_seq * page_size.  The params' k/v strides
 * are ignored.  Everything else -- outputs, precision, determinism, error
 * behaviour -- is that of the dense call: a paged call returns bit for bit
 * what the dense call returns on the same logical cache.
 * ---------------------------------------------------------------------- */
typedef struct {
    int32_t page_size, max_pages_per_seq, num_pages;
} asp_paged_kv;

/* a2+a3 over a paged K pool (k_pages: device bf16 pool; block_table: device
 * int32 [batch][max_pages_per_seq]).  Workspace as asyncspade_score_select. */
ASP_API asp_status asyncspade_score_select_paged(const asp_select_params *p, const asp_paged_kv *pk,
                                         const float *q_hat, const asp_bf16 *k_pages,
                                         const int32_t *block_table, const int32_t *seq_lens,
                                         int32_t *sel_idx, float *scores, void *workspace,
                                         size_t workspace_bytes, uint32_t *dev_flags,
                                         asp_stream stream);

/* a4 over paged K and V pools (same geometry and block table for both).
 * Workspace as asyncspade_sparse_decode. */
ASP_API asp_status asyncspade_sparse_decode_paged(const asp_decode_params *p, const asp_paged_kv *pk,
                                          const asp_bf16 *q, const asp_bf16 *k_pages,
                                          const asp_bf16 *v_pages, const int32_t *block_table,
                                          const int32_t *seq_lens, const int32_t *sel_idx,
                                          float *out, void *workspace, size_t workspace_bytes,
                                          asp_stream stream);

/* ------------------------------------------------------------------------
 * Quest-style page-bound selector -- the in-framework COMPARATOR of SURVEY
 * §8(f) NEXT-4: the paper's baseline (Quest, page size 16; P:78, P:356,
 * P:461-465) selects whole pages by an upper bound of the attention logit,
 * with the CURRENT query (so on the critical path).  SPEC's
 * page_level_select is the definition:
 *   tokens of row (b, h) are cut into consecutive pages of page_size (the
 *   last one may be short); per page and dimension the key max / min over
 *   its tokens are kept; the page bound is
 *     U = max_g sum_d max(q[b,hG+g,d] * maxK_d, q[b,hG+g,d] * minK_d)
 *   (ASP_AGG_SUM: sum_g); the top_k / page_size pages with the largest U
 *   are taken (ties to the lower page) and sel_idx[b,h,:] lists all their
 *   tokens in ascending order, -1 for positions past seq_lens[b] and for
 *   missing pages (fewer pages than top_k / page_size: ASP_FLAG_SHORT_ROW).
 * p         as asyncspade_score_select (dense strided K; top_k must be a
 *           multiple of page_size, else ASP_ERR_SHAPE).  1 <= page_size <= 128.
 * meta      device, >= asyncspade_quest_meta_bytes(p, page_size) bytes,
 *           16-B aligned: the page extremes, written by summarize (bf16,
 *           exact) and read by select.  In a serving engine it is
 *           maintained at KV append time; here it is rebuilt from the cache.
 * q         device fp32 [batch][n_q_heads][head_dim] (the current query).
 * sel_idx   device int32 [batch][n_kv_heads][top_k], written.
 * workspace >= asyncspade_quest_select_workspace(p, page_size), 256-B aligned.
 * Group sizes: G = n_q_heads / n_kv_heads in {1, 2, 4, 8}; others return
 * ASP_ERR_UNSUPPORTED (and a zero workspace size) before enqueuing anything.
 * Precision: fp32 FMA of the exact bf16 extremes (the bound is exact to
 * ~1e-6 relative); deterministic per row.
 * ---------------------------------------------------------------------- */
ASP_API size_t asyncspade_quest_meta_bytes(const asp_select_params *p, int32_t page_size);
ASP_API asp_status asyncspade_quest_summarize(const asp_select_params *p, int32_t page_size,
                                      const asp_bf16 *k_cache, const int32_t *seq_lens,
                                      void *meta, asp_stream stream);
ASP_API size_t asyncspade_quest_select_workspace(const asp_select_params *p, int32_t page_size);
ASP_API asp_status asyncspade_quest_select(const asp_select_params *p, int32_t page_size,
                                   const float *q, const void *meta, const int32_t *seq_lens,
                                   int32_t *sel_idx, void *workspace, size_t workspace_bytes,
                                   uint32_t *dev_flags, asp_stream stream);

/* Human-readable name of a status code (static storage). */
ASP_API const char *asyncspade_status_string(asp_status s);
/* ASYNCSPADE_ABI_VERSION the library was built with. */
ASP_API int32_t asyncspade_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ASYNCSPADE_H */
