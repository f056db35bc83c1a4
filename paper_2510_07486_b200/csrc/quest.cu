// quest.cu -- the Quest-style page-bound selector: the in-framework comparator
// of SURVEY §8(f) NEXT-4 (the paper's baseline at page size 16, P:356,
// P:461-465; SPEC page_level_select).
//
// Tokens are cut into consecutive pages of P (the last one may be short).
// Per (b, KV head, page) the per-dimension key max and min are kept (Quest's
// page metadata); a page's criticality is the upper bound of q . k over its
// keys,
//     U_g = sum_d max(q_gd * max_d, q_gd * min_d) = q_g+ . max + q_g- . min
// (q+ = max(q, 0), q- = min(q, 0)), reduced over the GQA group like the
// token scores (max, reading R10), the top k / P pages are selected with the
// token selector's exact radix select (ties to the lower page), and every
// token of a selected page is attended.
//
// Metadata layout (dim-chunk major, so lanes over pages read coalesced 16-B
// words): meta[row][c][page][8] bf16, row = b * Hkv + h, c in [0, 2 D / 8):
// c < D / 8 holds the max of dims 8c..8c+7, c >= D / 8 the min of dims
// 8(c - D/8)..; page in [0, n_pages_max).  Min / max of bf16 values are
// exact, so the bound is computed from the exact key extremes.
//
// Design (B200): page scoring is an fp32 CUDA-core contraction of 2 D G FMAs
// per page against 4 D bytes of metadata (1/8 of the K bytes at P = 16 and
// G = 8 it is ~4 FMA per byte -- CUDA cores, not tensor cores, at this
// intensity): one thread per page, the group's q+ / q- broadcast from shared
// memory, packed FFMA2.
#include "common.cuh"

namespace {

constexpr int kPagesPerCta = 128;

__host__ __device__ inline int n_pages_of(int len, int P) { return (len + P - 1) / P; }

// ---- page metadata: warp per page, lane over D/32 dims
template <int D>
__global__ void __launch_bounds__(128)
quest_summarize_kernel(asp_select_params p, int P, int npm, const asp_bf16 *__restrict__ k_cache,
                       const int32_t *__restrict__ seq_lens, asp_bf16 *__restrict__ meta) {
    constexpr int kPerLane = D / 32;                 // 4 (D = 128) or 2 (D = 64)
    constexpr int C = D / 8;
    const int row = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int page = blockIdx.y * 4 + warp;
    asp::pdl_wait();
    asp::pdl_trigger();
    const int b = row / p.n_kv_heads, h = row % p.n_kv_heads;
    const int len = min(max(seq_lens[b], 0), p.max_seq_len);
    if (page >= npm || page * P >= len) return;
    const asp_bf16 *kr = k_cache + b * p.k_stride_b + h * p.k_stride_h + lane * kPerLane;
    float mx[kPerLane], mn[kPerLane];
#pragma unroll
    for (int j = 0; j < kPerLane; j++) { mx[j] = -INFINITY; mn[j] = INFINITY; }
    const int t1 = min(len, (page + 1) * P);
    for (int t = page * P; t < t1; t++) {
        const asp_bf16 *src = kr + (int64_t)t * p.k_stride_t;
#pragma unroll
        for (int j = 0; j < kPerLane; j++) {
            const float v = asp::bf16f(src[j]);
            mx[j] = fmaxf(mx[j], v);
            mn[j] = fminf(mn[j], v);
        }
    }
    // lane's dims d0 = lane * kPerLane .. : chunk c = d0 / 8, offset d0 % 8
    const int d0 = lane * kPerLane, c = d0 / 8, o = d0 % 8;
    asp_bf16 *base = meta + ((size_t)row * 2 * C * npm) * 8;
#pragma unroll
    for (int j = 0; j < kPerLane; j++) {
        // bf16 of an exact bf16 value: the top half of its fp32 pattern
        base[((size_t)c * npm + page) * 8 + o + j] = (asp_bf16)(__float_as_uint(mx[j]) >> 16);
        base[((size_t)(C + c) * npm + page) * 8 + o + j] = (asp_bf16)(__float_as_uint(mn[j]) >> 16);
    }
}

// ---- page upper bounds: thread per page, group's q+ / q- in shared memory
template <int D, int G>
__global__ void __launch_bounds__(kPagesPerCta)
quest_score_kernel(asp_select_params p, int P, int npm, const float *__restrict__ q,
                   const asp_bf16 *__restrict__ meta, const int32_t *__restrict__ seq_lens,
                   float *__restrict__ page_scores, int32_t *__restrict__ page_lens) {
    constexpr int C = D / 8;
    __shared__ __align__(16) float s_q[2][D][G];      // [sign][d][g]
    const int row = blockIdx.x;
    const int b = row / p.n_kv_heads, h = row % p.n_kv_heads;
    asp::pdl_wait();
    asp::pdl_trigger();
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
        const int g = i / D, d = i % D;
        const float v = q[((size_t)b * p.n_q_heads + h * G + g) * D + d];
        s_q[0][d][g] = fmaxf(v, 0.0f);
        s_q[1][d][g] = fminf(v, 0.0f);
    }
    __syncthreads();
    const int len = min(max(seq_lens[b], 0), p.max_seq_len);
    const int np = n_pages_of(len, P);
    if (h == 0 && blockIdx.y == 0 && threadIdx.x == 0) page_lens[b] = np;
    const int page = blockIdx.y * kPagesPerCta + threadIdx.x;
    if (page >= np) return;
    const uint4 *mrow = reinterpret_cast<const uint4 *>(meta) + (size_t)row * 2 * C * npm + page;
    float2 acc[G / 2 > 0 ? G / 2 : 1];
    float acc1 = 0.0f;                                 // G == 1
#pragma unroll
    for (int g = 0; g < (G / 2 > 0 ? G / 2 : 1); g++) acc[g] = make_float2(0.0f, 0.0f);
#pragma unroll 2
    for (int c = 0; c < C; c++) {
        const uint4 wx = __ldg(mrow + (size_t)c * npm);          // max of dims 8c..8c+7
        const uint4 wn = __ldg(mrow + (size_t)(C + c) * npm);    // min
        const uint32_t ux[4] = {wx.x, wx.y, wx.z, wx.w}, un[4] = {wn.x, wn.y, wn.z, wn.w};
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int d = 8 * c + j;
            const float x = (j & 1) ? asp::bf16hi(ux[j >> 1]) : asp::bf16lo(ux[j >> 1]);
            const float n = (j & 1) ? asp::bf16hi(un[j >> 1]) : asp::bf16lo(un[j >> 1]);
            if (G == 1) {
                acc1 = fmaf(s_q[0][d][0], x, acc1);
                acc1 = fmaf(s_q[1][d][0], n, acc1);
            } else {
#pragma unroll
                for (int g2 = 0; g2 < G / 2; g2++) {
                    const float2 qp = *reinterpret_cast<const float2 *>(&s_q[0][d][2 * g2]);
                    const float2 qn = *reinterpret_cast<const float2 *>(&s_q[1][d][2 * g2]);
                    acc[g2] = asp::ffma2(qp, make_float2(x, x), acc[g2]);
                    acc[g2] = asp::ffma2(qn, make_float2(n, n), acc[g2]);
                }
            }
        }
    }
    float u;
    if (G == 1) {
        u = acc1;
    } else if (p.aggregation == ASP_AGG_SUM) {
        u = 0.0f;
#pragma unroll
        for (int g2 = 0; g2 < G / 2; g2++) u += acc[g2].x + acc[g2].y;
    } else {
        u = -INFINITY;
#pragma unroll
        for (int g2 = 0; g2 < G / 2; g2++) u = fmaxf(u, fmaxf(acc[g2].x, acc[g2].y));
    }
    page_scores[(size_t)row * npm + page] = u;
}

// ---- selected pages -> their tokens (ascending pages -> ascending tokens;
// positions past the row's length and unselected slots are -1)
__global__ void __launch_bounds__(256)
quest_expand_kernel(asp_select_params p, int P, int kp, const int32_t *__restrict__ page_idx,
                    const int32_t *__restrict__ seq_lens, int32_t *__restrict__ sel_idx) {
    const int row = blockIdx.x;
    asp::pdl_wait();
    asp::pdl_trigger();
    const int b = row / p.n_kv_heads;
    const int len = min(max(seq_lens[b], 0), p.max_seq_len);
    for (int e = threadIdx.x; e < p.top_k; e += blockDim.x) {
        const int pi = page_idx[(size_t)row * kp + e / P];
        int tok = pi >= 0 ? pi * P + e % P : -1;
        if (tok >= len) tok = -1;
        sel_idx[(size_t)row * p.top_k + e] = tok;
    }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

int asp_quest_pages_max(const asp_select_params &p, int P) { return n_pages_of(p.max_seq_len, P); }

size_t asp_quest_meta_bytes(const asp_select_params &p, int P) {
    return (size_t)p.batch * p.n_kv_heads * 2 * p.head_dim * asp_quest_pages_max(p, P) * sizeof(asp_bf16);
}

size_t asp_quest_workspace_bytes(const asp_select_params &p, int P) {
    const size_t npm = (size_t)asp_quest_pages_max(p, P);
    const size_t rows = (size_t)p.batch * p.n_kv_heads;
    return align256(rows * npm * sizeof(float)) + align256((size_t)p.batch * sizeof(int32_t)) +
           align256(rows * (size_t)(p.top_k / P) * sizeof(int32_t));
}

cudaError_t asp_launch_quest_summarize(const asp_select_params &p, int P, const asp_bf16 *k_cache,
                                       const int32_t *seq_lens, void *meta, cudaStream_t s) {
    const int npm = asp_quest_pages_max(p, P);
    const dim3 grid(p.batch * p.n_kv_heads, (npm + 3) / 4);
    auto *m = static_cast<asp_bf16 *>(meta);
    if (p.head_dim == 128)
        return asp_launch(quest_summarize_kernel<128>, grid, dim3(128), 0, s, 1, p, P, npm, k_cache, seq_lens, m);
    if (p.head_dim == 64)
        return asp_launch(quest_summarize_kernel<64>, grid, dim3(128), 0, s, 1, p, P, npm, k_cache, seq_lens, m);
    return cudaErrorInvalidValue;
}

cudaError_t asp_launch_quest_select(const asp_select_params &p, int P, const float *q,
                                    const void *meta, const int32_t *seq_lens, int32_t *sel_idx,
                                    void *workspace, uint32_t *dev_flags, cudaStream_t s) {
    const int npm = asp_quest_pages_max(p, P);
    const size_t rows = (size_t)p.batch * p.n_kv_heads;
    const int kp = p.top_k / P;
    char *ws = static_cast<char *>(workspace);
    float *page_scores = reinterpret_cast<float *>(ws);
    ws += align256(rows * npm * sizeof(float));
    int32_t *page_lens = reinterpret_cast<int32_t *>(ws);
    ws += align256((size_t)p.batch * sizeof(int32_t));
    int32_t *page_idx = reinterpret_cast<int32_t *>(ws);
    const int G = p.n_q_heads / p.n_kv_heads;
    const dim3 grid((unsigned)rows, (npm + kPagesPerCta - 1) / kPagesPerCta);
    const auto *m = static_cast<const asp_bf16 *>(meta);
    cudaError_t e = cudaErrorInvalidValue;
#define ASP_CASE(DD, GG)                                                                      \
    if (p.head_dim == DD && G == GG)                                                          \
        e = asp_launch(quest_score_kernel<DD, GG>, grid, dim3(kPagesPerCta), 0, s, 1, p, P, npm, q, m, \
                       seq_lens, page_scores, page_lens);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 4) ASP_CASE(64, 8)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 4) ASP_CASE(128, 8)
#undef ASP_CASE
    if (e != cudaSuccess) return e;
    // top k / P pages per row: the token selector over the rows of page bounds
    asp_select_params pp = p;
    pp.top_k = kp;
    pp.max_seq_len = npm;
    e = asp_launch_select(pp, page_scores, page_lens, page_idx, dev_flags, true, s);
    if (e != cudaSuccess) return e;
    return asp_launch(quest_expand_kernel, dim3((unsigned)rows), dim3(256), 0, s, 1, p, P, kp,
                      (const int32_t *)page_idx, seq_lens, sel_idx);
}
