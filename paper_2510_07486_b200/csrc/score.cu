// score.cu -- a2: token criticality q_hat . K per (sequence, KV head), reduced
// over the GQA group (Alg. 1 Step 7; GQA layout P:252-260).
//
//   s[b,h,n] = max_{g<G} sum_d q_hat[b,h*G+g,d] * K[b,h,n,d]      (R10, R11)
//
// v1: CUDA-core streaming kernel.  One thread per token; the token's 256-B
// key row is read with 16-B non-coherent loads (every fetched sector is
// consumed by the same thread), the G x D prediction sits in shared memory
// and is read as warp-wide broadcasts.  Per token the summation order is
// fixed (d ascending per head, then max over g ascending), so equal keys give
// equal scores anywhere in the cache and on any GPU shard.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;

template <int D, int G>
__global__ void __launch_bounds__(kThreads)
score_kernel_v1(asp_select_params p, const float *__restrict__ q_hat,
                const asp_bf16 *__restrict__ k_cache, const int32_t *__restrict__ seq_lens,
                float *__restrict__ scores, uint32_t *dev_flags) {
    __shared__ __align__(16) float qs[G][D];
    const int b = blockIdx.z, h = blockIdx.y;
    const float *qsrc = q_hat + ((size_t)b * p.n_q_heads + (size_t)h * G) * D;
    for (int i = threadIdx.x; i < G * D; i += kThreads) qs[i / D][i % D] = qsrc[i];
    __syncthreads();
    const int len = seq_lens[b];
    const int n = blockIdx.x * kThreads + threadIdx.x;
    if (n >= len) return;
    const uint4 *krow = reinterpret_cast<const uint4 *>(k_cache + (size_t)b * p.k_stride_b +
                                                        (size_t)h * p.k_stride_h +
                                                        (size_t)n * p.k_stride_t);
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; g++) acc[g] = 0.0f;
#pragma unroll 4
    for (int c = 0; c < D / 8; c++) {
        const uint4 w = __ldg(krow + c);
        const float k[8] = {asp::bf16lo(w.x), asp::bf16hi(w.x), asp::bf16lo(w.y), asp::bf16hi(w.y),
                            asp::bf16lo(w.z), asp::bf16hi(w.z), asp::bf16lo(w.w), asp::bf16hi(w.w)};
#pragma unroll
        for (int g = 0; g < G; g++) {
            const float4 qa = *reinterpret_cast<const float4 *>(&qs[g][c * 8]);
            const float4 qb = *reinterpret_cast<const float4 *>(&qs[g][c * 8 + 4]);
            float a = acc[g];
            a = fmaf(qa.x, k[0], a); a = fmaf(qa.y, k[1], a);
            a = fmaf(qa.z, k[2], a); a = fmaf(qa.w, k[3], a);
            a = fmaf(qb.x, k[4], a); a = fmaf(qb.y, k[5], a);
            a = fmaf(qb.z, k[6], a); a = fmaf(qb.w, k[7], a);
            acc[g] = a;
        }
    }
    float s = acc[0];
#pragma unroll
    for (int g = 1; g < G; g++) s = (p.aggregation == ASP_AGG_SUM) ? s + acc[g] : fmaxf(s, acc[g]);
    if (s != s || isinf(s)) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
    scores[((size_t)b * p.n_kv_heads + h) * p.max_seq_len + n] = s;
}

template <int D, int G>
cudaError_t launch(const asp_select_params &p, const float *q_hat, const asp_bf16 *k,
                   const int32_t *seq_lens, float *scores, uint32_t *dev_flags, cudaStream_t s) {
    dim3 grid((p.max_seq_len + kThreads - 1) / kThreads, p.n_kv_heads, p.batch);
    score_kernel_v1<D, G><<<grid, kThreads, 0, s>>>(p, q_hat, k, seq_lens, scores, dev_flags);
    return cudaGetLastError();
}

}  // namespace

cudaError_t asp_launch_score(const asp_select_params &p, const float *q_hat,
                             const asp_bf16 *k_cache, const int32_t *seq_lens, float *scores,
                             uint32_t *dev_flags, cudaStream_t s) {
    const int G = p.n_q_heads / p.n_kv_heads;
#define ASP_CASE(DD, GG) \
    if (p.head_dim == DD && G == GG) return launch<DD, GG>(p, q_hat, k_cache, seq_lens, scores, dev_flags, s);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 4) ASP_CASE(64, 8)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 4) ASP_CASE(128, 8)
#undef ASP_CASE
    return cudaErrorInvalidValue;
}
