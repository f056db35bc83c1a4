// score_cc.cu -- a2 (token criticality, Alg. 1 Step 7) for the
// attention shapes outside the tensor-core stream of score.cu: absorbed MLA
// -- "exactly transformed into MQA during the inference stage through matrix
// absorption": one KV head whose key is the 576-dim latent -- and
// query groups above 32 (multi-query attention with many heads):
//
//   s[b,h,n] = max_{g<G} sum_d q_hat[b,h*G+g,d] * K[b,h,n,d]      (R10, R11)
//
// fp32 FMA on the CUDA cores (bf16 keys widen exactly, fp32 q_hat), a fixed
// per-token summation order (d ascending), so equal keys give equal scores
// and shards reproduce the unsharded scores bit for bit.  These shapes are
// compute-heavier per byte than config [2] (MLA-16: 16 flop/B; MQA-64 at
// D = 128: 64 flop/B), so the kernel is organised as a small GEMM: a CTA
// owns contiguous (row, 64-token tile) items; q_hat of the row sits in
// shared memory (read as warp broadcasts), the key tile is double-buffered
// by cp.async into padded rows, and thread (token t, head group hg) forms
// the dot products of its token with heads hg, hg + 4, ...
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kTok = 64;                       // tokens per tile

template <int D, int G>
struct CcCfg {
    static constexpr int kHG = G < 4 ? G : 4;        // head groups (threads per token)
    static constexpr int kHPT = G / kHG;             // heads per thread
    static constexpr int kRow = D + 8;               // padded smem key row (bf16): no bank conflicts
    static constexpr int kQBytes = G * D * 4;
    static constexpr int kKBytes = kTok * kRow * 2;
    static constexpr int kSmem = kQBytes + 2 * kKBytes + kTok * 4 * 4;
};

template <int D, int G>
__global__ void __launch_bounds__(kThreads)
score_cc_kernel(asp_select_params p, const float *__restrict__ q_hat,
                const asp_bf16 *__restrict__ kc, const int32_t *__restrict__ seq_lens,
                float *__restrict__ scores, uint32_t *dev_flags, int tiles_per_row) {
    using C = CcCfg<D, G>;
    extern __shared__ __align__(16) unsigned char smem[];
    float *sq = reinterpret_cast<float *>(smem);                                  // [G][D]
    asp_bf16 *sk = reinterpret_cast<asp_bf16 *>(smem + C::kQBytes);               // [2][kTok][kRow]
    float *sred = reinterpret_cast<float *>(smem + C::kQBytes + 2 * C::kKBytes);  // [kTok][4]
    const int tid = threadIdx.x;
    const int tok = tid % kTok, hg = tid / kTok;
    const long total = (long)p.batch * p.n_kv_heads * tiles_per_row;
    const long i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;
    asp::pdl_wait();                       // q_hat and K may come from earlier kernels
    asp::pdl_trigger();
    auto len_of = [&](long row) { return min(max(seq_lens[row / p.n_kv_heads], 0), p.max_seq_len); };
    // cp.async one key tile (rows >= the capacity read as zeros) into buffer `buf`
    auto load_tile = [&](long i, int buf) {
        const long row = i / tiles_per_row;
        const int j = (int)(i % tiles_per_row);
        const int b = (int)(row / p.n_kv_heads), h = (int)(row % p.n_kv_heads);
        const asp_bf16 *base = kc + b * p.k_stride_b + h * p.k_stride_h;
        asp_bf16 *dst = sk + buf * (kTok * C::kRow);
        constexpr int kCh = D / 8;                       // 16-B chunks per key row
        for (int c = tid; c < kTok * kCh; c += kThreads) {
            const int r = c / kCh, cc = c % kCh;
            const int n = j * kTok + r;
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + r * C::kRow + cc * 8);
            if (n < p.max_seq_len) {
                const asp_bf16 *src = base + (int64_t)n * p.k_stride_t + cc * 8;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src));
            } else {
                *reinterpret_cast<uint4 *>(dst + r * C::kRow + cc * 8) = make_uint4(0, 0, 0, 0);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // skip tiles past the row's length
    auto next_valid = [&](long i) {
        while (i < i1 && (int)(i % tiles_per_row) * kTok >= len_of(i / tiles_per_row)) i++;
        return i;
    };
    bool nonfinite = false;
    long cur = next_valid(i0), cur_row = -1;
    int buf = 0;
    if (cur < i1) load_tile(cur, 0);
    while (cur < i1) {
        const long row = cur / tiles_per_row;
        const long nxt = next_valid(cur + 1);
        if (row != cur_row) {                           // q_hat of the new row -> smem
            __syncthreads();                            // everyone done with the old q_hat
            const float *qsrc = q_hat + ((size_t)(row / p.n_kv_heads) * p.n_q_heads +
                                         (size_t)(row % p.n_kv_heads) * G) * D;
            for (int c = tid; c < G * D / 4; c += kThreads)
                reinterpret_cast<float4 *>(sq)[c] = reinterpret_cast<const float4 *>(qsrc)[c];
            cur_row = row;
        }
        if (nxt < i1) {
            load_tile(nxt, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();                                // tile `buf` and q_hat visible
        const asp_bf16 *kr = sk + buf * (kTok * C::kRow) + tok * C::kRow;
        float acc[C::kHPT];
#pragma unroll
        for (int e = 0; e < C::kHPT; e++) acc[e] = 0.0f;
#pragma unroll 2
        for (int d = 0; d < D && hg < C::kHG; d += 8) {
            const uint4 kw = *reinterpret_cast<const uint4 *>(kr + d);
            const float k8[8] = {asp::bf16lo(kw.x), asp::bf16hi(kw.x), asp::bf16lo(kw.y),
                                 asp::bf16hi(kw.y), asp::bf16lo(kw.z), asp::bf16hi(kw.z),
                                 asp::bf16lo(kw.w), asp::bf16hi(kw.w)};
#pragma unroll
            for (int e = 0; e < C::kHPT; e++) {
                const float *qg = sq + (hg + e * C::kHG) * D + d;
                const float4 qa = *reinterpret_cast<const float4 *>(qg);
                const float4 qb = *reinterpret_cast<const float4 *>(qg + 4);
                float a = acc[e];
                a = fmaf(qa.x, k8[0], a);
                a = fmaf(qa.y, k8[1], a);
                a = fmaf(qa.z, k8[2], a);
                a = fmaf(qa.w, k8[3], a);
                a = fmaf(qb.x, k8[4], a);
                a = fmaf(qb.y, k8[5], a);
                a = fmaf(qb.z, k8[6], a);
                a = fmaf(qb.w, k8[7], a);
                acc[e] = a;
            }
        }
        // reduce over this thread's heads, then over the head groups (fixed order)
        float s = acc[0];
#pragma unroll
        for (int e = 1; e < C::kHPT; e++)
            s = p.aggregation == ASP_AGG_SUM ? __fadd_rn(s, acc[e]) : fmaxf(s, acc[e]);
        if (hg < C::kHG) sred[tok * 4 + hg] = s;
        __syncthreads();
        if (tid < kTok) {
            float v = sred[tid * 4];
#pragma unroll
            for (int g2 = 1; g2 < C::kHG; g2++)
                v = p.aggregation == ASP_AGG_SUM ? __fadd_rn(v, sred[tid * 4 + g2])
                                                 : fmaxf(v, sred[tid * 4 + g2]);
            const int n = (int)(cur % tiles_per_row) * kTok + tid;
            if (n < len_of(row)) {
                scores[(size_t)row * p.max_seq_len + n] = v;
                nonfinite |= !isfinite(v);
            }
        }
        buf ^= 1;
        cur = nxt;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (__syncthreads_or(nonfinite) && tid == 0) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
}

template <int D, int G>
cudaError_t launch(const asp_select_params &p, const float *q_hat, const asp_bf16 *k,
                   const int32_t *seq_lens, float *scores, uint32_t *dev_flags, cudaStream_t s) {
    using C = CcCfg<D, G>;
    auto kern = score_cc_kernel<D, G>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, C::kSmem);
    if (e != cudaSuccess) return e;
    const int tpr = (p.max_seq_len + kTok - 1) / kTok;
    const long total = (long)p.batch * p.n_kv_heads * tpr;
    const long slots = (long)asp_sm_count() * (per_sm > 0 ? per_sm : 1);
    const int grid = (int)(total < slots ? total : slots);
    return asp_launch(kern, dim3(grid), dim3(kThreads), C::kSmem, s, 1, p, q_hat, k, seq_lens,
                      scores, dev_flags, tpr);
}

}  // namespace

// Shapes: head_dim a multiple of 64 in [64, 576], G in {1, 2, ..., 128},
// G * head_dim <= 16384 (q_hat of a row in shared memory).
bool asp_score_cc_supported(int D, int G) {
    return D % 64 == 0 && D >= 64 && D <= 576 && G >= 1 && G <= 128 && (G & (G - 1)) == 0 &&
           G * D <= 16384;
}

cudaError_t asp_launch_score_cc(const asp_select_params &p, const float *q_hat,
                                const asp_bf16 *k_cache, const int32_t *seq_lens, float *scores,
                                uint32_t *dev_flags, cudaStream_t s) {
    const int G = p.n_q_heads / p.n_kv_heads, D = p.head_dim;
#define ASP_CC(DD, GG) \
    if (D == DD && G == GG) return launch<DD, GG>(p, q_hat, k_cache, seq_lens, scores, dev_flags, s);
    // absorbed MLA (latent 512 + rope 64) and MQA / large-group GQA
    ASP_CC(576, 1) ASP_CC(576, 2) ASP_CC(576, 4) ASP_CC(576, 8) ASP_CC(576, 16)
    ASP_CC(128, 64) ASP_CC(128, 128) ASP_CC(64, 64) ASP_CC(64, 128)
    ASP_CC(256, 1) ASP_CC(256, 8) ASP_CC(256, 16) ASP_CC(256, 32) ASP_CC(256, 64)
#undef ASP_CC
    return cudaErrorInvalidValue;
}
