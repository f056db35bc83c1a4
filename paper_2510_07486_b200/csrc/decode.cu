// decode.cu -- a4: sparse decode attention over only the selected K/V (P:190
// "the selected KV pairs ... participate in the attention computation";
// P:266), plus the always-attended fresh tail (reading R12).
//
//   out[b,hq] = sum_j softmax_j(sm_scale * q[b,hq] . K[b,h,t_j]) V[b,h,t_j],
//   t_j in {sel_idx valid} U [len - n_fresh, len),  h = hq / G.
//
// Design (B200), split-K: the E = top_k + n_fresh entries of a (b, KV head)
// row are cut into fixed 256-entry chunks, one CTA (4 warps x 64 entries) per
// chunk, so a row's arithmetic order depends only on (top_k, n_fresh).  All G
// query heads of the KV head share each gathered K/V row (GQA reuse).  Within
// a warp, lane j owns entry j of a 32-entry block: it gathers its key row with
// 16-B loads, computes the G logits in fp32 (bf16 x bf16 products are exact),
// and the block updates a running (max, sum) per head with warp-shuffle
// reductions; the value rows are then streamed coalesced (lane = 4 dims) and
// accumulated with per-entry weights broadcast by shuffle.  Warps, then
// chunks, are merged by the log-sum-exp rule in a fixed order; the chunk merge
// is a second small kernel.
#include "common.cuh"

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 256;                   // entries per CTA (fixed: determinism)
constexpr int kPerWarp = kChunk / kWarps;     // 64
constexpr float kLog2e = 1.4426950408889634f;

template <int D, int G>
__global__ void __launch_bounds__(kThreads)
decode_partial_kernel(asp_decode_params p, const asp_bf16 *__restrict__ q,
                      const asp_bf16 *__restrict__ k_cache, const asp_bf16 *__restrict__ v_cache,
                      const int32_t *__restrict__ seq_lens, const int32_t *__restrict__ sel_idx,
                      float *__restrict__ partials, int n_splits) {
    constexpr int DL = D / 32;               // dims per lane in the PV phase (4 or 2)
    __shared__ __align__(16) float qs[G][D];
    __shared__ float wm[kWarps][G], wl[kWarps][G];
    __shared__ __align__(16) float wo[kWarps][G][D];

    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Hq = p.n_q_heads;
    const float scale = p.sm_scale * kLog2e;
    const asp_bf16 *qsrc = q + ((size_t)b * Hq + (size_t)h * G) * D;
    for (int i = threadIdx.x; i < G * D; i += kThreads) qs[i / D][i % D] = asp::bf16f(qsrc[i]);
    __syncthreads();

    const int len = seq_lens[b];
    const int fresh_lo = max(len - p.n_fresh, 0);
    const int E = p.top_k + p.n_fresh;
    const asp_bf16 *kb = k_cache + (size_t)b * p.k_stride_b + (size_t)h * p.k_stride_h;
    const asp_bf16 *vb = v_cache + (size_t)b * p.v_stride_b + (size_t)h * p.v_stride_h;
    const int32_t *ib = sel_idx + ((size_t)b * p.n_kv_heads + h) * p.top_k;

    float m[G], l[G], o[G][DL];
#pragma unroll
    for (int g = 0; g < G; g++) {
        m[g] = -INFINITY;
        l[g] = 0.0f;
#pragma unroll
        for (int i = 0; i < DL; i++) o[g][i] = 0.0f;
    }

    for (int blk = 0; blk < kPerWarp / 32; blk++) {
        const int e = split * kChunk + warp * kPerWarp + blk * 32 + lane;
        int tok = -1;
        if (e < p.top_k) {
            const int t = ib[e];
            if (t >= 0 && t < fresh_lo) tok = t;
        } else if (e < E) {
            const int t = fresh_lo + (e - p.top_k);
            if (t < len) tok = t;
        }
        const unsigned valid_mask = __ballot_sync(0xffffffffu, tok >= 0);
        if (valid_mask == 0u) continue;
        // logits for this lane's entry, all G heads (log2 domain)
        float lg[G];
#pragma unroll
        for (int g = 0; g < G; g++) lg[g] = 0.0f;
        if (tok >= 0) {
            const uint4 *kr = reinterpret_cast<const uint4 *>(kb + (size_t)tok * p.k_stride_t);
#pragma unroll 4
            for (int c = 0; c < D / 8; c++) {
                const uint4 w = __ldg(kr + c);
                const float kk[8] = {asp::bf16lo(w.x), asp::bf16hi(w.x), asp::bf16lo(w.y),
                                     asp::bf16hi(w.y), asp::bf16lo(w.z), asp::bf16hi(w.z),
                                     asp::bf16lo(w.w), asp::bf16hi(w.w)};
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const float4 qa = *reinterpret_cast<const float4 *>(&qs[g][c * 8]);
                    const float4 qb = *reinterpret_cast<const float4 *>(&qs[g][c * 8 + 4]);
                    float a = lg[g];
                    a = fmaf(qa.x, kk[0], a); a = fmaf(qa.y, kk[1], a);
                    a = fmaf(qa.z, kk[2], a); a = fmaf(qa.w, kk[3], a);
                    a = fmaf(qb.x, kk[4], a); a = fmaf(qb.y, kk[5], a);
                    a = fmaf(qb.z, kk[6], a); a = fmaf(qb.w, kk[7], a);
                    lg[g] = a;
                }
            }
#pragma unroll
            for (int g = 0; g < G; g++) lg[g] *= scale;
        } else {
#pragma unroll
            for (int g = 0; g < G; g++) lg[g] = -INFINITY;
        }
        // block-wise online softmax update
        float pw[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            const float mb = asp::warp_max(lg[g]);
            const float mn = fmaxf(m[g], mb);
            const float alpha = exp2f(m[g] - mn);      // m = -inf first time -> 0
            pw[g] = (tok >= 0) ? exp2f(lg[g] - mn) : 0.0f;
            l[g] = l[g] * alpha + asp::warp_sum(pw[g]);
#pragma unroll
            for (int i = 0; i < DL; i++) o[g][i] *= alpha;
            m[g] = mn;
        }
        // PV: stream the value rows of the block's valid entries
        unsigned mask = valid_mask;
        while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const int tj = __shfl_sync(0xffffffffu, tok, j);
            const asp_bf16 *vr = vb + (size_t)tj * p.v_stride_t + lane * DL;
            float vv[DL];
            if constexpr (DL == 4) {
                const uint2 w = __ldg(reinterpret_cast<const uint2 *>(vr));
                vv[0] = asp::bf16lo(w.x); vv[1] = asp::bf16hi(w.x);
                vv[2] = asp::bf16lo(w.y); vv[3] = asp::bf16hi(w.y);
            } else {
                const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(vr));
                vv[0] = asp::bf16lo(w); vv[1] = asp::bf16hi(w);
            }
#pragma unroll
            for (int g = 0; g < G; g++) {
                const float pj = __shfl_sync(0xffffffffu, pw[g], j);
#pragma unroll
                for (int i = 0; i < DL; i++) o[g][i] = fmaf(pj, vv[i], o[g][i]);
            }
        }
    }
    // merge the 4 warps (fixed order)
    if (lane == 0) {
#pragma unroll
        for (int g = 0; g < G; g++) { wm[warp][g] = m[g]; wl[warp][g] = l[g]; }
    }
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
        for (int i = 0; i < DL; i++) wo[warp][g][lane * DL + i] = o[g][i];
    __syncthreads();
    float *dst_base = partials;
    for (int idx = threadIdx.x; idx < G * D; idx += kThreads) {
        const int g = idx / D, d = idx % D;
        float M = -INFINITY;
        for (int w = 0; w < kWarps; w++) M = fmaxf(M, wm[w][g]);
        float L = 0.0f, O = 0.0f;
        if (M != -INFINITY) {
            for (int w = 0; w < kWarps; w++) {
                const float a = exp2f(wm[w][g] - M);
                L = fmaf(wl[w][g], a, L);
                O = fmaf(wo[w][g][d], a, O);
            }
        }
        const int hq = h * G + g;
        float *dst = dst_base + (((size_t)b * Hq + hq) * n_splits + split) * (D + 2);
        dst[2 + d] = O;
        if (d == 0) { dst[0] = M; dst[1] = L; }
    }
}

template <int D>
__global__ void __launch_bounds__(D)
decode_combine_kernel(asp_decode_params p, const float *__restrict__ partials,
                      float *__restrict__ out, int n_splits) {
    const int hq = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
    const float *src = partials + ((size_t)b * p.n_q_heads + hq) * n_splits * (D + 2);
    float M = -INFINITY;
    for (int s = 0; s < n_splits; s++) M = fmaxf(M, src[(size_t)s * (D + 2)]);
    float L = 0.0f, O = 0.0f;
    if (M != -INFINITY) {
        for (int s = 0; s < n_splits; s++) {
            const float *ps = src + (size_t)s * (D + 2);
            const float a = exp2f(ps[0] - M);
            L = fmaf(ps[1], a, L);
            O = fmaf(ps[2 + d], a, O);
        }
    }
    out[((size_t)b * p.n_q_heads + hq) * D + d] = (L > 0.0f) ? O / L : 0.0f;
}

int n_splits_of(const asp_decode_params &p) {
    const int E = p.top_k + p.n_fresh;
    return E > 0 ? (E + kChunk - 1) / kChunk : 1;
}

template <int D, int G>
cudaError_t launch(const asp_decode_params &p, const asp_bf16 *q, const asp_bf16 *k,
                   const asp_bf16 *v, const int32_t *seq_lens, const int32_t *idx, float *out,
                   float *partials, cudaStream_t s) {
    const int ns = n_splits_of(p);
    dim3 grid(ns, p.n_kv_heads, p.batch);
    decode_partial_kernel<D, G><<<grid, kThreads, 0, s>>>(p, q, k, v, seq_lens, idx, partials, ns);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    decode_combine_kernel<D><<<dim3(p.n_q_heads, p.batch), D, 0, s>>>(p, partials, out, ns);
    return cudaGetLastError();
}

}  // namespace

size_t asp_decode_partials_bytes(const asp_decode_params &p) {
    return (size_t)p.batch * p.n_q_heads * n_splits_of(p) * (p.head_dim + 2) * sizeof(float);
}

cudaError_t asp_launch_decode(const asp_decode_params &p, const asp_bf16 *q,
                              const asp_bf16 *k_cache, const asp_bf16 *v_cache,
                              const int32_t *seq_lens, const int32_t *sel_idx, float *out,
                              float *partials, cudaStream_t s) {
    const int G = p.n_q_heads / p.n_kv_heads;
#define ASP_CASE(DD, GG) \
    if (p.head_dim == DD && G == GG) \
        return launch<DD, GG>(p, q, k_cache, v_cache, seq_lens, sel_idx, out, partials, s);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 4) ASP_CASE(64, 8)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 4) ASP_CASE(128, 8)
#undef ASP_CASE
    return cudaErrorInvalidValue;
}
