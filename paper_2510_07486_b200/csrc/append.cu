// append.cu -- a0: the new token enters the state the path reads (SURVEY
// §8(a) a0; "enqueues the query state to the sliding window"):
//   q_window[b][hq][ring_slot] = q_t[b][hq]            (fp32, the predictor's ring)
//   q_cur[b][hq]               = bf16_rn(q_t[b][hq])   (the query decode attends with)
//   K[b][h][pos[b]] = k_new[b][h],  V[b][h][pos[b]] = v_new[b][h]
// One launch instead of the caller's four strided copies, PDL-chained with the
// step's kernels.  Pure data movement: one CTA per sequence, 16-B accesses.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
append_kernel(asp_append_params p, const float *__restrict__ q_t, float *__restrict__ q_window,
              asp_bf16 *__restrict__ q_cur, const asp_bf16 *__restrict__ k_new,
              const asp_bf16 *__restrict__ v_new, asp_bf16 *__restrict__ k_cache,
              asp_bf16 *__restrict__ v_cache, const int32_t *__restrict__ pos) {
    const int b = blockIdx.x, t = threadIdx.x;
    const int D = p.head_dim, W = p.window;
    // every write below overwrites state an earlier kernel of the step reads
    // (the window slot, the current query, the cache row): wait for them
    // No early trigger: the kernels after append (predict, score) read the window
    // and K before their own programmatic-dependent-launch wait, which is safe
    // only because they cannot start before append has completed.
    asp::pdl_wait();
    const int nq4 = p.n_q_heads * D / 4;
    for (int i = t; i < nq4; i += kThreads) {
        const int hq = (4 * i) / D, d = (4 * i) % D;
        const float4 v = reinterpret_cast<const float4 *>(q_t + ((size_t)b * p.n_q_heads + hq) * D)[d / 4];
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t *>(&lo);
        w.y = *reinterpret_cast<const uint32_t *>(&hi);
        const size_t wo = (((size_t)b * p.n_q_heads + hq) * W + p.ring_slot) * D + d;
        if (!q_window) {
        } else if (p.window_bf16) {
            *reinterpret_cast<uint2 *>(reinterpret_cast<asp_bf16 *>(q_window) + wo) = w;
        } else {
            *reinterpret_cast<float4 *>(q_window + wo) = v;
        }
        if (q_cur) *reinterpret_cast<uint2 *>(q_cur + ((size_t)b * p.n_q_heads + hq) * D + d) = w;
    }
    const int n = pos ? pos[b] : -1;
    if (n < 0 || n >= p.max_seq_len) return;
    const int nkv8 = p.n_kv_heads * D / 8;
    for (int i = t; i < nkv8; i += kThreads) {
        const int h = (8 * i) / D, d = (8 * i) % D;
        const size_t src = ((size_t)b * p.n_kv_heads + h) * D + d;
        if (k_new)
            *reinterpret_cast<uint4 *>(k_cache + b * p.k_stride_b + h * p.k_stride_h + n * p.k_stride_t + d) =
                *reinterpret_cast<const uint4 *>(k_new + src);
        if (v_new)
            *reinterpret_cast<uint4 *>(v_cache + b * p.v_stride_b + h * p.v_stride_h + n * p.v_stride_t + d) =
                *reinterpret_cast<const uint4 *>(v_new + src);
    }
}

}  // namespace

cudaError_t asp_launch_append(const asp_append_params &p, const float *q_t, float *q_window,
                              asp_bf16 *q_cur, const asp_bf16 *k_new, const asp_bf16 *v_new,
                              asp_bf16 *k_cache, asp_bf16 *v_cache, const int32_t *pos,
                              cudaStream_t s) {
    return asp_launch(append_kernel, dim3(p.batch), dim3(kThreads), 0, s, 1, p, q_t, q_window, q_cur,
                      k_new, v_new, k_cache, v_cache, pos);
}
