// gather.cu -- the Cache Rank's transfer payload (P:187,
// P:190 "the selected KV entries are then immediately transferred back";
// SPEC gather_filtered S:286-293): the selected K and V rows of every
// (b, KV head) packed contiguously, bit-equal to the cache rows.
//   k_out[b][h][j][:] = K[b][h][sel_idx[b][h][j]][:]   (zeros for -1 entries)
//   idx_out[b][h][j]  = j if the entry is attended (0 <= t < len - n_fresh), else -1
// Pure data movement, bound by the random 256-B row reads: one warp per
// selected row pair (K and V), 16-B lanes, many rows in flight per SM.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;

template <int D>
__global__ void __launch_bounds__(kThreads)
gather_kernel(asp_decode_params p, const asp_bf16 *__restrict__ k_cache,
              const asp_bf16 *__restrict__ v_cache, const int32_t *__restrict__ seq_lens,
              const int32_t *__restrict__ sel_idx, asp_bf16 *__restrict__ k_out,
              asp_bf16 *__restrict__ v_out, int32_t *__restrict__ idx_out) {
    constexpr int kLanesPerRow = D / 8;                 // 16 (D = 128) or 8
    constexpr int kRowsPerWarp = 32 / kLanesPerRow;     // rows moved per warp step
    constexpr int kUnroll = 4;
    asp::pdl_wait();                                    // sel_idx comes from select
    asp::pdl_trigger();
    const long rows = (long)p.batch * p.n_kv_heads * p.top_k;
    const int lane = threadIdx.x & 31, sub = lane / kLanesPerRow, c = lane % kLanesPerRow;
    const long warps = (long)gridDim.x * (kThreads / 32);
    const long w0 = (long)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    for (long base = w0 * kRowsPerWarp * kUnroll; base < rows; base += warps * kRowsPerWarp * kUnroll) {
        uint4 kv[kUnroll], vv[kUnroll];
        long r[kUnroll];
        bool live[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {             // all loads first (rows in flight)
            r[u] = base + (long)u * kRowsPerWarp + sub;
            kv[u] = vv[u] = make_uint4(0, 0, 0, 0);
            live[u] = false;
            if (r[u] < rows) {
                const long row = r[u] / p.top_k;        // b * Hkv + h
                const int b = (int)(row / p.n_kv_heads), h = (int)(row % p.n_kv_heads);
                const int len = min(max(seq_lens[b], 0), p.max_seq_len);
                const int t = sel_idx[r[u]];
                live[u] = t >= 0 && t < len - p.n_fresh;
                if (t >= 0 && t < len) {
                    kv[u] = __ldg(reinterpret_cast<const uint4 *>(
                                      k_cache + b * p.k_stride_b + h * p.k_stride_h + (int64_t)t * p.k_stride_t) + c);
                    vv[u] = __ldg(reinterpret_cast<const uint4 *>(
                                      v_cache + b * p.v_stride_b + h * p.v_stride_h + (int64_t)t * p.v_stride_t) + c);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
            if (r[u] < rows) {
                // packed row (b, h, j): dense [B][Hkv][k][D], or (b, h) blocks at the
                // params' out strides (e.g. the Inference Rank's [B][Hkv][k + 1][D]
                // compact cache, row k left for its own fresh token)
                const long bh = r[u] / p.top_k, j = r[u] % p.top_k;
                const int64_t o = p.out_stride_b
                    ? (bh / p.n_kv_heads) * p.out_stride_b + (bh % p.n_kv_heads) * p.out_stride_h + j * D
                    : r[u] * D;
                reinterpret_cast<uint4 *>(k_out + o)[c] = kv[u];
                reinterpret_cast<uint4 *>(v_out + o)[c] = vv[u];
                if (idx_out && c == 0) idx_out[r[u]] = live[u] ? (int)(r[u] % p.top_k) : -1;
            }
        }
    }
}

}  // namespace

cudaError_t asp_launch_gather(const asp_decode_params &p, const asp_bf16 *k_cache,
                              const asp_bf16 *v_cache, const int32_t *seq_lens,
                              const int32_t *sel_idx, asp_bf16 *k_out, asp_bf16 *v_out,
                              int32_t *idx_out, cudaStream_t s) {
    const int grid = 8 * asp_sm_count();                 // 8 CTAs x 8 warps per SM
    if (p.head_dim == 128)
        return asp_launch(gather_kernel<128>, dim3(grid), dim3(kThreads), 0, s, 1, p, k_cache,
                          v_cache, seq_lens, sel_idx, k_out, v_out, idx_out);
    if (p.head_dim == 64)
        return asp_launch(gather_kernel<64>, dim3(grid), dim3(kThreads), 0, s, 1, p, k_cache,
                          v_cache, seq_lens, sel_idx, k_out, v_out, idx_out);
    return cudaErrorInvalidValue;
}
