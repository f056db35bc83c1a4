// common.cuh -- small device helpers shared by the sm_100a kernels of the
// product path.  (Nothing here is shared with oracle/.)
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "asyncspade.h"

#define ASP_DEV __device__ __forceinline__

namespace asp {

// bf16 pair packed in a 32-bit word -> two fp32 (exact: a bf16 is the top
// half of an fp32).
ASP_DEV float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
ASP_DEV float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
ASP_DEV float bf16f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

ASP_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
ASP_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Order-preserving map fp32 score -> uint32 key (larger score, larger key).
// -0.0 is canonicalised to +0.0 (they tie); NaN maps to 0, below every
// number including -inf (reading R14).
ASP_DEV uint32_t score_key(float f) {
    if (f != f) return 0u;
    if (f == 0.0f) f = 0.0f;
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Programmatic dependent launch (PDL): every kernel of the path is launched
// with programmatic stream serialization, so its prologue (barrier init,
// TMEM allocation, descriptor prefetch) overlaps the previous kernel's tail.
// pdl_wait() must precede the first global-memory access of every kernel
// (it returns once the preceding grid has completed and its writes are
// visible -- transitively, every earlier kernel in the stream; every input of
// the path -- window, caches, indices -- may come from an earlier kernel of
// this library, asyncspade_append included); reading caller-only inputs
// (seq_lens) to plan the work may precede it.  pdl_trigger() lets the next
// kernel in the stream start launching.
ASP_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
ASP_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

ASP_DEV void flag_or(uint32_t *dev_flags, uint32_t bits) {
    if (dev_flags && bits) atomicOr(dev_flags, bits);
}

// 2xfp32 packed FMA (Blackwell FFMA2): d = a * b + c on both halves.
ASP_DEV float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)),
          "l"(*reinterpret_cast<unsigned long long *>(&b)),
          "l"(*reinterpret_cast<unsigned long long *>(&c)));
    return d;
}

}  // namespace asp

// Launch `kern` with programmatic stream serialization (PDL) and an optional
// thread-block cluster size (1 = none).
template <typename... KArgs, typename... Args>
cudaError_t asp_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, unsigned cluster, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cluster > 1 ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<Args &&>(args)...);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Internal launchers (implemented per kernel file, called by abi.cu after
// host-side validation).  They return cudaGetLastError() of the launch.
cudaError_t asp_launch_append(const asp_append_params &p, const float *q_t, float *q_window,
                              asp_bf16 *q_cur, const asp_bf16 *k_new, const asp_bf16 *v_new,
                              asp_bf16 *k_cache, asp_bf16 *v_cache, const int32_t *pos,
                              cudaStream_t s);
cudaError_t asp_launch_predict(const asp_predict_params &p, const float *q_window, float *q_hat,
                               uint32_t *dev_flags, cudaStream_t s);
// pk / block_table: a paged pool (asyncspade_*_paged), or nullptr (dense cache)
cudaError_t asp_launch_score(const asp_select_params &p, const float *q_hat,
                             const asp_bf16 *k_cache, const int32_t *seq_lens, float *scores,
                             uint32_t *dev_flags, cudaStream_t s,
                             const asp_paged_kv *pk = nullptr, const int32_t *block_table = nullptr);
// discard_scores: the scores live in the caller's workspace and are dead
// after selection -- their L2 lines are dropped without write-back.
cudaError_t asp_launch_select(const asp_select_params &p, const float *scores,
                              const int32_t *seq_lens, int32_t *sel_idx, uint32_t *dev_flags,
                              bool discard_scores, cudaStream_t s);
// [split-K partials, 256-B aligned][per-(b, KV head) arrival counters, uint32]
size_t asp_decode_workspace_bytes(const asp_decode_params &p);
cudaError_t asp_launch_decode(const asp_decode_params &p, const asp_bf16 *q,
                              const asp_bf16 *k_cache, const asp_bf16 *v_cache,
                              const int32_t *seq_lens, const int32_t *sel_idx, float *out,
                              void *workspace, cudaStream_t s,
                              const asp_paged_kv *pk = nullptr, const int32_t *block_table = nullptr);
// CUDA-core kernels for absorbed MLA / large query groups (score_cc.cu, decode_cc.cu)
bool asp_score_cc_supported(int head_dim, int group);
cudaError_t asp_launch_score_cc(const asp_select_params &p, const float *q_hat,
                                const asp_bf16 *k_cache, const int32_t *seq_lens, float *scores,
                                uint32_t *dev_flags, cudaStream_t s);
bool asp_decode_cc_supported(int head_dim, int v_head_dim, int group);
size_t asp_decode_cc_workspace_bytes(const asp_decode_params &p, int v_head_dim);
cudaError_t asp_launch_decode_cc(const asp_decode_params &p, int v_head_dim, const asp_bf16 *q,
                                 const asp_bf16 *k_cache, const asp_bf16 *v_cache,
                                 const int32_t *seq_lens, const int32_t *sel_idx, float *out,
                                 void *workspace, cudaStream_t s);
// Quest-style page-bound comparator (quest.cu)
size_t asp_quest_meta_bytes(const asp_select_params &p, int page_size);
size_t asp_quest_workspace_bytes(const asp_select_params &p, int page_size);
cudaError_t asp_launch_quest_summarize(const asp_select_params &p, int page_size,
                                       const asp_bf16 *k_cache, const int32_t *seq_lens,
                                       void *meta, cudaStream_t s);
cudaError_t asp_launch_quest_select(const asp_select_params &p, int page_size, const float *q,
                                    const void *meta, const int32_t *seq_lens, int32_t *sel_idx,
                                    void *workspace, uint32_t *dev_flags, cudaStream_t s);
cudaError_t asp_launch_gather(const asp_decode_params &p, const asp_bf16 *k_cache,
                              const asp_bf16 *v_cache, const int32_t *seq_lens,
                              const int32_t *sel_idx, asp_bf16 *k_out, asp_bf16 *v_out,
                              int32_t *idx_out, cudaStream_t s);
int asp_sm_count();
