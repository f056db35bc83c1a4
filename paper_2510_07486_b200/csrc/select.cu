// select.cu -- a3: per-(sequence, KV head) top-k token selection (
// P:267 item (2) "top-k selection"), ties to the LOWER index (reading R9),
// output in ascending index order, -1 padded for short rows (R13).
//
// Definition: map every fp32 score to an order-preserving uint32 key, find
// the k-th largest key T, and emit every index with key > T plus the first
// `need` indices with key == T (need = k - #{key > T}), in index order.
//
// Design (B200).  Selection is latency- and issue-bound, not byte-bound (a
// 32k row is 128 KB), so the kernel keeps MANY rows in flight -- small
// 256-thread CTAs with ~57 KB of shared memory, 4 per SM, every row of
// config [2] resident at once -- and arranges each sweep over the row (read
// from L2 with coalesced 16-B lane loads, 4 in flight per lane) for few
// instructions per key:
//   1. SAMPLE: a 12-bit histogram (bits 31:20) of every s-th key (~16 per
//      thread) brackets T: the bins holding sample ranks r -/+ delta (r the
//      expected sample rank of T, delta ~3 sigma of its binomial spread).
//   2. CLASSIFY: a ballot sweep (32 consecutive keys per warp step) counts
//      the keys above the bracket and compacts the bracketed ones into
//      per-warp candidate lists (no shared counter).
//   3. EXACT T: if #above < k <= #above + #candidates, an MSB radix select
//      (12 + 12 + 8 bits) over the candidates alone finds T and `need`;
//      otherwise (an unlucky sample, massive ties, a candidate overflow) the
//      same radix select runs over every key.  Either way T is exact: the
//      sample only decides how much work finding it takes.
//   4. EMIT: per round of 32,768 keys, a ballot sweep writes two bitmaps
//      (key > T, key == T); a block scan of their popcounts gives every word
//      its output offset and each thread writes its words' indices in order.
//      No atomics touch the output, so it is independent of timing.
// A row may be split over a thread-block CLUSTER of C CTAs (C = 1..16, chosen
// on the host so that few long rows still fill the SMs: a long-CoT 512k row
// runs on 16 SMs): each CTA owns a contiguous segment, and histograms, counts
// and emission offsets are merged across the cluster through distributed
// shared memory in rank order (integer sums -- the result never depends on C).
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace cg = cooperative_groups;

#ifdef ASP_PROFILE_SELECT
__device__ unsigned long long g_sel_prof[8];
#define SPROF(idx)                                                                       \
    do {                                                                                 \
        if (threadIdx.x == 0) {                                                          \
            const long long _t = clock64();                                              \
            atomicAdd(&g_sel_prof[idx], (unsigned long long)(_t - _tp));                 \
            _tp = _t;                                                                    \
        }                                                                                \
    } while (0)
extern "C" __attribute__((visibility("default"))) int asp_select_prof_read(unsigned long long *h) {
    cudaMemcpyFromSymbol(h, g_sel_prof, sizeof(g_sel_prof));
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_sel_prof, z, sizeof(z));
    return 0;
}
#else
#define SPROF(idx) (void)0
#endif

namespace sel256 {
#define SEL_NT 256
#define SEL_MINB 4
#define SEL_ROUND 32768
#include "select_impl.cuh"
#undef SEL_NT
#undef SEL_MINB
#undef SEL_ROUND
}  // namespace sel256

namespace sel1024 {
#define SEL_NT 1024
#define SEL_MINB 1
#define SEL_ROUND 32768
#include "select_impl.cuh"
#undef SEL_NT
#undef SEL_MINB
#undef SEL_ROUND
}  // namespace sel1024

namespace sel1024w {              // 64k-key segments (long rows over a cluster)
#define SEL_NT 1024
#define SEL_MINB 1
#define SEL_ROUND 65536
#include "select_impl.cuh"
#undef SEL_NT
#undef SEL_MINB
#undef SEL_ROUND
}  // namespace sel1024w

namespace {

constexpr int kMaxCluster = 16;

long ceil_div(long a, long b) { return (a + b - 1) / b; }

}  // namespace

cudaError_t asp_launch_select_short(const asp_select_params &p, const float *scores,
                                    const int32_t *seq_lens, int32_t *sel_idx, uint32_t *dev_flags,
                                    bool discard_scores, cudaStream_t s);

cudaError_t asp_launch_select(const asp_select_params &p, const float *scores,
                              const int32_t *seq_lens, int32_t *sel_idx, uint32_t *dev_flags,
                              bool discard_scores, cudaStream_t s) {
    const long L = p.max_seq_len;
#ifndef ASP_SELECT_SHORT_MAX
#define ASP_SELECT_SHORT_MAX 4096
#endif
    // short rows (<= 4k keys): the whole row in one CTA's registers, exact radix
    // select with no sample / candidate phases (select_short.cu)
    if (L <= ASP_SELECT_SHORT_MAX)
        return asp_launch_select_short(p, scores, seq_lens, sel_idx, dev_flags, discard_scores, s);
    const long rows = (long)p.batch * p.n_kv_heads;
    // Cluster size (measured on B200): segments of <= 64k keys, then split
    // further only while the rows could not even occupy a quarter of the SMs,
    // keeping segments >= 16k keys (DSMEM merges cost more than they save on
    // shorter segments).
    const long target = asp_sm_count() / 4;
    int C = 1;
    while (C < kMaxCluster && ceil_div(L, C) > 65536) C *= 2;
    while (C < kMaxCluster && rows * C < target && ceil_div(L, 2 * C) >= 16384) C *= 2;
#ifdef ASP_PROFILE_SELECT
    if (const char *env = getenv("ASP_SELECT_CLUSTER")) C = atoi(env);   // experiments only
#endif
    const int seg = (int)(ceil_div(ceil_div(L, C), 128) * 128);
    // Few CTAs in total (each alone on an SM): 1024 threads per CTA shorten
    // every row's chain of sweeps and barriers; otherwise 256-thread CTAs,
    // four per SM, overlap the rows.
    const bool wide = rows * C < asp_sm_count();
#define ASP_SELECT_LAUNCH(NS)                                                              \
    do {                                                                                   \
        const int smem = (int)sizeof(NS::SelectSmem);                                      \
        cudaError_t e = cudaFuncSetAttribute(NS::select_kernel,                            \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        if (e != cudaSuccess) return e;                                                    \
        if (C > 8) {                                                                       \
            e = cudaFuncSetAttribute(NS::select_kernel,                                    \
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);   \
            if (e != cudaSuccess) return e;                                                \
        }                                                                                  \
        return asp_launch(NS::select_kernel, dim3(C * p.n_kv_heads, p.batch),              \
                          dim3(NS::kThreads), smem, s, (unsigned)C, p, scores, seq_lens,   \
                          sel_idx, dev_flags, C, seg, discard_scores ? 1 : 0);             \
    } while (0)
    if (wide && seg > 32768) ASP_SELECT_LAUNCH(sel1024w);
    if (wide) ASP_SELECT_LAUNCH(sel1024);
    ASP_SELECT_LAUNCH(sel256);
#undef ASP_SELECT_LAUNCH
}

#ifdef ASP_PROFILE_SELECT
// dev only (instrumented build): the select kernel alone on a caller-kept score buffer
extern "C" __attribute__((visibility("default"))) int asp_select_only(
    const asp_select_params *p, const float *scores, const int32_t *seq_lens, int32_t *sel_idx,
    uint32_t *dev_flags, void *stream) {
    return (int)asp_launch_select(*p, scores, seq_lens, sel_idx, dev_flags, false, (cudaStream_t)stream);
}
#endif
