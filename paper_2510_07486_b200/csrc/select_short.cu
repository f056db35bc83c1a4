// select_short.cu -- a3 (per-row top-k, ties to the lower index, ascending
// output; P:191, P:267 item (2); readings R9, R13, R14) for SHORT rows
// (<= 4096 tokens, the cut in select.cu: config [4]'s 4k-token rows, the
// short end of config [3]; 8k rows measured slower here than the general kernel).
//
// Many short rows (4096 rows of 4096 keys at config [4] batch 512) make the
// general select kernel latency-bound: its sample -> bracket -> classify ->
// candidate radix chain costs ~40 barrier-separated phases per row.  A short
// row fits in the registers of one CTA (16 or 32 keys per thread, in index
// order), so it is selected exactly with no sample and no candidates:
//   * an MSB-first radix select over all keys, 8 bits per pass (4 passes),
//     warp-private 256-bin histograms (`match.any`-aggregated shared atomics),
//     one 256-wide block scan per pass finds the digit holding the k-th key;
//   * emission: every thread owns a contiguous run of the row, so one block
//     scan of its (key > T, key == T) counts gives each selected index its
//     output slot in index order; the first `need` keys equal to T (lowest
//     index first) complete the set.
// The arithmetic is integer only (order-preserving keys), so the result is
// exactly the general kernel's.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
#ifndef ASP_SHORT_MINB
#define ASP_SHORT_MINB 4
#endif
constexpr int kWarps = kThreads / 32;

struct ShortSmem {
    uint32_t hist[kWarps][256];        // warp-private digit histograms
    uint32_t warp_sum[kWarps];
    uint32_t res[2];                   // chosen digit, rank inside it
};

// exclusive block scan of one value per thread (256 threads); total in *tot
__device__ __forceinline__ uint32_t scan256(ShortSmem &s, uint32_t v, uint32_t *tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s.warp_sum[warp] = x;
    __syncthreads();
    uint32_t before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; w++) {
        const uint32_t ws = s.warp_sum[w];
        before += w < warp ? ws : 0u;
        total += ws;
    }
    *tot = total;
    return before + x - v;
}

template <int KPT>
__global__ void __launch_bounds__(kThreads, KPT == 16 ? ASP_SHORT_MINB : 1)
select_short_kernel(asp_select_params p, const float *__restrict__ scores,
                    const int32_t *__restrict__ seq_lens, int32_t *__restrict__ sel_idx,
                    uint32_t *dev_flags, int discard) {
    __shared__ ShortSmem s;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int h = blockIdx.x, b = blockIdx.y;
    const int k = p.top_k;
    asp::pdl_wait();
    asp::pdl_trigger();
    const int len = min(max(seq_lens[b], 0), p.max_seq_len);
    const size_t row_id = (size_t)b * p.n_kv_heads + h;
    const float *row = scores + row_id * p.max_seq_len;
    int32_t *out = sel_idx + row_id * k;
    if (len <= k) {                          // degrade: all tokens, -1 padding (R13)
        bool nan = false;
        for (int i = t; i < k; i += kThreads) {
            out[i] = i < len ? i : -1;
            if (i < len) nan |= (row[i] != row[i]);
        }
        nan = __syncthreads_or(nan);
        if (t == 0) asp::flag_or(dev_flags, (len < k ? ASP_FLAG_SHORT_ROW : 0u) |
                                                (nan ? ASP_FLAG_NONFINITE : 0u));
        return;
    }
    // ---- the thread's run of the row: keys [t KPT, (t + 1) KPT), index order
    const int i0 = t * KPT;
    uint32_t key[KPT];
    uint32_t valid = 0;
    const bool vec = ((reinterpret_cast<uintptr_t>(row) & 15u) == 0) && i0 + KPT <= len;
    if (vec) {
#pragma unroll
        for (int j = 0; j < KPT; j += 4) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(row + i0 + j));
            key[j] = asp::score_key(v.x);
            key[j + 1] = asp::score_key(v.y);
            key[j + 2] = asp::score_key(v.z);
            key[j + 3] = asp::score_key(v.w);
        }
        valid = KPT == 32 ? 0xffffffffu : (1u << KPT) - 1u;
    } else {
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            const bool ok = i0 + j < len;
            key[j] = ok ? asp::score_key(__ldg(row + i0 + j)) : 0u;
            valid |= (uint32_t)ok << j;
        }
    }
    bool nan = false;
#pragma unroll
    for (int j = 0; j < KPT; j++) nan |= ((valid >> j) & 1u) && key[j] == 0u;   // NaN -> key 0
    // ---- T: MSB-first radix select, 8 bits per pass
    uint32_t prefix = 0, rank = (uint32_t)k;             // rank: 1-based from the top
#pragma unroll 1
    for (int pass = 0; pass < 4; pass++) {
        const int shift = 24 - 8 * pass;
#pragma unroll
        for (int i = lane; i < 256; i += 32) s.hist[warp][i] = 0u;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < KPT; j++) {
            const bool in = ((valid >> j) & 1u) &&
                            (pass == 0 || (key[j] >> (shift + 8)) == prefix);
            const uint32_t dg = in ? (key[j] >> shift) & 255u : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, dg);
            if (in && (__ffs(peers) - 1) == lane) atomicAdd(&s.hist[warp][dg], (uint32_t)__popc(peers));
        }
        __syncthreads();
        // thread t owns digit 255 - t (descending): keys in higher digits come first
        const int dig = 255 - t;
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) c += s.hist[w][dig];
        uint32_t tot;
        const uint32_t before = scan256(s, c, &tot);
        if (before < rank && before + c >= rank) {
            s.res[0] = (uint32_t)dig;
            s.res[1] = rank - before;
        }
        __syncthreads();
        prefix = (prefix << 8) | s.res[0];
        rank = s.res[1];
        __syncthreads();                                 // res / hist reused next pass
    }
    const uint32_t T = prefix, need = rank;              // need: keys == T to take
    // ---- emission in index order: one scan of the packed (gt, eq) counts
    uint32_t gt = 0, eq = 0;
#pragma unroll
    for (int j = 0; j < KPT; j++) {
        const bool ok = (valid >> j) & 1u;
        gt += ok && key[j] > T;
        eq += ok && key[j] == T;
    }
    uint32_t tot;
    const uint32_t pk = scan256(s, (gt << 16) | eq, &tot);
    uint32_t gt_before = pk >> 16, eq_before = pk & 0xFFFFu;
#pragma unroll
    for (int j = 0; j < KPT; j++) {
        if (!((valid >> j) & 1u)) continue;
        if (key[j] > T) {
            out[gt_before + min(eq_before, need)] = i0 + j;
            gt_before++;
        } else if (key[j] == T) {
            if (eq_before < need) out[gt_before + eq_before] = i0 + j;
            eq_before++;
        }
    }
    nan = __syncthreads_or(nan);
    if (t == 0 && nan) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
    if (discard) {
        // the scores are dead once selected: drop the row's whole 128-B lines
        const uintptr_t lo = (reinterpret_cast<uintptr_t>(row) + 127u) & ~(uintptr_t)127u;
        const uintptr_t hi = reinterpret_cast<uintptr_t>(row + len);
        for (uintptr_t x = lo + (uintptr_t)t * 128u; x + 128u <= hi; x += (uintptr_t)kThreads * 128u)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(x) : "memory");
    }
}

}  // namespace

// rows of at most 8192 keys (KPT 16 or 32; select.cu routes only <= 4096 here)
cudaError_t asp_launch_select_short(const asp_select_params &p, const float *scores,
                                    const int32_t *seq_lens, int32_t *sel_idx, uint32_t *dev_flags,
                                    bool discard_scores, cudaStream_t s) {
    const dim3 grid(p.n_kv_heads, p.batch);
    if (p.max_seq_len <= 16 * kThreads)
        return asp_launch(select_short_kernel<16>, grid, dim3(kThreads), 0, s, 1, p, scores,
                          seq_lens, sel_idx, dev_flags, discard_scores ? 1 : 0);
    return asp_launch(select_short_kernel<32>, grid, dim3(kThreads), 0, s, 1, p, scores, seq_lens,
                      sel_idx, dev_flags, discard_scores ? 1 : 0);
}
