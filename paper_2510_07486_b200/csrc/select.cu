// select.cu -- a3: per-(sequence, KV head) top-k token selection (
// P:267 item (2) "top-k selection"), ties to the LOWER index (reading R9),
// output in ascending index order, -1 padded for short rows (R13).
//
// Design (B200): one 1024-thread CTA per row.  The row's fp32 scores (written
// by the score kernel just before, so L2-resident) are mapped to
// order-preserving uint32 keys.  The k-th largest key T is found EXACTLY by a
// three-pass MSB radix select (12 + 12 + 8 bits; a 12-bit first digit leaves
// ~3-8% of a 32k row as candidates), each pass a shared-memory
// histogram plus one block suffix scan.  Emission takes every index with
// key > T plus the first `need` indices with key == T, in index order.
//
// Rows up to kMaxCached tokens live in shared memory for all passes, laid out
// as one contiguous segment per thread with an odd segment stride (so the 32
// lanes of a warp always hit 32 different banks): every pass is a
// conflict-free sweep of the thread's own segment, and emission needs a
// single block scan -- each thread then writes its segment's picks in order.
// Longer rows (long-CoT) stream their keys from L2 in every pass and emit
// chunk by chunk.  Either way the result is independent of thread timing.
#include "common.cuh"

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxSeg = 41;                    // odd segment stride bound
constexpr int kMaxCached = kThreads * 40;      // 40,960 tokens in smem
constexpr int kBins = 4096;

struct SelectSmem {
    uint32_t hist[kBins];
    uint32_t warp_tot[kWarps];
    uint32_t scan_total;
    uint32_t found_bin, found_rem;
    uint32_t keys[kThreads * kMaxSeg];
};

// Block-wide exclusive scan of one uint32 per thread; returns the exclusive
// prefix and the block total (every thread).
__device__ uint32_t block_excl_scan(SelectSmem &s, uint32_t v, uint32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s.warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t t = s.warp_tot[lane];
        uint32_t a = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= o) a += y;
        }
        s.warp_tot[lane] = a - t;
        if (lane == 31) s.scan_total = a;
    }
    __syncthreads();
    const uint32_t r = s.warp_tot[warp] + x - v;
    *total = s.scan_total;
    __syncthreads();
    return r;
}

// Find the bin holding the k_rem-th largest element (1-based), counting from
// the top bin; result in s.found_bin / s.found_rem (rank inside the bin).
__device__ void find_bucket(SelectSmem &s, int nbins, uint32_t k_rem) {
    const int per = nbins / kThreads > 0 ? nbins / kThreads : 1;
    const int t = threadIdx.x;
    const bool owns = t * per < nbins;
    uint32_t local = 0;
    if (owns)
        for (int i = 0; i < per; i++) local += s.hist[nbins - 1 - (t * per + i)];
    uint32_t total;
    uint32_t above = block_excl_scan(s, local, &total);
    if (owns) {
        for (int i = 0; i < per; i++) {
            const int bin = nbins - 1 - (t * per + i);
            const uint32_t c = s.hist[bin];
            if (above < k_rem && above + c >= k_rem) {
                s.found_bin = (uint32_t)bin;
                s.found_rem = k_rem - above;
            }
            above += c;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1)
select_kernel(asp_select_params p, const float *__restrict__ scores,
              const int32_t *__restrict__ seq_lens, int32_t *__restrict__ sel_idx,
              uint32_t *dev_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SelectSmem &s = *reinterpret_cast<SelectSmem *>(smem_raw);
    const int b = blockIdx.y, h = blockIdx.x, t = threadIdx.x;
    const int k = p.top_k;
    const int len = min(max(seq_lens[b], 0), p.max_seq_len);
    const float *row = scores + ((size_t)b * p.n_kv_heads + h) * p.max_seq_len;
    int32_t *out = sel_idx + ((size_t)b * p.n_kv_heads + h) * k;

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

    const bool cached = len <= kMaxCached;
    // segment of thread t: indices [t*seg, t*seg + seg), stored at t*stride (stride odd)
    const int seg = (len + kThreads - 1) / kThreads;
    const int stride = seg | 1;
    const int i0 = t * seg;
    const int i1 = min(i0 + seg, len);
    bool nan = false;
    for (int i = t; i < kBins; i += kThreads) s.hist[i] = 0;
    if (cached) {
        for (int i = t; i < len; i += kThreads) {
            const uint32_t key = asp::score_key(__ldcg(row + i));
            nan |= key == 0u;
            const int owner = i / seg;
            s.keys[owner * stride + (i - owner * seg)] = key;
        }
    }
    __syncthreads();

    // ---- pass 1: bits [31:20]
    if (cached) {
        for (int i = i0; i < i1; i++) atomicAdd(&s.hist[s.keys[t * stride + (i - i0)] >> 20], 1u);
    } else {
        for (int i = t; i < len; i += kThreads) {
            const uint32_t key = asp::score_key(__ldcg(row + i));
            nan |= key == 0u;
            atomicAdd(&s.hist[key >> 20], 1u);
        }
    }
    __syncthreads();
    find_bucket(s, kBins, (uint32_t)k);
    const uint32_t d1 = s.found_bin, rem1 = s.found_rem;
    for (int i = t; i < kBins; i += kThreads) s.hist[i] = 0;
    __syncthreads();
    // ---- pass 2: bits [19:8] among keys with top digit d1
    if (cached) {
        for (int i = i0; i < i1; i++) {
            const uint32_t key = s.keys[t * stride + (i - i0)];
            if ((key >> 20) == d1) atomicAdd(&s.hist[(key >> 8) & 0xFFFu], 1u);
        }
    } else {
        for (int i = t; i < len; i += kThreads) {
            const uint32_t key = asp::score_key(__ldcg(row + i));
            if ((key >> 20) == d1) atomicAdd(&s.hist[(key >> 8) & 0xFFFu], 1u);
        }
    }
    __syncthreads();
    find_bucket(s, kBins, rem1);
    const uint32_t pre24 = (d1 << 12) | s.found_bin, rem2 = s.found_rem;
    for (int i = t; i < 256; i += kThreads) s.hist[i] = 0;
    __syncthreads();
    // ---- pass 3: bits [7:0] among keys with prefix pre24
    if (cached) {
        for (int i = i0; i < i1; i++) {
            const uint32_t key = s.keys[t * stride + (i - i0)];
            if ((key >> 8) == pre24) atomicAdd(&s.hist[key & 0xFFu], 1u);
        }
    } else {
        for (int i = t; i < len; i += kThreads) {
            const uint32_t key = asp::score_key(__ldcg(row + i));
            if ((key >> 8) == pre24) atomicAdd(&s.hist[key & 0xFFu], 1u);
        }
    }
    __syncthreads();
    find_bucket(s, 256, rem2);
    const uint32_t T = (pre24 << 8) | s.found_bin;
    const uint32_t need = s.found_rem;       // keys == T to take, lowest index first

    // ---- emission: key > T, or key == T among the first `need` equal keys
    if (cached) {
        uint32_t gt = 0, eq = 0;
        for (int i = i0; i < i1; i++) {
            const uint32_t key = s.keys[t * stride + (i - i0)];
            gt += key > T;
            eq += key == T;
        }
        uint32_t total;                       // counts <= 40,960 < 2^16: pack (eq, gt)
        const uint32_t excl = block_excl_scan(s, (eq << 16) | gt, &total);
        uint32_t gt_before = excl & 0xFFFFu, eq_before = excl >> 16;
        for (int i = i0; i < i1; i++) {
            const uint32_t key = s.keys[t * stride + (i - i0)];
            if (key > T) {
                out[gt_before + min(eq_before, need)] = i;
                gt_before++;
            } else if (key == T) {
                if (eq_before < need) out[gt_before + eq_before] = i;
                eq_before++;
            }
        }
    } else {
        uint32_t carry_gt = 0, carry_eq = 0;
        for (int base = 0; base < len; base += kThreads) {
            const int i = base + t;
            uint32_t gt = 0, eq = 0;
            if (i < len) {
                const uint32_t key = asp::score_key(__ldcg(row + i));
                gt = key > T;
                eq = key == T;
            }
            uint32_t total;
            const uint32_t excl = block_excl_scan(s, (eq << 16) | gt, &total);
            const uint32_t eq_before = carry_eq + (excl >> 16);
            const uint32_t gt_before = carry_gt + (excl & 0xFFFFu);
            if (gt || (eq && eq_before < need)) out[gt_before + min(eq_before, need)] = i;
            carry_gt += total & 0xFFFFu;
            carry_eq += total >> 16;
        }
    }
    nan = __syncthreads_or(nan);
    if (t == 0 && nan) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
}

}  // namespace

cudaError_t asp_launch_select(const asp_select_params &p, const float *scores,
                              const int32_t *seq_lens, int32_t *sel_idx, uint32_t *dev_flags,
                              cudaStream_t s) {
    const int smem = (int)sizeof(SelectSmem);
    cudaError_t e =
        cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    dim3 grid(p.n_kv_heads, p.batch);
    select_kernel<<<grid, kThreads, smem, s>>>(p, scores, seq_lens, sel_idx, dev_flags);
    return cudaGetLastError();
}
