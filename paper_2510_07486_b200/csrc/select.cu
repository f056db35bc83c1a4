// select.cu -- a3: per-(sequence, KV head) top-k token selection (
// P:267 item (2) "top-k selection"), ties to the LOWER index (reading R9),
// output in ascending index order, -1 padded for short rows (R13).
//
// Design (B200): one 1024-thread CTA per row.  The row's fp32 scores (written
// by the score kernel moments earlier, so L2-resident) are mapped to
// order-preserving uint32 keys and -- for rows up to 40,960 tokens -- kept in
// shared memory for all passes.  The k-th largest key T is found EXACTLY by a
// three-pass MSB radix select (12 + 12 + 8 bits; a 12-bit first digit leaves
// ~3-8% of a 32k row as candidates), each pass a shared-memory
// histogram plus a block suffix scan.  A final ordered pass emits every index
// with key > T plus the first `need` indices with key == T, using one packed
// block scan per 1024-element chunk -- which yields the ascending order for
// free and makes the result independent of thread scheduling.
#include "common.cuh"

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kSmemKeys = 40960;         // 160 KB of cached keys
constexpr int kBins = 4096;

struct SelectSmem {
    uint32_t hist[kBins];
    uint32_t warp_tot[kWarps];
    uint32_t scan_total;
    uint32_t found_bin, found_rem;
    uint32_t keys[kSmemKeys];
};

// Block-wide exclusive scan of one uint32 per thread; returns the exclusive
// prefix and writes the block total to *total (every thread).
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t *warp_tot, uint32_t *total_smem,
                                    uint32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t t = warp_tot[lane];
        uint32_t s = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_tot[lane] = s - t;              // exclusive warp offsets
        if (lane == 31) *total_smem = s;
    }
    __syncthreads();
    const uint32_t r = warp_tot[warp] + x - v;
    *total = *total_smem;
    __syncthreads();                         // warp_tot / total reusable after return
    return r;
}

// Among `nbins` histogram bins (bin value = digit), find the bin holding the
// k_rem-th largest element (1-based) counting from the top bin; store it and
// the rank within the bin in s.found_bin / s.found_rem.
__device__ void find_bucket(SelectSmem &s, int nbins, uint32_t k_rem, uint32_t *total) {
    const int per = nbins / kThreads > 0 ? nbins / kThreads : 1;
    const int t = threadIdx.x;
    // thread t owns bins nbins-1-(t*per + i), i.e. descending order
    uint32_t local = 0;
    const bool owns = t * per < nbins;
    if (owns)
        for (int i = 0; i < per; i++) local += s.hist[nbins - 1 - (t * per + i)];
    uint32_t above = block_excl_scan(local, s.warp_tot, &s.scan_total, total);
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
    uint32_t total;

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

    const bool cached = len <= kSmemKeys;
    bool nan = false;
    if (cached) {
        for (int i = t; i < len; i += kThreads) {
            const uint32_t key = asp::score_key(row[i]);
            nan |= key == 0u;
            s.keys[i] = key;
        }
    }
    auto key_at = [&](int i) -> uint32_t { return cached ? s.keys[i] : asp::score_key(row[i]); };

    // ---- pass 1: bits [31:20]
    for (int i = t; i < kBins; i += kThreads) s.hist[i] = 0;
    __syncthreads();
    for (int i = t; i < len; i += kThreads) {
        const uint32_t key = key_at(i);
        if (!cached) nan |= key == 0u;
        atomicAdd(&s.hist[key >> 20], 1u);
    }
    __syncthreads();
    find_bucket(s, kBins, (uint32_t)k, &total);
    const uint32_t d1 = s.found_bin, rem1 = s.found_rem;
    __syncthreads();
    // ---- pass 2: bits [19:8] among keys with top digit d1
    for (int i = t; i < kBins; i += kThreads) s.hist[i] = 0;
    __syncthreads();
    for (int i = t; i < len; i += kThreads) {
        const uint32_t key = key_at(i);
        if ((key >> 20) == d1) atomicAdd(&s.hist[(key >> 8) & 0xFFFu], 1u);
    }
    __syncthreads();
    find_bucket(s, kBins, rem1, &total);
    const uint32_t d2 = s.found_bin, rem2 = s.found_rem;
    __syncthreads();
    // ---- pass 3: bits [7:0] among keys with prefix (d1, d2)
    const uint32_t pre24 = (d1 << 12) | d2;
    for (int i = t; i < 256; i += kThreads) s.hist[i] = 0;
    __syncthreads();
    for (int i = t; i < len; i += kThreads) {
        const uint32_t key = key_at(i);
        if ((key >> 8) == pre24) atomicAdd(&s.hist[key & 0xFFu], 1u);
    }
    __syncthreads();
    find_bucket(s, 256, rem2, &total);
    const uint32_t T = (pre24 << 8) | s.found_bin;
    const uint32_t need = s.found_rem;       // how many keys == T to take (lowest index first)
    __syncthreads();

    // ---- ordered emission: key > T, or key == T among the first `need` equal keys
    uint32_t carry_gt = 0, carry_eq = 0;
    for (int base = 0; base < len; base += kThreads) {
        const int i = base + t;
        uint32_t gt = 0, eq = 0;
        if (i < len) {
            const uint32_t key = key_at(i);
            gt = key > T;
            eq = key == T;
        }
        const uint32_t packed = (eq << 16) | gt;
        const uint32_t excl = block_excl_scan(packed, s.warp_tot, &s.scan_total, &total);
        const uint32_t eq_before = carry_eq + (excl >> 16);
        const uint32_t gt_before = carry_gt + (excl & 0xFFFFu);
        if (gt || (eq && eq_before < need)) out[gt_before + min(eq_before, need)] = i;
        carry_gt += total & 0xFFFFu;
        carry_eq += total >> 16;
    }
    nan = __syncthreads_or(nan);
    if (t == 0 && nan) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
}

}  // namespace

cudaError_t asp_launch_select(const asp_select_params &p, const float *scores,
                              const int32_t *seq_lens, int32_t *sel_idx, uint32_t *dev_flags,
                              cudaStream_t s) {
    const int smem = (int)sizeof(SelectSmem);
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid(p.n_kv_heads, p.batch);
    select_kernel<<<grid, kThreads, smem, s>>>(p, scores, seq_lens, sel_idx, dev_flags);
    return cudaGetLastError();
}
