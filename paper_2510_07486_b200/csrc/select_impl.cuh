// select_impl.cuh -- the select kernel body, instantiated by select.cu for
// SEL_NT threads per CTA (256: many rows, several CTAs per SM; 1024: few
// rows, one CTA per SM) inside a namespace of its own.  See select.cu.

constexpr int kThreads = SEL_NT;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 4096;
constexpr int kCand = 2048;                   // candidate slots per CTA
// keys per emission round (bitmap size): a segment of up to kRound keys is
// "direct" -- its classify sweep seeds the emission bitmaps, so the keys are
// read once.  32k, or 64k for the 64k-key segments of rows split over a
// cluster (1024-thread CTAs, one per SM, afford the bitmaps).
constexpr int kRound = SEL_ROUND;
constexpr int kSampleChunks = 32;             // 32 x 128 consecutive keys sampled per row
constexpr int kMaxCluster = 16;
constexpr int kUnroll = 8;                    // 16-B loads in flight per lane (classify)
struct SelectSmem {
    uint32_t hist[kBins];
    uint32_t red[kBins / 2];       // this rank's reduced slice of a cluster histogram (C >= 2)
    uint32_t cand[kCand];          // candidate keys (any order)
    uint32_t cand_idx[kCand];      // their segment offsets
    uint32_t bm_gt[kRound / 32];
    uint32_t bm_eq[kRound / 32];
    uint32_t n_cand;
    uint32_t warp_a[kWarps], warp_b[kWarps];
    uint32_t scan_total;
    uint32_t found_bin, found_rem, found_bin2;
    uint32_t cnt[4];                     // this CTA's counts (read by the cluster)
    uint32_t peer[kMaxCluster][4];       // every rank's counts, copied in
};

__device__ __forceinline__ uint32_t comp(const uint4 &k, int c) {
    return c == 0 ? k.x : c == 1 ? k.y : c == 2 ? k.z : k.w;
}
__device__ __forceinline__ float comp(const float4 &v, int c) {
    return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

// The smallest fp32 v with score_key(v) >= K (so v >= lb <=> key(v) >= K for
// every non-NaN v, -0 and +0 included); K beyond every key gives NaN (no v
// compares >=), K at or below key(-inf) gives -inf.
__device__ __forceinline__ float key_lower_bound(uint64_t K) {
    if (K > 0xFF800000ull) return __uint_as_float(0x7FC00000u);
    if (K <= 0x007FFFFFull) return -INFINITY;
    const uint32_t k = (uint32_t)K;
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Block sum of a warp-uniform per-warp value (every thread gets it).
__device__ uint32_t block_sum_warps(SelectSmem &s, uint32_t v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s.warp_b[warp] = v;
    __syncthreads();
    const uint32_t a = warp_sum_u32(lane < kWarps ? s.warp_b[lane] : 0u);
    __syncthreads();
    return a;
}

// Block-wide exclusive scan of one uint32 per thread; returns the exclusive
// prefix, *total = block sum (every thread).
__device__ uint32_t block_excl_scan(SelectSmem &s, uint32_t v, uint32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s.warp_a[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t t = lane < kWarps ? s.warp_a[lane] : 0u;
        uint32_t a = t;
#pragma unroll
        for (int o = 1; o < kWarps; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= o) a += y;
        }
        if (lane < kWarps) s.warp_a[lane] = a - t;
        if (lane == kWarps - 1) s.scan_total = a;
    }
    __syncthreads();
    const uint32_t r = s.warp_a[warp] + x - v;
    *total = s.scan_total;
    __syncthreads();
    return r;
}

// Bins holding the rank_a-th and rank_b-th largest elements (1-based,
// counted from the top bin; rank_a <= rank_b) -> s.found_bin with the rank
// inside it (s.found_rem), and s.found_bin2.  A rank beyond the total gives
// bin 0.  Thread t owns bins [nbins - PER (t+1), nbins - PER t), read as
// 16-B vectors; one block scan orders the threads from the top.
template <int PER>
__device__ __noinline__ void find_bucket_t(SelectSmem &s, int nbins, uint32_t rank_a, uint32_t rank_b) {
    const int t = threadIdx.x;
    const int lo = nbins - PER * (t + 1);          // < 0: this thread owns no bins
    if (t == 0) {
        s.found_bin = s.found_bin2 = 0;
        s.found_rem = rank_a;
    }
    uint32_t c[PER];
    if (lo < 0) {
#pragma unroll
        for (int i = 0; i < PER; i++) c[i] = 0;
    } else if constexpr (PER % 4 == 0) {
#pragma unroll
        for (int i = 0; i < PER; i += 4) {
            const uint4 v = *reinterpret_cast<const uint4 *>(&s.hist[lo + i]);
            c[i] = v.x;
            c[i + 1] = v.y;
            c[i + 2] = v.z;
            c[i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < PER; i++) c[i] = s.hist[lo + i];
    }
    uint32_t local = 0;
#pragma unroll
    for (int i = 0; i < PER; i++) local += c[i];
    uint32_t total;
    uint32_t above = block_excl_scan(s, local, &total);   // syncs: the init is visible first
    if (lo >= 0 && above < rank_b && above + local >= rank_a) {
#pragma unroll
        for (int i = PER - 1; i >= 0; i--) {
            const uint32_t cc = c[i];
            if (above < rank_a && above + cc >= rank_a) {
                s.found_bin = (uint32_t)(lo + i);
                s.found_rem = rank_a - above;
            }
            if (above < rank_b && above + cc >= rank_b) s.found_bin2 = (uint32_t)(lo + i);
            above += cc;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void find_bucket(SelectSmem &s, int nbins, uint32_t rank_a,
                                            uint32_t rank_b) {
    constexpr int kPerBig = kBins / kThreads > 0 ? kBins / kThreads : 1;
    constexpr int kPerSmall = 256 / kThreads > 0 ? 256 / kThreads : 1;
    if (nbins == kBins) find_bucket_t<kPerBig>(s, nbins, rank_a, rank_b);
    else find_bucket_t<kPerSmall>(s, nbins, rank_a, rank_b);
}

__device__ __forceinline__ void zero_hist(SelectSmem &s, int nbins) {
    for (int i = 4 * threadIdx.x; i < nbins; i += 4 * kThreads)
        *reinterpret_cast<uint4 *>(&s.hist[i]) = make_uint4(0u, 0u, 0u, 0u);
}

// Sum the first nbins bins of every cluster rank's histogram (rank order)
// into this CTA's histogram.
// (the cluster parts are out of line: single-CTA rows never run them, and
// inlined at every call site they would only lengthen the code a warp fetches)
__device__ __noinline__ void merge_hist_cluster(SelectSmem &s, int nbins, int C);
__device__ __forceinline__ void merge_hist(SelectSmem &s, int nbins, int C) {
    __syncthreads();
    if (C > 1) merge_hist_cluster(s, nbins, C);
}
__device__ __noinline__ void merge_hist_cluster(SelectSmem &s, int nbins, int C) {
    // reduce-scatter, then all-gather, through DSMEM: rank r sums its slice of
    // nbins / C bins over every rank (all C remote loads of a bin in flight at
    // once), then every rank reads the reduced slices back from their owners.
    // Integer sums in rank order: the result never depends on timing.
    cg::cluster_group cl = cg::this_cluster();
    const int me = (int)cl.block_rank();
    const int slice = nbins / C;                      // C | nbins (C, nbins powers of 2)
    cl.sync();                                        // every rank's histogram is final
    for (int i = threadIdx.x; i < slice; i += kThreads) {
        const int bin = me * slice + i;
        uint32_t v[kMaxCluster];
#pragma unroll
        for (int r = 0; r < kMaxCluster; r++) v[r] = r < C ? cl.map_shared_rank(s.hist, r)[bin] : 0u;
        uint32_t acc = 0;
#pragma unroll
        for (int r = 0; r < kMaxCluster; r++) acc += v[r];
        s.red[i] = acc;
    }
    cl.sync();                                        // slices reduced; hist no longer read remotely
    constexpr int kPer = kBins / kThreads;
    uint32_t acc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        const int bin = threadIdx.x + j * kThreads;
        acc[j] = bin < nbins ? cl.map_shared_rank(s.red, bin / slice)[bin % slice] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        const int bin = threadIdx.x + j * kThreads;
        if (bin < nbins) s.hist[bin] = acc[j];
    }
    __syncthreads();    // (red is next written after the next merge's first cluster barrier,
                        // which every rank reaches only after this gather)
}

// Cluster-wide totals of s.cnt[0..n) and their sums over earlier ranks
// (exclusive prefix), for every thread.  s.cnt must be written before.
__device__ __noinline__ void cluster_counts(SelectSmem &s, int C, int n, uint32_t *tot, uint32_t *before) {
    __syncthreads();
    if (C == 1) {
        for (int j = 0; j < n; j++) {
            tot[j] = s.cnt[j];
            before[j] = 0;
        }
        return;
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if ((int)threadIdx.x < C) {                      // one remote read per rank and count
        const SelectSmem *peer = cl.map_shared_rank(&s, (int)threadIdx.x);
        for (int j = 0; j < n; j++) s.peer[threadIdx.x][j] = peer->cnt[j];
    }
    cl.sync();                                       // peers may now overwrite cnt
    const int me = (int)cl.block_rank();
    for (int j = 0; j < n; j++) {
        tot[j] = before[j] = 0;
        for (int r = 0; r < C; r++) {
            tot[j] += s.peer[r][j];
            if (r < me) before[j] += s.peer[r][j];
        }
    }
}

__global__ void __launch_bounds__(kThreads, SEL_MINB)
select_kernel(asp_select_params p, const float *__restrict__ scores,
              const int32_t *__restrict__ seq_lens, int32_t *__restrict__ sel_idx,
              uint32_t *dev_flags, int C, int seg_len, int discard) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SelectSmem &s = *reinterpret_cast<SelectSmem *>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int crank = blockIdx.x % C;
    const int h = blockIdx.x / C, b = blockIdx.y;
    const int k = p.top_k;
    asp::pdl_wait();
    asp::pdl_trigger();
    const int len = min(max(seq_lens[b], 0), p.max_seq_len);
    const size_t row_id = (size_t)b * p.n_kv_heads + h;
    const float *row = scores + row_id * p.max_seq_len;
    int32_t *out = sel_idx + row_id * k;

    if (len <= k) {                          // degrade: all tokens, -1 padding (R13)
        if (crank != 0) return;              // uniform over the cluster: nobody syncs
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

    const int seg0 = min(crank * seg_len, len);
    const int n = min(seg0 + seg_len, len) - seg0;        // keys in this CTA's segment
    const float *srow = row + seg0;
    const bool vec = ((reinterpret_cast<uintptr_t>(row) & 15u) == 0);   // seg0 % 128 == 0
    auto key_at = [&](int o) -> uint32_t { return asp::score_key(__ldg(srow + o)); };
    // base[o..o+3] (o % 4 == 0), elements >= lim read as 0.  Callers issue
    // all their loads before converting any (in-order issue: a conversion
    // right after its load would serialise the loads).
    auto raw4 = [&](const float *base, int o, int lim) -> float4 {
        if (vec && o + 3 < lim) return __ldg(reinterpret_cast<const float4 *>(base + o));
        float4 v;
        v.x = o + 0 < lim ? __ldg(base + o + 0) : 0.f;
        v.y = o + 1 < lim ? __ldg(base + o + 1) : 0.f;
        v.z = o + 2 < lim ? __ldg(base + o + 2) : 0.f;
        v.w = o + 3 < lim ? __ldg(base + o + 3) : 0.f;
        return v;
    };
    auto keys4 = [](const float4 &v) -> uint4 {
        return make_uint4(asp::score_key(v.x), asp::score_key(v.y), asp::score_key(v.z),
                          asp::score_key(v.w));
    };
    const bool direct = n <= kRound;         // the classify sweep can seed the bitmaps

    zero_hist(s, kBins);
    for (int i = t; i < kRound / 32; i += kThreads) s.bm_eq[i] = 0;
    if (t == 0) s.n_cand = 0;
    __syncthreads();
#ifdef ASP_PROFILE_SELECT
    long long _tp = clock64();
#endif

    // ---- 1. sample: kSampleChunks blocks of 128 consecutive keys spread over
    // the ROW (every cluster rank draws the same sample: no merge needed),
    // kept in registers for the second-level histogram
    const int row_chunks = (len + 127) >> 7;
    const int ns = min(kSampleChunks, row_chunks);
    constexpr int kPerWarp = kSampleChunks / kWarps;
    uint4 sk[kPerWarp];
    int so[kPerWarp];
    {
        float4 sv[kPerWarp];
#pragma unroll
        for (int u = 0; u < kPerWarp; u++) {
            const int j = warp + u * kWarps;
            so[u] = j < ns ? ((j * row_chunks / ns) << 7) + 4 * lane : len;   // < 2^31
            sv[u] = raw4(row, so[u], len);
        }
#pragma unroll
        for (int u = 0; u < kPerWarp; u++) sk[u] = keys4(sv[u]);
    }
#pragma unroll
    for (int u = 0; u < kPerWarp; u++)
#pragma unroll
        for (int c = 0; c < 4; c++)
            if (so[u] + c < len) atomicAdd(&s.hist[comp(sk[u], c) >> 20], 1u);
    // sample size: ns full chunks, unless the last one sampled is the row's
    // partial last chunk
    uint32_t m = 128u * ns;
    if ((ns - 1) * row_chunks / ns == row_chunks - 1) m -= (uint32_t)(row_chunks * 128 - len);
    __syncthreads();
    SPROF(0);
    // bracket T between sample ranks r -/+ delta (1-based from the top)
    const double pk = (double)k / len;
    const double r = pk * m;
    const double delta = 3.0 * sqrt(r * (1.0 - pk)) + 4.0;
    const uint32_t rank_hi = (uint32_t)fmax(1.0, floor(r - delta));
    const uint32_t rank_lo = (uint32_t)fmax(1.0, fmin((double)m, ceil(r + delta)));
    find_bucket(s, kBins, rank_hi, rank_lo);
    const uint32_t bin_hi = s.found_bin, bin_lo = s.found_bin2;      // bin_lo <= bin_hi
    // samples above bin_hi
    const uint32_t above_s = rank_hi - s.found_rem;
    uint32_t key_lo = bin_lo << 20, key_hi = ((bin_hi + 1) << 20) - 1u;
    if (bin_hi - bin_lo < 16) {
        // second level: 8 more bits (19:12) over the bracketed samples
        zero_hist(s, kBins);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPerWarp; u++)
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const uint32_t key = comp(sk[u], c);
                if (so[u] + c < len && key >= key_lo && key <= key_hi)
                    atomicAdd(&s.hist[(key - key_lo) >> 12], 1u);
            }
        __syncthreads();
        find_bucket(s, kBins, rank_hi - above_s, rank_lo - above_s);
        const uint32_t f_hi = s.found_bin, f_lo = s.found_bin2;
        const uint32_t base = key_lo;
        key_lo = base + (f_lo << 12);
        key_hi = base + ((f_hi + 1) << 12) - 1u;
    }
    SPROF(1);

    // ---- 2. classify the segment: count the keys above the bracket and
    // collect the bracketed ones (key, offset) into the candidate list; NaN
    // detection rides along.  A warp step covers 128 consecutive keys, 4 per
    // lane (one 16-B load).  The bracket is compared in fp32 -- v >= lb(K)
    // <=> key(v) >= K -- so a key is only formed for the few candidates.
    // Direct segments (<= kRound keys) only mark both classes in bitmaps
    // (bm_gt: above, bm_eq: candidate) and gather the candidates afterwards.
    const int nchunks = (n + 127) >> 7;
    const float f_lo = key_lower_bound(key_lo);
    const float f_above = key_lower_bound((uint64_t)key_hi + 1);
    bool nan = false;
    {
        uint32_t above = 0;
        for (int c0 = warp; c0 < nchunks; c0 += kUnroll * kWarps) {
            const bool full = vec && ((c0 + (kUnroll - 1) * kWarps) << 7) + 128 <= n;
            float4 kv[kUnroll];
            if (full) {
#pragma unroll
                for (int u = 0; u < kUnroll; u++)
                    kv[u] = __ldg(reinterpret_cast<const float4 *>(srow + ((c0 + u * kWarps) << 7)) + lane);
            } else {
#pragma unroll
                for (int u = 0; u < kUnroll; u++) {
                    const int ch = c0 + u * kWarps;
                    kv[u] = raw4(srow, (ch << 7) + 4 * lane, ch < nchunks ? n : 0);
                }
            }
#pragma unroll
            for (int u = 0; u < kUnroll; u++) {
                const int ch = c0 + u * kWarps;
                if (ch >= nchunks) break;                      // warp-uniform
                const int o = (ch << 7) + 4 * lane;
                const uint32_t valid = full || o + 3 < n ? 0xFu : (0xFu >> min(4, o + 4 - n)) & 0xFu;
                uint32_t ab = 0, in = 0;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const float v = comp(kv[u], c);
                    nan |= v != v;
                    ab |= (uint32_t)(v >= f_above) << c;
                    in |= (uint32_t)(v >= f_lo) << c;
                }
                ab &= valid;
                in &= valid & ~ab;
                above += __popc(ab);
                if (direct) {                 // word ch*4 + lane/8 <- nibbles of 8 lanes
                    uint32_t wa = ab << (4 * (lane & 7)), wc = in << (4 * (lane & 7));
#pragma unroll
                    for (int d = 1; d < 8; d <<= 1) {
                        wa |= __shfl_xor_sync(0xffffffffu, wa, d);
                        wc |= __shfl_xor_sync(0xffffffffu, wc, d);
                    }
                    if ((lane & 7) == 0) {
                        s.bm_gt[(ch << 2) + (lane >> 3)] = wa;
                        s.bm_eq[(ch << 2) + (lane >> 3)] = wc;
                    }
                } else if (in) {              // order within the list is irrelevant
                    uint32_t slot = atomicAdd(&s.n_cand, (uint32_t)__popc(in));
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        if ((in >> c) & 1u) {
                            if (slot < (uint32_t)kCand) {
                                s.cand[slot] = asp::score_key(comp(kv[u], c));
                                s.cand_idx[slot] = (uint32_t)(o + c);
                            }
                            slot++;
                        }
                    }
                }
            }
        }
        above = warp_sum_u32(above);
        const uint32_t a = block_sum_warps(s, above);
        SPROF(5);
        if (direct) {                         // gather the marked candidates; clear bm_eq
            for (int w = t; w < ((nchunks << 2)); w += kThreads) {
                uint32_t bits = s.bm_eq[w];
                if (!bits) continue;
                s.bm_eq[w] = 0;
                uint32_t slot = atomicAdd(&s.n_cand, (uint32_t)__popc(bits));
                while (bits) {
                    const int o = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    if (slot < (uint32_t)kCand) {
                        s.cand[slot] = key_at(o);
                        s.cand_idx[slot] = (uint32_t)o;
                    }
                    slot++;
                }
            }
        }
        __syncthreads();
        if (t == 0) {
            s.cnt[0] = a;
            s.cnt[1] = s.n_cand;
            s.cnt[2] = s.n_cand > (uint32_t)kCand ? 1u : 0u;
        }
    }
    uint32_t tot[3], bef[3];
    cluster_counts(s, C, 3, tot, bef);
    const uint32_t cta_above = s.cnt[0];
    SPROF(2);
    const bool use_cand = tot[2] == 0 && tot[0] < (uint32_t)k && tot[0] + tot[1] >= (uint32_t)k;
    const uint32_t rank0 = use_cand ? (uint32_t)k - tot[0] : (uint32_t)k;
#ifdef ASP_PROFILE_SELECT
    if (t == 0 && !use_cand) atomicAdd(&g_sel_prof[7], 1ull);
    if (t == 0) atomicAdd(&g_sel_prof[6], (unsigned long long)tot[1]);
#endif

    // ---- 3. exact T: radix select over the candidates (relative to the
    // bracket, 8-bit digits) or, if the sample missed, over all keys (12 + 12 + 8)
    // fn(key, candidate slot or -1)
    auto for_each_key = [&](auto &&fn) {
        if (use_cand) {
            const int nc = (int)s.n_cand;
            for (int e = t; e < nc; e += kThreads) fn(s.cand[e], e);
        } else {
            for (int o = t; o < n; o += kThreads) fn(key_at(o), -1);
        }
    };
    uint32_t T;
    if (use_cand) {
        // the candidates lie in [key_lo, key_hi]: radix over key - key_lo, 8 bits
        // (256 bins: cheap zeroing, scans and cluster merges) per level, only as
        // many levels as the bracket is wide (usually 2)
        const uint32_t span = key_hi - key_lo;
        int bits = span ? 32 - __clz(span) : 1;
        uint32_t prefix = 0, rem = rank0;
        while (bits > 0) {
            const int shift = bits > 8 ? bits - 8 : 0;
            zero_hist(s, 256);
            __syncthreads();
            for_each_key([&](uint32_t key, int) {
                const uint32_t rel = key - key_lo;
                if (((uint64_t)rel >> bits) == ((uint64_t)prefix >> bits))
                    atomicAdd(&s.hist[(rel >> shift) & 0xFFu], 1u);
            });
            merge_hist(s, 256, C);
            find_bucket(s, 256, rem, rem);
            prefix |= s.found_bin << shift;
            rem = s.found_rem;
            bits = shift;
        }
        T = key_lo + prefix;
    } else {
        zero_hist(s, kBins);
        __syncthreads();
        for_each_key([&](uint32_t key, int) { atomicAdd(&s.hist[key >> 20], 1u); });
        merge_hist(s, kBins, C);
        find_bucket(s, kBins, rank0, rank0);
        const uint32_t d1 = s.found_bin, rem1 = s.found_rem;
        zero_hist(s, kBins);
        __syncthreads();
        for_each_key([&](uint32_t key, int) {
            if ((key >> 20) == d1) atomicAdd(&s.hist[(key >> 8) & 0xFFFu], 1u);
        });
        merge_hist(s, kBins, C);
        find_bucket(s, kBins, rem1, rem1);
        const uint32_t pre24 = (d1 << 12) | s.found_bin, rem2 = s.found_rem;
        zero_hist(s, 256);
        __syncthreads();
        for_each_key([&](uint32_t key, int) {
            if ((key >> 8) == pre24) atomicAdd(&s.hist[key & 0xFFu], 1u);
        });
        merge_hist(s, 256, C);
        find_bucket(s, 256, rem2, rem2);
        T = (pre24 << 8) | s.found_bin;
    }
    const uint32_t need = s.found_rem;       // keys == T to take, lowest index first
    SPROF(3);

    // ---- 4. cluster: this CTA's (key > T, key == T) counts -> offsets after
    // the earlier ranks' keys
    uint32_t gt_run = 0, eq_run = 0;
    if (C > 1) {
        uint32_t g = 0, e = 0;
        for_each_key([&](uint32_t key, int) {
            g += key > T;
            e += key == T;
        });
        g = block_sum_warps(s, warp_sum_u32(g));
        e = block_sum_warps(s, warp_sum_u32(e));
        if (use_cand) g += cta_above;        // keys above the bracket are all > T
        if (t == 0) {
            s.cnt[0] = g;
            s.cnt[1] = e;
        }
        uint32_t tot2[2], bef2[2];
        cluster_counts(s, C, 2, tot2, bef2);
        gt_run = bef2[0];
        eq_run = bef2[1];
    }

    // ---- 5. emission: bitmaps (key > T, key == T), word offsets, indices in order
    const bool seeded = direct && use_cand;  // bm_gt holds the keys above the bracket
    for (int r0 = 0; r0 < n; r0 += kRound) {
        const int rn = min(kRound, n - r0);
        const int rwords = (rn + 31) >> 5;
        if (seeded) {                        // + the candidates that made it
            for_each_key([&](uint32_t key, int e) {
                const uint32_t o = s.cand_idx[e];
                if (key > T) atomicOr(&s.bm_gt[o >> 5], 1u << (o & 31));
                else if (key == T) atomicOr(&s.bm_eq[o >> 5], 1u << (o & 31));
            });
        } else {
            const int rchunks = (rn + 127) >> 7;
            for (int c0 = warp; c0 < rchunks; c0 += 4 * kWarps) {
                float4 kv[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int ch = c0 + u * kWarps;
                    kv[u] = raw4(srow + r0, (ch << 7) + 4 * lane, ch < rchunks ? rn : 0);
                }
                uint4 kk[4];
#pragma unroll
                for (int u = 0; u < 4; u++) kk[u] = keys4(kv[u]);
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int ch = c0 + u * kWarps;
                    if (ch >= rchunks) break;                  // warp-uniform
                    const int o = (ch << 7) + 4 * lane;
                    uint32_t g = 0, e = 0;
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const uint32_t key = comp(kk[u], c);
                        const bool valid = o + c < rn;
                        g |= (uint32_t)(valid && key > T) << c;
                        e |= (uint32_t)(valid && key == T) << c;
                    }
                    g <<= 4 * (lane & 7);    // word ch*4 + lane/8 <- nibbles of 8 lanes
                    e <<= 4 * (lane & 7);
#pragma unroll
                    for (int d = 1; d < 8; d <<= 1) {
                        g |= __shfl_xor_sync(0xffffffffu, g, d);
                        e |= __shfl_xor_sync(0xffffffffu, e, d);
                    }
                    if ((lane & 7) == 0) {
                        s.bm_gt[(ch << 2) + (lane >> 3)] = g;
                        s.bm_eq[(ch << 2) + (lane >> 3)] = e;
                    }
                }
            }
        }
        __syncthreads();
        const int wpt = (rwords + kThreads - 1) / kThreads;           // words per thread
        const int wa = min(t * wpt, rwords), wb = min(wa + wpt, rwords);
        uint32_t cgt = 0, ceq = 0;
        for (int w = wa; w < wb; w++) {
            cgt += __popc(s.bm_gt[w]);
            ceq += __popc(s.bm_eq[w]);
        }
        uint32_t tg, te;
        uint32_t gt_before = gt_run + block_excl_scan(s, cgt, &tg);
        uint32_t eq_before = eq_run + block_excl_scan(s, ceq, &te);
        for (int w = wa; w < wb; w++) {
            const uint32_t g = s.bm_gt[w], e = s.bm_eq[w];
            uint32_t bits = g | e;
            while (bits) {
                const int bit = __ffs(bits) - 1;
                bits &= bits - 1;
                const int idx = seg0 + r0 + (w << 5) + bit;
                if ((g >> bit) & 1u) {
                    out[gt_before + min(eq_before, need)] = idx;
                    gt_before++;
                } else {
                    if (eq_before < need) out[gt_before + eq_before] = idx;
                    eq_before++;
                }
            }
        }
        gt_run += tg;
        eq_run += te;
        __syncthreads();                     // the bitmaps are rewritten next round
    }
    nan = __syncthreads_or(nan);
    SPROF(4);
    if (t == 0 && nan) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
    if (discard) {
        // The scores are dead once selected: drop this segment's L2 lines
        // without writing them back (only whole 128-B lines inside it).
        const uintptr_t lo = (reinterpret_cast<uintptr_t>(srow) + 127u) & ~(uintptr_t)127u;
        const uintptr_t hi = reinterpret_cast<uintptr_t>(srow + n);
        for (uintptr_t x = lo + (uintptr_t)t * 128u; x + 128u <= hi; x += (uintptr_t)kThreads * 128u)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(x) : "memory");
    }
}

