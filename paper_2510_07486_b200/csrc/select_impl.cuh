// select_impl.cuh -- the select kernel body, instantiated by select.cu for
// SEL_NT threads per CTA (256: many rows, several CTAs per SM; 1024: few
// rows, one CTA per SM) inside a namespace of its own.  See select.cu.

constexpr int kThreads = SEL_NT;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 4096;
constexpr int kCand = 2048;                   // candidate slots per CTA
constexpr int kRound = 65536;                 // keys per emission round (bitmap capacity)
constexpr int kRoundChunks = kRound / 128;    // 128-key chunks per round
constexpr int kSampleChunks = 32;             // 32 x 128 consecutive keys sampled per row
constexpr int kMaxCluster = 16;
constexpr int kUnroll = 8;                    // 16-B loads in flight per lane (classify)

// Bitmaps are in index order: word w bit j <-> key 32 w + j.  A warp reads a
// 128-key chunk as four coalesced 128-B loads (lane l takes keys 32 j + l,
// j = 0..3), so the ballot of load j IS bitmap word 4 * chunk + j:
// classification costs one compare + one ballot per key and no shuffles.
struct SelectSmem {
    uint32_t hist[kBins];
    uint32_t cand[kCand];          // candidate keys (any order)
    uint16_t cand_idx[kCand];      // their offsets inside the round (< kRound)
    uint32_t bm_gt[kRound / 32];   // key > T (seeded with the keys above the bracket)
    uint32_t bm_eq[kRound / 32];   // key == T
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
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    constexpr int kPer = kBins / kThreads;
    uint32_t acc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        const int bin = threadIdx.x + j * kThreads;
        acc[j] = 0;
        if (bin < nbins)
            for (int r = 0; r < C; r++) acc[j] += cl.map_shared_rank(s.hist, r)[bin];
    }
    cl.sync();
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        const int bin = threadIdx.x + j * kThreads;
        if (bin < nbins) s.hist[bin] = acc[j];
    }
    __syncthreads();
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

// Emit the selected indices of one round from the bitmaps (bm_gt: key > T,
// bm_eq: key == T; only the first `need` equal keys of the ROW, in index
// order, are taken): each thread owns a run of words, a block scan of their
// popcounts gives its output offsets, then it writes its indices in order.
// gt_run / eq_run: keys of this row before the round (earlier cluster ranks
// and rounds); updated.
__device__ __forceinline__ void emit_round(SelectSmem &s, int rwords, int base_idx, uint32_t need,
                                           uint32_t &gt_run, uint32_t &eq_run, int32_t *out) {
    const int t = threadIdx.x;
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
            const int idx = base_idx + (w << 5) + bit;
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
    __syncthreads();                       // the bitmaps are rewritten next round
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
    // base[o..o+3] (o % 4 == 0), elements >= lim read as 0 (callers mask them).
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
    const bool seeded = n <= kRound;         // the classify sweep can seed the bitmaps
    const int nchunks = (n + 127) >> 7;

    zero_hist(s, kBins);
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
    constexpr int kPerWarp = kSampleChunks / kWarps > 0 ? kSampleChunks / kWarps : 1;
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
        for (int c = 0; c < 4; c++) {                  // equal bins aggregated per warp
            const bool ok = so[u] + c < len;
            const uint32_t bin = ok ? comp(sk[u], c) >> 20 : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, bin);
            if (ok && (__ffs(peers) - 1) == lane) atomicAdd(&s.hist[bin], (uint32_t)__popc(peers));
        }
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

    // ---- 2. classify the segment against the bracket [key_lo, key_hi],
    // compared in fp32 (v >= lb(K) <=> key(v) >= K, NaN never): per 128-key
    // chunk, per float4 component c, one ballot for "above the bracket" and
    // one for "in it".  The above-words seed bm_gt (seeded segments); the
    // bracketed keys go to the candidate list (warp-aggregated slots).  NaN
    // detection rides along.
    const float f_lo = key_lower_bound(key_lo);
    const float f_above = key_lower_bound((uint64_t)key_hi + 1);
    bool nan = false;
    {
        uint32_t above = 0;                              // warp-uniform
        // one 128-key chunk: x[j] = key 32 j + lane (j = 0..3), `rem` keys valid
        auto chunk = [&](const float (&x)[4], int ch, int rem) {
            uint32_t ab[4], in[4], nn = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const bool ok = 32 * j + lane < rem;
                ab[j] = __ballot_sync(0xffffffffu, ok && x[j] >= f_above);
                in[j] = __ballot_sync(0xffffffffu, ok && x[j] >= f_lo) & ~ab[j];
                nn |= ok && x[j] != x[j];
            }
            nan |= nn != 0;
            above += __popc(ab[0]) + __popc(ab[1]) + __popc(ab[2]) + __popc(ab[3]);
            if (seeded) {                                // above -> bm_gt, bracketed -> bm_eq
                const uint32_t wa = lane == 0 ? ab[0] : lane == 1 ? ab[1] : lane == 2 ? ab[2] : ab[3];
                const uint32_t wc = lane == 0 ? in[0] : lane == 1 ? in[1] : lane == 2 ? in[2] : in[3];
                if (lane < 4) {
                    s.bm_gt[4 * ch + lane] = wa;
                    s.bm_eq[4 * ch + lane] = wc;
                }
                return;
            }
            const uint32_t any = in[0] | in[1] | in[2] | in[3];
            if (any) {                                   // unseeded (long) segments: warp-uniform
                const uint32_t lt = (1u << lane) - 1u;
                const uint32_t tot = __popc(in[0]) + __popc(in[1]) + __popc(in[2]) + __popc(in[3]);
                uint32_t slot = 0;
                if (lane == 0) slot = atomicAdd(&s.n_cand, tot);
                slot = __shfl_sync(0xffffffffu, slot, 0);
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    if ((in[j] >> lane) & 1u) {
                        const uint32_t sl = slot + __popc(in[j] & lt);
                        if (sl < (uint32_t)kCand) {
                            s.cand[sl] = asp::score_key(x[j]);
                            s.cand_idx[sl] = (uint16_t)(((ch << 7) + 32 * j + lane) & (kRound - 1));
                        }
                    }
                    slot += __popc(in[j]);
                }
            }
        };
        for (int c0 = warp; c0 < nchunks; c0 += kUnroll * kWarps) {
            const bool full = vec && ((c0 + (kUnroll - 1) * kWarps) << 7) + 128 <= n;
            float x[kUnroll][4];
            if (full) {
#pragma unroll
                for (int u = 0; u < kUnroll; u++)
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        x[u][j] = __ldg(srow + ((c0 + u * kWarps) << 7) + 32 * j + lane);
#pragma unroll
                for (int u = 0; u < kUnroll; u++) chunk(x[u], c0 + u * kWarps, 128);
            } else {
#pragma unroll
                for (int u = 0; u < kUnroll; u++)
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const int o = ((c0 + u * kWarps) << 7) + 32 * j + lane;
                        x[u][j] = o < n ? __ldg(srow + o) : 0.0f;
                    }
#pragma unroll
                for (int u = 0; u < kUnroll; u++) {
                    const int ch = c0 + u * kWarps;
                    if (ch >= nchunks) break;                      // warp-uniform
                    chunk(x[u], ch, n - (ch << 7));
                }
            }
        }
        const uint32_t a = block_sum_warps(s, above);
        if (seeded) {
            // gather the marked candidates (slots from one block scan of the
            // per-thread counts -- not a shared counter, whose atomics would
            // serialise) and clear bm_eq
            const int nw = 4 * nchunks, wpt = (nw + kThreads - 1) / kThreads;
            const int wa = min(t * wpt, nw), wb = min(wa + wpt, nw);
            uint32_t cnt = 0;
            for (int w = wa; w < wb; w++) cnt += __popc(s.bm_eq[w]);
            uint32_t total;
            uint32_t slot = block_excl_scan(s, cnt, &total);
            for (int w = wa; w < wb; w++) {
                uint32_t bits = s.bm_eq[w];
                if (!bits) continue;
                s.bm_eq[w] = 0u;
                while (bits) {
                    const int o = (w << 5) + __ffs(bits) - 1;
                    bits &= bits - 1;
                    if (slot < (uint32_t)kCand) {
                        s.cand[slot] = key_at(o);
                        s.cand_idx[slot] = (uint16_t)o;
                    }
                    slot++;
                }
            }
            if (t == 0) s.n_cand = total;
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

    // ---- 3. exact T: MSB-first radix select over (key - base), 12 bits per
    // pass, over the candidates (base = key_lo: the bracket's width bounds the
    // passes, usually 2) or, when the sample missed, over every key (base 0:
    // 12 + 12 + 8 bits).  fn(key, candidate slot or -1)
    auto for_each_key = [&](auto &&fn) {
        if (use_cand) {
            const int nc = (int)s.n_cand;
            for (int e = t; e < nc; e += kThreads) fn(s.cand[e], e);
        } else {
            for (int o = t; o < n; o += kThreads) fn(key_at(o), -1);
        }
    };
    const uint32_t kbase = use_cand ? key_lo : 0u;
    const uint64_t width = use_cand ? (uint64_t)key_hi - key_lo + 1 : (1ull << 32);
    int bits = width <= 1 ? 0 : 64 - __clzll((long long)(width - 1));
    uint32_t prefix = 0, rank = rank0;
    while (bits > 0) {
        const int d = min(12, bits);
        bits -= d;
        const int nb = d > 8 ? kBins : 256;
        zero_hist(s, nb);
        __syncthreads();
        const uint64_t pre = prefix;
        const int sh_hi = bits + d;
        if (use_cand) {
            // candidates crowd into a few bins: aggregate equal bins per warp
            // (one atomic per distinct bin) instead of serialising on them
            const int nc = (int)s.n_cand;
            for (int e0 = warp * 32; e0 < nc; e0 += kThreads) {
                const int e = e0 + lane;
                const uint64_t rel = e < nc ? (uint64_t)(s.cand[e] - kbase) : 0;
                const bool hit = e < nc && (rel >> sh_hi) == pre;
                const uint32_t bin = hit ? (uint32_t)((rel >> bits) & ((1u << d) - 1u)) : 0xFFFFFFFFu;
                const uint32_t peers = __match_any_sync(0xffffffffu, bin);
                if (hit && (__ffs(peers) - 1) == lane) atomicAdd(&s.hist[bin], (uint32_t)__popc(peers));
            }
        } else {
            for_each_key([&](uint32_t key, int) {
                const uint64_t rel = (uint64_t)(key - kbase);
                if ((rel >> sh_hi) == pre) atomicAdd(&s.hist[(rel >> bits) & ((1u << d) - 1u)], 1u);
            });
        }
        merge_hist(s, nb, C);
        find_bucket(s, nb, rank, rank);
        prefix = (prefix << d) | s.found_bin;
        rank = s.found_rem;
    }
    const uint32_t T = kbase + prefix;
    const uint32_t need = rank;              // keys == T to take, lowest index first
    SPROF(3);

    // ---- 4. this CTA's (key > T, key == T) counts; in a cluster, offsets
    // after the earlier ranks' keys.  Seeded candidate path: the candidates
    // that made it join the above-bracket keys in the bitmaps.
    const bool marked = seeded && use_cand;
    if (marked) {
        for_each_key([&](uint32_t key, int e) {
            const uint32_t o = s.cand_idx[e];
            if (key > T) atomicOr(&s.bm_gt[o >> 5], 1u << (o & 31u));
            else if (key == T) atomicOr(&s.bm_eq[o >> 5], 1u << (o & 31u));
        });
    }
    uint32_t gt_run = 0, eq_run = 0;
    if (C > 1) {
        uint32_t g = 0, e = 0;
        if (use_cand) {
            for_each_key([&](uint32_t key, int) {
                g += key > T;
                e += key == T;
            });
        } else {
            for (int o = t; o < n; o += kThreads) {
                const uint32_t key = key_at(o);
                g += key > T;
                e += key == T;
            }
        }
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
    __syncthreads();

    // ---- 5. emission, one round per kRound keys: bitmaps (seeded, or marked
    // here by re-reading the keys), chunk offsets, indices in order
    for (int r0 = 0; r0 < n; r0 += kRound) {
        const int rn = min(kRound, n - r0);
        const int rch = (rn + 127) >> 7;
        if (!marked) {                       // re-read the round's keys: compare with T
            for (int ch = warp; ch < rch; ch += kWarps) {
                uint32_t gw = 0, ew = 0;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int o = (ch << 7) + 32 * j + lane;
                    const bool ok = o < rn;
                    const uint32_t key = ok ? key_at(r0 + o) : 0u;
                    const uint32_t g = __ballot_sync(0xffffffffu, ok && key > T);
                    const uint32_t e = __ballot_sync(0xffffffffu, ok && key == T);
                    if (lane == j) { gw = g; ew = e; }
                }
                if (lane < 4) {
                    s.bm_gt[4 * ch + lane] = gw;
                    s.bm_eq[4 * ch + lane] = ew;
                }
            }
            __syncthreads();
        }
        emit_round(s, 4 * rch, seg0 + r0, need, gt_run, eq_run, out);
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
