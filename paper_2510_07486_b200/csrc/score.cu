// score.cu -- a2: token criticality q_hat . K per (sequence, KV head), reduced
// over the GQA group (Alg. 1 Step 7; GQA layout P:252-260):
//
//   s[b,h,n] = max_{g<G} sum_d q_hat[b,h*G+g,d] * K[b,h,n,d]      (R10, R11)
//
// The paper computes this as a flattened GEMM for GQA (Fig. 8).  On
// B200 the step is HBM-bound (it streams the whole bf16 K cache: ~88% of the
// path's bytes), but at G = 8 its fp32 FMA count would need ~70% of the SMs'
// FP32 issue just to keep pace with HBM.  So the contraction runs on the
// 5th-gen tensor cores, which leaves the SM pipes idle and the kernel a pure
// TMA stream:
//
//   * q_hat is fp32 and a bf16 q_hat fails the selection parity,
//     so each q_hat row is split exactly into three bf16 terms
//     q = hi + mid + lo (8+8+8 significand bits).  K is bf16, so every
//     product is exact; one tcgen05.mma (M = 128 tokens, N = 3G padded to
//     16/32, K = D) accumulates all three in fp32 TMEM columns, and the
//     epilogue forms s_g = (hi_g + mid_g) + lo_g, then the group max.
//   * Persistent CTAs (one per SM) own a contiguous range of the VALID
//     128-token tiles of the flattened (row, tile) space (balanced over the
//     rows' actual lengths, so ragged batches keep every SM busy).  Paged
//     pools stream page-sized TMA boxes, page ids fetched six tiles ahead.
//     Warp roles: warp 0 streams K tiles
//     with TMA (4-D tensor map over the strided cache, 128-B swizzle,
//     L2 evict-first) into a 6-stage mbarrier ring; warp 1 owns TMEM and
//     issues the MMAs (single thread); warps 2-3 build the swizzled bf16 B
//     operand for each new row into a 2-slot ring; warps 4-11 (two
//     warpgroups alternating tiles) drain TMEM (tcgen05.ld, 6 accumulator
//     stages) and store the fp32 scores.
//
// Every token's score is a fixed function of its key row and q_hat (the same
// MMA datapath and the same 3-term epilogue order wherever the tile falls),
// so equal keys give equal scores and any KV-head shard reproduces the
// unsharded scores bit for bit.
#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"
#include "tc.cuh"

#ifdef ASP_PROFILE_SCORE
__device__ unsigned long long g_score_prof[8];
#define PWAIT(acc, call)                       \
    do {                                       \
        const long long _t0 = clock64();       \
        call;                                  \
        acc += clock64() - _t0;                \
    } while (0)
#define PFLUSH(idx, acc) atomicAdd(&g_score_prof[idx], (unsigned long long)(acc))
#else
#define PWAIT(acc, call) call
#define PFLUSH(idx, acc) (void)(acc)
#endif

namespace {

using namespace asp::tc;

constexpr int kTileM = 128;           // tokens per tile (MMA M)
#ifndef ASP_SCORE_STAGES
#define ASP_SCORE_STAGES 6
#endif
constexpr int kStages = ASP_SCORE_STAGES;   // K-tile ring depth
constexpr int kAcc = 6;               // TMEM accumulator stages
constexpr int kGroup = 3;             // tiles whose MMA chains are interleaved
constexpr int kBSlots = 2;            // B-operand ring
constexpr int kThreads = 384;         // 12 warps: TMA, MMA, B build, spare, 2 x 4 epilogue

template <int D, int G>
struct Cfg {
    static constexpr int N = (3 * G + 15) / 16 * 16 < 16 ? 16 : (3 * G + 15) / 16 * 16;
    static constexpr int kRegions = D / 64;                       // 128-B swizzle rows per token
    // a ring stage holds one 128-token tile (D <= 128), or one 64-dim region of
    // it for wide keys (absorbed MLA, D = 576: a tile is 9 stages, accumulated
    // in TMEM across them)
#ifndef ASP_SCORE_WIDE_REGIONS
#define ASP_SCORE_WIDE_REGIONS 3
#endif
    static constexpr int kRegPerStage = D <= 128 ? kRegions
                                      : (kRegions % ASP_SCORE_WIDE_REGIONS == 0 ? ASP_SCORE_WIDE_REGIONS
                                         : (kRegions % 2 == 0 ? 2 : 1));
    static constexpr int kSub = kRegions / kRegPerStage;          // stages per tile
    static constexpr int kStageBytes = kTileM * 64 * kRegPerStage * 2;
    static constexpr int kBRegionBytes = N * 128;
    static constexpr int kBSlotBytes = kRegions * kBRegionBytes;
    // B-operand ring: two slots, one for wide keys (a row's operand is ~55 KB;
    // MLA has one KV head, so rows change every L / 128 tiles)
    static constexpr int kBSlots = D <= 128 ? ::kBSlots : 1;
    // accumulation chains per tile: even / odd k-steps in two TMEM halves (short
    // MMAs, latency-bound chains), one chain when N > 96 (G = 64: an N = 192 MMA
    // is long enough, and two halves would leave room for a single stage)
    static constexpr int kHalves = N <= 96 ? 2 : 1;
    // accumulator stages: 6, or as many as fit the 512 TMEM columns (G = 16: 5,
    // G = 32: 2, G = 64: 2)
    static constexpr int kAcc = (kHalves * ::kAcc * N) <= 512 ? ::kAcc : 512 / (kHalves * N);
    // K ring: 6 tile stages, fewer when the B-operand ring needs the room
    // (G = 32: 5); wide keys: as many region-group stages as fit, up to 12
    static constexpr int kFree = 227 * 1024 - 1024 - kBSlots * kBSlotBytes - 512;
    static constexpr int kStages = D <= 128 ? (kFree / kStageBytes < ::kStages ? kFree / kStageBytes : ::kStages)
                                            : (kFree / kStageBytes < 12 ? kFree / kStageBytes : 12);
    static constexpr uint32_t kTmemCols = (kHalves * kAcc * N) <= 64 ? 64
                                          : (kHalves * kAcc * N) <= 128 ? 128
                                          : (kHalves * kAcc * N) <= 256 ? 256 : 512;
    static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes +
                                      kBSlots * kBSlotBytes + 512 /*barriers*/;
    static_assert(kStages >= 2, "K ring");
};

// One group of 3 tiles x 8 k-steps (D = 128) in a single asm statement: the
// operands reach the uniform datapath once and the per-MMA offsets are
// uniform adds (the A start-address field is addr >> 4; the A tile's two
// 64-column regions are 16 KB apart, the B operand's N*128 bytes apart).
__device__ __forceinline__ void mma_group3_d128(uint64_t a0, uint64_t a1, uint64_t a2, uint64_t b0,
                                                uint32_t d0, uint32_t d1, uint32_t d2,
                                                uint32_t idesc, uint64_t b_region16,
                                                uint32_t n_cols) {
    asm volatile(
        "{\n\t.reg .pred e, p0, p1;\n\t.reg .b64 ta, tb;\n\t.reg .b32 td;\n\t"
        "setp.ne.b32 p0, %10, %10;\n\tsetp.eq.b32 p1, %10, %10;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "add.s64 tb, %3, 0;\n\t"
        "add.s64 ta, %0, 0;\n\t"
        "mov.u32 td, %4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p0;\n\t"
        "add.s64 ta, %1, 0;\n\t"
        "mov.u32 td, %5;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p0;\n\t"
        "add.s64 ta, %2, 0;\n\t"
        "mov.u32 td, %6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p0;\n\t"
        "add.s64 tb, %3, 2;\n\t"
        "add.s64 ta, %0, 2;\n\t"
        "add.u32 td, %4, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p0;\n\t"
        "add.s64 ta, %1, 2;\n\t"
        "add.u32 td, %5, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p0;\n\t"
        "add.s64 ta, %2, 2;\n\t"
        "add.u32 td, %6, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p0;\n\t"
        "add.s64 tb, %3, 4;\n\t"
        "add.s64 ta, %0, 4;\n\t"
        "mov.u32 td, %4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %1, 4;\n\t"
        "mov.u32 td, %5;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %2, 4;\n\t"
        "mov.u32 td, %6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 tb, %3, 6;\n\t"
        "add.s64 ta, %0, 6;\n\t"
        "add.u32 td, %4, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %1, 6;\n\t"
        "add.u32 td, %5, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %2, 6;\n\t"
        "add.u32 td, %6, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 tb, %3, %8;\n\tadd.s64 tb, tb, 0;\n\t"
        "add.s64 ta, %0, 1024;\n\t"
        "mov.u32 td, %4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %1, 1024;\n\t"
        "mov.u32 td, %5;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %2, 1024;\n\t"
        "mov.u32 td, %6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 tb, %3, %8;\n\tadd.s64 tb, tb, 2;\n\t"
        "add.s64 ta, %0, 1026;\n\t"
        "add.u32 td, %4, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %1, 1026;\n\t"
        "add.u32 td, %5, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %2, 1026;\n\t"
        "add.u32 td, %6, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 tb, %3, %8;\n\tadd.s64 tb, tb, 4;\n\t"
        "add.s64 ta, %0, 1028;\n\t"
        "mov.u32 td, %4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %1, 1028;\n\t"
        "mov.u32 td, %5;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %2, 1028;\n\t"
        "mov.u32 td, %6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 tb, %3, %8;\n\tadd.s64 tb, tb, 6;\n\t"
        "add.s64 ta, %0, 1030;\n\t"
        "add.u32 td, %4, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %1, 1030;\n\t"
        "add.u32 td, %5, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "add.s64 ta, %2, 1030;\n\t"
        "add.u32 td, %6, %9;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [td], ta, tb, %7, p1;\n\t"
        "}"
        ::"l"(a0), "l"(a1), "l"(a2), "l"(b0), "r"(d0), "r"(d1), "r"(d2), "r"(idesc),
        "l"(b_region16), "r"(n_cols), "r"(0u)
        : "memory");
}

struct TileIter {
    long start, end;
    int tpr, n_kv;
    const int32_t *seq_lens;
    int max_len;
    int crow = -1, clen = 0;                       // per-thread cache of the current row's length
    __device__ int len_of(int row) {
        if (row != crow) {                         // rows change rarely: one global load per row
            crow = row;
            clen = min(max(seq_lens[row / n_kv], 0), max_len);
        }
        return clen;
    }
    // Advance i to the next valid tile (token base < row length) in [i, end);
    // row / j of the returned tile are left in row, j.  Sequential calls
    // (i = previous + 1) step the cursor without any 64-bit division.
    long pos = -1;
    int row = 0, j = 0;
    __device__ long next(long i) {
        int r, jj;
        if (pos >= 0 && i == pos + 1) {
            r = row;
            jj = j + 1;
            if (jj == tpr) { r++; jj = 0; }
        } else {
            r = (int)(i / tpr);
            jj = (int)(i - (long)r * tpr);
        }
        while (i < end) {
            if (jj * kTileM < len_of(r)) { pos = i; row = r; j = jj; return i; }
            i += tpr - jj;                        // rest of the row is past its length
            r++;
            jj = 0;
        }
        pos = end;
        return end;
    }
};

// Paged pool (asyncspade_score_select_paged): the block table and the pool
// geometry; unused by the dense instantiation.
struct PagedArgs {
    const int32_t *block_table;
    int page_size, max_pages, num_pages;
};

template <int D, int G, bool PAGED>
__global__ void __launch_bounds__(kThreads, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap kmap, asp_select_params p,
                const float *__restrict__ q_hat, const int32_t *__restrict__ seq_lens,
                float *__restrict__ scores, uint32_t *dev_flags, int tiles_per_row,
                PagedArgs pg) {
    using C = Cfg<D, G>;
    constexpr int N = C::N;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char *gbase = smem_raw + (base - raw);
    const uint32_t stage0 = base;
    const uint32_t bslot0 = stage0 + C::kStages * C::kStageBytes;
    const uint32_t bar0 = bslot0 + C::kBSlots * C::kBSlotBytes;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (C::kStages + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * C::kStages + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * C::kStages + C::kAcc + a); };
    auto bfull_bar = [&](int s) { return bar0 + 8u * (2 * C::kStages + 2 * C::kAcc + s); };
    auto bempty_bar = [&](int s) { return bar0 + 8u * (2 * C::kStages + 2 * C::kAcc + C::kBSlots + s); };
    const uint32_t tmem_holder = bar0 + 8u * (2 * C::kStages + 2 * C::kAcc + 2 * C::kBSlots);
    unsigned char *gbslot0 = gbase + (bslot0 - base);
    volatile uint32_t *tmem_holder_g =
        reinterpret_cast<volatile uint32_t *>(gbase + (tmem_holder - base));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long total = (long)p.batch * p.n_kv_heads * tiles_per_row;
    TileIter it;
    // Balance the VALID tiles (token base < row length), not the capacity: CTA
    // i takes valid tiles [i T / grid, (i+1) T / grid), mapped back to the
    // flattened (row, tile) capacity index the iterator walks (it skips the
    // invalid tiles in between).  Ragged batches would otherwise leave the
    // CTAs over short rows idle.  (seq_lens is caller-written: no PDL wait.)
    __shared__ long long s_rng[2];
    if (warp == 3) {
        const int tpr = tiles_per_row, Hkv = p.n_kv_heads;
        auto vt = [&](int b) {                        // valid tiles of each row of batch b
            const int len = min(max(seq_lens[b], 0), p.max_seq_len);
            return (len + kTileM - 1) / kTileM;
        };
        long long T = 0;                              // all valid tiles
        for (int b0 = 0; b0 < p.batch; b0 += 32) {
            long long v = b0 + lane < p.batch ? (long long)vt(b0 + lane) * Hkv : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            T += v;
        }
        // capacity index of valid tile number v (v == T -> total)
        auto locate = [&](long long v) -> long long {
            if (v >= T) return total;
            long long before = 0;
            for (int b0 = 0; b0 < p.batch; b0 += 32) {
                const int b = b0 + lane;
                const int n = b < p.batch ? vt(b) : 0;
                long long inc = (long long)n * Hkv;   // inclusive scan over the chunk
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += t;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, b < p.batch && before + inc > v);
                if (hit) {
                    const int l = __ffs(hit) - 1;
                    const long long excl = __shfl_sync(0xffffffffu, inc, l) - (long long)__shfl_sync(0xffffffffu, n, l) * Hkv;
                    const int nb = __shfl_sync(0xffffffffu, n, l);
                    const long long off = v - before - excl;
                    const long long h = off / nb, j = off % nb;
                    return ((long long)(b0 + l) * Hkv + h) * tpr + j;
                }
                before += __shfl_sync(0xffffffffu, inc, 31);
            }
            return total;
        };
        const long long a = locate(T * blockIdx.x / gridDim.x);
        const long long e = locate(T * (blockIdx.x + 1) / gridDim.x);
        if (lane == 0) { s_rng[0] = a; s_rng[1] = e; }
    }
    it.tpr = tiles_per_row;
    it.n_kv = p.n_kv_heads;
    it.seq_lens = seq_lens;
    it.max_len = p.max_seq_len;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; s++) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 1); }
        for (int a = 0; a < C::kAcc; a++) { mbar_init(tfull_bar(a), 1); mbar_init(tempty_bar(a), 4); }
        for (int s = 0; s < C::kBSlots; s++) { mbar_init(bfull_bar(s), 2); mbar_init(bempty_bar(s), 1); }
        fence_mbar_init();
        prefetch_tmap(&kmap);
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder_g;
    it.start = s_rng[0];
    it.end = s_rng[1];
    // The TMA warp streams K before the programmatic-dependent-launch wait (K's
    // only writer in the library, asyncspade_append, does not trigger early, so
    // this kernel starts after it completed): the first tiles land while the
    // previous kernel (predict) finishes.  Everything that reads q_hat or writes
    // the scores waits.
    if (warp != 0 || PAGED) asp::pdl_wait();   // (the paged producer reads the block table)
    asp::pdl_trigger();
#ifdef ASP_PROFILE_SCORE
    const long long t_kernel0 = clock64();
#endif

    if (warp == 0 && !PAGED) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            long long pw_empty = 0;
            for (long i = it.next(it.start); i < it.end; i = it.next(i + 1)) {
                const int row = it.row, j = it.j;
                const int b = row / p.n_kv_heads, h = row % p.n_kv_heads;
                const int grow = (int)((b * p.k_stride_b + h * p.k_stride_h) / p.k_stride_t) +
                                 j * kTileM;
#pragma unroll 1
                for (int sub = 0; sub < C::kSub; sub++) {
                    PWAIT(pw_empty, mbar_wait(empty_bar(s), ph ^ 1));
                    mbar_arrive_expect_tx(full_bar(s), C::kStageBytes);
                    const uint32_t dst = stage0 + s * C::kStageBytes;
#pragma unroll
                    for (int r = 0; r < C::kRegPerStage; r++)
                        tma_load_2d(dst + r * (kTileM * 128), &kmap, full_bar(s),
                                    (sub * C::kRegPerStage + r) * 64, grow, kEvictFirst);
                    if (++s == C::kStages) { s = 0; ph ^= 1; }
                }
            }
            PFLUSH(0, pw_empty);
        }
        __syncwarp();
    } else if (warp == 0) {
        // ------------------------------------------------ TMA producer, paged pool
        // A 128-token tile is NP = 128 / page_size pages; each page is a
        // [page_size][D] box of the pool's [rows][D] view (row = (page * Hkv +
        // h) * page_size + t), landing at its token offset in the stage (the
        // 128-B swizzle repeats every 8 rows, so the boxes compose).  The whole
        // warp walks the tile sequence: lanes < NP fetch the page ids of the
        // tile kAhead positions ahead (one block-table word each), so the
        // lookups never stall the stream, and issue that page's copies.
        constexpr int kAhead = 6;
        const int P = pg.page_size, NP = kTileM / pg.page_size;
        TileIter ahead = it;
        long ia = ahead.next(it.start);
        // (the id is clamped where it is used, not here: the load stays in
        // flight for kAhead tiles instead of stalling the warp right away)
        auto fetch = [&]() -> int {
            int id = 0;
            if (ia < it.end) {
                const int row = ahead.row, b = row / p.n_kv_heads;
                const int lp = ahead.j * NP + lane;
                if (lane < NP && lp * P < ahead.len_of(row))
                    id = __ldg(pg.block_table + (size_t)b * pg.max_pages + lp);
                ia = ahead.next(ia + 1);
            }
            return id;
        };
        int q[kAhead];
#pragma unroll
        for (int u = 0; u < kAhead; u++) q[u] = fetch();
        int s = 0;
        uint32_t ph = 0;
        for (long i = it.next(it.start); i < it.end; i = it.next(i + 1)) {
            const int cur = min(max(q[0], 0), pg.num_pages - 1);   // never fault on a bad entry
#pragma unroll
            for (int u = 0; u + 1 < kAhead; u++) q[u] = q[u + 1];
            q[kAhead - 1] = fetch();
            const int h = it.row % p.n_kv_heads;
            mbar_wait(empty_bar(s), ph ^ 1);
            if (lane == 0) mbar_arrive_expect_tx(full_bar(s), C::kStageBytes);
            __syncwarp();
            // lane l < NP copies its own page (issue spread over the lanes)
            const uint32_t dst = stage0 + s * C::kStageBytes;
            if (lane < NP) {
#pragma unroll
                for (int r = 0; r < C::kRegions; r++)
                    tma_load_2d(dst + r * (kTileM * 128) + lane * P * 128, &kmap, full_bar(s),
                                r * 64, (cur * p.n_kv_heads + h) * P, kEvictFirst);
            }
            if (++s == C::kStages) { s = 0; ph ^= 1; }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (whole warp, one elected lane)
        // A tile's D/16 MMAs are a dependent accumulation chain and each MMA is far
        // shorter than the tensor pipe's latency, so chains are interleaved: every
        // tile accumulates into two TMEM halves (even / odd k-steps) and tiles are
        // issued in groups of up to kGroup (same row), k-step outer / tile inner
        // -- 2 x kGroup independent chains in flight.
        {
            constexpr uint32_t idesc = idesc_bf16_f32(kTileM, N);
            int s = 0, a = 0, bs = -1;
            uint32_t ph = 0, aph = 0, bph = 0;
            int cur_row = -1;
            long long pm_full = 0, pm_tempty = 0, pm_issue = 0, pm_b = 0;
            long i = it.next(it.start);
            if constexpr (C::kSub > 1) {
                // wide keys: a tile is kSub region stages accumulated in one TMEM
                // stage (two chains: even / odd k-steps), tile after tile
                while (i < it.end) {
                    const int row = it.row;
                    if (row != cur_row) {
                        if (bs >= 0) mma_commit_warp(bempty_bar(bs));
                        bs = (bs + 1) % C::kBSlots;
                        if (bs == 0 && cur_row != -1) bph ^= 1;
                        mbar_wait(bfull_bar(bs), bph);
                        cur_row = row;
                    }
                    mbar_wait(tempty_bar(a), aph ^ 1);
                    const uint32_t dcol = tmem_base + a * (C::kHalves * N);
                    const uint64_t bdesc0 = desc_sw128_kmajor(bslot0 + bs * C::kBSlotBytes);
#pragma unroll 1
                    for (int sub = 0; sub < C::kSub; sub++) {
                        mbar_wait(full_bar(s), ph);
                        tc_fence_after();
                        const uint64_t adesc = desc_sw128_kmajor(stage0 + s * C::kStageBytes);
#pragma unroll
                        for (int kk = 0; kk < 4 * C::kRegPerStage; kk++) {
                            const int r = kk / 4, ko = (kk % 4) * 32;
                            const int kg = sub * 4 * C::kRegPerStage + kk;   // k-step in the tile
                            const uint64_t aoff = (uint64_t)((r * (kTileM * 128) + ko) >> 4);
                            const uint64_t boff = (uint64_t)(((sub * C::kRegPerStage + r) *
                                                              C::kBRegionBytes + ko) >> 4);
                            if constexpr (C::kHalves == 2)
                                mma_bf16_warp(dcol + (kg & 1) * N, adesc + aoff, bdesc0 + boff, idesc,
                                              kg > 1 ? 1u : 0u);
                            else
                                mma_bf16_warp(dcol, adesc + aoff, bdesc0 + boff, idesc, kg > 0 ? 1u : 0u);
                        }
                        mma_commit_warp(empty_bar(s));
                        if (++s == C::kStages) { s = 0; ph ^= 1; }
                    }
                    mma_commit_warp(tfull_bar(a));
                    if (++a == C::kAcc) { a = 0; aph ^= 1; }
                    i = it.next(i + 1);
                }
            } else
            while (i < it.end) {
                const int row = it.row;
                if (row != cur_row) {
                    if (bs >= 0) mma_commit_warp(bempty_bar(bs));   // previous row's B slot free
                    bs = (bs + 1) % C::kBSlots;
                    if (bs == 0 && cur_row != -1) bph ^= 1;
                    PWAIT(pm_b, mbar_wait(bfull_bar(bs), bph));
                    cur_row = row;
                }
                // collect a group of consecutive valid tiles of this row
                int gs[kGroup], ga[kGroup], ng = 0;
                // (a group never needs more accumulator stages than exist: every
                // tile of it waits for its stage before any of them is issued)
                // (one-chain tiles -- G = 64 -- are long MMAs on their own: issue each as
                // soon as its stage and an accumulator are free, never wait for a group)
                constexpr int kGroupMax = C::kHalves == 1 ? 1 : (C::kAcc < kGroup ? C::kAcc : kGroup);
                while (ng < kGroupMax && i < it.end && it.row == row) {
                    PWAIT(pm_full, mbar_wait(full_bar(s), ph));
                    PWAIT(pm_tempty, mbar_wait(tempty_bar(a), aph ^ 1));
                    gs[ng] = s;
                    ga[ng] = a;
                    ng++;
                    if (++s == C::kStages) { s = 0; ph ^= 1; }
                    if (++a == C::kAcc) { a = 0; aph ^= 1; }
                    i = it.next(i + 1);
                }
#ifdef ASP_PROFILE_SCORE
                const long long t_issue = clock64();
#endif
                tc_fence_after();
                const uint32_t b_base = bslot0 + bs * C::kBSlotBytes;
                // descriptors: the start-address field is addr >> 4 in the low
                // bits (no carry for addresses < 256 KB), so offsets add directly
                uint64_t adesc[kGroup];
                uint32_t dcol[kGroup];
#pragma unroll
                for (int t = 0; t < kGroup; t++) {
                    adesc[t] = desc_sw128_kmajor(stage0 + gs[t < ng ? t : 0] * C::kStageBytes);
                    dcol[t] = tmem_base + ga[t < ng ? t : 0] * (C::kHalves * N);
                }
                const uint64_t bdesc0 = desc_sw128_kmajor(b_base);
                auto issue = [&](auto NG) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; kk++) {
                        const int r = kk / 4, ko = (kk % 4) * 32;
                        const uint64_t aoff = (uint64_t)((r * (kTileM * 128) + ko) >> 4);
                        const uint64_t bdesc = bdesc0 + (uint64_t)((r * C::kBRegionBytes + ko) >> 4);
#pragma unroll
                        for (int t = 0; t < decltype(NG)::value; t++) {
                            if constexpr (C::kHalves == 2)
                                mma_bf16_warp(dcol[t] + (kk & 1) * N, adesc[t] + aoff, bdesc, idesc,
                                              kk > 1 ? 1u : 0u);
                            else
                                mma_bf16_warp(dcol[t], adesc[t] + aoff, bdesc, idesc, kk > 0 ? 1u : 0u);
                        }
                    }
                };
                if (D == 128 && ng == 3 && C::kHalves == 2)
                    mma_group3_d128(adesc[0], adesc[1], adesc[2], bdesc0, dcol[0], dcol[1], dcol[2],
                                    idesc, (uint64_t)(C::kBRegionBytes >> 4), (uint32_t)N);
                else if (ng == kGroup) issue(std::integral_constant<int, kGroup>{});
                else if (ng == 2) issue(std::integral_constant<int, 2>{});
                else issue(std::integral_constant<int, 1>{});
                for (int t = 0; t < ng; t++) {
                    mma_commit_warp(empty_bar(gs[t]));
                    mma_commit_warp(tfull_bar(ga[t]));
                }
#ifdef ASP_PROFILE_SCORE
                pm_issue += clock64() - t_issue;
#endif
            }
            PFLUSH(1, pm_full); PFLUSH(2, pm_tempty); PFLUSH(3, pm_issue); PFLUSH(7, pm_b);
        }
        __syncwarp();
    } else if (warp == 2 || warp == 3) {
        // ------------------------------------------------ B-operand builders (two warps)
        const int bl = lane + 32 * (warp - 2);                // 0..63
        int bs = -1;
        uint32_t bph = 0;
        int cur_row = -1;
        for (long i = it.next(it.start); i < it.end; i = it.next(i + 1)) {
            const int row = it.row;
            if (row == cur_row) continue;
            cur_row = row;
            bs = (bs + 1) % C::kBSlots;
            if (bs == 0 && i != it.next(it.start)) bph ^= 1;
            mbar_wait(bempty_bar(bs), bph ^ 1);
            const int b = row / p.n_kv_heads, h = row % p.n_kv_heads;
            const float *qsrc = q_hat + ((size_t)b * p.n_q_heads + (size_t)h * G) * D;
            unsigned char *slot = gbslot0 + bs * C::kBSlotBytes;
            // One (head g, 8 consecutive d) pair per lane-iteration: ONE load of q_hat
            // feeds the pair's three 16-B chunks (rows g, G + g, 2G + g: the hi /
            // mid / lo terms), and the loads of kBatch iterations are issued before
            // any is used -- the row's first MMA waits for this build (at G = 64 a
            // load-use loop over the 3G x D chunks cost ~37 us per CTA).
            auto put = [&](int n, int d0, uint4 w) {
                const int region = d0 / 64, chunk = (d0 % 64) / 8;
                *reinterpret_cast<uint4 *>(slot + region * C::kBRegionBytes + n * 128 +
                                           ((chunk ^ (n & 7)) * 16)) = w;
            };
            for (int c = bl; c < (N - 3 * G) * (D / 8); c += 64)          // padding rows: zero
                put(3 * G + c / (D / 8), (c % (D / 8)) * 8, make_uint4(0u, 0u, 0u, 0u));
            constexpr int kPairs = G * D / 8;
            constexpr int kPer = (kPairs + 63) / 64;                      // iterations per thread
            constexpr int kBatch = kPer < 8 ? kPer : 8;
            for (int p0 = 0; p0 < kPer; p0 += kBatch) {
                float4 x0[kBatch], x1[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; u++) {
                    const int pc = bl + 64 * (p0 + u);
                    if (pc < kPairs) {
                        const int g = pc / (D / 8), d0 = (pc % (D / 8)) * 8;
                        x0[u] = *reinterpret_cast<const float4 *>(qsrc + g * D + d0);
                        x1[u] = *reinterpret_cast<const float4 *>(qsrc + g * D + d0 + 4);
                    }
                }
#pragma unroll
                for (int u = 0; u < kBatch; u++) {
                    const int pc = bl + 64 * (p0 + u);
                    if (pc >= kPairs) continue;
                    const int g = pc / (D / 8), d0 = (pc % (D / 8)) * 8;
                    const float xs[8] = {x0[u].x, x0[u].y, x0[u].z, x0[u].w,
                                         x1[u].x, x1[u].y, x1[u].z, x1[u].w};
                    uint32_t wh[4], wm[4], wl[4];
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        uint16_t hv[2], mv[2], lv[2];
#pragma unroll
                        for (int f = 0; f < 2; f++) {
                            // exact 3-way split q = hi + mid + lo (each residual is exact in fp32)
                            const float q = xs[e + f];
                            const __nv_bfloat16 hi = __float2bfloat16_rn(q);
                            const float r1 = q - __bfloat162float(hi);
                            const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
                            const float r2 = r1 - __bfloat162float(mid);
                            const __nv_bfloat16 lo = __float2bfloat16_rn(r2);
                            hv[f] = *reinterpret_cast<const uint16_t *>(&hi);
                            mv[f] = *reinterpret_cast<const uint16_t *>(&mid);
                            lv[f] = *reinterpret_cast<const uint16_t *>(&lo);
                        }
                        wh[e / 2] = (uint32_t)hv[0] | ((uint32_t)hv[1] << 16);
                        wm[e / 2] = (uint32_t)mv[0] | ((uint32_t)mv[1] << 16);
                        wl[e / 2] = (uint32_t)lv[0] | ((uint32_t)lv[1] << 16);
                    }
                    put(g, d0, make_uint4(wh[0], wh[1], wh[2], wh[3]));
                    put(G + g, d0, make_uint4(wm[0], wm[1], wm[2], wm[3]));
                    put(2 * G + g, d0, make_uint4(wl[0], wl[1], wl[2], wl[3]));
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(bfull_bar(bs));
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue: TMEM -> scores
        // two warpgroups alternate tiles (each warp drains its 32-lane quadrant)
        const int quad = warp & 3;                  // TMEM lanes 32*quad .. +31
        const int group = (warp - 4) >> 2;
        bool nonfinite = false;
        long long pe_full = 0;
        long k = 0;                                 // index of the tile in this CTA's sequence
        // the scores are read back by the select kernel right after: keep them
        // L2-resident against the evict-first key stream
        const uint64_t keep = l2_policy_evict_last();
        for (long i = it.next(it.start); i < it.end; i = it.next(i + 1), k++) {
            if ((k & 1) != group) continue;
            const int a = (int)(k % C::kAcc);
            const uint32_t aph = (uint32_t)((k / C::kAcc) & 1);
            const int row = it.row, j = it.j;
            PWAIT(pe_full, mbar_wait(tfull_bar(a), aph));
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + a * (C::kHalves * N);
            float v[N <= 96 ? N : 32];                  // even + odd k-step halves (fixed order)
            float s_big = 0.0f;                         // G >= 64: reduced block by block
            if constexpr (N > 96) {
                // one chain; heads in blocks of 32: s_g = (hi_g + mid_g) + lo_g, then
                // the group reduction block by block (fixed order)
#pragma unroll 1
                for (int gb = 0; gb < G / 32; gb++) {
                    uint32_t rh[32], rm[32], rl[32];
                    tmem_ld32(taddr + 32 * gb, rh);
                    tmem_ld32(taddr + G + 32 * gb, rm);
                    tmem_ld32(taddr + 2 * G + 32 * gb, rl);
                    tmem_wait_ld();
#pragma unroll
                    for (int g = 0; g < 32; g++) {
                        const float sg = __fadd_rn(__fadd_rn(__uint_as_float(rh[g]), __uint_as_float(rm[g])),
                                                   __uint_as_float(rl[g]));
                        s_big = (gb == 0 && g == 0) ? sg
                              : (p.aggregation == ASP_AGG_SUM ? __fadd_rn(s_big, sg) : fmaxf(s_big, sg));
                    }
                }
            } else if constexpr (N == 32) {
                uint32_t r0[32], r1[32];
                tmem_ld32(taddr, r0);
                tmem_ld32(taddr + N, r1);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 32; c++) v[c] = __fadd_rn(__uint_as_float(r0[c]), __uint_as_float(r1[c]));
            } else if constexpr (N == 96) {
                // G = 32: the three 32-column chunks are the hi / mid / lo terms;
                // s_g = (hi_g + mid_g) + lo_g accumulated chunk by chunk
                uint32_t r0[32], r1[32];
                float acc32[32];
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    tmem_ld32(taddr + 32 * c, r0);
                    tmem_ld32(taddr + N + 32 * c, r1);
                    tmem_wait_ld();
#pragma unroll
                    for (int g = 0; g < 32; g++) {
                        const float x = __fadd_rn(__uint_as_float(r0[g]), __uint_as_float(r1[g]));
                        acc32[g] = c == 0 ? x : __fadd_rn(acc32[g], x);
                    }
                }
#pragma unroll
                for (int g = 0; g < 32; g++) v[g] = acc32[g];
            } else if constexpr (N == 48) {
                uint32_t r0[32], r1[32], r2[16], r3[16];
                tmem_ld32(taddr, r0);
                tmem_ld16(taddr + 32, r2);
                tmem_ld32(taddr + N, r1);
                tmem_ld16(taddr + N + 32, r3);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 32; c++) v[c] = __fadd_rn(__uint_as_float(r0[c]), __uint_as_float(r1[c]));
#pragma unroll
                for (int c = 0; c < 16; c++) v[32 + c] = __fadd_rn(__uint_as_float(r2[c]), __uint_as_float(r3[c]));
            } else {
                uint32_t r0[16], r1[16];
                tmem_ld16(taddr, r0);
                tmem_ld16(taddr + N, r1);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 16; c++) v[c] = __fadd_rn(__uint_as_float(r0[c]), __uint_as_float(r1[c]));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(a));
            float s = s_big;
            if constexpr (N <= 96) {
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const float sg = N == 96 ? v[g] : __fadd_rn(__fadd_rn(v[g], v[G + g]), v[2 * G + g]);
                    s = g == 0 ? sg : (p.aggregation == ASP_AGG_SUM ? __fadd_rn(s, sg) : fmaxf(s, sg));
                }
            }
            const int tok = j * kTileM + quad * 32 + lane;
            const int len = it.len_of(row);
            if (tok < len) {
                st_global_hint(scores + (size_t)row * p.max_seq_len + tok, s, keep);
                nonfinite |= !isfinite(s);
            }
        }
        if (__any_sync(0xffffffffu, nonfinite) && lane == 0) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
        if (warp == 4 && lane == 0) PFLUSH(4, pe_full);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem_base);
#ifdef ASP_PROFILE_SCORE
    if (threadIdx.x == 0) atomicAdd(&g_score_prof[6], (unsigned long long)(clock64() - t_kernel0));
#endif
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

template <int D, int G>
cudaError_t launch(const asp_select_params &p, const float *q_hat, const asp_bf16 *k,
                   const int32_t *seq_lens, float *scores, uint32_t *dev_flags, cudaStream_t s,
                   const asp_paged_kv *pk, const int32_t *block_table) {
    using C = Cfg<D, G>;
    auto encode = get_encode();
    if (!encode) return cudaErrorNotSupported;
    // 2-D row view [rows][D]: dense cache row(b, h, t) = (b*sb + h*sh)/st + t
    // (the ABI requires sb, sh to be multiples of st), a tile is one 128-row
    // box; paged pool row(page, h, t) = (page * Hkv + h) * page_size + t, a
    // tile is 128 / page_size boxes of page_size rows.
    CUtensorMap map;
    const bool paged = pk != nullptr;
    const int64_t rows = paged ? (int64_t)pk->num_pages * p.n_kv_heads * pk->page_size
                               : ((int64_t)(p.batch - 1) * p.k_stride_b +
                                  (int64_t)(p.n_kv_heads - 1) * p.k_stride_h) / p.k_stride_t +
                                     p.max_seq_len;
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(paged ? D : p.k_stride_t) * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)(paged ? pk->page_size : kTileM)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<asp_bf16 *>(k), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    const int tpr = (p.max_seq_len + kTileM - 1) / kTileM;
    const long total = (long)p.batch * p.n_kv_heads * tpr;
    const int grid = (int)(total < asp_sm_count() ? total : asp_sm_count());
    PagedArgs pg{block_table, paged ? pk->page_size : 0, paged ? pk->max_pages_per_seq : 0,
                 paged ? pk->num_pages : 0};
    auto kern = paged ? score_tc_kernel<D, G, true> : score_tc_kernel<D, G, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    return asp_launch(kern, dim3(grid), dim3(kThreads), C::kSmemBytes, s, 1, map, p, q_hat,
                      seq_lens, scores, dev_flags, tpr, pg);
}

}  // namespace

#ifdef ASP_PROFILE_SCORE
extern "C" __attribute__((visibility("default"))) int asp_score_prof_read(unsigned long long *host) {
    cudaMemcpyFromSymbol(host, g_score_prof, sizeof(g_score_prof));
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_score_prof, z, sizeof(z));
    return 0;
}
#endif

cudaError_t asp_launch_score(const asp_select_params &p, const float *q_hat,
                             const asp_bf16 *k_cache, const int32_t *seq_lens, float *scores,
                             uint32_t *dev_flags, cudaStream_t s, const asp_paged_kv *pk,
                             const int32_t *block_table) {
    const int G = p.n_q_heads / p.n_kv_heads;
#define ASP_CASE(DD, GG) \
    if (p.head_dim == DD && G == GG) \
        return launch<DD, GG>(p, q_hat, k_cache, seq_lens, scores, dev_flags, s, pk, block_table);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 4) ASP_CASE(64, 8)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 4) ASP_CASE(128, 8)
    ASP_CASE(64, 16) ASP_CASE(128, 16) ASP_CASE(64, 32) ASP_CASE(128, 32)
    ASP_CASE(64, 64) ASP_CASE(128, 64)
    // absorbed MLA (576-dim latent + rope keys) and 256-dim heads: region stages
    ASP_CASE(576, 1) ASP_CASE(576, 2) ASP_CASE(576, 4) ASP_CASE(576, 8) ASP_CASE(576, 16)
    ASP_CASE(256, 8) ASP_CASE(256, 16)
#undef ASP_CASE
    return cudaErrorInvalidValue;
}
