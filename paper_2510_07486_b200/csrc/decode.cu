// decode.cu -- a4: sparse decode attention over only the selected K/V (P:190
// "the selected KV pairs ... participate in the attention computation";
// P:266), plus the always-attended fresh tail (reading R12).
//
//   out[b,hq] = sum_j softmax_j(sm_scale * q[b,hq] . K[b,h,t_j]) V[b,h,t_j],
//   t_j in {sel_idx valid} U [len - n_fresh, len),  h = hq / G.
//
// Design (B200): split-K over fixed 256-entry chunks of a (b, KV head) row --
// a chunk's arithmetic depends only on the row, never on the grid -- with
// the chunk partials merged in chunk order by a small combine kernel.  Each
// chunk is one work item of a persistent, warp-specialised kernel:
//
//   warps 0-7  producers: resolve the chunk's token list (indices fetched one
//            item ahead), build the bf16 Q operand when the row changes, and
//            GATHER the selected key / value rows with cp.async (16 lanes per
//            256-B row, coalesced) straight into the 128-B-swizzled UMMA
//            layout; 128-token tiles in a 5-stage ring; each producer waits
//            its copies two tiles later, fences them to the async proxy and
//            arrives on the stage's mbarrier.  (TMA tile::gather4 was measured
//            ~2.5x slower for 256-B random rows.)
//   warp 12  TMEM owner + tcgen05.mma issuer (warp-uniform, one elected lane):
//              S^T[128 tok x 16] = K_tile . Q^T          (q is bf16: exact)
//              O^T[D x 16]      += V_tile^T . P^T        (V tile MN-major)
//            P = [p_hi; p_lo] is the fp32 softmax weight split into two bf16
//            terms (rel. error 2^-17), so the P.V products stay fp32-exact;
//   warps 8-11 softmax (chunk max / exp2 / sums with warp shuffles and one
//            named barrier) writing the P operand, then the epilogue that
//            drains O from TMEM and stores the chunk partial (m, l, o).
//
// All G query heads of a KV head share every gathered row (GQA reuse); the
// contraction runs on the tensor cores so the SM pipes only orchestrate the
// gather stream (537 MB of K/V rows at the Qwen3-32B shape).
#include "common.cuh"
#include "tc.cuh"

#ifdef ASP_PROFILE_DECODE
__device__ unsigned long long g_dec_prof[16];
#define DWAIT(idx, call)                                                                 \
    do {                                                                                 \
        const long long _t0 = clock64();                                                 \
        call;                                                                            \
        if (threadIdx.x == 0 || threadIdx.x == kMmaWarp * 32 || threadIdx.x == kProducerThreads) \
            atomicAdd(&g_dec_prof[idx], (unsigned long long)(clock64() - _t0));          \
    } while (0)
#else
#define DWAIT(idx, call) call
#endif

namespace {

using namespace asp::tc;

constexpr int kTile = 128;                  // tokens per tile
constexpr int kChunk = 256;                 // entries per work item (fixed: determinism)
// A row of up to kTilesMax tiles of entries (384 when G <= 16) is ONE item of
// up to 3 tiles, so a 257-entry row (high concurrency: k = 256 plus the fresh
// token) is one item written straight to out -- not a full item plus a
// one-entry item and a combine.  Item sizes depend only on (top_k, n_fresh,
// G): never on the grid.
template <int G>
constexpr int tiles_max() { return G <= 16 ? 3 : 2; }   // G = 32: the P slots would not fit

constexpr int kProducerWarps = 8;
constexpr int kProducerThreads = kProducerWarps * 32;
constexpr int kMmaWarp = kProducerWarps + 4;
constexpr int kThreads = (kProducerWarps + 5) * 32;   // producers, 4 softmax/epilogue, 1 MMA warp
constexpr float kLog2e = 1.4426950408889634f;

template <int D, int G, int NT>
struct DCfg {
    static constexpr int kRegions = D / 64;
    static constexpr int kStageBytes = kRegions * kTile * 128;      // one K or V tile
    static constexpr int kN = G <= 16 ? 16 : 32;                    // MMA1 N: the G query heads
    static constexpr int kN2 = 2 * G <= 16 ? 16 : 2 * G;            // MMA2 N: 2G hi/lo P rows
    // K/V ring: 5 (D = 128) / 8 (D = 64) stages, 4 when G = 32's P and Q slots need the room
    static constexpr int kStages = G > 16 ? (D == 128 ? 4 : 6) : (D == 128 ? 5 : 8);

    static constexpr int kGR = G <= 8 ? 8 : G;                      // reduction row stride
    static constexpr int kQSlotBytes = kRegions * kN * 128;
    static constexpr int kPTileBytes = 2 * kN2 * 128;               // 128 tokens = 2 regions
    static constexpr int kTiles = NT;                               // tiles of the largest item
    static constexpr int kChunkMax = kTiles * kTile;
    static constexpr uint32_t kTmemCols = 2 * kTiles * kN + 2 * kN2 <= 128 ? 128
                                        : 2 * kTiles * kN + 2 * kN2 <= 256 ? 256 : 512;
    static constexpr int kPSlotBytes = kTiles * kPTileBytes;
    static constexpr int kZeroBytes = D == 64 ? 16384 : 0;          // MN-block 1 of V^T for D=64
    static constexpr int kTokBytes = 2 * kChunkMax * 4;
    static constexpr int kRedBytes = 2 * 2 * 4 * kGR * 4 + 2 * kGR * 4; // wmax, wsum, mrow
    static constexpr int kBarBytes = 256;
    static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + 2 * kQSlotBytes +
                                      2 * kPSlotBytes + kZeroBytes + kTokBytes + kRedBytes +
                                      kBarBytes;
};

struct Item {
    int row, chunk, nt;     // nt: tiles of this item (1..kTiles)
};

// Paged pools (asyncspade_sparse_decode_paged); unused by the dense instantiation.
struct PagedArgs {
    const int32_t *block_table;
    int page_size, max_pages, num_pages;
};

template <int D, int G, bool PAGED, int NT>
__global__ void __launch_bounds__(kThreads, 1)
decode_tc_kernel(asp_decode_params p, const asp_bf16 *__restrict__ q,
                 const asp_bf16 *__restrict__ k_cache, const asp_bf16 *__restrict__ v_cache,
                 const int32_t *__restrict__ seq_lens, const int32_t *__restrict__ sel_idx,
                 float *__restrict__ partials, float *__restrict__ out, int n_splits, PagedArgs pg,
                 int vshift) {
    using C = DCfg<D, G, NT>;
    constexpr int kGR = C::kGR;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char *gb = smem_raw + (base - raw);
    // ---- shared memory carve-up (all operand regions 1024-B aligned)
    const uint32_t stage0 = base;
    const uint32_t qslot0 = stage0 + C::kStages * C::kStageBytes;
    const uint32_t pslot0 = qslot0 + 2 * C::kQSlotBytes;
    const uint32_t zero0 = pslot0 + 2 * C::kPSlotBytes;
    const uint32_t tok0 = zero0 + C::kZeroBytes;
    const uint32_t red0 = tok0 + C::kTokBytes;
    const uint32_t bar0 = red0 + C::kRedBytes;
    int32_t *s_tok = reinterpret_cast<int32_t *>(gb + (tok0 - base));          // [2][256]
    float *s_wmax = reinterpret_cast<float *>(gb + (red0 - base));             // [2][4][kGR]
    float *s_wsum = s_wmax + 2 * 4 * kGR;                                      // [2][4][kGR]
    float *s_mrow = s_wsum + 2 * 4 * kGR;                                      // [2][kGR]
    auto bar = [&](int i) { return bar0 + 8u * i; };
    // barrier indices
    const int B_FULL = 0, B_EMPTY = C::kStages;
    const int B_QFULL = 2 * C::kStages, B_QEMPTY = B_QFULL + 2;
    const int B_TOKFULL = B_QEMPTY + 2, B_TOKEMPTY = B_TOKFULL + 2;
    const int B_SFULL = B_TOKEMPTY + 2, B_PFULL = B_SFULL + 2;
    const int B_OFULL = B_PFULL + 2, B_OEMPTY = B_OFULL + 2;
    const int B_COUNT = B_OEMPTY + 2;
    const uint32_t tmem_holder = bar(B_COUNT);
    volatile uint32_t *tmem_holder_g = reinterpret_cast<volatile uint32_t *>(gb + (tmem_holder - base));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Hq = p.n_q_heads, Hkv = p.n_kv_heads;
    const int E = p.top_k + p.n_fresh;
    const long total = (long)p.batch * Hkv * n_splits;
    const long i_start = total * blockIdx.x / gridDim.x;
    const long i_end = total * (blockIdx.x + 1) / gridDim.x;
    const int n_items = (int)(i_end - i_start);
    // the last chunk's entries (1..kChunkMax); every other chunk has kChunk
    const int last_entries = E - (n_splits - 1) * kChunk;
    auto item = [&](int i) -> Item {               // total items < 2^31: 32-bit math
        const int g = (int)i_start + i;
        const int c = g % n_splits;
        const int ne = c == n_splits - 1 ? last_entries : kChunk;
        return Item{g / n_splits, c, ne > 0 ? (ne + kTile - 1) / kTile : 1};
    };
    auto chunk_end = [&](const Item &it) {         // one past the item's last entry
        return it.chunk == n_splits - 1 ? E : (it.chunk + 1) * kChunk;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; s++) {
            mbar_init(bar(B_FULL + s), kProducerThreads);   // one cp.async arrival per producer
            mbar_init(bar(B_EMPTY + s), 1);
        }
        for (int s = 0; s < 2; s++) {
            mbar_init(bar(B_QFULL + s), 1);
            mbar_init(bar(B_QEMPTY + s), 1);
            mbar_init(bar(B_TOKFULL + s), 1);
            mbar_init(bar(B_TOKEMPTY + s), 4);
            mbar_init(bar(B_SFULL + s), 1);
            mbar_init(bar(B_PFULL + s), 4);
            mbar_init(bar(B_OFULL + s), 1);
            mbar_init(bar(B_OEMPTY + s), 4);
        }
        fence_mbar_init();
    }
    // zero the P operand slots (rows >= 2G stay zero) and the D=64 zero region
    for (uint32_t o = threadIdx.x * 16; o < 2u * C::kPSlotBytes + C::kZeroBytes; o += kThreads * 16)
        *reinterpret_cast<uint4 *>(gb + (pslot0 - base) + o) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (warp == kMmaWarp) tmem_alloc<C::kTmemCols>(tmem_holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder_g;
    asp::pdl_wait();                        // q, the caches, idx and partials are ours now
    asp::pdl_trigger();
#ifdef ASP_PROFILE_DECODE
    const long long t_k0 = clock64();
#endif
    // TMEM columns: S[slot][tile] at (slot*kTiles + tile)*kN, O[slot] after them
    auto s_col = [](int slot, int t) { return (uint32_t)((slot * C::kTiles + t) * C::kN); };
    auto o_col = [](int slot) { return (uint32_t)(2 * C::kTiles * C::kN + slot * C::kN2); };

    if (warp < kProducerWarps) {
        // ================================================= producers (8 warps)
        // Gather the selected K / V rows with cp.async (16 B per thread-op, one
        // token row per 16 consecutive lanes -> coalesced 256-B rows) straight into
        // the 128-B-swizzled UMMA layout; completion arrives on the stage's
        // mbarrier (cp.async.mbarrier.arrive.noinc).  Also builds the Q operand.
        const int pt = threadIdx.x;                           // 0..127
        int s = 0, qs = -1, cur_row = -1;
        uint32_t ph = 0, qph = 0;
        // software pipeline: the selection indices and row length of the NEXT item
        // are loaded while the current one is being gathered
        constexpr int kEntriesPerThread = (C::kChunkMax + kProducerThreads - 1) / kProducerThreads;
        int pre_raw[kEntriesPerThread] = {};
        int pre_len = 0;
        auto fetch = [&](int i) {
            const Item it = item(i);
            pre_len = seq_lens[it.row / Hkv];
            // (virtual KV heads of an MQA split share their batch's index row)
            const int32_t *ib = sel_idx + (size_t)(it.row >> vshift) * p.top_k;
#pragma unroll
            for (int u = 0; u < kEntriesPerThread; u++) {
                const int e = it.chunk * kChunk + pt + u * kProducerThreads;
                pre_raw[u] = e < p.top_k && e < chunk_end(it) ? __ldg(ib + e) : -1;
            }
        };
        // the attended token of entry u of item `it` (-1: none): a selected index
        // below the fresh tail, or a fresh-tail position (reading R12)
        auto logical_tok = [&](const Item &it, int len, int raw_u, int u) {
            const int fresh_lo = max(len - p.n_fresh, 0);
            const int e = it.chunk * kChunk + pt + u * kProducerThreads;
            int tok = -1;
            if (e >= chunk_end(it)) {
                // past this item (the next chunk's entries)
            } else if (e < p.top_k) {
                if (raw_u >= 0 && raw_u < fresh_lo) tok = raw_u;
            } else if (e < E) {
                const int t = fresh_lo + (e - p.top_k);
                if (t < len) tok = t;
            }
            return tok;
        };
        // Paged pools: s_tok holds the token's POOL row, (page * Hkv + h) *
        // page_size + slot.  The block-table lookups of item i+1 are issued
        // while item i is prepared (indices fetched two items ahead), so the
        // dependent loads never stall the gather.
        int x_tok[kEntriesPerThread] = {};
        auto xlate = [&](int i) {                             // uses pre_* of item i
            const Item it = item(i);
            const int b = it.row / Hkv, h = it.row % Hkv;
            const int len = min(max(pre_len, 0), p.max_seq_len);
#pragma unroll
            for (int u = 0; u < kEntriesPerThread; u++) {
                const int tok = logical_tok(it, len, pre_raw[u], u);
                int id = 0;
                if (tok >= 0) {
                    id = __ldg(pg.block_table + (size_t)b * pg.max_pages + tok / pg.page_size);
                    id = min(max(id, 0), pg.num_pages - 1);   // never fault on a bad entry
                }
                x_tok[u] = tok < 0 ? -1 : (id * Hkv + h) * pg.page_size + tok % pg.page_size;
            }
        };
        if (n_items > 0) fetch(0);
        if (PAGED && n_items > 0) {
            xlate(0);
            if (n_items > 1) fetch(1);
        }
        constexpr int kLag = 2;                               // < kStages
        int pending[kLag + 1];
        int npend = 0;
        auto release_oldest = [&]() {
            DWAIT(11, asm volatile("cp.async.wait_group %0;" ::"n"(kLag) : "memory"));
            fence_proxy_async_smem();
            mbar_arrive(bar(B_FULL + pending[0]));
            for (int u = 1; u < npend; u++) pending[u - 1] = pending[u];
            npend--;
        };
        auto prepare = [&](int i) {
            const int slot = i & 1;
            const Item it = item(i);
            const int b = it.row / Hkv, h = it.row % Hkv;
            const bool new_row = it.row != cur_row;
            if (new_row) {                                    // new row: Q operand
                qs = (qs + 1) & 1;
                if (qs == 0 && cur_row != -1) qph ^= 1;
                cur_row = it.row;
                DWAIT(0, mbar_wait(bar(B_QEMPTY + qs), qph ^ 1));
                const asp_bf16 *qsrc = q + ((size_t)b * Hq + (size_t)h * G) * D;
                unsigned char *qslot = gb + (qslot0 - base) + qs * C::kQSlotBytes;
                for (int c = pt; c < C::kN * D / 8; c += kProducerThreads) {
                    const int n = c / (D / 8), d0 = (c % (D / 8)) * 8;
                    uint4 v = make_uint4(0, 0, 0, 0);
                    if (n < G) v = *reinterpret_cast<const uint4 *>(qsrc + n * D + d0);
                    const int region = d0 / 64, chunk = (d0 % 64) / 8;
                    *reinterpret_cast<uint4 *>(qslot + region * (C::kN * 128) + n * 128 +
                                               ((chunk ^ (n & 7)) * 16)) = v;
                }
                fence_proxy_async_smem();
            }
            int toks[kEntriesPerThread];
            if (PAGED) {
                // this item's pool rows were resolved one item ahead (x_tok);
                // resolve the next one and fetch the indices of the one after
#pragma unroll
                for (int u = 0; u < kEntriesPerThread; u++) toks[u] = x_tok[u];
                if (i + 1 < n_items) xlate(i + 1);
                if (i + 2 < n_items) fetch(i + 2);
            } else {
                // this item's indices were fetched one item ahead (pre_*); fetch the next
                const int len = min(max(pre_len, 0), p.max_seq_len);
#pragma unroll
                for (int u = 0; u < kEntriesPerThread; u++) toks[u] = logical_tok(it, len, pre_raw[u], u);
                if (i + 1 < n_items) fetch(i + 1);
            }
            DWAIT(1, mbar_wait(bar(B_TOKEMPTY + slot), ((i >> 1) & 1) ^ 1));
            // WAR: every producer thread must be done reading this slot for the
            // previous item's V gather before anyone overwrites it
            asm volatile("bar.sync 2, %0;" ::"n"(kProducerThreads) : "memory");
#pragma unroll
            for (int u = 0; u < kEntriesPerThread; u++)
                if (pt + u * kProducerThreads < C::kChunkMax)
                    s_tok[slot * C::kChunkMax + pt + u * kProducerThreads] = toks[u];
            asm volatile("bar.sync 2, %0;" ::"n"(kProducerThreads) : "memory");
            if (pt == 0) {
                mbar_arrive(bar(B_TOKFULL + slot));
                if (new_row) mbar_arrive(bar(B_QFULL + qs));
            }
        };
        auto load = [&](int i, const asp_bf16 *cache, int64_t sb, int64_t sh, int64_t st) {
            const int slot = i & 1;
            const Item it = item(i);
            const int b = it.row / Hkv, h = it.row % Hkv;
            const asp_bf16 *rowbase = PAGED ? cache : cache + b * sb + h * sh;
            if (PAGED) st = D;                                // pool rows
            constexpr int kChunksPerRow = D / 8;              // 16-B chunks per token row
            constexpr int kRowsPerPass = kProducerThreads / kChunksPerRow;
            const int chunk = pt % kChunksPerRow;
            const int region = chunk / 8, cc = chunk % 8;
            constexpr int kPerThread = kTile / kRowsPerPass;  // rows r0 + kRowsPerPass * u
            const int r0 = pt / kChunksPerRow;
            const asp_bf16 *src0 = rowbase + chunk * 8;
            for (int t = 0; t < it.nt; t++) {
                DWAIT(2, mbar_wait(bar(B_EMPTY + s), ph ^ 1));
                // rows r0 + 8u share (r & 7): one swizzle per thread
                const uint32_t dst0 = stage0 + s * C::kStageBytes + region * (kTile * 128) +
                                      r0 * 128 + ((cc ^ (r0 & 7)) * 16);
                const int32_t *tk = s_tok + slot * C::kChunkMax + t * kTile + r0;
                // all token loads first, then the copies back to back (no memory
                // clobber on the copies: they are ordered by commit / wait_group)
                // an empty entry (-1: past a short row's selection, or the padding of
                // a row's last chunk) is zero-filled without a memory read (src-size
                // 0): its weight is 0, and a zero V row keeps 0 * V finite
                int tok[kPerThread];
#pragma unroll
                for (int u = 0; u < kPerThread; u++) tok[u] = tk[u * kRowsPerPass];
#pragma unroll
                for (int u = 0; u < kPerThread; u++) {
                    const asp_bf16 *src = src0 + (int64_t)max(tok[u], 0) * st;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                                 ::"r"(dst0 + (uint32_t)(u * kRowsPerPass * 128)), "l"(src),
                                 "r"(tok[u] >= 0 ? 16 : 0));
                }
                // cp.async writes are generic-proxy: each producer waits for its group
                // from kLag tiles ago, fences it to the async proxy (tensor core), and
                // only then arrives -- kLag + 1 tiles of copies stay in flight per thread
                asm volatile("cp.async.commit_group;" ::: "memory");
                pending[npend++] = s;
                if (npend > kLag) release_oldest();
                if (++s == C::kStages) { s = 0; ph ^= 1; }
            }
        };
        if (n_items > 0) {
            prepare(0);
            load(0, k_cache, p.k_stride_b, p.k_stride_h, p.k_stride_t);
        }
        for (int i = 0; i < n_items; i++) {
            if (i + 1 < n_items) {
                prepare(i + 1);
                load(i + 1, k_cache, p.k_stride_b, p.k_stride_h, p.k_stride_t);
            }
            load(i, v_cache, p.v_stride_b, p.v_stride_h, p.v_stride_t);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");   // drain the lagged stages
        fence_proxy_async_smem();
        for (int u = 0; u < npend; u++) mbar_arrive(bar(B_FULL + pending[u]));
    } else if (warp == kMmaWarp) {
        // ================================================= MMA issuer
        {                                   // whole warp; one elected lane issues
            constexpr uint32_t idesc1 = idesc_bf16_f32(kTile, C::kN);                 // K-major A, B
            constexpr uint32_t idesc2 = idesc_bf16_f32(kTile, C::kN2) | (1u << 15); // A MN-major
            int s = 0, qs = -1, cur_row = -1;
            uint32_t ph = 0, qph = 0;
            auto wait_stage = [&]() {
                DWAIT(3, mbar_wait(bar(B_FULL + s), ph));
                fence_proxy_async_smem();        // cp.async (generic proxy) -> tensor core reads
                tc_fence_after();
            };
            auto mma1 = [&](int i) {
                const int slot = i & 1;
                const Item it = item(i);
                if (it.row != cur_row) {
                    if (qs >= 0) mma_commit_warp(bar(B_QEMPTY + qs));
                    qs = (qs + 1) & 1;
                    if (qs == 0 && cur_row != -1) qph ^= 1;
                    DWAIT(4, mbar_wait(bar(B_QFULL + qs), qph));
                    cur_row = it.row;
                }
                const uint32_t qb = qslot0 + qs * C::kQSlotBytes;
                for (int t = 0; t < it.nt; t++) {
                    wait_stage();
                    const uint32_t ab = stage0 + s * C::kStageBytes;
#pragma unroll
                    for (int kk = 0; kk < D / 16; kk++) {
                        const int r = kk / 4, ko = (kk % 4) * 32;
                        mma_bf16_warp(tmem_base + s_col(slot, t),
                                 desc_sw128_kmajor(ab + r * (kTile * 128) + ko),
                                 desc_sw128_kmajor(qb + r * (C::kN * 128) + ko), idesc1, kk > 0 ? 1u : 0u);
                    }
                    mma_commit_warp(bar(B_EMPTY + s));
                    if (++s == C::kStages) { s = 0; ph ^= 1; }
                }
                mma_commit_warp(bar(B_SFULL + slot));
            };
            auto mma2 = [&](int i) {
                const int slot = i & 1;
                const uint32_t use = (uint32_t)((i >> 1) & 1);
                DWAIT(5, mbar_wait(bar(B_PFULL + slot), use));
                DWAIT(6, mbar_wait(bar(B_OEMPTY + slot), use ^ 1));
                tc_fence_after();
                const uint32_t pb = pslot0 + slot * C::kPSlotBytes;
                const int nt = item(i).nt;
                for (int t = 0; t < nt; t++) {
                    wait_stage();
                    const uint32_t vb = stage0 + s * C::kStageBytes;
                    // V tile as the MN-major A operand of O^T = V^T P^T: MN blocks of 64
                    // dims (LBO) and 8-token swizzle atoms (SBO = 1024 B)
                    const uint32_t lbo = D == 128 ? (uint32_t)(kTile * 128) : (zero0 - vb);
#pragma unroll
                    for (int kk = 0; kk < kTile / 16; kk++) {
                        uint64_t ad = desc_sw128_kmajor(vb + kk * 2048);
                        ad = (ad & ~(0x3FFFull << 16)) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16);
                        const uint64_t bd = desc_sw128_kmajor(pb + t * C::kPTileBytes +
                                                              (kk / 4) * (C::kN2 * 128) + (kk % 4) * 32);
                        mma_bf16_warp(tmem_base + o_col(slot), ad, bd, idesc2, (t | kk) ? 1u : 0u);
                    }
                    mma_commit_warp(bar(B_EMPTY + s));
                    if (++s == C::kStages) { s = 0; ph ^= 1; }
                }
                mma_commit_warp(bar(B_OFULL + slot));
            };
            if (n_items > 0) mma1(0);
            for (int i = 0; i < n_items; i++) {
                if (i + 1 < n_items) mma1(i + 1);
                mma2(i);
            }
        }
        __syncwarp();
    } else {
        // ================================================= softmax + epilogue (warps 8-11)
        const int quad = warp & 3;
        const float scale = p.sm_scale * kLog2e;
        auto softmax = [&](int i) {
            const int slot = i & 1;
            const uint32_t use = (uint32_t)((i >> 1) & 1);
            DWAIT(7, mbar_wait(bar(B_TOKFULL + slot), use));
            DWAIT(8, mbar_wait(bar(B_SFULL + slot), use));
            tc_fence_after();
            const int nt = item(i).nt;
            float l[C::kTiles][G];
            int tok[C::kTiles];
#pragma unroll
            for (int t = 0; t < C::kTiles; t++) {
                if (t >= nt) {                   // no such tile in this item
                    tok[t] = -1;
#pragma unroll
                    for (int g = 0; g < G; g++) l[t][g] = -INFINITY;
                    continue;
                }
                uint32_t r[C::kN];
                if constexpr (C::kN == 32)
                    tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + s_col(slot, t), r);
                else
                    tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + s_col(slot, t), r);
                tmem_wait_ld();
                tok[t] = s_tok[slot * C::kChunkMax + t * kTile + quad * 32 + lane];
#pragma unroll
                for (int g = 0; g < G; g++)
                    l[t][g] = tok[t] >= 0 ? __uint_as_float(r[g]) * scale : -INFINITY;
#ifdef ASP_DEBUG_DECODE
                if (tok[t] >= 0) {               // recompute S on CUDA cores from global K
                    const Item itd = item(i);
                    const int bd = itd.row / Hkv, hd = itd.row % Hkv;
                    const asp_bf16 *kr = k_cache + bd * p.k_stride_b + hd * p.k_stride_h +
                                         (int64_t)tok[t] * p.k_stride_t;
                    const asp_bf16 *qr = q + ((size_t)bd * Hq + (size_t)hd * G) * D;
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        float acc = 0.f;
                        for (int d = 0; d < D; d++)
                            acc += asp::bf16f(qr[g * D + d]) * asp::bf16f(kr[d]);
                        if (fabsf(acc - __uint_as_float(r[g])) > 1e-3f * (1.f + fabsf(acc)))
                            atomicAdd(&g_dec_prof[12], 1ull);
                    }
                    atomicAdd(&g_dec_prof[13], 1ull);
                }
#endif
            }
            float mx[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                float m = l[0][g];
#pragma unroll
                for (int t = 1; t < C::kTiles; t++) m = fmaxf(m, l[t][g]);
                mx[g] = asp::warp_max(m);
            }
            if (lane == 0)
#pragma unroll
                for (int g = 0; g < G; g++) s_wmax[(slot * 4 + quad) * kGR + g] = mx[g];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            float M[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                float m = s_wmax[(slot * 4 + 0) * kGR + g];
#pragma unroll
                for (int w = 1; w < 4; w++) m = fmaxf(m, s_wmax[(slot * 4 + w) * kGR + g]);
                M[g] = m;
            }
            unsigned char *pb = gb + (pslot0 - base) + slot * C::kPSlotBytes;
            const int x = quad * 32 + lane;                      // token column within a tile
            const int region = x / 64, within = x % 64;
            float sum[G];
#pragma unroll
            for (int g = 0; g < G; g++) sum[g] = 0.0f;
#pragma unroll
            for (int t = 0; t < C::kTiles; t++) {
                if (t >= nt) continue;           // (its P tile is not read)
                unsigned char *ptile = pb + t * C::kPTileBytes + region * (C::kN2 * 128);
#pragma unroll
                for (int g = 0; g < G; g++) {
                    const float pv = (tok[t] >= 0 && M[g] != -INFINITY) ? exp2f(l[t][g] - M[g]) : 0.0f;
                    sum[g] += pv;
                    const __nv_bfloat16 hi = __float2bfloat16_rn(pv);
                    const __nv_bfloat16 lo = __float2bfloat16_rn(pv - __bfloat162float(hi));
                    const int nh = g, nl = G + g;
                    *reinterpret_cast<__nv_bfloat16 *>(
                        ptile + nh * 128 + (((within >> 3) ^ (nh & 7)) * 16) + (within & 7) * 2) = hi;
                    *reinterpret_cast<__nv_bfloat16 *>(
                        ptile + nl * 128 + (((within >> 3) ^ (nl & 7)) * 16) + (within & 7) * 2) = lo;
                }
            }
#pragma unroll
            for (int g = 0; g < G; g++) sum[g] = asp::warp_sum(sum[g]);
            if (lane == 0)
#pragma unroll
                for (int g = 0; g < G; g++) s_wsum[(slot * 4 + quad) * kGR + g] = sum[g];
            if (quad == 0 && lane < G) s_mrow[slot * kGR + lane] = M[lane];
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(bar(B_PFULL + slot));
                mbar_arrive(bar(B_TOKEMPTY + slot));
            }
        };
        const uint64_t keep = l2_policy_evict_last();
        auto epilogue = [&](int i) {
            const int slot = i & 1;
            const uint32_t use = (uint32_t)((i >> 1) & 1);
            DWAIT(9, mbar_wait(bar(B_OFULL + slot), use));
            tc_fence_after();
            uint32_t r[C::kN2];
            if constexpr (C::kN2 == 64) {
                uint32_t (&ra)[32] = *reinterpret_cast<uint32_t (*)[32]>(&r[0]);
                uint32_t (&rb)[32] = *reinterpret_cast<uint32_t (*)[32]>(&r[32]);
                tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + o_col(slot), ra);
                tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + o_col(slot) + 32, rb);
            } else if constexpr (C::kN2 == 32) {
                tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + o_col(slot),
                          *reinterpret_cast<uint32_t (*)[32]>(&r[0]));
            } else {
                tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + o_col(slot),
                          *reinterpret_cast<uint32_t (*)[16]>(&r[0]));
            }
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(B_OEMPTY + slot));
            const Item it = item(i);
            const int b = it.row / Hkv, h = it.row % Hkv;
            const int d = quad * 32 + lane;
            if (n_splits == 1) {
                // a row of one chunk: out = o / l, exactly what the combine's merge
                // of a single partial gives (exp2f(0) = 1, fmaf(x, 1, 0) = x)
                const int64_t osb = p.out_stride_b ? p.out_stride_b : (int64_t)Hq * D;
                const int64_t osh = p.out_stride_h ? p.out_stride_h : (int64_t)D;
#pragma unroll
                for (int g = 0; g < G; g++) {
                    float L = 0.0f;
#pragma unroll
                    for (int w = 0; w < 4; w++) L += s_wsum[(slot * 4 + w) * kGR + g];
                    const float O = __fadd_rn(__uint_as_float(r[g]), __uint_as_float(r[G + g]));
                    if (d < D) out[b * osb + (int64_t)(h * G + g) * osh + d] = (L > 0.0f) ? O / L : 0.0f;
                }
                return;
            }
#pragma unroll
            for (int g = 0; g < G; g++) {
                // partials are read back by the combine kernel right after:
                // keep them in L2 (it drops them once merged)
                float *dst = partials + (((size_t)b * Hq + h * G + g) * n_splits + it.chunk) * (D + 2);
                if (d < D)
                    st_global_hint(dst + 2 + d,
                                   __fadd_rn(__uint_as_float(r[g]), __uint_as_float(r[G + g])), keep);
                if (d == 0) {
                    float L = 0.0f;
#pragma unroll
                    for (int w = 0; w < 4; w++) L += s_wsum[(slot * 4 + w) * kGR + g];
                    st_global_hint(dst, s_mrow[slot * kGR + g], keep);
                    st_global_hint(dst + 1, L, keep);
                }
            }
        };
        if (n_items > 0) softmax(0);
        for (int i = 0; i < n_items; i++) {
            if (i + 1 < n_items) softmax(i + 1);
            epilogue(i);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) tmem_dealloc<C::kTmemCols>(tmem_base);
#ifdef ASP_PROFILE_DECODE
    if (threadIdx.x == 0) atomicAdd(&g_dec_prof[10], (unsigned long long)(clock64() - t_k0));
#endif
}

// Few chunks (<= kCombineShort, e.g. config [2]'s 9): one sequential pass
// per thread, the loads of 8 chunks in flight -- no barriers.
constexpr int kCombineShort = 16;
template <int D>
__global__ void __launch_bounds__(D)
decode_combine_short_kernel(asp_decode_params p, const float *__restrict__ partials,
                            float *__restrict__ out, int n_splits) {
    const int hq = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
    asp::pdl_wait();
    asp::pdl_trigger();
    const float *src = partials + ((size_t)b * p.n_q_heads + hq) * n_splits * (D + 2);
    float M = -INFINITY;
#pragma unroll 8
    for (int s = 0; s < n_splits; s++) M = fmaxf(M, src[(size_t)s * (D + 2)]);
    float L = 0.0f, O = 0.0f;
    if (M != -INFINITY) {
#pragma unroll 8
        for (int s = 0; s < n_splits; s++) {
            const float *ps = src + (size_t)s * (D + 2);
            const float a = exp2f(ps[0] - M);
            L = fmaf(ps[1], a, L);
            O = fmaf(ps[2 + d], a, O);
        }
    }
    const int64_t osb = p.out_stride_b ? p.out_stride_b : (int64_t)p.n_q_heads * D;
    const int64_t osh = p.out_stride_h ? p.out_stride_h : (int64_t)D;
    out[b * osb + hq * osh + d] = (L > 0.0f) ? O / L : 0.0f;
    __syncthreads();
    const uintptr_t lo = (reinterpret_cast<uintptr_t>(src) + 127u) & ~(uintptr_t)127u;
    const uintptr_t hi = reinterpret_cast<uintptr_t>(src + (size_t)n_splits * (D + 2));
    for (uintptr_t x = lo + (uintptr_t)d * 128u; x + 128u <= hi; x += (uintptr_t)D * 128u)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(x) : "memory");
}

// Many chunks (long-CoT rows: 128): the chunk scales are computed once, in
// parallel, and staged in shared memory; the merge keeps the same order and
// the same fma chains (bit-identical to the short kernel), with only the
// partial-output loads on each thread's critical path.
template <int D>
__global__ void __launch_bounds__(D)
decode_combine_kernel(asp_decode_params p, const float *__restrict__ partials,
                      float *__restrict__ out, int n_splits) {
    extern __shared__ float s_comb[];           // [n_splits] scales a_s, [n_splits] l_s
    __shared__ float s_wmax[D / 32];
    const int hq = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
    asp::pdl_wait();
    asp::pdl_trigger();
    const float *src = partials + ((size_t)b * p.n_q_heads + hq) * n_splits * (D + 2);
    // 1. every chunk's (m_s, l_s) once, thread s of each block of D chunks
    //    (one round trip for up to D chunks), the row max by a block reduction
    float M = -INFINITY;
    for (int s = d; s < n_splits; s += D) {
        const float m = src[(size_t)s * (D + 2)];
        s_comb[s] = m;
        s_comb[n_splits + s] = src[(size_t)s * (D + 2) + 1];
        M = fmaxf(M, m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    if ((d & 31) == 0) s_wmax[d >> 5] = M;
    __syncthreads();
    M = s_wmax[0];
#pragma unroll
    for (int w = 1; w < D / 32; w++) M = fmaxf(M, s_wmax[w]);
    // 2. the scale of each chunk, a_s = 2^(m_s - M), computed once
    if (M != -INFINITY)
        for (int s = d; s < n_splits; s += D) s_comb[s] = exp2f(s_comb[s] - M);
    __syncthreads();
    // 3. the merge in chunk order (the same sequential fma chains as ever); the
    //    partial-output loads are independent of the chain: 16 in flight
    float L = 0.0f, O = 0.0f;
    if (M != -INFINITY) {
#pragma unroll 16
        for (int s = 0; s < n_splits; s++) {
            const float a = s_comb[s];
            L = fmaf(s_comb[n_splits + s], a, L);
            O = fmaf(src[(size_t)s * (D + 2) + 2 + d], a, O);
        }
    }
    const int64_t osb = p.out_stride_b ? p.out_stride_b : (int64_t)p.n_q_heads * D;
    const int64_t osh = p.out_stride_h ? p.out_stride_h : (int64_t)D;
    out[b * osb + hq * osh + d] = (L > 0.0f) ? O / L : 0.0f;
    // the partials are dead once merged: drop their L2 lines without write-back
    // (whole 128-B lines inside this (b, hq) block only)
    __syncthreads();
    const uintptr_t lo = (reinterpret_cast<uintptr_t>(src) + 127u) & ~(uintptr_t)127u;
    const uintptr_t hi = reinterpret_cast<uintptr_t>(src + (size_t)n_splits * (D + 2));
    for (uintptr_t x = lo + (uintptr_t)d * 128u; x + 128u <= hi; x += (uintptr_t)D * 128u)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(x) : "memory");
}

int n_splits_of(const asp_decode_params &p) {
    const int E = p.top_k + p.n_fresh;
    const int G = p.n_q_heads / p.n_kv_heads;
    const int max_last = (G <= 16 ? 3 : 2) * kTile;     // tiles_max<G>() tiles: 384 / 256 entries
    // one item up to max_last entries (no combine); else chunks of kChunk.
    // (Folding a longer row's remainder into a 3-tile last chunk -- config [2]'s
    // 2049 entries as 8 items instead of 9 -- measured SLOWER: 104 -> 113 us.)
    if (E <= max_last) return 1;
    return (E + kChunk - 1) / kChunk;
}

template <int D, int G, int NT>
cudaError_t launch_nt(const asp_decode_params &p, const asp_bf16 *q, const asp_bf16 *k,
                      const asp_bf16 *v, const int32_t *seq_lens, const int32_t *idx, float *out,
                      float *partials, cudaStream_t s, const asp_paged_kv *pk,
                      const int32_t *block_table, int vshift) {
    using C = DCfg<D, G, NT>;
    const int ns = n_splits_of(p);
    const long total = (long)p.batch * p.n_kv_heads * ns;
    const int grid = (int)(total < asp_sm_count() ? total : asp_sm_count());
    PagedArgs pg{block_table, pk ? pk->page_size : 1, pk ? pk->max_pages_per_seq : 0,
                 pk ? pk->num_pages : 0};
    auto kern = pk ? decode_tc_kernel<D, G, true, NT> : decode_tc_kernel<D, G, false, NT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    e = asp_launch(kern, dim3(grid), dim3(kThreads), C::kSmemBytes, s, 1, p, q, k, v, seq_lens,
                   idx, partials, out, ns, pg, vshift);
    if (e != cudaSuccess || ns == 1) return e;            // one chunk: written directly
    if (ns <= kCombineShort)
        return asp_launch(decode_combine_short_kernel<D>, dim3(p.n_q_heads, p.batch), dim3(D), 0, s, 1,
                          p, (const float *)partials, out, ns);
    const int csmem = (int)(2 * ns * sizeof(float));     // chunk scales + sums (top_k < ~7M)
    if (csmem > 48 * 1024) {
        e = cudaFuncSetAttribute(decode_combine_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem);
        if (e != cudaSuccess) return e;
    }
    return asp_launch(decode_combine_kernel<D>, dim3(p.n_q_heads, p.batch), dim3(D), csmem, s, 1, p,
                      (const float *)partials, out, ns);
}

// Two instantiations: 2-tile items (every multi-chunk row), and one item of up
// to 3 tiles for rows of 257..384 entries (G <= 16).  The 3-tile structure in
// the 2-tile case measured 104 -> 113 us at config [2] (wider softmax state,
// two index loads per producer thread), so it is used only where it saves a
// whole item and the combine.
template <int D, int G>
cudaError_t launch(const asp_decode_params &p, const asp_bf16 *q, const asp_bf16 *k,
                   const asp_bf16 *v, const int32_t *seq_lens, const int32_t *idx, float *out,
                   float *partials, cudaStream_t s, const asp_paged_kv *pk,
                   const int32_t *block_table, int vshift = 0) {
    if constexpr (tiles_max<G>() == 3) {
        if (p.top_k + p.n_fresh > kChunk)
            if (n_splits_of(p) == 1)
                return launch_nt<D, G, 3>(p, q, k, v, seq_lens, idx, out, partials, s, pk, block_table,
                                          vshift);
    }
    return launch_nt<D, G, 2>(p, q, k, v, seq_lens, idx, out, partials, s, pk, block_table, vshift);
}

}  // namespace

#ifdef ASP_PROFILE_DECODE
extern "C" __attribute__((visibility("default"))) int asp_decode_prof_read(unsigned long long *host) {
    cudaMemcpyFromSymbol(host, g_dec_prof, sizeof(g_dec_prof));
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_dec_prof, z, sizeof(z));
    return 0;
}
#endif

size_t asp_decode_workspace_bytes(const asp_decode_params &p) {
    const size_t b = (size_t)p.batch * p.n_q_heads * n_splits_of(p) * (p.head_dim + 2) * sizeof(float);
    return (b + 255) & ~(size_t)255;
}

cudaError_t asp_launch_decode(const asp_decode_params &p, const asp_bf16 *q,
                              const asp_bf16 *k_cache, const asp_bf16 *v_cache,
                              const int32_t *seq_lens, const int32_t *sel_idx, float *out,
                              void *workspace, cudaStream_t s, const asp_paged_kv *pk,
                              const int32_t *block_table) {
    float *partials = static_cast<float *>(workspace);
    const int G = p.n_q_heads / p.n_kv_heads;
    if (G > 32 && p.n_kv_heads == 1 && pk == nullptr && (G == 64 || G == 128)) {
        // MQA with 64 / 128 query heads: G / 32 "virtual" KV heads of 32 query
        // heads each over the SAME key / value rows (head stride 0) and the same
        // index row (row >> vshift).  Every virtual head gathers the selected rows
        // again, but its neighbour runs at the same time on the next SM, so the
        // second read is mostly an L2 hit; the arithmetic is the G = 32 kernel's.
        asp_decode_params v = p;
        v.n_kv_heads = G / 32;
        v.k_stride_h = v.v_stride_h = 0;
        const int vshift = G == 64 ? 1 : 2;
        if (p.head_dim == 64)
            return launch<64, 32>(v, q, k_cache, v_cache, seq_lens, sel_idx, out, partials, s, nullptr,
                                  nullptr, vshift);
        if (p.head_dim == 128)
            return launch<128, 32>(v, q, k_cache, v_cache, seq_lens, sel_idx, out, partials, s, nullptr,
                                   nullptr, vshift);
    }
#define ASP_CASE(DD, GG) \
    if (p.head_dim == DD && G == GG) \
        return launch<DD, GG>(p, q, k_cache, v_cache, seq_lens, sel_idx, out, partials, s, pk, block_table);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 4) ASP_CASE(64, 8)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 4) ASP_CASE(128, 8)
    ASP_CASE(64, 16) ASP_CASE(128, 16) ASP_CASE(64, 32) ASP_CASE(128, 32)
#undef ASP_CASE
    return cudaErrorInvalidValue;
}
