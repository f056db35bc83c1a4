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
//   * Persistent CTAs (one per SM) own a contiguous range of 128-token tiles
//     of the flattened (row, tile) space.  Warp roles: warp 0 streams K tiles
//     with TMA (4-D tensor map over the strided cache, 128-B swizzle,
//     L2 evict-first) into a 6-stage mbarrier ring; warp 1 owns TMEM and
//     issues the MMAs (single thread); warp 2 builds the swizzled bf16 B
//     operand for each new row into a 2-slot ring; warps 4-7 drain TMEM
//     (tcgen05.ld, 4 accumulator stages) and store the fp32 scores.
//
// Every token's score is a fixed function of its key row and q_hat (the same
// MMA datapath and the same 3-term epilogue order wherever the tile falls),
// so equal keys give equal scores and any KV-head shard reproduces the
// unsharded scores bit for bit.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc.cuh"

namespace {

using namespace asp::tc;

constexpr int kTileM = 128;           // tokens per tile (MMA M)
constexpr int kStages = 6;            // K-tile ring depth
constexpr int kAcc = 4;               // TMEM accumulator stages
constexpr int kBSlots = 2;            // B-operand ring
constexpr int kThreads = 256;         // 8 warps

template <int D, int G>
struct Cfg {
    static constexpr int N = (3 * G + 15) / 16 * 16 < 16 ? 16 : (3 * G + 15) / 16 * 16;
    static constexpr int kRegions = D / 64;                       // 128-B swizzle rows per token
    static constexpr int kStageBytes = kTileM * D * 2;
    static constexpr int kBRegionBytes = N * 128;
    static constexpr int kBSlotBytes = kRegions * kBRegionBytes;
    static constexpr uint32_t kTmemCols = (kAcc * N) <= 32 ? 32 : (kAcc * N) <= 64 ? 64
                                          : (kAcc * N) <= 128 ? 128 : 256;
    static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes +
                                      kBSlots * kBSlotBytes + 256 /*barriers*/;
};

struct TileIter {
    long start, end;
    int tpr, n_kv;
    const int32_t *seq_lens;
    int max_len;
    __device__ int len_of(int row) const {
        return min(max(seq_lens[row / n_kv], 0), max_len);
    }
    // advance i to the next valid tile (token base < row length) in [i, end)
    __device__ long next(long i) const {
        while (i < end) {
            const int row = (int)(i / tpr), j = (int)(i % tpr);
            if (j * kTileM < len_of(row)) return i;
            i = (long)(row + 1) * tpr;             // rest of the row is past its length
        }
        return end;
    }
};

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap kmap, asp_select_params p,
                const float *__restrict__ q_hat, const int32_t *__restrict__ seq_lens,
                float *__restrict__ scores, uint32_t *dev_flags, int tiles_per_row) {
    using C = Cfg<D, G>;
    constexpr int N = C::N;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char *gbase = smem_raw + (base - raw);
    const uint32_t stage0 = base;
    const uint32_t bslot0 = stage0 + kStages * C::kStageBytes;
    const uint32_t bar0 = bslot0 + kBSlots * C::kBSlotBytes;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * kStages + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * kStages + kAcc + a); };
    auto bfull_bar = [&](int s) { return bar0 + 8u * (2 * kStages + 2 * kAcc + s); };
    auto bempty_bar = [&](int s) { return bar0 + 8u * (2 * kStages + 2 * kAcc + kBSlots + s); };
    const uint32_t tmem_holder = bar0 + 8u * (2 * kStages + 2 * kAcc + 2 * kBSlots);
    unsigned char *gbslot0 = gbase + (bslot0 - base);
    volatile uint32_t *tmem_holder_g =
        reinterpret_cast<volatile uint32_t *>(gbase + (tmem_holder - base));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long total = (long)p.batch * p.n_kv_heads * tiles_per_row;
    TileIter it;
    it.start = total * blockIdx.x / gridDim.x;
    it.end = total * (blockIdx.x + 1) / gridDim.x;
    it.tpr = tiles_per_row;
    it.n_kv = p.n_kv_heads;
    it.seq_lens = seq_lens;
    it.max_len = p.max_seq_len;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 1); }
        for (int a = 0; a < kAcc; a++) { mbar_init(tfull_bar(a), 1); mbar_init(tempty_bar(a), 4); }
        for (int s = 0; s < kBSlots; s++) { mbar_init(bfull_bar(s), 1); mbar_init(bempty_bar(s), 1); }
        fence_mbar_init();
        prefetch_tmap(&kmap);
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder_g;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (long i = it.next(it.start); i < it.end; i = it.next(i + 1)) {
                const int row = (int)(i / it.tpr), j = (int)(i % it.tpr);
                const int b = row / p.n_kv_heads, h = row % p.n_kv_heads;
                mbar_wait(empty_bar(s), ph ^ 1);
                mbar_arrive_expect_tx(full_bar(s), C::kStageBytes);
                const uint32_t dst = stage0 + s * C::kStageBytes;
#pragma unroll
                for (int r = 0; r < C::kRegions; r++)
                    tma_load_4d(dst + r * (kTileM * 128), &kmap, full_bar(s), r * 64, j * kTileM,
                                h, b, kEvictFirst);
                if (++s == kStages) { s = 0; ph ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(kTileM, N);
            int s = 0, a = 0, bs = -1;
            uint32_t ph = 0, aph = 0, bph = 0;
            int cur_row = -1;
            for (long i = it.next(it.start); i < it.end; i = it.next(i + 1)) {
                const int row = (int)(i / it.tpr);
                if (row != cur_row) {
                    if (bs >= 0) mma_commit(bempty_bar(bs));        // previous row's B slot free
                    bs = (bs + 1) % kBSlots;
                    if (bs == 0 && cur_row != -1) bph ^= 1;
                    mbar_wait(bfull_bar(bs), bph);
                    cur_row = row;
                }
                mbar_wait(full_bar(s), ph);
                mbar_wait(tempty_bar(a), aph ^ 1);
                tc_fence_after();
                const uint32_t a_base = stage0 + s * C::kStageBytes;
                const uint32_t b_base = bslot0 + bs * C::kBSlotBytes;
                const uint32_t d_tmem = tmem_base + a * N;
#pragma unroll
                for (int kk = 0; kk < D / 16; kk++) {
                    const int r = kk / 4, ko = (kk % 4) * 32;
                    mma_bf16(d_tmem, desc_sw128_kmajor(a_base + r * (kTileM * 128) + ko),
                             desc_sw128_kmajor(b_base + r * C::kBRegionBytes + ko), idesc,
                             kk > 0 ? 1u : 0u);
                }
                mma_commit(empty_bar(s));
                mma_commit(tfull_bar(a));
                if (++s == kStages) { s = 0; ph ^= 1; }
                if (++a == kAcc) { a = 0; aph ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ------------------------------------------------ B-operand builder
        int bs = -1;
        uint32_t bph = 0;
        int cur_row = -1;
        for (long i = it.next(it.start); i < it.end; i = it.next(i + 1)) {
            const int row = (int)(i / it.tpr);
            if (row == cur_row) continue;
            cur_row = row;
            bs = (bs + 1) % kBSlots;
            if (bs == 0 && i != it.next(it.start)) bph ^= 1;
            mbar_wait(bempty_bar(bs), bph ^ 1);
            const int b = row / p.n_kv_heads, h = row % p.n_kv_heads;
            const float *qsrc = q_hat + ((size_t)b * p.n_q_heads + (size_t)h * G) * D;
            unsigned char *slot = gbslot0 + bs * C::kBSlotBytes;
            // one 16-B chunk (8 consecutive d of one B row) per lane-iteration
            constexpr int kChunks = N * D / 8;
            for (int c = lane; c < kChunks; c += 32) {
                const int n = c / (D / 8), d0 = (c % (D / 8)) * 8;
                uint32_t w[4] = {0u, 0u, 0u, 0u};
                if (n < 3 * G) {
                    const int g = n % G, term = n / G;
                    const float4 x0 = *reinterpret_cast<const float4 *>(qsrc + g * D + d0);
                    const float4 x1 = *reinterpret_cast<const float4 *>(qsrc + g * D + d0 + 4);
                    const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                    uint16_t hv[8];
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        // exact 3-way split q = hi + mid + lo (each residual is exact in fp32)
                        const float q = xs[e];
                        const __nv_bfloat16 hi = __float2bfloat16_rn(q);
                        const float r1 = q - __bfloat162float(hi);
                        const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
                        const float r2 = r1 - __bfloat162float(mid);
                        const __nv_bfloat16 lo = __float2bfloat16_rn(r2);
                        const __nv_bfloat16 t = term == 0 ? hi : term == 1 ? mid : lo;
                        hv[e] = *reinterpret_cast<const uint16_t *>(&t);
                    }
#pragma unroll
                    for (int e = 0; e < 4; e++) w[e] = (uint32_t)hv[2 * e] | ((uint32_t)hv[2 * e + 1] << 16);
                }
                const int region = d0 / 64, chunk = (d0 % 64) / 8;
                const int off = region * C::kBRegionBytes + n * 128 + ((chunk ^ (n & 7)) * 16);
                *reinterpret_cast<uint4 *>(slot + off) = make_uint4(w[0], w[1], w[2], w[3]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(bfull_bar(bs));
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue: TMEM -> scores
        const int quad = warp & 3;                  // TMEM lanes 32*quad .. +31
        int a = 0;
        uint32_t aph = 0;
        bool nonfinite = false;
        for (long i = it.next(it.start); i < it.end; i = it.next(i + 1)) {
            const int row = (int)(i / it.tpr), j = (int)(i % it.tpr);
            mbar_wait(tfull_bar(a), aph);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + a * N;
            float v[N];
            if constexpr (N == 32) {
                uint32_t r[32];
                tmem_ld32(taddr, r);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 32; c++) v[c] = __uint_as_float(r[c]);
            } else {
                uint32_t r[16];
                tmem_ld16(taddr, r);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 16; c++) v[c] = __uint_as_float(r[c]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(a));
            if (++a == kAcc) { a = 0; aph ^= 1; }
            float s = 0.0f;
#pragma unroll
            for (int g = 0; g < G; g++) {
                const float sg = __fadd_rn(__fadd_rn(v[g], v[G + g]), v[2 * G + g]);
                s = g == 0 ? sg : (p.aggregation == ASP_AGG_SUM ? __fadd_rn(s, sg) : fmaxf(s, sg));
            }
            const int tok = j * kTileM + quad * 32 + lane;
            const int len = it.len_of(row);
            if (tok < len) {
                scores[(size_t)row * p.max_seq_len + tok] = s;
                nonfinite |= !isfinite(s);
            }
        }
        if (__any_sync(0xffffffffu, nonfinite) && lane == 0) asp::flag_or(dev_flags, ASP_FLAG_NONFINITE);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem_base);
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
                   const int32_t *seq_lens, float *scores, uint32_t *dev_flags, cudaStream_t s) {
    using C = Cfg<D, G>;
    auto encode = get_encode();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap map;
    const cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)p.max_seq_len,
                                (cuuint64_t)p.n_kv_heads, (cuuint64_t)p.batch};
    const cuuint64_t strides[3] = {(cuuint64_t)p.k_stride_t * 2, (cuuint64_t)p.k_stride_h * 2,
                                   (cuuint64_t)p.k_stride_b * 2};
    const cuuint32_t box[4] = {64, (cuuint32_t)kTileM, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<asp_bf16 *>(k), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    const int tpr = (p.max_seq_len + kTileM - 1) / kTileM;
    const long total = (long)p.batch * p.n_kv_heads * tpr;
    const int grid = (int)(total < asp_sm_count() ? total : asp_sm_count());
    cudaError_t e = cudaFuncSetAttribute(score_tc_kernel<D, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    score_tc_kernel<D, G><<<grid, kThreads, C::kSmemBytes, s>>>(map, p, q_hat, seq_lens, scores,
                                                                dev_flags, tpr);
    return cudaGetLastError();
}

}  // namespace

cudaError_t asp_launch_score(const asp_select_params &p, const float *q_hat,
                             const asp_bf16 *k_cache, const int32_t *seq_lens, float *scores,
                             uint32_t *dev_flags, cudaStream_t s) {
    const int G = p.n_q_heads / p.n_kv_heads;
#define ASP_CASE(DD, GG) \
    if (p.head_dim == DD && G == GG) return launch<DD, GG>(p, q_hat, k_cache, seq_lens, scores, dev_flags, s);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 4) ASP_CASE(64, 8)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 4) ASP_CASE(128, 8)
#undef ASP_CASE
    return cudaErrorInvalidValue;
}
