// decode_cc.cu -- a4 (sparse decode attention over the selected tokens, P:190,
// P:266; R12 fresh tail) for the shapes outside decode.cu's tensor-core
// kernel: absorbed MLA -- one KV head whose key is the 576-dim latent and
// whose value is its first 512 dims (v_head_dim < head_dim, the
// value rows read from the key rows when the caches alias) -- and query
// groups above 32 (MQA with many heads).
//
//   out[b,hq] = sum_j softmax_j(sm_scale * q[b,hq] . K[b,h,t_j]) V[b,h,t_j][:Dv]
//
// Same split-K contract as decode.cu: fixed 256-entry chunks of a row (a
// chunk's arithmetic depends only on the row), partials (m, l, o) in the
// workspace, merged in chunk order by the combine kernel below.  Inside a
// chunk, 32-token sub-tiles are gathered by cp.async into padded shared rows
// (double-buffered); logits on the CUDA cores (bf16 x bf16 products exact,
// fp32 sums), online softmax in exp2 units, P.V accumulated in fp32
// registers (each thread owns Dv / (256 / G) output dims of one head).
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kChunk = 256;                    // entries per work item (as decode.cu)
constexpr int kSub = 32;                       // tokens per gathered sub-tile
constexpr float kLog2e = 1.4426950408889634f;

template <int DK, int DV, int G>
struct DccCfg {
    static constexpr int kRowK = DK + 8;                         // padded bf16 rows
    static constexpr int kRowV = DV + 8;
    static constexpr int kTPH = kThreads / G;                    // threads per head (P.V)
    static constexpr int kDPT = DV / kTPH;                       // output dims per thread
    // ... in kNG groups of kVW contiguous dims (vector loads of V)
    static constexpr int kVW = kDPT % 8 == 0 ? 8 : kDPT % 4 == 0 ? 4 : 2;
    static constexpr int kNG = kDPT / kVW;
    static constexpr int kLG = G < 8 ? G : 8;                    // logit head groups
    static constexpr int kLHPT = G / kLG;                        // logit heads per thread
    static constexpr int kQBytes = G * DK * 4;
    static constexpr int kKBytes = kSub * kRowK * 2;
    static constexpr int kVBytes = kSub * kRowV * 2;
    static constexpr int kSmem = kQBytes + 2 * (kKBytes + kVBytes) + G * kSub * 4 /*p*/ +
                                 3 * G * 4 /*m, l, scale*/ + kChunk * 4 /*tokens*/;
    static_assert(kThreads % G == 0 && DV % kTPH == 0, "thread mapping");
};

template <int DK, int DV, int G>
__global__ void __launch_bounds__(kThreads)
decode_cc_kernel(asp_decode_params p, const asp_bf16 *__restrict__ q,
                 const asp_bf16 *__restrict__ kc, const asp_bf16 *__restrict__ vc,
                 const int32_t *__restrict__ seq_lens, const int32_t *__restrict__ sel_idx,
                 float *__restrict__ partials, int n_splits, int v_from_k) {
    using C = DccCfg<DK, DV, G>;
    extern __shared__ __align__(16) unsigned char smem[];
    float *sq = reinterpret_cast<float *>(smem);                                   // [G][DK]
    asp_bf16 *sk = reinterpret_cast<asp_bf16 *>(smem + C::kQBytes);                // [2][kSub][kRowK]
    asp_bf16 *sv = reinterpret_cast<asp_bf16 *>(smem + C::kQBytes + 2 * C::kKBytes);   // [2][kSub][kRowV]
    float *sp = reinterpret_cast<float *>(smem + C::kQBytes + 2 * (C::kKBytes + C::kVBytes));  // [G][kSub]
    float *sm = sp + G * kSub;                                                     // [G] running max
    float *sl = sm + G;                                                            // [G] running sum
    float *ss = sl + G;                                                            // [G] rescale
    int32_t *stok = reinterpret_cast<int32_t *>(ss + G);                           // [kChunk]
    const int tid = threadIdx.x;
    const int Hq = p.n_q_heads, Hkv = p.n_kv_heads;
    const int E = p.top_k + p.n_fresh;
    const long total = (long)p.batch * Hkv * n_splits;
    const long i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;
    const float scale = p.sm_scale * kLog2e;
    // P.V ownership: head og, dims od + kTPH * e
    const int og = tid / C::kTPH, od = tid % C::kTPH;
    // logits: token lt, heads lg + kLG * e
    const int lt = tid % kSub, lg = tid / kSub;
    asp::pdl_wait();                       // q, the caches and the selection
    asp::pdl_trigger();
    long cur_row = -1;
    for (long it = i0; it < i1; it++) {
        const long row = it / n_splits;
        const int chunk = (int)(it % n_splits);
        const int b = (int)(row / Hkv), h = (int)(row % Hkv);
        const int len = min(max(seq_lens[b], 0), p.max_seq_len);
        const int fresh_lo = max(len - p.n_fresh, 0);
        __syncthreads();                   // the previous item is done with smem
        if (row != cur_row) {
            const asp_bf16 *qs = q + ((size_t)b * Hq + (size_t)h * G) * DK;
            for (int c = tid; c < G * DK; c += kThreads) sq[c] = asp::bf16f(qs[c]);
            cur_row = row;
        }
        // the chunk's attended tokens (R12): selected below the fresh tail, then the tail
        int ntok_local = 0;
        {
            const int e = chunk * kChunk + tid;
            int tk = -1;
            if (e < p.top_k) {
                const int t = sel_idx[(size_t)row * p.top_k + e];
                if (t >= 0 && t < fresh_lo) tk = t;
            } else if (e < E) {
                const int t = fresh_lo + (e - p.top_k);
                if (t < len) tk = t;
            }
            stok[tid] = tk;
            ntok_local = tk >= 0;
        }
        if (tid < G) {
            sm[tid] = -INFINITY;
            sl[tid] = 0.0f;
        }
        const int any = __syncthreads_count(ntok_local);
        float acc[C::kDPT];
#pragma unroll
        for (int e = 0; e < C::kDPT; e++) acc[e] = 0.0f;
        const asp_bf16 *kb = kc + b * p.k_stride_b + h * p.k_stride_h;
        const asp_bf16 *vb = vc + b * p.v_stride_b + h * p.v_stride_h;
        auto gather = [&](int s, int buf) {
            asp_bf16 *dk = sk + buf * (kSub * C::kRowK);
            asp_bf16 *dv = sv + buf * (kSub * C::kRowV);
            constexpr int kCk = DK / 8, kCv = DV / 8;
            for (int c = tid; c < kSub * kCk; c += kThreads) {
                const int r = c / kCk, cc = c % kCk;
                const int t = max(stok[s * kSub + r], 0);          // -1 -> row 0 (masked below)
                const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dk + r * C::kRowK + cc * 8);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             ::"r"(sa), "l"(kb + (int64_t)t * p.k_stride_t + cc * 8));
            }
            if (!v_from_k) {
                for (int c = tid; c < kSub * kCv; c += kThreads) {
                    const int r = c / kCv, cc = c % kCv;
                    const int t = max(stok[s * kSub + r], 0);
                    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dv + r * C::kRowV + cc * 8);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                                 ::"r"(sa), "l"(vb + (int64_t)t * p.v_stride_t + cc * 8));
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        constexpr int kNSub = kChunk / kSub;
        if (any) gather(0, 0);
        for (int s = 0; any && s < kNSub; s++) {
            const int buf = s & 1;
            if (s + 1 < kNSub) {
                gather(s + 1, buf ^ 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();                                      // sub-tile `buf` landed
            const asp_bf16 *kt = sk + buf * (kSub * C::kRowK);
            // ---- logits (log2 units) of token lt against heads lg + kLG e
            {
                const bool valid = stok[s * kSub + lt] >= 0;
                const asp_bf16 *kr = kt + lt * C::kRowK;
                float dot[C::kLHPT];
#pragma unroll
                for (int e = 0; e < C::kLHPT; e++) dot[e] = 0.0f;
                if (lg < C::kLG) {
#pragma unroll 2
                    for (int d = 0; d < DK; d += 8) {
                        const uint4 kw = *reinterpret_cast<const uint4 *>(kr + d);
                        const float k8[8] = {asp::bf16lo(kw.x), asp::bf16hi(kw.x), asp::bf16lo(kw.y),
                                             asp::bf16hi(kw.y), asp::bf16lo(kw.z), asp::bf16hi(kw.z),
                                             asp::bf16lo(kw.w), asp::bf16hi(kw.w)};
#pragma unroll
                        for (int e = 0; e < C::kLHPT; e++) {
                            const float *qg = sq + (lg + C::kLG * e) * DK + d;
                            const float4 qa = *reinterpret_cast<const float4 *>(qg);
                            const float4 qb = *reinterpret_cast<const float4 *>(qg + 4);
                            float a = dot[e];
                            a = fmaf(qa.x, k8[0], a);
                            a = fmaf(qa.y, k8[1], a);
                            a = fmaf(qa.z, k8[2], a);
                            a = fmaf(qa.w, k8[3], a);
                            a = fmaf(qb.x, k8[4], a);
                            a = fmaf(qb.y, k8[5], a);
                            a = fmaf(qb.z, k8[6], a);
                            a = fmaf(qb.w, k8[7], a);
                            dot[e] = a;
                        }
                    }
#pragma unroll
                    for (int e = 0; e < C::kLHPT; e++)
                        sp[(lg + C::kLG * e) * kSub + lt] = valid ? dot[e] * scale : -INFINITY;
                }
            }
            __syncthreads();
            // ---- online softmax per head (thread g < G): new max, rescale, weights
            if (tid < G) {
                float mx = sm[tid];
                for (int j = 0; j < kSub; j++) mx = fmaxf(mx, sp[tid * kSub + j]);
                const float sc = mx == -INFINITY ? 1.0f : exp2f(sm[tid] - mx);
                float sum = 0.0f;
                for (int j = 0; j < kSub; j++) {
                    const float l = sp[tid * kSub + j];
                    const float w = l == -INFINITY ? 0.0f : exp2f(l - mx);
                    sp[tid * kSub + j] = w;
                    sum += w;
                }
                sl[tid] = sl[tid] * sc + sum;
                sm[tid] = mx;
                ss[tid] = sc;
            }
            __syncthreads();
            // ---- o[og][dims of group e] = o * scale + sum_j w_j V_j; thread od owns
            // the kVW-dim groups (od + kTPH e) (vector loads of the V rows)
            {
                const asp_bf16 *vt = v_from_k ? kt : sv + buf * (kSub * C::kRowV);
                const int vrow = v_from_k ? C::kRowK : C::kRowV;
                const float sc = ss[og];
#pragma unroll
                for (int e = 0; e < C::kDPT; e++) acc[e] *= sc;
                for (int j = 0; j < kSub; j++) {
                    const float w = sp[og * kSub + j];
                    if (w == 0.0f) continue;                      // uniform per head group
                    const asp_bf16 *vr = vt + j * vrow;
#pragma unroll
                    for (int e = 0; e < C::kNG; e++) {
                        const asp_bf16 *vg = vr + (od + C::kTPH * e) * C::kVW;
                        uint32_t w4[C::kVW / 2];
                        if constexpr (C::kVW == 8) {
                            const uint4 x = *reinterpret_cast<const uint4 *>(vg);
                            w4[0] = x.x; w4[1] = x.y; w4[2] = x.z; w4[3] = x.w;
                        } else if constexpr (C::kVW == 4) {
                            const uint2 x = *reinterpret_cast<const uint2 *>(vg);
                            w4[0] = x.x; w4[1] = x.y;
                        } else {
                            w4[0] = *reinterpret_cast<const uint32_t *>(vg);
                        }
#pragma unroll
                        for (int v = 0; v < C::kVW / 2; v++) {
                            acc[e * C::kVW + 2 * v] = fmaf(w, asp::bf16lo(w4[v]), acc[e * C::kVW + 2 * v]);
                            acc[e * C::kVW + 2 * v + 1] = fmaf(w, asp::bf16hi(w4[v]), acc[e * C::kVW + 2 * v + 1]);
                        }
                    }
                }
            }
            __syncthreads();                                      // sub-tile buffers reusable
        }
        // ---- the chunk's partial: m (log2 units), l, o for every head
        float *dst = partials + (((size_t)b * Hq + (size_t)h * G + og) * n_splits + chunk) * (DV + 2);
#pragma unroll
        for (int e = 0; e < C::kDPT; e++)
            dst[2 + (od + C::kTPH * (e / C::kVW)) * C::kVW + e % C::kVW] = any ? acc[e] : 0.0f;
        if (od == 0) {
            dst[0] = any ? sm[og] : -INFINITY;
            dst[1] = any ? sl[og] : 0.0f;
        }
    }
}

// chunk partials -> out, in chunk order (the same two-pass merge as decode.cu)
__global__ void decode_cc_combine_kernel(asp_decode_params p, int dv, const float *__restrict__ partials,
                                         float *__restrict__ out, int n_splits) {
    const int hq = blockIdx.x, b = blockIdx.y;
    asp::pdl_wait();
    asp::pdl_trigger();
    const float *src = partials + ((size_t)b * p.n_q_heads + hq) * n_splits * (dv + 2);
    float M = -INFINITY;
#pragma unroll 8
    for (int s = 0; s < n_splits; s++) M = fmaxf(M, src[(size_t)s * (dv + 2)]);
    const int64_t osb = p.out_stride_b ? p.out_stride_b : (int64_t)p.n_q_heads * dv;
    const int64_t osh = p.out_stride_h ? p.out_stride_h : (int64_t)dv;
    for (int d = threadIdx.x; d < dv; d += blockDim.x) {
        float L = 0.0f, O = 0.0f;
        if (M != -INFINITY) {
#pragma unroll 8
            for (int s = 0; s < n_splits; s++) {
                const float *ps = src + (size_t)s * (dv + 2);
                const float a = exp2f(ps[0] - M);
                L = fmaf(ps[1], a, L);
                O = fmaf(ps[2 + d], a, O);
            }
        }
        out[b * osb + hq * osh + d] = (L > 0.0f) ? O / L : 0.0f;
    }
}

int n_splits_cc(const asp_decode_params &p) {
    const int E = p.top_k + p.n_fresh;
    return E > 0 ? (E + kChunk - 1) / kChunk : 1;
}

template <int DK, int DV, int G>
cudaError_t launch(const asp_decode_params &p, const asp_bf16 *q, const asp_bf16 *k,
                   const asp_bf16 *v, const int32_t *seq_lens, const int32_t *idx, float *out,
                   void *workspace, cudaStream_t s) {
    using C = DccCfg<DK, DV, G>;
    auto kern = decode_cc_kernel<DK, DV, G>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, C::kSmem);
    if (e != cudaSuccess) return e;
    const int ns = n_splits_cc(p);
    const long total = (long)p.batch * p.n_kv_heads * ns;
    const long slots = (long)asp_sm_count() * (per_sm > 0 ? per_sm : 1);
    const int grid = (int)(total < slots ? total : slots);
    // MLA: the value rows are the key rows' first DV dims (the caches alias)
    const int v_from_k = (k == v && p.k_stride_b == p.v_stride_b && p.k_stride_h == p.v_stride_h &&
                          p.k_stride_t == p.v_stride_t) ? 1 : 0;
    float *partials = static_cast<float *>(workspace);
    e = asp_launch(kern, dim3(grid), dim3(kThreads), C::kSmem, s, 1, p, q, k, v, seq_lens, idx,
                   partials, ns, v_from_k);
    if (e != cudaSuccess) return e;
    return asp_launch(decode_cc_combine_kernel, dim3(p.n_q_heads, p.batch), dim3(DV < 256 ? DV : 256),
                      0, s, 1, p, DV, (const float *)partials, out, ns);
}

}  // namespace

size_t asp_decode_cc_workspace_bytes(const asp_decode_params &p, int dv) {
    const size_t b = (size_t)p.batch * p.n_q_heads * n_splits_cc(p) * (dv + 2) * sizeof(float);
    return (b + 255) & ~(size_t)255;
}

#define ASP_DCC_SHAPES(X)                                                                     \
    X(576, 512, 1) X(576, 512, 2) X(576, 512, 4) X(576, 512, 8) X(576, 512, 16)              \
    X(576, 576, 16) X(128, 128, 64) X(128, 128, 128) X(64, 64, 64) X(64, 64, 128)            \
    X(256, 256, 8) X(256, 256, 16)

bool asp_decode_cc_supported(int dk, int dv, int G) {
#define ASP_DCC_Q(DK, DV, GG) if (dk == DK && dv == DV && G == GG) return true;
    ASP_DCC_SHAPES(ASP_DCC_Q)
#undef ASP_DCC_Q
    return false;
}

cudaError_t asp_launch_decode_cc(const asp_decode_params &p, int dv, const asp_bf16 *q,
                                 const asp_bf16 *k_cache, const asp_bf16 *v_cache,
                                 const int32_t *seq_lens, const int32_t *sel_idx, float *out,
                                 void *workspace, cudaStream_t s) {
    const int G = p.n_q_heads / p.n_kv_heads, dk = p.head_dim;
#define ASP_DCC_L(DK, DV, GG)                                                                     \
    if (dk == DK && dv == DV && G == GG)                                                         \
        return launch<DK, DV, GG>(p, q, k_cache, v_cache, seq_lens, sel_idx, out, workspace, s);
    ASP_DCC_SHAPES(ASP_DCC_L)
#undef ASP_DCC_L
    return cudaErrorInvalidValue;
}
