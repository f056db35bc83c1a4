// predict.cu -- a1: temporal-regressive next-query prediction on sm_100a.
//
// AsyncSpade predicts q_hat_{t+1} from the window of recent query states by a
// softmax-normalised ridge regression applied to the one-step-shifted window
// (Eq. 2-4) assembled over window sizes and average
// pooled (Eq. 5; Alg. 1 Steps 1-6), with the readings
// R1-R8 of DESIGN.md §3 (masked-shared default).  All regression arithmetic
// is fp64 (reading R16).
//
// Design (B200).  Two kernels:
//   * predict_pair_kernel (2 <= W <= 16, masked-shared / single assembly --
//     every configured workload): TWO rows per warp; see the comment at the
//     kernel below.
//   * predict_kernel (every other case: W = 1 or W > 16, the per-window
//     assembly): one warp per (batch, q-head) row, eight independent rows per
//     CTA, no CTA-wide barriers, built for occupancy (~5 KB of shared memory
//     and <= 64 registers per warp) so the rows' dependent chains overlap:
//   * The augmented Gram matrix G' = Q Q^T (W x W) -- the history Gram G0
//     AND beta = H y in its last row -- runs on the fp64 tensor cores
//     (mma.sync m8n8k4 f64), all 8x8 tiles interleaved per k-step; the
//     fragments are read straight from the window in global memory in
//     logical ring order (each element once; lines reused through L1).
//   * For W <= 17 the ridge system lives in registers (lane i: row i of
//     [G0 + eps I | beta]) and is solved by Gauss-Jordan elimination with
//     shuffled pivot rows; longer windows use a shared-memory Cholesky.
//   * Cholesky of G0 + eps I is lane-parallel over the rows below each pivot;
//     forward / backward substitution keep the right-hand side in registers
//     (lane j owns component j) and broadcast pivots by shuffle.
//   * The masked-shared weights collapse to W coefficients c_p (one exp per
//     history weight, prefix sums by shuffle; a row-prefix softmax is the
//     prefix's normalised exponentials), so q_hat = sum_p c_p Q[p] / m is one
//     coalesced pass over the (cache-hot) window, rounded once to fp32.
// The step is ~0.7% of the path's bytes ("negligible runtime").
#include "common.cuh"

#include <math.h>

#ifdef ASP_PROFILE_PREDICT
__device__ unsigned long long g_pred_prof[8];
#define PPROF(idx)                                                                       \
    do {                                                                                 \
        if ((threadIdx.x & 31) == 0) {                                                   \
            const long long _t = clock64();                                              \
            atomicAdd(&g_pred_prof[idx], (unsigned long long)(_t - _tp));                \
            _tp = _t;                                                                    \
        }                                                                                \
    } while (0)
extern "C" __attribute__((visibility("default"))) int asp_predict_prof_read(unsigned long long *h) {
    cudaMemcpyFromSymbol(h, g_pred_prof, sizeof(g_pred_prof));
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_pred_prof, z, sizeof(z));
    return 0;
}
#else
#define PPROF(idx) (void)0
#endif

namespace {

constexpr int kWarps = 8;

__host__ __device__ size_t warp_smem_bytes(int W) {
    const size_t b = (size_t)W * W * sizeof(double)                  // augmented Gram G'
                     + (size_t)(W > 1 ? (W - 1) * (W - 1) : 1) * sizeof(double)  // Cholesky
                     + (size_t)(64 + 32 + 32) * sizeof(double);      // scratch, exps, coeffs
    return (b + 15) & ~(size_t)15;                                   // next warp: 16-B aligned
}

struct WarpSmem {
    double *G;      // [W][W] augmented Gram
    double *A;      // [nh][nh] Cholesky working copy
    double *vec;    // [64]
    double *e;      // [32]
    double *c;      // [32]
};

__device__ __forceinline__ double shfl_d(double v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// G' = Q Q^T over the window (NB 8-row blocks of logical rows; physical
// row of logical i = (ring_start + i) % W), fp64 tensor cores.  Every window
// element is loaded exactly once (by the lane owning its fragment slot), so
// the finiteness check rides along; returns it (warp-uniform).
template <int D, int NB>
__device__ bool gram_dmma(const WarpSmem &s, const float *__restrict__ win, int W, int ring_start) {
    const int lane = threadIdx.x & 31;
    const int fr = lane >> 2, fc = lane & 3;
    constexpr int kTiles = NB * (NB + 1) / 2;
    double acc[kTiles][2];
#pragma unroll
    for (int t = 0; t < kTiles; t++) acc[t][0] = acc[t][1] = 0.0;
    const float *rp[NB];
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const int i = 8 * b + fr;                     // logical row of this lane's fragment
        int phys = i + ring_start;
        if (phys >= W) phys -= W;
        rp[b] = i < W ? win + (size_t)phys * D + fc : nullptr;
    }
    bool finite = true;
#pragma unroll 4
    for (int k = 0; k < D; k += 4) {
        double f[NB];
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const float x = rp[b] ? __ldg(rp[b] + k) : 0.0f;
            finite = finite && isfinite(x);
            f[b] = (double)x;
        }
        int t = 0;
#pragma unroll
        for (int bi = 0; bi < NB; bi++)
#pragma unroll
            for (int bj = bi; bj < NB; bj++, t++) dmma(acc[t][0], acc[t][1], f[bi], f[bj]);
    }
    // lane holds C[8bi + fr][8bj + 2fc + e]
    int t = 0;
#pragma unroll
    for (int bi = 0; bi < NB; bi++)
#pragma unroll
        for (int bj = bi; bj < NB; bj++, t++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int i = 8 * bi + fr, j = 8 * bj + 2 * fc + e;
                if (i < W && j < W) {
                    s.G[i * W + j] = acc[t][e];
                    s.G[j * W + i] = acc[t][e];
                }
            }
    return __all_sync(0xffffffffu, finite);
}

// Ridge solve over history rows [h0, h0 + nh) regressing the newest row W-1
// (Alg. 1 Step 3): omega = (G0 + eps I)^{-1} beta.  Lane i < nh
// returns omega_i; ok is warp-uniform (false: not positive definite).
__device__ double ridge_solve(const WarpSmem &s, int W, int h0, int nh, float eps, bool absolute,
                              bool &ok) {
    const int lane = threadIdx.x & 31;
    double *A = s.A;
    for (int u = lane; u < nh * nh; u += 32) {
        const int i = u / nh, j = u - (u / nh) * nh;
        A[u] = s.G[(h0 + i) * W + (h0 + j)];
    }
    const double beta_lane = lane < nh ? s.G[(W - 1) * W + h0 + lane] : 0.0;
    __syncwarp();
    // eps relative to mean diag(G0) (reading R7) unless absolute; zero floor.
    double e = (double)eps;
    if (!absolute) {
        double tr = 0.0;
        for (int i = 0; i < nh; i++) tr += A[i * nh + i];
        e = (double)eps * (tr / nh);
    }
    if (e == 0.0) e = 1e-30;
    __syncwarp();
    if (lane < nh) A[lane * nh + lane] += e;
    __syncwarp();
    // Right-looking Cholesky G = L L^T: per pivot, scale the column (lanes over
    // rows) and apply the rank-1 update to the trailing lower triangle (lanes
    // over its elements) -- constant dependency depth per column.
    double inv_d_lane = 0.0;
    ok = true;
    for (int j = 0; j < nh; j++) {
        const double ajj = A[j * nh + j];
        if (!(ajj > 0.0) || !isfinite(ajj)) { ok = false; break; }   // warp-uniform
        const double dj = sqrt(ajj);
        const double inv = 1.0 / dj;
        if (lane == j) inv_d_lane = inv;
        __syncwarp();
        if (lane == 0) A[j * nh + j] = dj;
        for (int i = j + 1 + lane; i < nh; i += 32) A[i * nh + j] *= inv;
        __syncwarp();
        const int m = nh - j - 1;                       // trailing block size
        for (int u = lane; u < m * (m + 1) / 2; u += 32) {
            // u -> (ii, kk), kk <= ii, row-major over the lower triangle
            int ii = (int)((sqrtf(8.0f * u + 1.0f) - 1.0f) * 0.5f);
            if ((ii + 1) * (ii + 2) / 2 <= u) ii++;
            if (ii * (ii + 1) / 2 > u) ii--;
            const int kk = u - ii * (ii + 1) / 2;
            const int i = j + 1 + ii, k = j + 1 + kk;
            A[i * nh + k] = fma(-A[i * nh + j], A[k * nh + j], A[i * nh + k]);
        }
        __syncwarp();
    }
    if (!ok) return 0.0;
    // forward: L y = beta (lane j owns component j)
    double r = beta_lane;
    for (int i = 0; i < nh; i++) {
        const double yi = shfl_d(r * inv_d_lane, i);
        if (lane == i) r = yi;
        else if (lane > i && lane < nh) r = fma(-A[lane * nh + i], yi, r);
    }
    // backward: L^T x = y
    for (int i = nh - 1; i >= 0; i--) {
        const double xi = shfl_d(r * inv_d_lane, i);
        if (lane == i) r = xi;
        else if (lane < i) r = fma(-A[i * nh + lane], xi, r);
    }
    ok = __all_sync(0xffffffffu, lane >= nh || isfinite(r));
    return lane < nh ? r : 0.0;
}

// The same ridge solve for the full history (h0 = 0, nh <= 16) with the
// system in registers: lane i holds row i of [G0 + eps I | beta] and
// Gauss-Jordan elimination (no pivoting: the matrix is SPD, its pivots are
// Cholesky's squared diagonal -- a pivot <= 0 means not positive definite)
// broadcasts one pivot row per step by shuffle.  ~15 dependent steps of
// independent shuffles and FMAs instead of the shared-memory Cholesky.
__device__ double ridge_solve_regs(const WarpSmem &s, int W, int nh, float eps, bool absolute,
                                   bool &ok) {
    constexpr int kMax = 16;
    const int lane = threadIdx.x & 31;
    const bool own = lane < nh;
    double r[kMax];
#pragma unroll
    for (int k = 0; k < kMax; k++) r[k] = (own && k < nh) ? s.G[lane * W + k] : 0.0;
    double rb = own ? s.G[(W - 1) * W + lane] : 0.0;
    // eps relative to mean diag(G0) (reading R7) unless absolute; zero floor
    double e = (double)eps;
    if (!absolute) {
        double tr = own ? s.G[lane * W + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
        e = (double)eps * (tr / nh);
    }
    if (e == 0.0) e = 1e-30;
#pragma unroll
    for (int k = 0; k < kMax; k++) if (k == lane && own) r[k] += e;
    ok = true;
    double diag = 1.0;                                                 // lane j: pivot j
#pragma unroll
    for (int j = 0; j < kMax; j++) {
        if (j >= nh) break;
        const double d = __shfl_sync(0xffffffffu, r[j], j);
        const double pb = __shfl_sync(0xffffffffu, rb, j);
        if (!(d > 0.0) || !isfinite(d)) { ok = false; break; }        // warp-uniform
        if (lane == j) diag = d;
        const double f = lane != j ? r[j] / d : 0.0;                   // the pivot row stays
#pragma unroll
        for (int k = j; k < kMax; k++) r[k] = fma(-f, __shfl_sync(0xffffffffu, r[k], j), r[k]);
        rb = fma(-f, pb, rb);
    }
    if (!ok) return 0.0;
    const double x = own ? rb / diag : 0.0;
    ok = __all_sync(0xffffffffu, !own || isfinite(x));
    return x;
}

// Collapse the masked-shared assembly (Alg. 1 Steps 4-6, readings R4-R6) of
// the weights v[0..n) (lane i holds v_i) into coefficients c[0..W) (smem):
// row j = 1..W uses r_j = softmax(v[0..n_j)), n_j = min(j, n), on the newest
// n_j queries; c_p = sum_j r_j[p - W + n_j] (the 1/W is applied by the caller).
__device__ void masked_shared_coeffs(const WarpSmem &s, int W, int n, double v_lane) {
    const int lane = threadIdx.x & 31;
    double m = lane < n ? v_lane : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const double e = lane < n ? exp(v_lane - m) : 0.0;
    double S = e;                                 // inclusive prefix sums S_{lane+1}
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, S, o);
        if (lane >= o) S += t;
    }
    s.e[lane] = e;
    s.vec[32 + lane] = 1.0 / S;                   // reciprocal prefix sums (lane-parallel)
    const bool tiny = __any_sync(0xffffffffu, lane == 0 && !(S > 1e-280));
    s.vec[lane] = v_lane;
    __syncwarp();
    if (lane < W) {
        const int p = lane;
        double acc = 0.0;
        for (int mm = W - p; mm <= n; mm++) {
            if (mm < 1) continue;
            const double mult = (mm == n) ? 2.0 : 1.0;      // rows j = W-1 and W share n_j = n
            if (!tiny) {
                acc += mult * s.e[p - W + mm] * s.vec[32 + mm - 1];
            } else {
                // a prefix's exponentials underflowed against the global max
                double mx = s.vec[0];
                for (int i = 1; i < mm; i++) mx = fmax(mx, s.vec[i]);
                double den = 0.0;
                for (int i = 0; i < mm; i++) den += exp(s.vec[i] - mx);
                acc += mult * exp(s.vec[p - W + mm] - mx) / den;
            }
        }
        s.c[p] = acc;
    }
    __syncwarp();
}

// full softmax of v over lanes < n (lane i returns its weight, 0 beyond n)
__device__ double lane_softmax(double v_lane, int n) {
    const int lane = threadIdx.x & 31;
    double m = lane < n ? v_lane : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const double e = lane < n ? exp(v_lane - m) : 0.0;
    double S = e;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    return e / S;
}

template <int D, int NB>
__global__ void __launch_bounds__(kWarps * 32, 4)
predict_kernel(asp_predict_params p, const float *__restrict__ q_window,
               float *__restrict__ q_hat, uint32_t *dev_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int W = p.window, n = W - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long rows = (long)p.batch * p.n_q_heads;
    const long row = (long)blockIdx.x * (blockDim.x >> 5) + warp;   // 1..kWarps rows per CTA
    asp::pdl_wait();
    asp::pdl_trigger();
    if (row >= rows) return;

    unsigned char *base = smem_raw + warp_smem_bytes(W) * warp;
    WarpSmem s;
    size_t off = 0;
    s.G = reinterpret_cast<double *>(base + off);
    off += (size_t)W * W * sizeof(double);
    s.A = reinterpret_cast<double *>(base + off);
    off += (size_t)(W > 1 ? (W - 1) * (W - 1) : 1) * sizeof(double);
    s.vec = reinterpret_cast<double *>(base + off);
    s.e = s.vec + 64;
    s.c = s.e + 32;
    s.c[lane] = 0.0;

    // Step 1: the window's logical row i is physical row
    // (ring_start + i) % W; row W-1 is the newest query.
    const float *src = q_window + (size_t)row * W * D;
    auto phys_of = [&](int i) {
        const int ph = i + p.ring_start;
        return ph >= W ? ph - W : ph;
    };
    float *out = q_hat + (size_t)row * D;
    const uint32_t mode = p.flags & 0xFu;
    const double sgn = (p.flags & ASP_SIGN_NEGATED) ? -1.0 : 1.0;
    const bool absolute = (p.flags & ASP_EPS_ABSOLUTE) != 0;

#ifdef ASP_PROFILE_PREDICT
    long long _tp = clock64();
#endif
    const bool finite = W > 1 ? gram_dmma<D, NB>(s, src, W, p.ring_start) : true;
    PPROF(0);
    bool ok = finite && W > 1;
    double denom = 1.0;
    if (ok) {
        __syncwarp();
        if (mode == ASP_ASSEMBLY_PER_WINDOW) {
            // Eq. 5 literal: one solve per window size k = 1..n on Q[W-1-k..W-2],
            // softmax weights applied to Q[W-k..W-1]; m = n.
            double cacc = 0.0;                        // lane p accumulates c_p
            for (int k = 1; k <= n && ok; k++) {
                const double om = ridge_solve(s, W, W - 1 - k, k, p.eps, absolute, ok);
                if (!ok) break;
                const double w = lane_softmax(sgn * om, k);
                s.e[lane] = w;
                __syncwarp();
                if (lane >= W - k && lane < W) cacc += s.e[lane - (W - k)];
                __syncwarp();
            }
            s.c[lane] = cacc;
            denom = (double)n;
        } else {
            const double om = n <= 16 ? ridge_solve_regs(s, W, n, p.eps, absolute, ok)
                                      : ridge_solve(s, W, 0, n, p.eps, absolute, ok);
            PPROF(1);
            if (ok && mode == ASP_ASSEMBLY_SINGLE) {
                // Eq. 4: omega[i] (history row i) weights Q[i+1].
                const double w = (p.flags & ASP_NORM_NONE) ? om : lane_softmax(sgn * om, n);
                if (lane < n) s.c[lane + 1] = w;
                denom = 1.0;
            } else if (ok) {
                double v = sgn * om;
                if (p.flags & ASP_DOUBLE_SOFTMAX) v = lane_softmax(v, n);  // literal Step 3
                masked_shared_coeffs(s, W, n, v);
                denom = (double)W;
            }
        }
        __syncwarp();
    }
    PPROF(2);
    if (ok) {
        const double inv_m = 1.0 / denom;
        double acc[D / 32];
#pragma unroll
        for (int j = 0; j < D / 32; j++) acc[j] = 0.0;
        for (int q = 0; q < W; q++) {
            const double cq = s.c[q];
            const float *rq = src + (size_t)phys_of(q) * D + lane;
#pragma unroll
            for (int j = 0; j < D / 32; j++) acc[j] = fma(cq, (double)__ldg(rq + 32 * j), acc[j]);
        }
#pragma unroll
        for (int j = 0; j < D / 32; j++) out[lane + 32 * j] = (float)(acc[j] * inv_m);
        PPROF(3);
    } else {
        // Passthrough q_hat = Q_t; flag why.
        const float *rq = src + (size_t)phys_of(W - 1) * D;
        for (int d = lane; d < D; d += 32) out[d] = rq[d];
        if (lane == 0 && W > 1) asp::flag_or(dev_flags, finite ? ASP_FLAG_NOT_PD : ASP_FLAG_NONFINITE);
    }
}

// ---------------------------------------------------------------------------
// Fast path for the common case (2 <= W <= 16, masked-shared or single-window
// assembly): TWO rows per warp.  The W x W Gram of both rows runs on the fp64
// tensor cores from 128-bit loads (the contraction index d is permuted
// identically in both operands, so each lane's float4 feeds four k-steps and
// the two rows give six independent accumulator chains); then each half-warp
// owns one row for the branch-free register Gauss-Jordan solve (lane l = row l
// of [G0 + eps I | beta], padded to 16 with identity rows that change
// nothing), the shuffle-only masked-shared coefficient assembly and the
// weighted sum -- so every instruction of the sequential part serves two
// rows.  Non-finite windows are caught by the Gram diagonal (sum of squares:
// finite iff every element is) instead of a per-element test.
ASP_DEV double rcp_nr(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}

// one Newton step: relative error ~2^-44 (the pivots of the elimination)
ASP_DEV double rcp_nr1(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    return fma(y, fma(-d, y, 1.0), y);
}

ASP_DEV double shfl16(double v, int src) { return __shfl_sync(0xffffffffu, v, src, 16); }
ASP_DEV double shfl16_up(double v, unsigned dl) { return __shfl_up_sync(0xffffffffu, v, dl, 16); }
ASP_DEV double half_max(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o, 16));
    return v;
}
ASP_DEV double half_sum(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, 16);
    return v;
}
// softmax over lanes l < n of the half-warp (0 beyond n)
ASP_DEV double half_softmax(double v, int l, int n) {
    const double m = half_max(l < n ? v : -INFINITY);
    const double e = l < n ? exp(v - m) : 0.0;
    return e / half_sum(e);
}

// four consecutive window elements at element offset `off` (a multiple of 4)
// as fp32: the ring is fp32, or bf16 with ASP_WINDOW_BF16 (exact widening)
template <bool BF>
ASP_DEV float4 ld4(const float *__restrict__ win, int off) {
    if constexpr (BF) {
        const uint2 w = __ldg(reinterpret_cast<const uint2 *>(reinterpret_cast<const asp_bf16 *>(win) + off));
        return make_float4(asp::bf16lo(w.x), asp::bf16hi(w.x), asp::bf16lo(w.y), asp::bf16hi(w.y));
    } else {
        return __ldg(reinterpret_cast<const float4 *>(win + off));
    }
}

constexpr int kPairWarps = 8;
constexpr int kGS = 17;                            // smem row stride of a Gram (doubles)

// Steps 3-6 for the two rows of a warp, one per half-warp (h =
// lane / 16, l = lane % 16) on the augmented Gram G (row stride kGS) of row h:
// the ridge solve by register Gauss-Jordan and the masked-shared / single
// coefficients.  Lane l returns c = c_{l+1} of q_hat = sum_p c_p Q[p] / denom
// (c_0 = 0); ok = the half's system was finite and positive definite.
ASP_DEV void solve_coeffs(const asp_predict_params &p, const double *G, int W, double &c,
                          double &denom, bool &ok, bool &finite) {
    const int n = W - 1;
    const int lane = threadIdx.x & 31;
    // ---- from here each half-warp owns one row: h = row, l = lane within the half
    const int h = lane >> 4, l = lane & 15;
    const unsigned hmask = 0xFFFFu << (16 * h);
    const bool own = l < n;
    const double gdiag = l < W ? G[l * kGS + l] : 0.0;
    finite = (__ballot_sync(0xffffffffu, isfinite(gdiag)) & hmask) == hmask;

    // ---- Step 3: omega = (G0 + eps I)^{-1} beta, Gauss-Jordan in registers.
    double tr = half_sum(own && finite ? gdiag : 0.0);
    double e = (p.flags & ASP_EPS_ABSOLUTE) ? (double)p.eps : (double)p.eps * (tr / n);
    if (e == 0.0) e = 1e-30;                                           // reading R7
    // (a non-finite window solves the identity system instead, so no NaN or
    // inf flows through the shared arithmetic below; its output is the
    // passthrough either way)
    const bool sys = own && finite;
    double r[16];
#pragma unroll
    for (int k = 0; k < 16; k++)
        r[k] = sys ? (k < n ? G[l * kGS + k] + (k == l ? e : 0.0) : 0.0) : (k == l ? 1.0 : 0.0);
    double rb = sys ? G[n * kGS + l] : 0.0;                             // beta_l = (H y)_l
    bool pd = true;
    double diag = 1.0;
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const double d = shfl16(r[j], j);
        const double pb = shfl16(rb, j);
        const bool good = d > 0.0 && d < INFINITY;                     // SPD: pivots > 0
        pd = pd && good;
        const double f = l != j ? r[j] * rcp_nr1(good ? d : 1.0) : 0.0; // the pivot row stays
        diag = l == j ? d : diag;
#pragma unroll
        for (int k = j + 1; k < 16; k++) r[k] = fma(-f, shfl16(r[k], j), r[k]);
        rb = fma(-f, pb, rb);
    }
    const double x = own ? rb * rcp_nr(diag) : 0.0;
    // (the ballot runs on every lane: never behind a short-circuit)
    const unsigned solved = __ballot_sync(0xffffffffu, pd && (!own || isfinite(x)));
    ok = finite && (solved & hmask) == hmask;

    // ---- Steps 4-6: coefficients c_p of q_hat = sum_p c_p Q[p] / m;
    // lane l holds c_{l+1} (c_0 = 0 in both assemblies).
    const double sgn = (p.flags & ASP_SIGN_NEGATED) ? -1.0 : 1.0;
    const uint32_t mode = p.flags & 0xFu;
    c = 0.0;
    denom = 1.0;
    if (mode == ASP_ASSEMBLY_SINGLE) {
        // Eq. 4: omega[i] (history row i) weights Q[i+1].
        const double w = (p.flags & ASP_NORM_NONE) ? x : half_softmax(sgn * x, l, n);
        c = own ? w : 0.0;
    } else {
        // masked-shared (readings R4-R6): row j = 1..W uses softmax(v[0..n_j)),
        // n_j = min(j, n), on the newest n_j queries; rows W-1 and W share n_j = n.
        double v = sgn * x;
        if (p.flags & ASP_DOUBLE_SOFTMAX) v = half_softmax(v, l, n);    // literal Step 3
        const double m = half_max(own ? v : -INFINITY);
        const double ev = own ? exp(v - m) : 0.0;
        double S = ev;                                                // inclusive prefix: S_{l+1}
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const double t = shfl16_up(S, o);
            if (l >= o) S += t;
        }
        const double invS = rcp_nr(S > 0.0 ? S : 1.0);
        const bool tiny = (__ballot_sync(0xffffffffu, l == 0 && !(S > 1e-280)) & hmask) != 0;
        const bool tiny_any = __any_sync(0xffffffffu, tiny);           // warp-uniform
        double c2 = 0.0;
#pragma unroll
        for (int mm = 1; mm < 16; mm++) {
            if (mm > n) break;                                        // n is warp-uniform
            const unsigned sh = (unsigned)(n - mm);
            double t = ev * shfl16(invS, mm - 1);
            if (mm == n) t *= 2.0;
            const double u = shfl16_up(t, sh);
            if (l >= (int)sh && own) {
                if (mm & 1) c += u;
                else c2 += u;
            }
        }
        if (tiny_any) {
            // a prefix's exponentials underflowed against the global max: redo
            // the half that needs it with each prefix's own max (rolled -- rare,
            // and kept out of the hot straight-line code)
            double ct = 0.0;
#pragma unroll 1
            for (int mm = 1; mm <= n; mm++) {
                const unsigned sh = (unsigned)(n - mm);
                const double mx = half_max(l < mm ? v : -INFINITY);
                const double ex = l < mm ? exp(v - mx) : 0.0;
                double t = ex / half_sum(ex);
                if (mm == n) t *= 2.0;
                const double u = shfl16_up(t, sh);
                if (l >= (int)sh && own) ct += u;
            }
            if (tiny) {
                c = ct;
                c2 = 0.0;
            }
        }
        c += c2;
        denom = (double)W;
    }

}


template <int D, int NB, bool BF>
__global__ void __launch_bounds__(kPairWarps * 32)
predict_pair_kernel(asp_predict_params p, const float *__restrict__ q_window,
                    float *__restrict__ q_hat, uint32_t *dev_flags) {
    extern __shared__ double sG_raw[];
    double (*sG)[2][16 * kGS] = reinterpret_cast<double (*)[2][16 * kGS]>(sG_raw);
    const int W = p.window, n = W - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long rows = (long)p.batch * p.n_q_heads;
    const long row0 = ((long)blockIdx.x * (blockDim.x >> 5) + warp) * 2;
    // The window is read before the programmatic-dependent-launch wait: its only
    // writer in the library, asyncspade_append, does not trigger its dependents
    // early, so a kernel after it starts only once it has completed (and a
    // caller's own kernels never trigger early).  q_hat / the flags are written
    // after the wait (the previous step's kernels may still run).
    asp::pdl_trigger();
    if (row0 >= rows) return;
    const bool has1 = row0 + 1 < rows;
    const int rs = p.ring_start;
#ifdef ASP_PROFILE_PREDICT
    long long _tp = clock64();
#endif
    auto phys_of = [&](int i) {
        const int ph = i + rs;
        return ph >= W ? ph - W : ph;
    };

    // ---- Step 2: augmented Gram G' = Q Q^T of both rows, fp64 MMA.
    {
        const int fr = lane >> 2, fc = lane & 3;
        constexpr int T = NB * (NB + 1) / 2;
        double acc[2][T][2], acc2[2][T][2];             // even / odd groups: shorter chains
#pragma unroll
        for (int r = 0; r < 2; r++)
#pragma unroll
            for (int t = 0; t < T; t++) acc[r][t][0] = acc[r][t][1] = acc2[r][t][0] = acc2[r][t][1] = 0.0;
        int rp[2][NB];                                  // element offsets (-1: padding;
#pragma unroll                                          //  the window is < 2^31 elements)
        for (int r = 0; r < 2; r++)
#pragma unroll
            for (int b = 0; b < NB; b++) {
                const int i = 8 * b + fr;
                const bool live = i < W && (r == 0 || has1);
                rp[r][b] = live ? ((int)row0 + r) * W * D + phys_of(i) * D + 4 * fc : -1;
            }
        // software-pipelined: the next two groups' fragments are in flight while
        // this pair's MMAs run (the loads, not the MMAs, set the latency).  The
        // loop stays rolled: at small row counts instruction fetch of long
        // straight-line code, not arithmetic, is what a warp waits on.
        auto load = [&](float4 (&f)[2][2][NB], int s) {
#pragma unroll
            for (int hh = 0; hh < 2; hh++)
#pragma unroll
                for (int r = 0; r < 2; r++)
#pragma unroll
                    for (int b = 0; b < NB; b++)
                        f[hh][r][b] = rp[r][b] >= 0 ? ld4<BF>(q_window, rp[r][b] + 16 * (s + hh))
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        float4 fa[2][2][NB], fb[2][2][NB];
        load(fa, 0);
#pragma unroll 1
        for (int s = 0; s < D / 16; s += 2) {
            if (s + 2 < D / 16) load(fb, s + 2);
            // each fragment element converted to fp64 once
            double x[2][2][NB][4];
#pragma unroll
            for (int hh = 0; hh < 2; hh++)
#pragma unroll
                for (int r = 0; r < 2; r++)
#pragma unroll
                    for (int b = 0; b < NB; b++) {
                        x[hh][r][b][0] = (double)fa[hh][r][b].x;
                        x[hh][r][b][1] = (double)fa[hh][r][b].y;
                        x[hh][r][b][2] = (double)fa[hh][r][b].z;
                        x[hh][r][b][3] = (double)fa[hh][r][b].w;
                    }
            // k-step j of group s pairs d = 16 s + 4 fc + j in both operands
#pragma unroll
            for (int j = 0; j < 4; j++)
#pragma unroll
                for (int hh = 0; hh < 2; hh++)
#pragma unroll
                    for (int r = 0; r < 2; r++) {
                        int t = 0;
#pragma unroll
                        for (int bi = 0; bi < NB; bi++)
#pragma unroll
                            for (int bj = bi; bj < NB; bj++, t++) {
                                double *c = hh ? acc2[r][t] : acc[r][t];
                                dmma(c[0], c[1], x[hh][r][bi][j], x[hh][r][bj][j]);
                            }
                    }
#pragma unroll
            for (int hh = 0; hh < 2; hh++)
#pragma unroll
                for (int r = 0; r < 2; r++)
#pragma unroll
                    for (int b = 0; b < NB; b++) fa[hh][r][b] = fb[hh][r][b];
        }
#pragma unroll
        for (int r = 0; r < 2; r++)
#pragma unroll
            for (int t = 0; t < T; t++) {
                acc[r][t][0] += acc2[r][t][0];
                acc[r][t][1] += acc2[r][t][1];
            }
        // lane holds C[8 bi + fr][8 bj + 2 fc + e]
#pragma unroll
        for (int r = 0; r < 2; r++) {
            int t = 0;
#pragma unroll
            for (int bi = 0; bi < NB; bi++)
#pragma unroll
                for (int bj = bi; bj < NB; bj++, t++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int i = 8 * bi + fr, j = 8 * bj + 2 * fc + e;
                        if (i < W && j < W) {
                            sG[warp][r][i * kGS + j] = acc[r][t][e];
                            sG[warp][r][j * kGS + i] = acc[r][t][e];
                        }
                    }
        }
    }
    __syncwarp();
    PPROF(0);

    // ---- from here each half-warp owns one row: h = row, l = lane within the half
    const int h = lane >> 4, l = lane & 15;
    double c, denom;
    bool ok, finite;
    solve_coeffs(p, sG[warp][h], W, c, denom, ok, finite);
    PPROF(1);
    PPROF(2);
    // ---- q_hat = (1/m) sum_p c_p Q[p] (one pass over the cache-hot window), or
    // the passthrough Q_t.
    const bool live = h == 0 || has1;
    const int src = ((int)row0 + h) * W * D;                           // element offset
    float *out = q_hat + (size_t)(row0 + h) * D;
    constexpr int kV = D / 64;                                          // float4 per lane
    // (all lanes run the loop -- its shuffles span both halves -- even when a
    // half falls back to the passthrough)
    double acc[kV][4], acc2[kV][4];
#pragma unroll
    for (int u = 0; u < kV; u++)
#pragma unroll
        for (int z = 0; z < 4; z++) acc[u][z] = acc2[u][z] = 0.0;
    auto axpy = [&](double (&a)[kV][4], int q) {
        const double cq = shfl16(c, q - 1);
        const int rq = src + phys_of(q) * D + 4 * l;
#pragma unroll
        for (int u = 0; u < kV; u++) {
            const float4 v4 = live ? ld4<BF>(q_window, rq + 64 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
            a[u][0] = fma(cq, (double)v4.x, a[u][0]);
            a[u][1] = fma(cq, (double)v4.y, a[u][1]);
            a[u][2] = fma(cq, (double)v4.z, a[u][2]);
            a[u][3] = fma(cq, (double)v4.w, a[u][3]);
        }
    };
    int q = 1;
    for (; q + 1 < W; q += 2) {
        axpy(acc, q);
        axpy(acc2, q + 1);
    }
    if (q < W) axpy(acc, q);
#pragma unroll
    for (int u = 0; u < kV; u++)
#pragma unroll
        for (int z = 0; z < 4; z++) acc[u][z] += acc2[u][z];
    asp::pdl_wait();
    if (live && ok) {
        const double inv_m = 1.0 / denom;
#pragma unroll
        for (int u = 0; u < kV; u++)
            reinterpret_cast<float4 *>(out)[l + 16 * u] =
                make_float4((float)(acc[u][0] * inv_m), (float)(acc[u][1] * inv_m),
                            (float)(acc[u][2] * inv_m), (float)(acc[u][3] * inv_m));
    } else if (live) {
        const int rq = src + phys_of(W - 1) * D + 4 * l;
#pragma unroll
        for (int u = 0; u < kV; u++) reinterpret_cast<float4 *>(out)[l + 16 * u] = ld4<BF>(q_window, rq + 64 * u);
        if (l == 0) asp::flag_or(dev_flags, finite ? ASP_FLAG_NOT_PD : ASP_FLAG_NONFINITE);
    }
    PPROF(3);
}

// Few rows (a KV-head shard, small batches): a row pair per CTA of kSplit
// warps, the head dimension sliced over the warps.  Each warp loads its slice
// of both windows ONCE, all at once (<= 8 float4 per lane in flight), keeps
// it in registers for the weighted sum, and runs its slice of the Gram on the
// fp64 tensor cores; the partial Grams are summed in smem in warp order
// (deterministic), warp 0 solves both rows (solve_coeffs), and every warp
// writes its slice of q_hat.  The latency chain is one DRAM round trip plus
// the solve, instead of a row pair's whole window streamed through one warp.
// kSplit warps: 4 (D = 64 / 128 / 256), 12 for the 576-dim absorbed-MLA query
// (three 16-dim groups per warp; the partial Grams then need dynamic smem).
template <int D>
constexpr int split_warps() { return D == 576 ? 12 : 4; }

template <int D, int NB, bool BF>
__global__ void __launch_bounds__(split_warps<D>() * 32)
predict_split_kernel(asp_predict_params p, const float *__restrict__ q_window,
                     float *__restrict__ q_hat, uint32_t *dev_flags) {
    constexpr int kSplit = split_warps<D>();
    constexpr int kG = D / (16 * kSplit);               // 16-dim groups per warp (2, 1 or 3)
    static_assert(kG * 16 * kSplit == D, "head-dim slices");
    constexpr int T = NB * (NB + 1) / 2;
    extern __shared__ double sP_raw[];
    double (*sP)[2][16 * kGS] = reinterpret_cast<double (*)[2][16 * kGS]>(sP_raw);   // partial Grams
    __shared__ double sC[2][16];                       // c_{l+1} per row
    __shared__ double sDen[2];
    __shared__ int sOk[2];
    const int W = p.window;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long rows = (long)p.batch * p.n_q_heads;
    const long row0 = (long)blockIdx.x * 2;
    asp::pdl_trigger();              // window read before the wait: see predict_pair_kernel
    const bool has1 = row0 + 1 < rows;
    const int rs = p.ring_start;
#ifdef ASP_PROFILE_PREDICT
    long long _tp = clock64();
#endif
    auto phys_of = [&](int i) {
        const int ph = i + rs;
        return ph >= W ? ph - W : ph;
    };
    const int fr = lane >> 2, fc = lane & 3;
    // this lane's fragment rows i = 8 b + fr (logical) of both windows, dims
    // 16 (warp kG + g) + 4 fc + j of this warp's slice
    float4 f[2][NB][kG];
#pragma unroll
    for (int r = 0; r < 2; r++)
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const int i = 8 * b + fr;
            const bool live = i < W && (r == 0 || has1);
            const int base = ((int)row0 + r) * W * D + phys_of(i < W ? i : 0) * D + 4 * fc;
#pragma unroll
            for (int g = 0; g < kG; g++)
                f[r][b][g] = live ? ld4<BF>(q_window, base + 16 * (warp * kG + g))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    // ---- Step 2: this slice's share of G' = Q Q^T, fp64 MMA
    double acc[2][T][2];
#pragma unroll
    for (int r = 0; r < 2; r++)
#pragma unroll
        for (int t = 0; t < T; t++) acc[r][t][0] = acc[r][t][1] = 0.0;
#pragma unroll
    for (int g = 0; g < kG; g++)
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int r = 0; r < 2; r++) {
                double x[NB];
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    const float4 v = f[r][b][g];
                    x[b] = (double)(j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w);
                }
                int t = 0;
#pragma unroll
                for (int bi = 0; bi < NB; bi++)
#pragma unroll
                    for (int bj = bi; bj < NB; bj++, t++) dmma(acc[r][t][0], acc[r][t][1], x[bi], x[bj]);
            }
#pragma unroll
    for (int r = 0; r < 2; r++) {
        int t = 0;
#pragma unroll
        for (int bi = 0; bi < NB; bi++)
#pragma unroll
            for (int bj = bi; bj < NB; bj++, t++)
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int i = 8 * bi + fr, j = 8 * bj + 2 * fc + e;
                    if (i < W && j < W) {
                        sP[warp][r][i * kGS + j] = acc[r][t][e];
                        sP[warp][r][j * kGS + i] = acc[r][t][e];
                    }
                }
    }
    PPROF(0);
    __syncthreads();
    // sum the slices in warp order into sP[0]
    for (int x = threadIdx.x; x < 2 * 16 * kGS; x += kSplit * 32) {
        double v = (&sP[0][0][0])[x];
#pragma unroll
        for (int w = 1; w < kSplit; w++) v += (&sP[w][0][0])[x];
        (&sP[0][0][0])[x] = v;
    }
    __syncthreads();
    PPROF(4);
    // ---- Steps 3-6: warp 0 solves both rows (one per half-warp)
    if (warp == 0) {
        const int h = lane >> 4, l = lane & 15;
        double c, denom;
        bool ok, finite;
        solve_coeffs(p, sP[0][h], W, c, denom, ok, finite);
        sC[h][l] = c;
        if (l == 0) {
            sDen[h] = denom;
            sOk[h] = ok ? 1 : (finite ? 2 : 3);        // 2: not PD, 3: non-finite
        }
    }
    __syncthreads();
    PPROF(1);
    asp::pdl_wait();                 // q_hat / flags written from here on
    PPROF(2);
    // ---- q_hat slice = (1/m) sum_p c_p Q[p]: each lane weights its two rows,
    // the 8 lanes of a column (same fc) reduce by shuffle
#pragma unroll
    for (int r = 0; r < 2; r++) {
        if (r == 1 && !has1) break;
        const int st = sOk[r];
        float *out = q_hat + (size_t)(row0 + r) * D;
        if (st == 1) {
            const double inv_m = 1.0 / sDen[r];
            double cb[NB];
#pragma unroll
            for (int b = 0; b < NB; b++) {
                const int i = 8 * b + fr;                 // logical row; c_0 = 0
                cb[b] = (i >= 1 && i < W) ? sC[r][i - 1] : 0.0;
            }
#pragma unroll
            for (int g = 0; g < kG; g++) {
                double a[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    double v = 0.0;
#pragma unroll
                    for (int b = 0; b < NB; b++) {
                        const float4 q4 = f[r][b][g];
                        v = fma(cb[b], (double)(j == 0 ? q4.x : j == 1 ? q4.y : j == 2 ? q4.z : q4.w), v);
                    }
#pragma unroll
                    for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    a[j] = v;
                }
                if (fr == 0)
                    reinterpret_cast<float4 *>(out + 16 * (warp * kG + g))[fc] =
                        make_float4((float)(a[0] * inv_m), (float)(a[1] * inv_m),
                                    (float)(a[2] * inv_m), (float)(a[3] * inv_m));
            }
        } else {                                          // passthrough Q_t
            const int q_off = ((int)row0 + r) * W * D + phys_of(W - 1) * D;
            for (int d4 = threadIdx.x; d4 < D / 4; d4 += kSplit * 32)
                reinterpret_cast<float4 *>(out)[d4] = ld4<BF>(q_window, q_off + 4 * d4);
            if (threadIdx.x == 0) asp::flag_or(dev_flags, st == 2 ? ASP_FLAG_NOT_PD : ASP_FLAG_NONFINITE);
        }
    }
    PPROF(3);
}

template <int D, int NB>
cudaError_t launch_split(const asp_predict_params &p, const float *q_window, float *q_hat,
                         uint32_t *dev_flags, cudaStream_t s) {
    auto kern = (p.flags & ASP_WINDOW_BF16) ? predict_split_kernel<D, NB, true>
                                            : predict_split_kernel<D, NB, false>;
    const long rows = (long)p.batch * p.n_q_heads;
    constexpr int kSplit = split_warps<D>();
    const int smem = (int)(sizeof(double) * kSplit * 2 * 16 * kGS);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    return asp_launch(kern, dim3((unsigned)((rows + 1) / 2)), dim3(kSplit * 32), smem, s, 1, p,
                      q_window, q_hat, dev_flags);
}

template <int D, int NB>
cudaError_t launch_pair(const asp_predict_params &p, const float *q_window, float *q_hat,
                        uint32_t *dev_flags, cudaStream_t s) {
    auto kern = (p.flags & ASP_WINDOW_BF16) ? predict_pair_kernel<D, NB, true>
                                            : predict_pair_kernel<D, NB, false>;
    const long rows = (long)p.batch * p.n_q_heads;
    const long warps = (rows + 1) / 2;
    // as many CTAs as it takes to cover the SMs twice before packing 8 warps each
    const long target = 2L * asp_sm_count();
    int wpc = 1;
    while (wpc < kPairWarps && (warps + 2 * wpc - 1) / (2 * wpc) >= target) wpc *= 2;
    const unsigned grid = (unsigned)((warps + wpc - 1) / wpc);
    const size_t smem = (size_t)wpc * 2 * 16 * kGS * sizeof(double);
    return asp_launch(kern, dim3(grid), dim3(wpc * 32), smem, s, 1, p,
                      q_window, q_hat, dev_flags);
}

template <int D, int NB>
cudaError_t launch(const asp_predict_params &p, const float *q_window, float *q_hat,
                   uint32_t *dev_flags, cudaStream_t s) {
    const long rows = (long)p.batch * p.n_q_heads;
    // rows per CTA: kWarps, or fewer so that few rows (absorbed MLA's 256, say)
    // still spread over twice the SMs instead of sharing a few SMs' fp64 pipes
    int wpc = kWarps;
    while (wpc > 1 && (rows + wpc - 1) / wpc < 2L * asp_sm_count()) wpc /= 2;
    const size_t smem = warp_smem_bytes(p.window) * wpc;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(predict_kernel<D, NB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)((rows + wpc - 1) / wpc);
    return asp_launch(predict_kernel<D, NB>, dim3(grid), dim3(wpc * 32), smem, s, 1, p, q_window,
                      q_hat, dev_flags);
}

}  // namespace

cudaError_t asp_launch_predict(const asp_predict_params &p, const float *q_window, float *q_hat,
                               uint32_t *dev_flags, cudaStream_t s) {
    const int nb = (p.window + 7) / 8;
    const uint32_t mode = p.flags & 0xFu;
    const bool small = (long)p.batch * p.n_q_heads * p.window * p.head_dim < (1L << 31);
    if (p.window >= 2 && p.window <= 16 && small &&
        (mode == ASP_ASSEMBLY_MASKED_SHARED || mode == ASP_ASSEMBLY_SINGLE)) {
        // few row pairs: slice the head dimension over a CTA's warps (latency);
        // many: two rows per warp (throughput)
#ifndef ASP_PREDICT_SPLIT_ROWS_PER_SM
#define ASP_PREDICT_SPLIT_ROWS_PER_SM 8
#endif
        const bool split = (long)p.batch * p.n_q_heads < (long)ASP_PREDICT_SPLIT_ROWS_PER_SM * asp_sm_count();
        if (split) {
            if (p.head_dim == 64) return nb == 1 ? launch_split<64, 1>(p, q_window, q_hat, dev_flags, s)
                                                 : launch_split<64, 2>(p, q_window, q_hat, dev_flags, s);
            if (p.head_dim == 128) return nb == 1 ? launch_split<128, 1>(p, q_window, q_hat, dev_flags, s)
                                                  : launch_split<128, 2>(p, q_window, q_hat, dev_flags, s);
            // wide queries (absorbed MLA's 576-dim latent, 256-dim heads): the same
            // slicing over 12 / 4 warps instead of a whole window per warp
            if (p.head_dim == 576) return nb == 1 ? launch_split<576, 1>(p, q_window, q_hat, dev_flags, s)
                                                  : launch_split<576, 2>(p, q_window, q_hat, dev_flags, s);
            if (p.head_dim == 256) return nb == 1 ? launch_split<256, 1>(p, q_window, q_hat, dev_flags, s)
                                                  : launch_split<256, 2>(p, q_window, q_hat, dev_flags, s);
        }
        if (p.head_dim == 64) return nb == 1 ? launch_pair<64, 1>(p, q_window, q_hat, dev_flags, s)
                                             : launch_pair<64, 2>(p, q_window, q_hat, dev_flags, s);
        if (p.head_dim == 128) return nb == 1 ? launch_pair<128, 1>(p, q_window, q_hat, dev_flags, s)
                                              : launch_pair<128, 2>(p, q_window, q_hat, dev_flags, s);
    }
#define ASP_CASE(DD, NBB) \
    if (p.head_dim == DD && nb == NBB) return launch<DD, NBB>(p, q_window, q_hat, dev_flags, s);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 3) ASP_CASE(64, 4)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 3) ASP_CASE(128, 4)
    // absorbed MLA queries (the 576-dim latent + rope space) and 256-dim heads
    ASP_CASE(256, 1) ASP_CASE(256, 2) ASP_CASE(256, 3) ASP_CASE(256, 4)
    ASP_CASE(576, 1) ASP_CASE(576, 2) ASP_CASE(576, 3) ASP_CASE(576, 4)
#undef ASP_CASE
    return cudaErrorInvalidValue;
}
