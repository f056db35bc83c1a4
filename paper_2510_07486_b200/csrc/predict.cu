// predict.cu -- a1: temporal-regressive next-query prediction on sm_100a.
//
// AsyncSpade predicts q_hat_{t+1} from the window of recent query states by a
// softmax-normalised ridge regression applied to the one-step-shifted window
// (Eq. 2-4) assembled over window sizes and average
// pooled (Eq. 5; Alg. 1 Steps 1-6), with the readings
// R1-R8 of DESIGN.md §3 (masked-shared default).  All regression arithmetic
// is fp64 (reading R16).
//
// Design (B200): one warp per (batch, q-head) row, four independent rows per
// CTA, no CTA-wide barriers.
//   * The W x D window is staged once in shared memory (fp32, logical ring
//     order, row stride D+4 so the tensor-core fragment loads are
//     bank-conflict free) with 8 x 16-B loads in flight per lane.
//   * The augmented Gram matrix G' = Q Q^T (W x W) -- the history Gram G0
//     AND beta = H y in its last row -- runs on the fp64 tensor cores
//     (mma.sync m8n8k4 f64), all 8x8 tiles interleaved per k-step.
//   * Cholesky of G0 + eps I is lane-parallel over the rows below each pivot;
//     forward / backward substitution keep the right-hand side in registers
//     (lane j owns component j) and broadcast pivots by shuffle.
//   * The masked-shared weights collapse to W coefficients c_p (one exp per
//     history weight, prefix sums by shuffle; a row-prefix softmax is the
//     prefix's normalised exponentials), so q_hat = sum_p c_p Q[p] / m is one
//     pass over the staged window, rounded once to fp32.
// The step is ~0.7% of the path's bytes ("negligible runtime").
#include "common.cuh"

#include <math.h>

namespace {

constexpr int kWarps = 4;

__host__ __device__ size_t warp_smem_bytes(int W, int D) {
    const int Wp = (W + 7) & ~7;
    const size_t b = (size_t)Wp * (D + 4) * sizeof(float)            // staged window
                     + (size_t)W * W * sizeof(double)                // augmented Gram G'
                     + (size_t)(W > 1 ? (W - 1) * (W - 1) : 1) * sizeof(double)  // Cholesky
                     + (size_t)(64 + 32 + 32) * sizeof(double);      // scratch, exps, coeffs
    return (b + 15) & ~(size_t)15;                                   // next warp: 16-B aligned
}

struct WarpSmem {
    float *win;     // [Wp][D+4]
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

// G' = Q Q^T over the staged window (NB 8-row blocks), fp64 tensor cores.
template <int D, int NB>
__device__ void gram_dmma(const WarpSmem &s, int W) {
    const int lane = threadIdx.x & 31;
    const int fr = lane >> 2, fc = lane & 3;
    constexpr int kTiles = NB * (NB + 1) / 2;
    double acc[kTiles][2];
#pragma unroll
    for (int t = 0; t < kTiles; t++) acc[t][0] = acc[t][1] = 0.0;
    const float *base = s.win + fr * (D + 4) + fc;
#pragma unroll 4
    for (int k = 0; k < D; k += 4) {
        double f[NB];
#pragma unroll
        for (int b = 0; b < NB; b++) f[b] = (double)base[b * 8 * (D + 4) + k];
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
__global__ void __launch_bounds__(kWarps * 32)
predict_kernel(asp_predict_params p, const float *__restrict__ q_window,
               float *__restrict__ q_hat, uint32_t *dev_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int LD = D + 4;
    const int W = p.window, n = W - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long rows = (long)p.batch * p.n_q_heads;
    const long row = (long)blockIdx.x * kWarps + warp;
    if (row >= rows) return;

    unsigned char *base = smem_raw + warp_smem_bytes(W, D) * warp;
    WarpSmem s;
    s.win = reinterpret_cast<float *>(base);
    size_t off = (size_t)NB * 8 * LD * sizeof(float);
    s.G = reinterpret_cast<double *>(base + off);
    off += (size_t)W * W * sizeof(double);
    s.A = reinterpret_cast<double *>(base + off);
    off += (size_t)(W > 1 ? (W - 1) * (W - 1) : 1) * sizeof(double);
    s.vec = reinterpret_cast<double *>(base + off);
    s.e = s.vec + 64;
    s.c = s.e + 32;

    // Step 1: stage the window in logical order (physical slot
    // ring_start + j holds logical j); zero the padding rows.
    const float *src = q_window + (size_t)row * W * D;
    bool finite = true;
    constexpr int kVecsPerRow = D / 4;
    const int vecs = W * kVecsPerRow;
    constexpr int kBatch = 8;
    for (int v0 = 0; v0 < vecs; v0 += 32 * kBatch) {
        float4 x[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; u++) {
            const int v = v0 + u * 32 + lane;
            x[u] = v < vecs ? __ldg(reinterpret_cast<const float4 *>(src) + v)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kBatch; u++) {
            const int v = v0 + u * 32 + lane;
            if (v >= vecs) break;
            const int phys = v / kVecsPerRow, d = (v % kVecsPerRow) * 4;
            int logical = phys - p.ring_start;
            if (logical < 0) logical += W;
            *reinterpret_cast<float4 *>(s.win + logical * LD + d) = x[u];
            finite = finite && isfinite(x[u].x) && isfinite(x[u].y) && isfinite(x[u].z) &&
                     isfinite(x[u].w);
        }
    }
    for (int i = W * LD + lane * 4; i < NB * 8 * LD; i += 128)
        *reinterpret_cast<float4 *>(s.win + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    finite = __all_sync(0xffffffffu, finite);
    s.c[lane] = 0.0;
    __syncwarp();

    float *out = q_hat + (size_t)row * D;
    const uint32_t mode = p.flags & 0xFu;
    const double sgn = (p.flags & ASP_SIGN_NEGATED) ? -1.0 : 1.0;
    const bool absolute = (p.flags & ASP_EPS_ABSOLUTE) != 0;

    bool ok = finite && W > 1;
    double denom = 1.0;
    if (ok) {
        gram_dmma<D, NB>(s, W);
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
            const double om = ridge_solve(s, W, 0, n, p.eps, absolute, ok);
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
    if (ok) {
        const double inv_m = 1.0 / denom;
        for (int d = lane; d < D; d += 32) {
            double acc = 0.0;
            for (int q = 0; q < W; q++) acc = fma(s.c[q], (double)s.win[q * LD + d], acc);
            out[d] = (float)(acc * inv_m);
        }
    } else {
        // Passthrough q_hat = Q_t; flag why.
        for (int d = lane; d < D; d += 32) out[d] = s.win[(W - 1) * LD + d];
        if (lane == 0 && W > 1) asp::flag_or(dev_flags, finite ? ASP_FLAG_NOT_PD : ASP_FLAG_NONFINITE);
    }
}

template <int D, int NB>
cudaError_t launch(const asp_predict_params &p, const float *q_window, float *q_hat,
                   uint32_t *dev_flags, cudaStream_t s) {
    const long rows = (long)p.batch * p.n_q_heads;
    const size_t smem = warp_smem_bytes(p.window, D) * kWarps;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(predict_kernel<D, NB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
    predict_kernel<D, NB><<<grid, kWarps * 32, smem, s>>>(p, q_window, q_hat, dev_flags);
    return cudaGetLastError();
}

}  // namespace

cudaError_t asp_launch_predict(const asp_predict_params &p, const float *q_window, float *q_hat,
                               uint32_t *dev_flags, cudaStream_t s) {
    const int nb = (p.window + 7) / 8;
#define ASP_CASE(DD, NBB) \
    if (p.head_dim == DD && nb == NBB) return launch<DD, NBB>(p, q_window, q_hat, dev_flags, s);
    ASP_CASE(64, 1) ASP_CASE(64, 2) ASP_CASE(64, 3) ASP_CASE(64, 4)
    ASP_CASE(128, 1) ASP_CASE(128, 2) ASP_CASE(128, 3) ASP_CASE(128, 4)
#undef ASP_CASE
    return cudaErrorInvalidValue;
}
