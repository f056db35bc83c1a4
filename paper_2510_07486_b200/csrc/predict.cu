// predict.cu -- a1: temporal-regressive next-query prediction on sm_100a.
//
// AsyncSpade predicts q_hat_{t+1} from the window of recent query states by a
// softmax-normalised ridge regression applied to the one-step-shifted window
// (Eq. 2-4) assembled over window sizes and average
// pooled (Eq. 5; Alg. 1 Steps 1-6), with the readings
// R1-R8 of DESIGN.md §3 (masked-shared default).
//
// Design (B200): one warp per (batch, q-head) row, four rows per CTA.  The
// row's W x D window is staged once into shared memory as fp64 (reading R16:
// fp64 regression; converting once keeps the F2F pipe out of the Gram loop),
// with a padded row stride so lanes reading different rows hit different
// banks.  Then, all lane-parallel:
//   * the (W-1)(W-1) Gram triangle + (W-1) beta dot products, one per lane;
//   * Cholesky, one lane per row below each pivot, reciprocal pivots kept;
//   * forward / backward substitution with the right-hand side in registers
//     (lane j owns component j, pivots broadcast by shuffle);
//   * the masked-shared weights collapse to W coefficients c_p: one exp per
//     history weight (shifted by the global max), prefix sums by shuffle,
//     c_p = (1/W) sum_m mult(m) e_{p-W+m} / S_m  (a row-prefix softmax is the
//     prefix's normalised exponentials); if a prefix sum underflows the rows
//     fall back to per-row max-shifted softmaxes;
//   * q_hat = sum_p c_p Q[p] / m, lanes over d, rounded once to fp32.
// The step is ~0.7% of the path's bytes ("negligible runtime").
#include "common.cuh"

#include <math.h>

namespace {

constexpr int kWarps = 4;

struct WarpSmem {
    double *win;    // [W][D+1] fp64, logical order
    double *A;      // [n][n] Gram / Cholesky factor (lower)
    double *vec;    // [64] scratch
    double *e;      // [32] exponentials / scratch
    double *c;      // [32] collapsed coefficients
};

__host__ __device__ size_t warp_smem_bytes(int W, int D) {
    const int n = W - 1;
    return (size_t)W * (D + 1) * sizeof(double) + (size_t)(n > 0 ? n * n : 1) * sizeof(double) +
           (64 + 32 + 32) * sizeof(double);
}

__device__ __forceinline__ double shfl_d(double v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}

// Ridge solve over history rows [h0, h0 + nh) of the staged window with the
// newest row W-1 as target (Alg. 1 Step 3):
//   omega = (G0 + eps I)^{-1} beta,  G0 = H H^T,  beta = H y.
// Returns omega_lane (lane i < nh holds omega_i) and ok (warp-uniform).
__device__ double ridge_solve(const WarpSmem &s, int W, int D, int h0, int nh, float eps,
                              bool absolute, bool &ok) {
    const int lane = threadIdx.x & 31;
    const int ld = D + 1;
    const double *y = s.win + (size_t)(W - 1) * ld;
    double *A = s.A;
    const int tri = nh * (nh + 1) / 2;
    // Gram triangle (unit u -> (i, j), i <= j) and beta, one dot product per lane-unit
    for (int u = lane; u < tri + nh; u += 32) {
        const double *a, *b;
        int i = 0, j = 0;
        if (u < tri) {
            int v = u;
            while (v >= nh - i) { v -= nh - i; i++; }
            j = i + v;
            a = s.win + (size_t)(h0 + i) * ld;
            b = s.win + (size_t)(h0 + j) * ld;
        } else {
            i = u - tri;
            a = s.win + (size_t)(h0 + i) * ld;
            b = y;
        }
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 8
        for (int d = 0; d < D; d += 2) {
            acc0 = fma(a[d], b[d], acc0);
            acc1 = fma(a[d + 1], b[d + 1], acc1);
        }
        const double acc = acc0 + acc1;
        if (u < tri) {
            A[i * nh + j] = acc;
            A[j * nh + i] = acc;
        } else {
            s.e[i] = acc;                         // beta staged through smem
        }
    }
    __syncwarp();
    const double beta_lane = lane < nh ? s.e[lane] : 0.0;
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
    // Cholesky G = L L^T, lane-parallel over rows below the pivot.
    double inv_d_lane = 0.0;
    ok = true;
    for (int j = 0; j < nh; j++) {
        double sjj = A[j * nh + j];
        for (int k = 0; k < j; k++) sjj = fma(-A[j * nh + k], A[j * nh + k], sjj);
        if (!(sjj > 0.0) || !isfinite(sjj)) { ok = false; break; }   // warp-uniform
        const double dj = sqrt(sjj);
        const double inv = 1.0 / dj;
        if (lane == j) inv_d_lane = inv;
        const int i = j + 1 + lane;
        double t = 0.0;
        if (i < nh) {
            t = A[i * nh + j];
            for (int k = 0; k < j; k++) t = fma(-A[i * nh + k], A[j * nh + k], t);
        }
        __syncwarp();
        if (i < nh) A[i * nh + j] = t * inv;
        if (lane == 0) A[j * nh + j] = dj;
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
    // inclusive prefix sums S_{lane+1} = sum_{i <= lane} e_i
    double S = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, S, o);
        if (lane >= o) S += t;
    }
    s.e[lane] = e;
    s.vec[32 + lane] = S;                         // S_m for m = lane + 1
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
                acc += mult * s.e[p - W + mm] / s.vec[32 + mm - 1];
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

__global__ void __launch_bounds__(kWarps * 32)
predict_kernel(asp_predict_params p, const float *__restrict__ q_window,
               float *__restrict__ q_hat, uint32_t *dev_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int W = p.window, D = p.head_dim, n = W - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long rows = (long)p.batch * p.n_q_heads;
    const long row = (long)blockIdx.x * kWarps + warp;
    if (row >= rows) return;

    unsigned char *base = smem_raw + warp_smem_bytes(W, D) * warp;
    WarpSmem s;
    s.win = reinterpret_cast<double *>(base);
    size_t off = (size_t)W * (D + 1) * sizeof(double);
    s.A = reinterpret_cast<double *>(base + off);
    off += (size_t)(n > 0 ? n * n : 1) * sizeof(double);
    s.vec = reinterpret_cast<double *>(base + off);
    s.e = s.vec + 64;
    s.c = s.e + 32;

    // Step 1: stage the window in logical order, fp32 -> fp64 once.
    const float *src = q_window + (size_t)row * W * D;
    bool finite = true;
    const int vecs = W * D / 4;
    for (int v = lane; v < vecs; v += 32) {
        const int phys = (v * 4) / D, d = (v * 4) - phys * D;
        const int logical = ((phys - p.ring_start) % W + W) % W;
        const float4 x = __ldg(reinterpret_cast<const float4 *>(src) + v);
        double *dst = s.win + (size_t)logical * (D + 1) + d;
        dst[0] = x.x; dst[1] = x.y; dst[2] = x.z; dst[3] = x.w;
        finite = finite && isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w);
    }
    finite = __all_sync(0xffffffffu, finite);
    s.c[lane] = 0.0;
    __syncwarp();

    float *out = q_hat + (size_t)row * D;
    const double *newest = s.win + (size_t)(W - 1) * (D + 1);
    const uint32_t mode = p.flags & 0xFu;
    const double sgn = (p.flags & ASP_SIGN_NEGATED) ? -1.0 : 1.0;
    const bool absolute = (p.flags & ASP_EPS_ABSOLUTE) != 0;

    bool ok = finite && W > 1;
    double denom = 1.0;
    if (ok) {
        if (mode == ASP_ASSEMBLY_PER_WINDOW) {
            // Eq. 5 literal: one solve per window size k = 1..n on Q[W-1-k..W-2],
            // softmax weights applied to Q[W-k..W-1]; m = n.
            double cacc = 0.0;                        // lane p accumulates c_p
            for (int k = 1; k <= n && ok; k++) {
                const double om = ridge_solve(s, W, D, W - 1 - k, k, p.eps, absolute, ok);
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
            const double om = ridge_solve(s, W, D, 0, n, p.eps, absolute, ok);
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
        for (int d = lane; d < D; d += 32) {
            double acc = 0.0;
            for (int q = 0; q < W; q++) acc = fma(s.c[q], s.win[(size_t)q * (D + 1) + d], acc);
            out[d] = (float)(acc / denom);
        }
    } else {
        // Passthrough q_hat = Q_t; flag why.
        for (int d = lane; d < D; d += 32) out[d] = (float)newest[d];
        if (lane == 0 && W > 1) asp::flag_or(dev_flags, finite ? ASP_FLAG_NOT_PD : ASP_FLAG_NONFINITE);
    }
}

}  // namespace

cudaError_t asp_launch_predict(const asp_predict_params &p, const float *q_window, float *q_hat,
                               uint32_t *dev_flags, cudaStream_t s) {
    const long rows = (long)p.batch * p.n_q_heads;
    const size_t smem = warp_smem_bytes(p.window, p.head_dim) * kWarps;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(predict_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
    predict_kernel<<<grid, kWarps * 32, smem, s>>>(p, q_window, q_hat, dev_flags);
    return cudaGetLastError();
}
