// predict.cu -- a1: temporal-regressive next-query prediction on sm_100a.
//
// AsyncSpade predicts q_hat_{t+1} from the window of recent query states by a
// softmax-normalised ridge regression applied to the one-step-shifted window
// (Eq. 2-4) assembled over window sizes and average
// pooled (Eq. 5; Alg. 1 Steps 1-6), with the readings
// R1-R8 of DESIGN.md §3 (masked-shared default).
//
// Design (B200): one warp per (batch, q-head) row, four rows per CTA.  The
// row's W x D window is staged once into shared memory (coalesced float4 global
// reads, padded row stride so lanes reading different rows hit different
// banks).  Everything downstream is fp64 (reading R16): lanes split the
// (W-1)(W-1) Gram + (W-1) beta dot products; Cholesky is lane-parallel over
// rows of each column; the masked-shared rows' softmaxes run one per lane; the
// result is collapsed to W coefficients c_p so q_hat = sum_p c_p Q[p] / m is
// a single pass over the window.  The step is ~0.7% of the path's bytes and
// well under 100 M DFMA at the Qwen3-32B shape ("negligible runtime").
#include "common.cuh"

#include <math.h>

namespace {

constexpr int kWarps = 4;
constexpr int kMaxW = 32;

struct WarpSmem {
    float *win;     // [W][D+1] fp32, logical order
    double *A;      // [n][n] Gram / Cholesky factor
    double *vec;    // beta / omega scratch [64]
    double *r;      // [W][n] per-row softmax weights
    double *c;      // [W] collapsed coefficients
};

__device__ size_t warp_smem_bytes(int W, int D) {
    const int n = W - 1;
    size_t b = (size_t)W * (D + 1) * sizeof(float);
    b = (b + 15) & ~(size_t)15;
    b += (size_t)(n > 0 ? n * n : 1) * sizeof(double);
    b += 64 * sizeof(double);
    b += (size_t)W * (n > 0 ? n : 1) * sizeof(double);
    b += (size_t)kMaxW * sizeof(double);
    return b;
}

// Ridge solve over history rows [h0, h0 + nh) of the staged window with the
// newest row W-1 as target (Alg. 1 Step 3).  Result omega[0..nh)
// in s.vec.  Returns true (warp-uniform) if the matrix was positive definite.
__device__ bool ridge_solve(const WarpSmem &s, int W, int D, int h0, int nh, float eps,
                            bool absolute) {
    const int lane = threadIdx.x & 31;
    const int ld = D + 1;
    const float *y = s.win + (size_t)(W - 1) * ld;
    double *A = s.A;          // nh x nh, row-major
    double *beta = s.vec;     // reuse: beta then omega (in place)
    const int units = nh * nh + nh;
    for (int u = lane; u < units; u += 32) {
        const float *a, *b;
        int i, j = 0;
        if (u < nh * nh) {
            i = u / nh;
            j = u - i * nh;
            if (j < i) continue;
            a = s.win + (size_t)(h0 + i) * ld;
            b = s.win + (size_t)(h0 + j) * ld;
        } else {
            i = u - nh * nh;
            a = s.win + (size_t)(h0 + i) * ld;
            b = y;
        }
        double acc = 0.0;
        for (int d = 0; d < D; d++) acc = fma((double)a[d], (double)b[d], acc);
        if (u < nh * nh) {
            A[i * nh + j] = acc;
            A[j * nh + i] = acc;
        } else {
            beta[i] = acc;
        }
    }
    __syncwarp();
    // eps: relative to the mean of diag(G0) (reading R7) unless absolute.
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
    // Cholesky, lane-parallel over the rows below each pivot.
    bool ok = true;
    for (int j = 0; j < nh; j++) {
        double sjj = A[j * nh + j];
        for (int k = 0; k < j; k++) sjj -= A[j * nh + k] * A[j * nh + k];
        const bool piv_ok = (sjj > 0.0) && isfinite(sjj);
        if (!piv_ok) { ok = false; break; }        // warp-uniform (same value in every lane)
        const double dj = sqrt(sjj);
        const int i = j + 1 + lane;
        double t = 0.0;
        if (i < nh) {
            t = A[i * nh + j];
            for (int k = 0; k < j; k++) t -= A[i * nh + k] * A[j * nh + k];
        }
        __syncwarp();
        if (i < nh) A[i * nh + j] = t / dj;
        if (lane == 0) A[j * nh + j] = dj;
        __syncwarp();
    }
    if (!ok) return false;
    // Triangular solves (tiny: lane 0), omega overwrites beta.
    if (lane == 0) {
        double yv[kMaxW];
        for (int i = 0; i < nh; i++) {
            double t = beta[i];
            for (int k = 0; k < i; k++) t -= A[i * nh + k] * yv[k];
            yv[i] = t / A[i * nh + i];
        }
        for (int i = nh - 1; i >= 0; i--) {
            double t = yv[i];
            for (int k = i + 1; k < nh; k++) t -= A[k * nh + i] * beta[k];
            beta[i] = t / A[i * nh + i];
        }
    }
    __syncwarp();
    bool fin = true;
    for (int i = 0; i < nh; i++) fin = fin && isfinite(beta[i]);
    return fin;
}

// softmax of v[0..n) (max-subtracted, fp64) into out[0..n).
__device__ void softmax_serial(const double *v, int n, double *out) {
    double m = v[0];
    for (int i = 1; i < n; i++) m = fmax(m, v[i]);
    double sum = 0.0;
    for (int i = 0; i < n; i++) {
        out[i] = exp(v[i] - m);
        sum += out[i];
    }
    for (int i = 0; i < n; i++) out[i] /= sum;
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
    s.win = reinterpret_cast<float *>(base);
    size_t off = ((size_t)W * (D + 1) * sizeof(float) + 15) & ~(size_t)15;
    s.A = reinterpret_cast<double *>(base + off);
    off += (size_t)(n > 0 ? n * n : 1) * sizeof(double);
    s.vec = reinterpret_cast<double *>(base + off);
    off += 64 * sizeof(double);
    s.r = reinterpret_cast<double *>(base + off);
    off += (size_t)W * (n > 0 ? n : 1) * sizeof(double);
    s.c = reinterpret_cast<double *>(base + off);

    // Step 1: stage the window in logical order.
    const float *src = q_window + (size_t)row * W * D;
    bool finite = true;
    const int vecs = W * D / 4;
    for (int v = lane; v < vecs; v += 32) {
        const int phys = (v * 4) / D, d = (v * 4) - phys * D;
        const int logical = ((phys - p.ring_start) % W + W) % W;
        const float4 x = __ldg(reinterpret_cast<const float4 *>(src) + v);
        float *dst = s.win + (size_t)logical * (D + 1) + d;
        dst[0] = x.x; dst[1] = x.y; dst[2] = x.z; dst[3] = x.w;
        finite = finite && isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w);
    }
    finite = __all_sync(0xffffffffu, finite);
    __syncwarp();

    float *out = q_hat + (size_t)row * D;
    const float *newest = s.win + (size_t)(W - 1) * (D + 1);
    const uint32_t mode = p.flags & 0xFu;
    const double sgn = (p.flags & ASP_SIGN_NEGATED) ? -1.0 : 1.0;
    const bool absolute = (p.flags & ASP_EPS_ABSOLUTE) != 0;

    bool ok = finite && W > 1;
    double denom = 1.0;
    if (ok) {
        if (lane < W) s.c[lane] = 0.0;
        __syncwarp();
        if (mode == ASP_ASSEMBLY_PER_WINDOW) {
            // Eq. 5 literal: one solve per window size k = 1..n, m = n.
            for (int k = 1; k <= n && ok; k++) {
                ok = ridge_solve(s, W, D, W - 1 - k, k, p.eps, absolute);
                if (!ok) break;
                if (lane == 0) {
                    double v[kMaxW], r[kMaxW];
                    for (int i = 0; i < k; i++) v[i] = sgn * s.vec[i];
                    softmax_serial(v, k, r);
                    for (int i = 0; i < k; i++) s.c[W - k + i] += r[i];
                }
                __syncwarp();
            }
            denom = (double)n;
        } else {
            ok = ridge_solve(s, W, D, 0, n, p.eps, absolute);
            if (ok && mode == ASP_ASSEMBLY_SINGLE) {
                // Eq. 4: omega[i] (history row i) weights Q[i+1].
                if (lane == 0) {
                    double v[kMaxW], r[kMaxW];
                    if (p.flags & ASP_NORM_NONE) {
                        for (int i = 0; i < n; i++) s.c[i + 1] = s.vec[i];
                    } else {
                        for (int i = 0; i < n; i++) v[i] = sgn * s.vec[i];
                        softmax_serial(v, n, r);
                        for (int i = 0; i < n; i++) s.c[i + 1] = r[i];
                    }
                }
                __syncwarp();
                denom = 1.0;
            } else if (ok) {
                // Masked-shared (Alg. 1 Steps 4-6; R4-R6).  Row j = 1..W keeps the
                // first n_j = min(j, n) weights, softmaxed over just those, and
                // applies them to Q[W-n_j .. W-1]; m = W.
                if (lane == 0) {
                    for (int i = 0; i < n; i++) s.vec[32 + i] = sgn * s.vec[i];
                    if (p.flags & ASP_DOUBLE_SOFTMAX) {
                        double tmp[kMaxW];
                        softmax_serial(s.vec + 32, n, tmp);
                        for (int i = 0; i < n; i++) s.vec[32 + i] = tmp[i];
                    }
                }
                __syncwarp();
                if (lane < W) {
                    const int j = lane + 1, nj = j < n ? j : n;
                    softmax_serial(s.vec + 32, nj, s.r + (size_t)lane * n);
                }
                __syncwarp();
                // c_p = sum_j r_j[p - W + n_j] over rows with n_j >= W - p (fixed order).
                if (lane < W) {
                    const int pidx = lane;
                    double acc = 0.0;
                    for (int j = 1; j <= W; j++) {
                        const int nj = j < n ? j : n;
                        const int i = pidx - W + nj;
                        if (i >= 0) acc += s.r[(size_t)(j - 1) * n + i];
                    }
                    s.c[pidx] = acc;
                }
                __syncwarp();
                denom = (double)W;
            }
        }
    }
    if (ok) {
        for (int d = lane; d < D; d += 32) {
            double acc = 0.0;
            for (int q = 0; q < W; q++) acc = fma(s.c[q], (double)s.win[(size_t)q * (D + 1) + d], acc);
            out[d] = (float)(acc / denom);
        }
    } else {
        // Passthrough q_hat = Q_t; flag why.
        for (int d = lane; d < D; d += 32) out[d] = newest[d];
        if (lane == 0 && W > 1) asp::flag_or(dev_flags, finite ? ASP_FLAG_NOT_PD : ASP_FLAG_NONFINITE);
    }
}

size_t host_warp_smem_bytes(int W, int D) {
    const int n = W - 1;
    size_t b = (size_t)W * (D + 1) * sizeof(float);
    b = (b + 15) & ~(size_t)15;
    b += (size_t)(n > 0 ? n * n : 1) * sizeof(double);
    b += 64 * sizeof(double);
    b += (size_t)W * (n > 0 ? n : 1) * sizeof(double);
    b += (size_t)kMaxW * sizeof(double);
    return b;
}

}  // namespace

cudaError_t asp_launch_predict(const asp_predict_params &p, const float *q_window, float *q_hat,
                               uint32_t *dev_flags, cudaStream_t s) {
    const long rows = (long)p.batch * p.n_q_heads;
    const size_t smem = host_warp_smem_bytes(p.window, p.head_dim) * kWarps;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
    predict_kernel<<<grid, kWarps * 32, smem, s>>>(p, q_window, q_hat, dev_flags);
    return cudaGetLastError();
}
