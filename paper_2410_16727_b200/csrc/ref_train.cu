// Training step of the reference profile's denoiser (planseed/diffusion.py:357-508: _batch_loss,
// loss_eq2, train; planseed/autodiff.py: the ops' backward rules and Adam), float64 on the GPU.
// The host (paper_2410_16727_b200/ref/train.py) sequences the forward pass, keeps the activations,
// runs the backward pass through the same layers in reverse and applies Adam; the kernels here are
// the layer-level building blocks: a tiled fp64 GEMM with transposes (linear layers forward and
// backward), bias / activation / FiLM forward+backward, the strided valid-mode conv1d of the scan
// encoder forward+backward, the FK-weighted + plain noise MSE with its gradient, and the Adam update.
#include <cstdint>

#include "common.cuh"

namespace {

constexpr int GT = 16;   // GEMM tile

// C[M x N] = alpha * op(A)[M x K] op(B)[K x N] + (accumulate ? C : 0), row-major with leading dims;
// op(A)(i, k) = TA ? A[k * lda + i] : A[i * lda + k], op(B)(k, j) = TB ? B[j * ldb + k] : B[k * ldb + j]
__global__ void gemm_f64_kernel(const double* __restrict__ A, int lda, int TA, const double* __restrict__ B, int ldb,
                                int TB, double* __restrict__ C, int ldc, int M, int N, int K, int accumulate) {
    __shared__ double sa[GT][GT + 1], sb[GT][GT + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int i = blockIdx.y * GT + ty, j = blockIdx.x * GT + tx;
    double acc = 0.0;
    for (int k0 = 0; k0 < K; k0 += GT) {
        const int ka = k0 + tx, kb = k0 + ty;
        sa[ty][tx] = (i < M && ka < K) ? (TA ? A[(size_t)ka * lda + i] : A[(size_t)i * lda + ka]) : 0.0;
        sb[ty][tx] = (kb < K && j < N) ? (TB ? B[(size_t)j * ldb + kb] : B[(size_t)kb * ldb + j]) : 0.0;
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GT; ++kk) acc = fma(sa[ty][kk], sb[kk][tx], acc);
        __syncthreads();
    }
    if (i < M && j < N) {
        double* c = C + (size_t)i * ldc + j;
        *c = accumulate ? *c + acc : acc;
    }
}

// y = pre = y + b (row broadcast); act 1: y = silu(pre) with pre kept for the backward pass
__global__ void bias_act_kernel(double* __restrict__ y, int ldy, const double* __restrict__ b, int R, int N, int act,
                                double* __restrict__ pre) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (j >= N || r >= R) return;
    const double v = y[(size_t)r * ldy + j] + b[j];
    if (act) {
        pre[(size_t)r * N + j] = v;
        const double s = 1.0 / (1.0 + exp(-v));
        y[(size_t)r * ldy + j] = v * s;
    } else {
        y[(size_t)r * ldy + j] = v;
    }
}

// g <- g * silu'(pre) = g * s (1 + x (1 - s))   (autodiff.py:166-171)
__global__ void silu_bwd_kernel(double* __restrict__ g, int ldg, const double* __restrict__ pre, int R, int N) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (j >= N || r >= R) return;
    const double x = pre[(size_t)r * N + j];
    const double s = 1.0 / (1.0 + exp(-x));
    g[(size_t)r * ldg + j] *= s * (1.0 + x * (1.0 - s));
}

// db (+)= column sums of g (R x N)
__global__ void colsum_kernel(const double* __restrict__ g, int ldg, int R, int N, double* __restrict__ db,
                              int accumulate) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    double s = 0.0;
    for (int r = 0; r < R; ++r) s += g[(size_t)r * ldg + j];
    db[j] = accumulate ? db[j] + s : s;
}

// FiLM: out = a * (1 + sc) + sh (all (R x N)); backward: da = g (1 + sc), dsc = g a, dsh = g
__global__ void film_fwd_kernel(const double* __restrict__ a, const double* __restrict__ sc,
                                const double* __restrict__ sh, int n, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i] * (1.0 + sc[i]) + sh[i];
}
__global__ void film_bwd_kernel(const double* __restrict__ g, const double* __restrict__ a,
                                const double* __restrict__ sc, int n, double* __restrict__ da,
                                double* __restrict__ dsc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    da[i] = g[i] * (1.0 + sc[i]);
    dsc[i] = g[i] * a[i];
}

// valid-mode strided conv1d (B, C, L) x (O, C, K) -> (B, O, Lo) + bias, then silu (pre kept)
__global__ void conv1d_fwd_kernel(const double* __restrict__ x, int B, int C, int L, const double* __restrict__ w,
                                  const double* __restrict__ b, int O, int K, int S, int Lo, double* __restrict__ pre,
                                  double* __restrict__ y) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)B * O * Lo) return;
    const int l = (int)(i % Lo), o = (int)((i / Lo) % O), bb = (int)(i / ((size_t)Lo * O));
    double acc = 0.0;
    for (int c = 0; c < C; ++c)
        for (int k = 0; k < K; ++k) acc = fma(x[((size_t)bb * C + c) * L + l * S + k], w[((size_t)o * C + c) * K + k], acc);
    const double v = acc + b[o];
    pre[i] = v;
    y[i] = v / (1.0 + exp(-v));
}

// conv1d backward: gy (B, O, Lo) -> dw (O, C, K), db (O), gx (B, C, L) (gx optional)
__global__ void conv1d_bwd_w_kernel(const double* __restrict__ gy, const double* __restrict__ x, int B, int C, int L,
                                    int O, int K, int S, int Lo, double* __restrict__ dw, double* __restrict__ db) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < O * C * K) {
        const int k = i % K, c = (i / K) % C, o = i / (K * C);
        double acc = 0.0;
        for (int bb = 0; bb < B; ++bb)
            for (int l = 0; l < Lo; ++l)
                acc = fma(gy[((size_t)bb * O + o) * Lo + l], x[((size_t)bb * C + c) * L + l * S + k], acc);
        dw[i] = acc;
    } else if (i < O * C * K + O) {
        const int o = i - O * C * K;
        double acc = 0.0;
        for (int bb = 0; bb < B; ++bb)
            for (int l = 0; l < Lo; ++l) acc += gy[((size_t)bb * O + o) * Lo + l];
        db[o] = acc;
    }
}
__global__ void conv1d_bwd_x_kernel(const double* __restrict__ gy, const double* __restrict__ w, int B, int C, int L,
                                    int O, int K, int S, int Lo, double* __restrict__ gx) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)B * C * L) return;
    const int p = (int)(i % L), c = (int)((i / L) % C), bb = (int)(i / ((size_t)L * C));
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
        const int q = p - k;
        if (q < 0 || q % S) continue;
        const int l = q / S;
        if (l >= Lo) continue;
        for (int o = 0; o < O; ++o) acc = fma(gy[((size_t)bb * O + o) * Lo + l], w[((size_t)o * C + c) * K + k], acc);
    }
    gx[i] = acc;
}

// FK point sets of normalised joint rows u (T rows of D) for the planar chain
// (_batch_loss / fk_weighted_mse, diffusion.py:304-338): q = lo + u span, th = cumsum q,
// px = base + prefix + frac * l_k cos th_k.  One thread per (b, t) row.
template <int D, int M>
__device__ __forceinline__ void fk_row(const double* u, const double* lo, const double* span, const double* len,
                                       const double* fr, double bx, double by, double (&px)[D][M], double (&py)[D][M],
                                       double (&s)[D], double (&c)[D]) {
    double th = 0.0, prx = 0.0, pry = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        th += lo[d] + u[d] * span[d];
        c[d] = cos(th);
        s[d] = sin(th);
        const double lx = c[d] * len[d], ly = s[d] * len[d];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            px[d][m] = bx + prx + lx * fr[m];
            py[d][m] = by + pry + ly * fr[m];
        }
        prx += lx;
        pry += ly;
    }
}

// per-sample loss terms and d loss / d eps_pred:
//   loss = mean_b w_b [ sum_{t,d,m} |P(pred) - P(true)|^2 / (T D M) + mse_w * sum (pred - true)^2 / (T D) ]
template <int D, int M>
__global__ void fk_loss_kernel(const double* __restrict__ eps_t, const double* __restrict__ eps_p, int B, int T,
                               const double* __restrict__ w, const double* __restrict__ lo,
                               const double* __restrict__ span, const double* __restrict__ len,
                               const double* __restrict__ fr, double bx, double by, double mse_w,
                               double* __restrict__ row_fk, double* __restrict__ row_mse, double* __restrict__ grad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * T) return;
    const int bb = i / T;
    const double* ut = eps_t + (size_t)i * D;
    const double* up = eps_p + (size_t)i * D;
    double pxt[D][M], pyt[D][M], pxp[D][M], pyp[D][M], st[D], ct[D], sp[D], cp[D];
    fk_row<D, M>(ut, lo, span, len, fr, bx, by, pxt, pyt, st, ct);
    fk_row<D, M>(up, lo, span, len, fr, bx, by, pxp, pyp, sp, cp);
    const double n_pts = (double)T * D * M, n_el = (double)T * D;
    const double cfk = 2.0 * w[bb] / (n_pts * B), cms = 2.0 * mse_w * w[bb] / (n_el * B);
    double fk = 0.0, ms = 0.0;
    // dL/dth_j = sum over points (d, m) with j <= d of (gx dpx/dth_j + gy dpy/dth_j):
    //   dpx(d, m)/dth_j = -s_j l_j (j < d) or -s_d l_d fr_m (j = d); dpy: +c_j l_j / c_d l_d fr_m
    double gth[D];
#pragma unroll
    for (int d = 0; d < D; ++d) gth[d] = 0.0;
    double sgx = 0.0, sgy = 0.0;   // suffix sums of the point gradients over links > j
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
        double gx_d = 0.0, gy_d = 0.0, gxf = 0.0, gyf = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const double ex = pxp[d][m] - pxt[d][m], ey = pyp[d][m] - pyt[d][m];
            fk += ex * ex + ey * ey;
            gx_d += cfk * ex;
            gy_d += cfk * ey;
            gxf += cfk * ex * fr[m];
            gyf += cfk * ey * fr[m];
        }
        gth[d] = (-sp[d] * len[d]) * (gxf + sgx) + (cp[d] * len[d]) * (gyf + sgy);
        sgx += gx_d;
        sgy += gy_d;
    }
    // th_j = sum_{i <= j} q_i  ->  dL/dq_i = sum_{j >= i} dL/dth_j;  q = lo + u span
    double acc = 0.0;
    for (int d = D - 1; d >= 0; --d) {
        acc += gth[d];
        const double e = up[d] - ut[d];
        ms += e * e;
        grad[(size_t)i * D + d] = acc * span[d] + cms * e;
    }
    row_fk[i] = fk;
    row_mse[i] = ms;
}

// Adam (autodiff.py:254-284): m = b1 m + (1 - b1) g; v = b2 v + (1 - b2) g^2;
// p -= lr (m / b1t) / (sqrt(v / b2t) + eps)
__global__ void adam_kernel(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                            double* __restrict__ v, size_t n, double lr, double b1, double b2, double b1t, double b2t,
                            double eps) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double mi = m[i] * b1;
    mi += (1.0 - b1) * g[i];
    double vi = v[i] * b2;
    vi += (1.0 - b2) * (g[i] * g[i]);
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / b1t) / (sqrt(vi / b2t) + eps);
}

inline unsigned blocks_for(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

extern "C" int ps_train_gemm(const double* A, int lda, int ta, const double* B, int ldb, int tb, double* C, int ldc,
                             int M, int N, int K, int accumulate, void* stream) {
    if (M < 0 || N < 0 || K < 0) return PS_FAIL(PS_ERR_SHAPE);
    if (M == 0 || N == 0) return PS_OK;
    gemm_f64_kernel<<<dim3((N + GT - 1) / GT, (M + GT - 1) / GT), dim3(GT, GT), 0, (cudaStream_t)stream>>>(
        A, lda, ta, B, ldb, tb, C, ldc, M, N, K, accumulate);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_bias_act(double* y, int ldy, const double* b, int R, int N, int act, double* pre, void* stream) {
    if (R <= 0 || N <= 0) return PS_FAIL(PS_ERR_SHAPE);
    bias_act_kernel<<<dim3(blocks_for(N, 128), R), 128, 0, (cudaStream_t)stream>>>(y, ldy, b, R, N, act, pre);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_silu_bwd(double* g, int ldg, const double* pre, int R, int N, void* stream) {
    if (R <= 0 || N <= 0) return PS_FAIL(PS_ERR_SHAPE);
    silu_bwd_kernel<<<dim3(blocks_for(N, 128), R), 128, 0, (cudaStream_t)stream>>>(g, ldg, pre, R, N);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_colsum(const double* g, int ldg, int R, int N, double* db, int accumulate, void* stream) {
    if (R <= 0 || N <= 0) return PS_FAIL(PS_ERR_SHAPE);
    colsum_kernel<<<blocks_for(N, 128), 128, 0, (cudaStream_t)stream>>>(g, ldg, R, N, db, accumulate);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_film(const double* a, const double* sc, const double* sh, int n, double* out, void* stream) {
    if (n <= 0) return PS_FAIL(PS_ERR_SHAPE);
    film_fwd_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(a, sc, sh, n, out);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_film_bwd(const double* g, const double* a, const double* sc, int n, double* da, double* dsc,
                                 void* stream) {
    if (n <= 0) return PS_FAIL(PS_ERR_SHAPE);
    film_bwd_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(g, a, sc, n, da, dsc);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_conv1d(const double* x, int B, int C, int L, const double* w, const double* b, int O, int K,
                               int S, double* pre, double* y, void* stream) {
    if (B <= 0 || L < K || S <= 0) return PS_FAIL(PS_ERR_SHAPE);
    const int Lo = (L - K) / S + 1;
    conv1d_fwd_kernel<<<blocks_for((size_t)B * O * Lo, 256), 256, 0, (cudaStream_t)stream>>>(x, B, C, L, w, b, O, K,
                                                                                            S, Lo, pre, y);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_conv1d_bwd(const double* gy, const double* x, const double* w, int B, int C, int L, int O,
                                   int K, int S, double* dw, double* db, double* gx, void* stream) {
    if (B <= 0 || L < K || S <= 0) return PS_FAIL(PS_ERR_SHAPE);
    const int Lo = (L - K) / S + 1;
    conv1d_bwd_w_kernel<<<blocks_for((size_t)O * C * K + O, 128), 128, 0, (cudaStream_t)stream>>>(gy, x, B, C, L, O,
                                                                                                 K, S, Lo, dw, db);
    PS_CHECK_LAUNCH();
    if (gx) {
        conv1d_bwd_x_kernel<<<blocks_for((size_t)B * C * L, 256), 256, 0, (cudaStream_t)stream>>>(gy, w, B, C, L, O,
                                                                                                 K, S, Lo, gx);
        PS_CHECK_LAUNCH();
    }
    return PS_OK;
}

extern "C" int ps_train_fk_loss(const double* eps_true, const double* eps_pred, int B, int T, int D, int M,
                                const double* w, const double* lo, const double* span, const double* len,
                                const double* fr, double base_x, double base_y, double mse_w, double* row_fk,
                                double* row_mse, double* grad, void* stream) {
    if (D != 7 || M != 4 || B <= 0 || T <= 0) return PS_FAIL(PS_ERR_SHAPE);
    fk_loss_kernel<7, 4><<<blocks_for((size_t)B * T, 128), 128, 0, (cudaStream_t)stream>>>(
        eps_true, eps_pred, B, T, w, lo, span, len, fr, base_x, base_y, mse_w, row_fk, row_mse, grad);
    PS_CHECK_LAUNCH();
    return PS_OK;
}

extern "C" int ps_train_adam(double* p, const double* g, double* m, double* v, long long n, double lr, double b1,
                             double b2, double b1t, double b2t, double eps, void* stream) {
    if (n < 0) return PS_FAIL(PS_ERR_SHAPE);
    if (n == 0) return PS_OK;
    adam_kernel<<<blocks_for((size_t)n, 256), 256, 0, (cudaStream_t)stream>>>(p, g, m, v, (size_t)n, lr, b1, b2, b1t,
                                                                             b2t, eps);
    PS_CHECK_LAUNCH();
    return PS_OK;
}
