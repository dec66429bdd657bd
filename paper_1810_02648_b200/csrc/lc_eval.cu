// Tracking-quality metrics on the device (reference metrics.py:26-106,
// evaluation.py:16-40): centred mean vertex error and the Umeyama
// (Procrustes) similarity alignment behind aligned_joint_error, batched over
// frames.  Used by sequence evaluation and by bench.py's tracking block.
//
// mean_vertex_error is bit-identical to numpy: the axis-0 means of an (N,3)
// array are sequential row sums (numpy's reduction over a non-contiguous
// axis), np.linalg.norm(axis=1) is sqrt((x^2 + y^2) + z^2), and np.mean of
// the distances is numpy's pairwise summation (`pairwise_sum_DOUBLE`: blocks
// of <= 128 elements with 8 accumulators, halves rounded to multiples of 8),
// all unfused (--fmad=false).  umeyama_alignment replaces LAPACK's SVD with
// a one-sided Jacobi SVD of the 3x3 cross-covariance (agreement ~1e-15).
#include <cuda_runtime.h>
#include <cstdint>
#include "lc_internal.h"

namespace {

// numpy pairwise_sum_DOUBLE (numpy/_core/src/umath/loops_utils.h.src) over
// a[0], a[s], ..., a[(n-1)s]
__device__ double np_pairwise_sum(const double *a, long long n, long long s) {
    if (n < 8) {
        double r = 0.0;
        for (long long i = 0; i < n; ++i) r += a[i * s];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j * s];
        long long i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * s];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * s];
        return res;
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2, s) + np_pairwise_sum(a + n2 * s, n - n2, s);
}

// column means of an (n, 3) row-major block (ndarray.mean(axis=0))
__device__ void col_means3(const double *x, long long n, double mu[3]) {
    for (int c = 0; c < 3; ++c) {
        double acc = x[c];
        for (long long i = 1; i < n; ++i) acc += x[3 * i + c];
        mu[c] = acc / (double)n;
    }
}

// one-sided Jacobi SVD of a 3x3: A = U diag(s) V^T, s descending, U and V
// orthonormal (columns of zero singular values completed to a basis)
__device__ void svd3(const double A[9], double U[9], double s[3], double V[9]) {
    for (int k = 0; k < 9; ++k) {
        U[k] = A[k];
        V[k] = (k % 4 == 0) ? 1.0 : 0.0;
    }
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int r = 0; r < 3; ++r) {
                    al += U[3 * r + p] * U[3 * r + p];
                    be += U[3 * r + q] * U[3 * r + q];
                    ga += U[3 * r + p] * U[3 * r + q];
                }
                if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
                rotated = true;
                const double ze = (be - al) / (2.0 * ga);
                const double t = (ze >= 0.0 ? 1.0 : -1.0) / (fabs(ze) + sqrt(1.0 + ze * ze));
                const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
                for (int r = 0; r < 3; ++r) {
                    const double up = U[3 * r + p], uq = U[3 * r + q];
                    U[3 * r + p] = c * up - sn * uq;
                    U[3 * r + q] = sn * up + c * uq;
                    const double vp = V[3 * r + p], vq = V[3 * r + q];
                    V[3 * r + p] = c * vp - sn * vq;
                    V[3 * r + q] = sn * vp + c * vq;
                }
            }
        if (!rotated) break;
    }
    for (int k = 0; k < 3; ++k)
        s[k] = sqrt(U[k] * U[k] + U[3 + k] * U[3 + k] + U[6 + k] * U[6 + k]);
    // descending order (selection sort on three columns, U and V together)
    for (int a = 0; a < 2; ++a) {
        int m = a;
        for (int b = a + 1; b < 3; ++b)
            if (s[b] > s[m]) m = b;
        if (m != a) {
            const double ts = s[a]; s[a] = s[m]; s[m] = ts;
            for (int r = 0; r < 3; ++r) {
                double t = U[3 * r + a]; U[3 * r + a] = U[3 * r + m]; U[3 * r + m] = t;
                t = V[3 * r + a]; V[3 * r + a] = V[3 * r + m]; V[3 * r + m] = t;
            }
        }
    }
    const double tiny = 1e-300 + 1e-15 * s[0];
    int rank = 0;
    for (int k = 0; k < 3; ++k) {
        if (s[k] > tiny) {
            for (int r = 0; r < 3; ++r) U[3 * r + k] /= s[k];
            ++rank;
        }
    }
    // complete U's columns of (numerically) zero singular values
    for (int k = rank; k < 3; ++k) {
        double best[3] = {0, 0, 0};
        if (k == 2 && rank == 2) {   // cross product of the first two
            best[0] = U[3] * U[7] - U[6] * U[4];
            best[1] = U[6] * U[1] - U[0] * U[7];
            best[2] = U[0] * U[4] - U[3] * U[1];
        } else {                     // Gram-Schmidt of the unit axis least aligned with the basis so far
            double bn = -1.0;
            for (int e = 0; e < 3; ++e) {
                double v[3] = {0, 0, 0};
                v[e] = 1.0;
                for (int j = 0; j < k; ++j) {
                    const double d = U[3 * e + j];
                    for (int r = 0; r < 3; ++r) v[r] -= d * U[3 * r + j];
                }
                const double nn = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
                if (nn > bn) { bn = nn; best[0] = v[0]; best[1] = v[1]; best[2] = v[2]; }
            }
        }
        const double nn = sqrt(best[0] * best[0] + best[1] * best[1] + best[2] * best[2]);
        for (int r = 0; r < 3; ++r) U[3 * r + k] = best[r] / nn;
    }
}

__device__ double det3(const double m[9]) {
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}

}  // namespace

// metrics.mean_vertex_error per frame: one CTA per frame.  `dist` is scratch
// (F * n_sel doubles).  idx == nullptr selects every vertex.
__global__ void k_vertex_error(int F, long long N, const double *pred, const double *gt, const long long *idx,
                               long long n_sel, int center, double *dist, double *out) {
    lc_pdl_wait();
    const int f = blockIdx.x;
    const double *P = pred + (size_t)f * N * 3, *G = gt + (size_t)f * N * 3;
    __shared__ double mu[6];
    if (threadIdx.x < 6) {
        const int c = threadIdx.x % 3;
        if (center) {
            double m[3];
            col_means3(threadIdx.x < 3 ? P : G, N, m);
            mu[threadIdx.x] = m[c];
        } else {
            mu[threadIdx.x] = 0.0;
        }
    }
    __syncthreads();
    double *D = dist + (size_t)f * n_sel;
    for (long long k = threadIdx.x; k < n_sel; k += blockDim.x) {
        const long long i = idx ? idx[k] : k;
        double d2[3];
        for (int c = 0; c < 3; ++c) {
            const double a = center ? P[3 * i + c] - mu[c] : P[3 * i + c];
            const double b = center ? G[3 * i + c] - mu[3 + c] : G[3 * i + c];
            const double d = a - b;
            d2[c] = d * d;
        }
        D[k] = sqrt((d2[0] + d2[1]) + d2[2]);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[f] = np_pairwise_sum(D, n_sel, 1) / (double)n_sel;
}

// metrics.umeyama_alignment + aligned_joint_error per frame: one thread per
// frame, M points of dimension 3.  scratch: F * M doubles.
__global__ void k_umeyama(int F, int M, const double *src_all, const double *dst_all, int with_scaling,
                          double *scale_out, double *rot_out, double *t_out, double *err_out, double *scratch) {
    lc_pdl_wait();
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    const double *S = src_all + (size_t)f * M * 3, *D = dst_all + (size_t)f * M * 3;
    double *tmp = scratch + (size_t)f * M;
    double ms[3], md[3];
    col_means3(S, M, ms);
    col_means3(D, M, md);
    // cov = xd^T @ xs / n
    double cov[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int i = 0; i < M; ++i) acc += (D[3 * i + a] - md[a]) * (S[3 * i + b] - ms[b]);
            cov[3 * a + b] = acc / (double)M;
        }
    double U[9], s[3], V[9];
    svd3(cov, U, s, V);
    double sign[3] = {1.0, 1.0, 1.0};
    if (det3(U) * det3(V) < 0.0) sign[2] = -1.0;
    double R[9];   // (u * sign) @ vt
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            R[3 * a + b] = U[3 * a + 0] * sign[0] * V[3 * b + 0] + U[3 * a + 1] * sign[1] * V[3 * b + 1] +
                           U[3 * a + 2] * sign[2] * V[3 * b + 2];
    double scale = 1.0;
    if (with_scaling) {
        for (int i = 0; i < M; ++i) {
            const double x = S[3 * i] - ms[0], y = S[3 * i + 1] - ms[1], z = S[3 * i + 2] - ms[2];
            tmp[i] = (x * x + y * y) + z * z;
        }
        const double var_s = np_pairwise_sum(tmp, M, 1) / (double)M;
        scale = var_s > 0.0 ? ((s[0] * sign[0] + s[1] * sign[1]) + s[2] * sign[2]) / var_s : 1.0;
    }
    double t[3];
    for (int a = 0; a < 3; ++a)
        t[a] = md[a] - scale * ((R[3 * a] * ms[0] + R[3 * a + 1] * ms[1]) + R[3 * a + 2] * ms[2]);
    for (int i = 0; i < M; ++i) {
        double d2[3];
        for (int a = 0; a < 3; ++a) {
            const double al = ((scale * S[3 * i]) * R[3 * a] + (scale * S[3 * i + 1]) * R[3 * a + 1]) +
                              (scale * S[3 * i + 2]) * R[3 * a + 2] + t[a];
            const double d = al - D[3 * i + a];
            d2[a] = d * d;
        }
        tmp[i] = sqrt((d2[0] + d2[1]) + d2[2]);
    }
    err_out[f] = np_pairwise_sum(tmp, M, 1) / (double)M;
    scale_out[f] = scale;
    for (int k = 0; k < 9; ++k) rot_out[9 * (size_t)f + k] = R[k];
    for (int a = 0; a < 3; ++a) t_out[3 * (size_t)f + a] = t[a];
}
