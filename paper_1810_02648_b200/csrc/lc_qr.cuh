// Dense normal-equation solve (dense_solve, reference solvers.py:41-56):
// Householder QR of A, rank test min|R_ii| < 1e-10 max|R_ii|, Tikhonov
// damping 1e-6 tr(A)/n (or 1e-6) and a second QR, back substitution.
//
// Block-cooperative, everything in shared memory: one warp owns each column
// (rows over lanes), so a Householder step is one broadcast of v and one
// column update per warp.  n <= 64.
#pragma once
#include "lc_device.cuh"

#define LC_QR_MAXN 64

template <int MAXN>
struct QrSmemT {
    double a[MAXN][MAXN + 1];   // augmented [A | b], row-major
    double v[MAXN];
    double rdiag[MAXN];
    double x[MAXN];
    double w[MAXN + 1];
    double tau;
    int skip;
};
using QrSmem = QrSmemT<LC_QR_MAXN>;

// Householder on columns 0..n-1 of the augmented (n x n+1) matrix.
// Per column: warp 0 forms the reflector (shuffle-reduced norm), one thread
// per trailing column forms w_j = v . a_j serially (no shuffle chains on the
// critical path), then every thread updates the trailing block.
template <int NT, typename S>
__device__ void qr_factor(S &s, int n) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = 0; k < n; ++k) {
        if (w == 0) {
            double ss = 0.0;
            for (int i = k + lane; i < n; i += 32) ss += s.a[i][k] * s.a[i][k];
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            const double akk = s.a[k][k];
            const double nrm = sqrt(ss);
            const double alpha = akk >= 0.0 ? -nrm : nrm;
            const double v0 = akk - alpha;
            const double vn2 = ss - akk * akk + v0 * v0;
            for (int i = k + lane; i < n; i += 32) s.v[i] = i == k ? v0 : s.a[i][k];
            if (lane == 0) {
                s.skip = !(nrm > 0.0) || !(vn2 > 0.0);
                s.tau = s.skip ? 0.0 : 2.0 / vn2;
                s.rdiag[k] = s.skip ? akk : alpha;
            }
        }
        __syncthreads();
        const int m = n - k;            // rows k..n-1
        const int ncol = n - k;         // columns k+1..n (incl. the rhs column n)
        if (!s.skip) {
            for (int jj = threadIdx.x; jj < ncol; jj += NT) {
                const int j = k + 1 + jj;
                double d = 0.0;
                for (int i = k; i < n; ++i) d += s.v[i] * s.a[i][j];
                s.w[jj] = s.tau * d;
            }
            __syncthreads();
            for (int e = threadIdx.x; e < m * ncol; e += NT) {
                const int i = k + e / ncol, jj = e % ncol;
                s.a[i][k + 1 + jj] -= s.w[jj] * s.v[i];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) s.a[k][k] = s.rdiag[k];
    }
    __syncthreads();
}

// back substitution R x = (Q^T b) on warp 0 (column n holds Q^T b)
template <typename S>
__device__ inline void qr_backsolve(S &s, int n) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    for (int k = n - 1; k >= 0; --k) {
        double acc = 0.0;
        for (int j = k + 1 + lane; j < n; j += 32) acc += s.a[k][j] * s.x[j];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) s.x[k] = (s.a[k][n] - acc) / s.a[k][k];
        __syncwarp();
    }
}

// Solve with the reference's rank test / damping.  A is read from `A` (n*n
// row-major, symmetric) and `b`; result in s.x.  Returns damped flag.
template <int NT, typename S>
__device__ bool dense_solve_block(S &s, const double *A, const double *b, int n,
                                  double &damping) {
    for (int i = threadIdx.x; i < n * n; i += NT) s.a[i / n][i % n] = A[i];
    for (int i = threadIdx.x; i < n; i += NT) s.a[i][n] = b[i];
    __syncthreads();
    qr_factor<NT, S>(s, n);
    __shared__ int damped_flag;
    __shared__ double lam;
    if (threadIdx.x == 0) {
        double mx = 0.0, mn = LC_INF;
        for (int i = 0; i < n; ++i) {
            const double d = fabs(s.rdiag[i]);
            mx = fmax(mx, d);
            mn = fmin(mn, d);
        }
        damped_flag = mn < 1e-10 * fmax(mx, 1e-300);
        double tr = 0.0;
        for (int i = 0; i < n; ++i) tr += A[i * n + i];
        double l = 1e-6 * tr / n;
        if (l <= 0.0) l = 1e-6;
        lam = damped_flag ? l : 0.0;
    }
    __syncthreads();
    if (damped_flag) {
        for (int i = threadIdx.x; i < n * n; i += NT) {
            const int r = i / n, c = i % n;
            s.a[r][c] = r == c ? A[i] + lam : A[i];
        }
        for (int i = threadIdx.x; i < n; i += NT) s.a[i][n] = b[i];
        __syncthreads();
        qr_factor<NT, S>(s, n);
    }
    qr_backsolve(s, n);
    __syncthreads();
    damping = lam;
    return damped_flag != 0;
}
