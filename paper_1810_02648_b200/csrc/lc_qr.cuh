// Dense normal-equation solve (dense_solve, reference solvers.py:41-56):
// Householder QR of A, rank test min|R_ii| < 1e-10 max|R_ii|, Tikhonov
// damping 1e-6 tr(A)/n (or 1e-6) and a second QR, back substitution.
//
// The augmented matrix [A | b] is stored column-major in shared memory (row
// stride MAXN + 1 doubles); a quad of threads owns each column.  A
// Householder step is one batched read of the pivot column, 2-step quad
// butterflies for the norm and the dot products, and an update of each
// quad's column from registers, with one block barrier.  Back substitution
// is column-oriented on one warp with the right-hand side held in
// registers.  n <= 64.
#pragma once
#include "lc_device.cuh"

#define LC_QR_MAXN 64

template <int MAXN>
struct QrSmemT {
    double c[MAXN + 1][MAXN + 1];   // c[j][i] = column j, row i; column n is the rhs
    double rdiag[MAXN];
    double x[MAXN];
    int damped;
    double lam;
};
using QrSmem = QrSmemT<LC_QR_MAXN>;

// Householder on columns 0..n-1 of the augmented n x (n+1) matrix by all NT
// threads of the block.  A quad of 4 threads owns a column (quad q owns
// columns q, q + NT/4, ...); lane r of the quad owns rows i = 4m + r.  The
// reflector of column k is v = (a_kk - alpha, a_k+1,k, ...), tau = 2/|v|^2,
// applied as a_j -= tau (v . a_j) v; R's diagonal goes to rdiag and to
// c[k][k] (so R_ij = c[j][i] for i <= j).  Each quad reads column k and
// forms |a_k|^2 with a 2-step xor butterfly (commutative, so every thread of
// every quad holds the same bits), then updates its column from registers.
// NB (a multiple of 4) bounds n at compile time: the row loops are unrolled
// and predicated so each step issues its shared loads in one batch.  One
// block barrier per step.
template <int NB, int NT, typename S>
__device__ void qr_factor_quad(S &s, int n) {
    static_assert(NB % 4 == 0, "NB must be a multiple of 4");
    constexpr int R = NB / 4, NQ = NT / 4;
    const int r = threadIdx.x & 3, q = threadIdx.x >> 2;
    // every quad runs the same number of passes so the butterflies stay
    // warp-uniform; inactive quads read the pivot column as a dummy
    const int passes = (n + 1 + NQ - 1) / NQ;
    for (int k = 0; k < n; ++k) {
        // the pivot column, and (first pass) this quad's column, in one batch;
        // the dot product v . a_j (rows > k) does not depend on the
        // reflector's leading entry, so it is reduced together with the norm
        const double akk = s.c[k][k];
        double v[R], col[R];
        int j = q;
        bool act = j > k && j <= n;
        double *cj = s.c[act ? j : k];
        double ck = act ? cj[k] : 0.0;
        double p = 0.0, d = 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int i = 4 * m + r;
            const bool row = i > k && i < n;
            v[m] = row ? s.c[k][i] : 0.0;
            col[m] = (act && row) ? cj[i] : 0.0;
        }
#pragma unroll
        for (int m = 0; m < R; ++m) {
            p = fma(v[m], v[m], p);
            d = fma(v[m], col[m], d);
        }
        p += __shfl_xor_sync(0xffffffffu, p, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        p += __shfl_xor_sync(0xffffffffu, p, 2);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        const double ss = akk * akk + p;
        const double nrm = sqrt(ss);
        const double alpha = akk >= 0.0 ? -nrm : nrm;
        const double v0 = akk - alpha;
        const double vn2 = p + v0 * v0;
        const bool skip = !(nrm > 0.0) || !(vn2 > 0.0);
        if (!skip) {
            const double tau = 2.0 / vn2;
            for (int ps = 0; ps < passes; ++ps) {
                if (ps > 0) {
                    j = q + ps * NQ;
                    act = j > k && j <= n;
                    cj = s.c[act ? j : k];
                    ck = act ? cj[k] : 0.0;
                    d = 0.0;
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        const int i = 4 * m + r;
                        col[m] = (act && i > k && i < n) ? cj[i] : 0.0;
                        d = fma(v[m], col[m], d);
                    }
                    d += __shfl_xor_sync(0xffffffffu, d, 1);
                    d += __shfl_xor_sync(0xffffffffu, d, 2);
                }
                // the quad's lanes have all read their rows of column j (and
                // a_jk) before lane 0 overwrites a_jk: the shuffles above
                // converge the warp, __syncwarp makes that ordering explicit
                __syncwarp();
                if (act) {
                    const double w = tau * fma(v0, ck, d);
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        const int i = 4 * m + r;
                        if (i > k && i < n) cj[i] = fma(-w, v[m], col[m]);
                    }
                    if (r == 0) cj[k] = fma(-w, v0, ck);
                }
            }
        }
        if (threadIdx.x == 0) s.rdiag[k] = skip ? akk : alpha;
        __syncthreads();
    }
    // R's diagonal into place (column k's rows > k keep the reflector)
    for (int k = threadIdx.x; k < n; k += NT) s.c[k][k] = s.rdiag[k];
    __syncthreads();
}

// R x = Q^T b (column n), column-oriented on warp 0: x_k = c_k / R_kk, then
// every remaining c_i -= R_ik x_k.  The result goes to s.x.
template <typename S>
__device__ void qr_backsolve_warp(S &s, int n) {
    const int lane = threadIdx.x & 31;
    double c0 = lane < n ? s.c[n][lane] : 0.0;
    double c1 = lane + 32 < n ? s.c[n][lane + 32] : 0.0;
    for (int k = n - 1; k >= 0; --k) {
        const double ck = __shfl_sync(0xffffffffu, k < 32 ? c0 : c1, k & 31);
        const double xk = ck / s.c[k][k];
        if (lane == 0) s.x[k] = xk;
        const double *rk = s.c[k];
        if (lane < k) c0 = fma(-rk[lane], xk, c0);
        if (lane + 32 < k) c1 = fma(-rk[lane + 32], xk, c1);
    }
    __syncwarp();
}

template <int NT, typename S>
__device__ __forceinline__ void qr_load_block(S &s, const double *A, const double *b, int n, double lam) {
    for (int e = threadIdx.x; e < n * n; e += NT) {
        const int i = e / n, j = e % n;
        s.c[j][i] = (i == j) ? A[e] + lam : A[e];
    }
    for (int i = threadIdx.x; i < n; i += NT) s.c[n][i] = b[i];
    __syncthreads();
}

// Solve with the reference's rank test / damping, entirely on warp 0.  A is
// read from `A` (n*n row-major) and `b`; the result is in s.x.  Every thread
// of the block must call it (one trailing __syncthreads).  Returns the damped flag.
template <int NT, typename S>
__device__ bool dense_solve_block(S &s, const double *A, const double *b, int n, double &damping) {
    static_assert(NT % 32 == 0, "whole warps");
    const int t = threadIdx.x;
    qr_load_block<NT>(s, A, b, n, 0.0);
    if (n <= 36) qr_factor_quad<36, NT>(s, n);
    else qr_factor_quad<LC_QR_MAXN, NT>(s, n);
    if (t < 32) {
        const int lane = t;
        double mx = 0.0, mn = LC_INF;
        for (int i = lane; i < n; i += 32) {
            const double d = fabs(s.rdiag[i]);
            mx = fmax(mx, d);
            mn = fmin(mn, d);
        }
        for (int o = 16; o > 0; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        const bool damped = mn < 1e-10 * fmax(mx, 1e-300);
        double lam = 0.0;
        if (damped) {
            double tr = 0.0;
            for (int i = 0; i < n; ++i) tr += A[i * n + i];   // sequential trace (np.trace order)
            lam = 1e-6 * tr / n;
            if (lam <= 0.0) lam = 1e-6;
        }
        if (lane == 0) {
            s.damped = damped;
            s.lam = lam;
        }
    }
    __syncthreads();
    if (s.damped) {
        qr_load_block<NT>(s, A, b, n, s.lam);
        if (n <= 36) qr_factor_quad<36, NT>(s, n);
        else qr_factor_quad<LC_QR_MAXN, NT>(s, n);
    }
    if (t < 32) qr_backsolve_warp(s, n);
    __syncthreads();
    damping = s.lam;
    return s.damped != 0;
}
