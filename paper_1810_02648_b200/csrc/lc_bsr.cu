// Kernel-level seams with the reference's explicit layouts:
//   pcg_solve(BlockSparseSystem)  (solvers.py:59-145) -- full 3x3 diag blocks,
//       full 3x3 off-diagonal blocks with (row, col) lists, block-Jacobi PCG;
//   dense_solve(DenseNormalSystem) (solvers.py:41-56).
// The off-diagonal list is row-sorted on the device (stable radix sort, so
// each row accumulates its blocks in the reference's np.add.at order).
#include <cub/cub.cuh>
#include "livecap.h"
#include "lc_device.cuh"
#include "lc_qr.cuh"
#include "lc_bsr.cuh"

namespace {
constexpr int NT = 1024;

// general 3x3 inverse (np.linalg.inv per block); false when singular
__device__ bool inv3(const double *a, double *o) {
    const double c00 = a[4] * a[8] - a[5] * a[7], c01 = a[5] * a[6] - a[3] * a[8],
                 c02 = a[3] * a[7] - a[4] * a[6];
    const double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
    if (det == 0.0 || !isfinite(det)) return false;
    const double id = 1.0 / det;
    o[0] = c00 * id; o[1] = (a[2] * a[7] - a[1] * a[8]) * id; o[2] = (a[1] * a[5] - a[2] * a[4]) * id;
    o[3] = c01 * id; o[4] = (a[0] * a[8] - a[2] * a[6]) * id; o[5] = (a[2] * a[3] - a[0] * a[5]) * id;
    o[6] = c02 * id; o[7] = (a[1] * a[6] - a[0] * a[7]) * id; o[8] = (a[0] * a[4] - a[1] * a[3]) * id;
    return true;
}

__device__ __forceinline__ V3 m3v(const double *m, V3 v) { return mat_vec(m, v); }
}  // namespace

__global__ void k_bsr_keys(int m, const long long *rows, int *keys, int *vals, int *count) {
    lc_pdl_wait();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        keys[i] = (int)rows[i];
        vals[i] = i;
        atomicAdd(count + rows[i], 1);
    }
}

template <int T>
__device__ int scan_block(const int *in, int *out, int n) {
    __shared__ int wt[T / 32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += T) {
        const int i = base + threadIdx.x;
        const int v = i < n ? in[i] : 0;
        int s = v;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
        }
        if (lane == 31) wt[w] = s;
        __syncthreads();
        if (w == 0) {
            int t = lane < T / 32 ? wt[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            if (lane < T / 32) wt[lane] = t;
        }
        __syncthreads();
        const int before = (w > 0 ? wt[w - 1] : 0) + carry;
        if (i < n) out[i] = before + s - v;
        __syncthreads();
        if (threadIdx.x == T - 1) carry = before + s;
        __syncthreads();
    }
    return carry;
}

__global__ void k_bsr_rowptr(int n, const int *count, int *rowptr) {
    lc_pdl_wait();
    const int tot = scan_block<1024>(count, rowptr, n);
    if (threadIdx.x == 0) rowptr[n] = tot;
}

__global__ void __launch_bounds__(NT, 1) k_pcg_bsr(BsrJob J) {
    lc_pdl_wait();
    __shared__ double red[8 * 32 + 16];
    const int n = J.n;
    // M^-1 = inv(diag); every block pseudo-inverted when one is exactly singular
    __shared__ int singular;
    if (threadIdx.x == 0) singular = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) {
        double o[9];
        if (!lu_inv3(J.diag + 9 * (size_t)i, o)) {
            singular = 1;
            for (int k = 0; k < 9; ++k) o[k] = 0.0;
        }
        for (int k = 0; k < 9; ++k) J.minv[9 * (size_t)i + k] = o[k];
    }
    __syncthreads();
    // np.linalg.inv raised: the reference pseudo-inverts the whole batch
    if (singular)
        for (int i = threadIdx.x; i < n; i += NT) pinv3(J.diag + 9 * (size_t)i, J.minv + 9 * (size_t)i);
    __syncthreads();
    double part[2] = {0, 0};
    for (int i = threadIdx.x; i < n; i += NT) {
        const V3 r = ld3(J.rhs + 3 * (size_t)i);
        const V3 z = m3v(J.minv + 9 * (size_t)i, r);
        st3(J.x + 3 * (size_t)i, v3(0, 0, 0));
        st3(J.best + 3 * (size_t)i, v3(0, 0, 0));
        st3(J.r + 3 * (size_t)i, r);
        st3(J.z + 3 * (size_t)i, z);
        st3(J.p + 3 * (size_t)i, z);
        part[0] += r.x * z.x + r.y * z.y + r.z * z.z;
        part[1] += r.x * r.x + r.y * r.y + r.z * r.z;
    }
    block_sums<NT, 2>(part, red);
    double rz = part[0];
    double best_norm = sqrt(part[1]);
    int done = 0, breakdown = 0;
    if (threadIdx.x == 0) J.norms[0] = best_norm;
    for (int it = 0; it < J.iters; ++it) {
        double s1[2] = {0, 0};
        for (int i = threadIdx.x; i < n; i += NT) {
            const V3 pi = ld3(J.p + 3 * (size_t)i);
            V3 y = m3v(J.diag + 9 * (size_t)i, pi);
            for (int k = J.rowptr[i]; k < J.rowptr[i + 1]; ++k) {
                const int m = J.order[k];
                y = y + m3v(J.off + 9 * (size_t)m, ld3(J.p + 3 * (size_t)J.cols[m]));
            }
            st3(J.ap + 3 * (size_t)i, y);
            s1[0] += pi.x * y.x + pi.y * y.y + pi.z * y.z;
            s1[1] += pi.x * pi.x + pi.y * pi.y + pi.z * pi.z;
        }
        block_sums<NT, 2>(s1, red);
        if (s1[0] <= 1e-14 * fmax(s1[1], 1e-300)) { breakdown = 1; break; }
        const double alpha = rz / s1[0];
        double s2[2] = {0, 0};
        for (int i = threadIdx.x; i < n; i += NT) {
            const V3 x = ld3(J.x + 3 * (size_t)i) + alpha * ld3(J.p + 3 * (size_t)i);
            const V3 r = ld3(J.r + 3 * (size_t)i) - alpha * ld3(J.ap + 3 * (size_t)i);
            const V3 z = m3v(J.minv + 9 * (size_t)i, r);
            st3(J.x + 3 * (size_t)i, x);
            st3(J.r + 3 * (size_t)i, r);
            st3(J.z + 3 * (size_t)i, z);
            s2[0] += r.x * z.x + r.y * z.y + r.z * z.z;
            s2[1] += r.x * r.x + r.y * r.y + r.z * r.z;
        }
        block_sums<NT, 2>(s2, red);
        ++done;
        const double nrm = sqrt(s2[1]);
        if (threadIdx.x == 0 && done < LC_MAX_LOG) J.norms[done] = nrm;
        const bool better = nrm < best_norm;
        if (better) best_norm = nrm;
        const bool stop = rz <= 0.0;
        const double beta = stop ? 0.0 : s2[0] / rz;
        for (int i = threadIdx.x; i < n; i += NT) {
            if (better) st3(J.best + 3 * (size_t)i, ld3(J.x + 3 * (size_t)i));
            if (!stop) st3(J.p + 3 * (size_t)i, ld3(J.z + 3 * (size_t)i) + beta * ld3(J.p + 3 * (size_t)i));
        }
        __syncthreads();
        if (stop) { breakdown = 1; break; }
        rz = s2[0];
    }
    if (threadIdx.x == 0) {
        J.info[0] = done;
        J.info[1] = breakdown;
        J.info[2] = singular;
    }
}

__global__ void __launch_bounds__(256, 1) k_dense_solve(int n, const double *A, const double *b,
                                                       double *x, double *info) {
    lc_pdl_wait();
    __shared__ QrSmem s;
    double damping;
    const bool damped = dense_solve_block<256>(s, A, b, n, damping);
    for (int i = threadIdx.x; i < n; i += 256) x[i] = s.x[i];
    if (threadIdx.x == 0) {
        info[0] = damped ? 1.0 : 0.0;
        info[1] = damping;
    }
}

size_t bsr_sort_temp_bytes(int m) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int *)nullptr, (int *)nullptr,
                                    (const int *)nullptr, (int *)nullptr, m);
    return bytes;
}

cudaError_t bsr_sort(void *temp, size_t temp_bytes, const int *keys_in, int *keys_out,
                     const int *vals_in, int *vals_out, int m, int key_bits, cudaStream_t st) {
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, m,
                                           0, key_bits, st);
}
