// Offline post-processing of tracked sequences (reference pipeline.py:308-325
// smooth_trajectory; metrics.py iou / mean_vertex_error).
//
// smooth_trajectory: a centred weighted average along the frame axis,
// truncated and renormalised at the ends.  The reference accumulates
// out[lo:hi] += w_k * arr[lo+off:hi+off] and norm[lo:hi] += w_k in stencil
// order, then divides; the kernel does the same per element in the same
// order (unfused, --fmad=false), so the result is bit-identical.
#include <cuda_runtime.h>
#include <cstdint>
#include "lc_internal.h"

__global__ void k_smooth_trajectory(const double *v, int F, long long D, const double *w, int K, double *out) {
    lc_pdl_wait();
    const int half = K / 2;
    const long long n = (long long)F * D;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(idx / D);
        const long long d = idx - (long long)f * D;
        double acc = 0.0, norm = 0.0;
        for (int k = 0; k < K; ++k) {
            const int src = f + (k - half);
            if (src < 0 || src >= F) continue;
            acc = acc + w[k] * v[(long long)src * D + d];
            norm = norm + w[k];
        }
        out[idx] = acc / norm;
    }
}

// per-frame |a & b| and |a | b| of two mask stacks (iou), one CTA per frame
__global__ void k_mask_overlap(const uint8_t *a, const uint8_t *b, long long HW, unsigned long long *inter,
                               unsigned long long *uni) {
    lc_pdl_wait();
    const int f = blockIdx.y;
    const uint8_t *pa = a + (long long)f * HW, *pb = b + (long long)f * HW;
    unsigned long long i0 = 0, u0 = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < HW; i += (long long)gridDim.x * blockDim.x) {
        const bool x = pa[i] != 0, y = pb[i] != 0;
        i0 += (x && y) ? 1 : 0;
        u0 += (x || y) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        i0 += __shfl_xor_sync(0xffffffffu, i0, o);
        u0 += __shfl_xor_sync(0xffffffffu, u0, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(inter + f, i0);
        atomicAdd(uni + f, u0);
    }
}
