// Exact squared Euclidean distance transform of a feature image
// (reference imageproc.py:52-124 `_edt_squared`, numba) and the contour
// distance `euclidean_dt` / `DistanceField.dt` (:117-124, :182).
//
// The reference's two passes, restated per thread: one thread per column
// runs the forward / backward vertical sweeps (distances counted in +1.0
// steps, then squared), one thread per row builds the lower envelope of
// parabolas (Felzenszwalb-Huttenlocher) with the same floating-point
// expressions in the same order (compiled --fmad=false), so every output
// bit equals the reference's.  Squared distances are integers below 2^53:
// the transform is exact, and sqrt is correctly rounded.
#include <cuda_runtime.h>
#include <cstdint>
#include "lc_internal.h"

#define LC_EDT_BIG 1e18

// feature = contour_mask(mask) when contour != 0 (foreground with a
// background 4-neighbour, the border counting as background), else mask
__device__ __forceinline__ bool edt_feature(const uint8_t *m, int H, int W, int x, int y, int contour) {
    const bool on = m[(size_t)y * W + x] != 0;
    if (!contour || !on) return on;
    const bool l = x > 0 && m[(size_t)y * W + x - 1], r = x + 1 < W && m[(size_t)y * W + x + 1];
    const bool u = y > 0 && m[(size_t)(y - 1) * W + x], d = y + 1 < H && m[(size_t)(y + 1) * W + x];
    return !(l && r && u && d);
}

__global__ void k_edt_cols(const uint8_t *mask, int H, int W, int contour, double *g) {
    lc_pdl_wait();
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= W) return;
    double dist = LC_EDT_BIG;
    for (int y = 0; y < H; ++y) {
        if (edt_feature(mask, H, W, x, y, contour)) dist = 0.0;
        else if (dist < LC_EDT_BIG) dist += 1.0;
        g[(size_t)y * W + x] = dist;
    }
    dist = LC_EDT_BIG;
    for (int y = H - 1; y >= 0; --y) {
        if (edt_feature(mask, H, W, x, y, contour)) dist = 0.0;
        else if (dist < LC_EDT_BIG) dist += 1.0;
        double &gy = g[(size_t)y * W + x];
        if (dist < gy) gy = dist;
        if (gy < LC_EDT_BIG) gy = gy * gy;
    }
}

// one thread per row; v / z are per-row scratch (W and W+1 entries)
__global__ void k_edt_rows(const double *g, int H, int W, int take_sqrt, long long *vs, double *zs, double *out) {
    lc_pdl_wait();
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= H) return;
    const double *f = g + (size_t)y * W;
    long long *v = vs + (size_t)y * W;
    double *z = zs + (size_t)y * (W + 1);
    double *o = out + (size_t)y * W;
    int k = -1;
    for (int q = 0; q < W; ++q) {
        if (f[q] >= LC_EDT_BIG) continue;
        double s = 0.0;
        if (k >= 0) {
            s = ((f[q] + (double)q * q) - (f[v[k]] + (double)(v[k] * v[k]))) / (2.0 * (double)(q - v[k]));
            while (k >= 0 && s <= z[k]) {
                --k;
                if (k >= 0)
                    s = ((f[q] + (double)q * q) - (f[v[k]] + (double)(v[k] * v[k]))) / (2.0 * (double)(q - v[k]));
            }
        }
        if (k < 0) {
            k = 0;
            v[0] = q;
            z[0] = -LC_EDT_BIG;
            z[1] = LC_EDT_BIG;
        } else {
            ++k;
            v[k] = q;
            z[k] = s;
            z[k + 1] = LC_EDT_BIG;
        }
    }
    if (k < 0) {
        for (int x = 0; x < W; ++x) o[x] = take_sqrt ? sqrt(LC_EDT_BIG) : LC_EDT_BIG;
        return;
    }
    int j = 0;
    for (int x = 0; x < W; ++x) {
        while (z[j + 1] < (double)x) ++j;
        const long long dx = x - v[j];
        const double d2 = (double)(dx * dx) + f[v[j]];
        o[x] = take_sqrt ? sqrt(d2) : d2;
    }
}
