// Device-side building blocks shared by the kernels.
//
// Everything here is fp64.  The library is compiled with --fmad=false so
// `a*b + c` is never contracted: numpy and the numba kernels of the reference
// evaluate it unfused, and several discrete decisions (raster coverage,
// colour pruning, rim / inside tests, e1 <= e0) depend on the exact bits.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "lc_internal.h"

#define LC_INF (__longlong_as_double(0x7ff0000000000000LL))

// nanosecond device clock (phase timing of the persistent solvers)
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define LC_NPHASE 64

struct V3 { double x, y, z; };

__device__ __forceinline__ V3 v3(double x, double y, double z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 ld3(const double *p) { return V3{p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double *p, V3 v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(double s, V3 a) { return V3{s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 operator*(V3 a, double s) { return V3{a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ V3 cross3(V3 a, V3 b) {
    return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// numpy add.reduce over a length-3 axis: (x0 + x1) + x2
__device__ __forceinline__ double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double norm3(V3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

// 3x3 row-major matrices
__device__ __forceinline__ V3 mat_vec(const double *m, V3 v) {
    return V3{m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
              m[6] * v.x + m[7] * v.y + m[8] * v.z};
}
__device__ __forceinline__ void mat_mul(const double *a, const double *b, double *c) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

// ---------------------------------------------------------------------------
// camera (reference camera.py:45-83)

__device__ __forceinline__ bool project(const CamDev &c, V3 p, double &px, double &py) {
    const bool ok = p.z > 1e-9;
    const double zs = ok ? p.z : 1.0;
    px = ok ? c.fx * p.x / zs + c.cx : 0.0;
    py = ok ? c.fy * p.y / zs + c.cy : 0.0;
    return ok;
}
// rows of d(pix)/d(p): (a0, 0, a2) and (0, b1, b2); zero when invalid
__device__ __forceinline__ void proj_jac(const CamDev &c, V3 p, double &a0, double &a2,
                                         double &b1, double &b2) {
    if (!(p.z > 1e-9)) { a0 = a2 = b1 = b2 = 0.0; return; }
    const double zs = p.z;
    a0 = c.fx / zs;
    a2 = -c.fx * p.x / (zs * zs);
    b1 = c.fy / zs;
    b2 = -c.fy * p.y / (zs * zs);
}

// ---------------------------------------------------------------------------
// quaternions (w, x, y, z)  (skinning.py:85-112)

struct Q4 { double w, x, y, z; };
__device__ __forceinline__ Q4 qmul(Q4 a, Q4 b) {
    return Q4{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
              a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
              a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
              a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
__device__ __forceinline__ Q4 qconj(Q4 q) { return Q4{q.w, -q.x, -q.y, -q.z}; }
__device__ __forceinline__ V3 qrot(Q4 q, V3 v) {
    const V3 u{q.x, q.y, q.z};
    const V3 t = 2.0 * cross3(u, v);
    return v + q.w * t + cross3(u, t);
}

// ---------------------------------------------------------------------------
// deterministic block reduction (fixed thread -> value mapping, fixed tree)

template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = (l < NT / 32) ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (l == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// several sums at once (M <= 8)
template <int NT, int M>
__device__ __forceinline__ void block_sums(double (&v)[M], double *red) {
    for (int m = 0; m < M; ++m)
        for (int o = 16; o > 0; o >>= 1) v[m] += __shfl_down_sync(0xffffffffu, v[m], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0)
        for (int m = 0; m < M; ++m) red[m * 32 + w] = v[m];
    __syncthreads();
    if (threadIdx.x < 32) {
        for (int m = 0; m < M; ++m) {
            double s = (l < NT / 32) ? red[m * 32 + l] : 0.0;
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if (l == 0) red[8 * 32 + m] = s;
        }
    }
    __syncthreads();
    for (int m = 0; m < M; ++m) v[m] = red[8 * 32 + m];
    __syncthreads();
}

// ---------------------------------------------------------------------------
// exact nearest contour-pixel centre (DistanceField._nearest, imageproc.py:195-213)
//
// Uniform grid of LC_GRID_CELL-pixel cells with Chebyshev ring search.  Ties
// on the squared distance break toward the lowest point index (argwhere
// order).  Queries outside the grid fall back to a linear scan.

__device__ __forceinline__ void nn_consider(const NnGridDev &g, int pid, double qx, double qy,
                                            double &best, int &bi) {
    const int2 p = g.pts[pid];
    const double dx = qx - (double)p.x, dy = qy - (double)p.y;
    const double d2 = dx * dx + dy * dy;
    if (d2 < best || (d2 == best && pid < bi)) { best = d2; bi = pid; }
}

// packed candidate: one 8-byte load carries the coordinates and the id
__device__ __forceinline__ void nn_consider_packed(int2 c, double qx, double qy, double &best, int &bi) {
    const double dx = qx - (double)(c.x & 0xffff), dy = qy - (double)(c.x >> 16);
    const double d2 = dx * dx + dy * dy;
    if (d2 < best || (d2 == best && c.y < bi)) { best = d2; bi = c.y; }
}

__device__ __forceinline__ double box_dist2(double qx, double qy, double x0, double y0, double s) {
    const double dx = qx < x0 ? x0 - qx : (qx > x0 + s ? qx - (x0 + s) : 0.0);
    const double dy = qy < y0 ? y0 - qy : (qy > y0 + s ? qy - (y0 + s) : 0.0);
    return dx * dx + dy * dy;
}

// Exact best-first search of the site-count quadtree: a subtree is skipped
// only when its box is strictly farther than the best distance so far, so
// equidistant sites are still all seen and the lowest index wins.
__device__ inline void nn_quadtree(const NnGridDev &g, double qx, double qy, double &best, int &bi) {
    int stack[3 * 12 + 2];
    int sp = 0;
    stack[sp++] = g.qL << 24;                       // root: level qL, (0, 0)
    while (sp > 0) {
        const int e = stack[--sp];
        const int l = e >> 24, ny = (e >> 12) & 0xfff, nx = e & 0xfff;
        const int side = g.qP >> l;
        if (g.quad[quad_off(g.qP, l) + ny * side + nx] == 0) continue;
        const double s = (double)(LC_GRID_CELL << l);
        if (box_dist2(qx, qy, nx * s, ny * s, s) > best) continue;
        if (l == 0) {
            if (nx < g.ncx && ny < g.ncy) {
                const int c = ny * g.ncx + nx;
                for (int k = g.cell_start[c]; k < g.cell_start[c + 1]; ++k) nn_consider(g, g.cell_pts[k], qx, qy, best, bi);
            }
            continue;
        }
        // push the 4 children, nearest last (popped first)
        int ch[4];
        double d[4];
        const double cs = s * 0.5;
        for (int k = 0; k < 4; ++k) {
            const int cx = 2 * nx + (k & 1), cy = 2 * ny + (k >> 1);
            ch[k] = ((l - 1) << 24) | (cy << 12) | cx;
            d[k] = box_dist2(qx, qy, cx * cs, cy * cs, cs);
        }
        for (int i = 1; i < 4; ++i)      // sort descending by distance
            for (int j = i; j > 0 && d[j] > d[j - 1]; --j) {
                const double td = d[j]; d[j] = d[j - 1]; d[j - 1] = td;
                const int tc = ch[j]; ch[j] = ch[j - 1]; ch[j - 1] = tc;
            }
        for (int k = 0; k < 4; ++k) stack[sp++] = ch[k];
    }
}

// `hint` (a site id or -1) only seeds the search bound: the result is the
// exact nearest site with the lowest-index tie break whatever the hint.
__device__ inline int nn_query(const NnGridDev &g, double qx, double qy, double &d2out, int hint = -1) {
    double best = LC_INF;
    int bi = 0x7fffffff;
    if (hint >= 0 && hint < g.K) nn_consider(g, hint, qx, qy, best, bi);
    const double gx = (double)(g.ncx * LC_GRID_CELL), gy = (double)(g.ncy * LC_GRID_CELL);
    const bool in_grid = qx >= 0.0 && qy >= 0.0 && qx < gx && qy < gy;
    if (in_grid && g.cand_range) {
        const int cx = (int)qx >> LC_GRID_SHIFT, cy = (int)qy >> LC_GRID_SHIFT;
        const int2 rg = g.cand_range[cy * g.ncx + cx];
        if (rg.y >= 0) {
            // 4 independent (best, id) chains expose memory-level parallelism;
            // merging keeps the minimum with the lowest id on ties (exact)
            double b1 = LC_INF, b2 = LC_INF, b3 = LC_INF;
            int i1 = 0x7fffffff, i2 = 0x7fffffff, i3 = 0x7fffffff;
            const int2 *cp = g.cand_pts + rg.x;
            int k = 0;
            for (; k + 4 <= rg.y; k += 4) {
                const int2 c0 = __ldg(cp + k), c1 = __ldg(cp + k + 1), c2 = __ldg(cp + k + 2), c3 = __ldg(cp + k + 3);
                nn_consider_packed(c0, qx, qy, best, bi);
                nn_consider_packed(c1, qx, qy, b1, i1);
                nn_consider_packed(c2, qx, qy, b2, i2);
                nn_consider_packed(c3, qx, qy, b3, i3);
            }
            for (; k < rg.y; ++k) nn_consider_packed(__ldg(cp + k), qx, qy, best, bi);
            if (b1 < best || (b1 == best && i1 < bi)) { best = b1; bi = i1; }
            if (b2 < best || (b2 == best && i2 < bi)) { best = b2; bi = i2; }
            if (b3 < best || (b3 == best && i3 < bi)) { best = b3; bi = i3; }
            d2out = best;
            return bi;
        }
    }
    if (g.quad) {
        nn_quadtree(g, qx, qy, best, bi);
        d2out = best;
        return bi;
    }
    for (int k = 0; k < g.K; ++k) nn_consider(g, k, qx, qy, best, bi);
    d2out = best;
    return bi;
}

// ---- per-cell candidate lists (built once per mask) ----------------------
// squared farthest / nearest distance from cell c's square to point p
__device__ __forceinline__ double cell_far2(int cx, int cy, int2 p) {
    const double x0 = (double)(cx * LC_GRID_CELL), y0 = (double)(cy * LC_GRID_CELL);
    const double x1 = x0 + LC_GRID_CELL, y1 = y0 + LC_GRID_CELL;
    const double dx = fmax(fabs(p.x - x0), fabs(p.x - x1)), dy = fmax(fabs(p.y - y0), fabs(p.y - y1));
    return dx * dx + dy * dy;
}
__device__ __forceinline__ double cell_near2(int cx, int cy, int2 p) {
    const double x0 = (double)(cx * LC_GRID_CELL), y0 = (double)(cy * LC_GRID_CELL);
    const double x1 = x0 + LC_GRID_CELL, y1 = y0 + LC_GRID_CELL;
    const double dx = p.x < x0 ? x0 - p.x : (p.x > x1 ? p.x - x1 : 0.0);
    const double dy = p.y < y0 ? y0 - p.y : (p.y > y1 ? p.y - y1 : 0.0);
    return dx * dx + dy * dy;
}

// Visit every grid point within Chebyshev cell-rings [0, rmax] of (cx, cy),
// lanes striding over the cells of each ring.  Returns when `done(r)` after ring r.
template <typename F, typename D>
__device__ __forceinline__ void ring_visit_warp(const NnGridDev &g, int cx, int cy, F &&f, D &&done) {
    const int lane = threadIdx.x & 31;
    const int rmax = max(max(cx, g.ncx - 1 - cx), max(cy, g.ncy - 1 - cy));
    for (int r = 0; r <= rmax; ++r) {
        const int side = 2 * r + 1;
        const int ncell = r == 0 ? 1 : 8 * r;
        for (int k = lane; k < ncell; k += 32) {
            int xx, yy;
            if (r == 0) { xx = cx; yy = cy; }
            else if (k < side) { xx = cx - r + k; yy = cy - r; }
            else if (k < 2 * side) { xx = cx - r + (k - side); yy = cy + r; }
            else { const int m = k - 2 * side; xx = (m & 1) ? cx + r : cx - r; yy = cy - r + 1 + (m >> 1); }
            if (xx < 0 || yy < 0 || xx >= g.ncx || yy >= g.ncy) continue;
            const int c = yy * g.ncx + xx;
            for (int q = g.cell_start[c]; q < g.cell_start[c + 1]; ++q) f(g.cell_pts[q]);
        }
        if (done(r)) return;
    }
}

// continuous distance + unit direction away from the nearest contour point
struct NnResult { double dist, vx, vy; bool clamped; };

__device__ __forceinline__ NnResult field_nearest(const NnGridDev &g, double qx, double qy,
                                                  int *hint = nullptr) {
    NnResult r;
    const bool fin = isfinite(qx) && isfinite(qy);
    if (!fin) { qx = 0.0; qy = 0.0; }
    double d2;
    const int k = nn_query(g, qx, qy, d2, hint ? *hint : -1);
    if (hint && k >= 0 && k < g.K) *hint = k;
    if (k < 0 || k >= g.K) { r.dist = LC_INF; r.vx = r.vy = 0.0; r.clamped = true; return r; }
    const double d = sqrt(d2);
    const int2 p = g.pts[k];
    const double safe = d > 1e-12 ? d : 1e-12;
    const bool dirok = (d > 1e-12) && fin;
    r.vx = dirok ? (qx - (double)p.x) / safe : 0.0;
    r.vy = dirok ? (qy - (double)p.y) / safe : 0.0;
    r.dist = fin ? d : 0.0;
    r.clamped = !fin;
    return r;
}

// C^1 interface residual (DistanceField.sample_residual, imageproc.py:225-243)
__device__ __forceinline__ void field_residual(const NnResult &n, double &res, double &gx,
                                               double &gy) {
    const double lo = 0.5 - 0.15, hi = 0.5 + 0.15;
    double t = n.dist - lo;
    t = t < 0.0 ? 0.0 : (t > hi - lo ? hi - lo : t);
    const bool far = n.dist >= hi;
    res = far ? n.dist - 0.5 : t * t / (4.0 * 0.15);
    const double slope = far ? 1.0 : t / (2.0 * 0.15);
    gx = n.vx * slope;
    gy = n.vy * slope;
}

__device__ __forceinline__ double field_interface(const NnResult &n) {
    const double v = n.dist - 0.5;
    return v > 0.0 ? v : 0.0;
}

// nearest-pixel foreground test (DistanceField.inside, imageproc.py:254-261); np.round == rint
__device__ __forceinline__ bool field_inside(const NnGridDev &g, double x, double y) {
    const double xr = rint(x), yr = rint(y);
    if (!(xr >= 0.0 && xr < (double)g.W && yr >= 0.0 && yr < (double)g.H)) return false;
    return g.mask[(int)yr * g.W + (int)xr] != 0;
}

// contour side sign (pose_stage.py:194-215): -1 iff inside and n . dir < 0
__device__ __forceinline__ double side_sign(const NnGridDev &g, const NnResult &n, double px,
                                            double py, double n2x, double n2y) {
    if (!field_inside(g, px, py)) return 1.0;
    return (n2x * n.vx + n2y * n.vy) < 0.0 ? -1.0 : 1.0;
}

// ---------------------------------------------------------------------------
// bilinear sample of an (H,W,3) image with the analytic gradient
// (sample_bilinear, imageproc.py:127-174)

__device__ __forceinline__ bool bilinear3(const double *img, int W, int H, double x, double y,
                                          double val[3], double gx[3], double gy[3]) {
    const bool clamped = (x < 0) || (x > W - 1) || (y < 0) || (y > H - 1);
    const double xc = fmin(fmax(x, 0.0), (double)(W - 1));
    const double yc = fmin(fmax(y, 0.0), (double)(H - 1));
    const int x0 = min((int)floor(xc), W - 2), y0 = min((int)floor(yc), H - 2);
    const double fx = xc - x0, fy = yc - y0;
    const double *p00 = img + ((size_t)y0 * W + x0) * 3;
    const double *p10 = p00 + (size_t)W * 3;
    const bool inx = (x >= 0) && (x <= W - 1), iny = (y >= 0) && (y <= H - 1);
    for (int c = 0; c < 3; ++c) {
        const double c00 = p00[c], c01 = p00[3 + c], c10 = p10[c], c11 = p10[3 + c];
        const double top = c00 * (1 - fx) + c01 * fx;
        const double bot = c10 * (1 - fx) + c11 * fx;
        val[c] = top * (1 - fy) + bot * fy;
        gx[c] = inx ? (c01 - c00) * (1 - fy) + (c11 - c10) * fy : 0.0;
        gy[c] = iny ? bot - top : 0.0;
    }
    return clamped;
}

// ---------------------------------------------------------------------------
// symmetric 3x3 inverse via the adjugate; s = (xx, xy, xz, yy, yz, zz)
__device__ __forceinline__ bool sym3_inverse(const double s[6], double o[6]) {
    const double a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5];
    const double A = d * f - e * e, B = c * e - b * f, C = b * e - c * d;
    const double det = a * A + b * B + c * C;
    if (det == 0.0 || !isfinite(det)) return false;
    const double id = 1.0 / det;
    o[0] = A * id;
    o[1] = B * id;
    o[2] = C * id;
    o[3] = (a * f - c * c) * id;
    o[4] = (b * c - a * e) * id;
    o[5] = (a * d - b * b) * id;
    return true;
}
__device__ __forceinline__ V3 sym3_mul(const double s[6], V3 v) {
    return V3{s[0] * v.x + s[1] * v.y + s[2] * v.z, s[1] * v.x + s[3] * v.y + s[4] * v.z,
              s[2] * v.x + s[4] * v.y + s[5] * v.z};
}
