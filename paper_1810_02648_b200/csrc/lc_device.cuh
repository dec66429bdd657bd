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

// A site is identified by its key y << 16 | x.  Contour pixels are indexed
// in np.argwhere (row-major) order, so ascending keys are ascending indices
// and the lowest-index tie break is the lowest-key tie break.
__device__ __forceinline__ int site_key(int2 p) { return (p.y << 16) | p.x; }
__device__ __forceinline__ int2 site_xy(int key) { return make_int2(key & 0xffff, key >> 16); }

__device__ __forceinline__ void nn_consider_key(int key, double qx, double qy, double &best, int &bk) {
    const double dx = qx - (double)(key & 0xffff), dy = qy - (double)(key >> 16);
    const double d2 = dx * dx + dy * dy;
    if (d2 < best || (d2 == best && key < bk)) { best = d2; bk = key; }
}

__device__ __forceinline__ void nn_consider(const NnGridDev &g, int pid, double qx, double qy,
                                            double &best, int &bk) {
    nn_consider_key(site_key(g.pts[pid]), qx, qy, best, bk);
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

#ifdef LC_NN_STATS
__device__ unsigned long long g_nn_stats[16];   // queries, list entries read, quadtree queries, hinted, max walk cycles, its steps, max steps, total steps
#endif

// Up to 16 keys of a sorted candidate list at once.  A single-precision
// pass (no serial chain through the running best; fp32 issues far faster
// than fp64) bounds the batch: with |q| < 2^11 the float distance is within
// 1e-3 px of the exact one, so only keys whose float squared distance is
// within thr = m (1 + 1e-5) + 1e-2 of the smaller of the batch's float
// minimum and the running best can win or tie, and only those are measured
// exactly in fp64 (the reference's arithmetic) and merged into (best, bk)
// in (distance, key) order.  `stop` is set when the batch's last key is
// farther from the cell than best: every later key of the sorted list is
// then strictly farther than the answer.  Exact and order-independent.
__device__ __forceinline__ void nn_batch16(const int *e, int n, int x0, int y0, double qx, double qy,
                                           float qxf, float qyf, double &best, int &bk, bool &stop) {
    float df[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const float dx = qxf - (float)(e[u] & 0xffff), dy = qyf - (float)(e[u] >> 16);
        df[u] = u < n ? fmaf(dx, dx, dy * dy) : __int_as_float(0x7f800000);
    }
    float m = df[0];
#pragma unroll
    for (int u = 1; u < 16; ++u) m = fminf(m, df[u]);
    const float lim = fminf(m, (float)best);
    const float thr = fmaf(lim, 1e-5f, lim) + 1e-2f;
#pragma unroll
    for (int u = 0; u < 16; ++u)
        if (df[u] <= thr) nn_consider_key(e[u], qx, qy, best, bk);
    int last = e[0];
#pragma unroll
    for (int u = 1; u < 16; ++u) if (u < n) last = e[u];
    const int px = last & 0xffff, py = last >> 16;
    const int ex = px < x0 ? x0 - px : (px > x0 + LC_GRID_CELL ? px - (x0 + LC_GRID_CELL) : 0);
    const int ey = py < y0 ? y0 - py : (py > y0 + LC_GRID_CELL ? py - (y0 + LC_GRID_CELL) : 0);
    if ((double)(ex * ex + ey * ey) > best) stop = true;
}

// Returns the key of the nearest site (INT_MAX if there is none).  `hint`
// (a site key of this grid, or -1) only seeds the search bound: the result
// is the exact nearest site with the lowest-key tie break whatever the hint.
static __device__ __noinline__ int nn_query(const NnGridDev &g, double qx, double qy, double &d2out, int hint = -1) {
    double best = LC_INF;
    int bk = 0x7fffffff;
    if (hint >= 0) nn_consider_key(hint, qx, qy, best, bk);
    const double gx = (double)(g.ncx * LC_GRID_CELL), gy = (double)(g.ncy * LC_GRID_CELL);
    const bool in_grid = qx >= 0.0 && qy >= 0.0 && qx < gx && qy < gy;
    if (in_grid && g.cand_blk) {
        // One 128 B line holds the cell's list range and the first
        // LC_CAND_HEAD keys.  The list is sorted by (cell distance, key):
        // stop at the first entry whose distance to the cell exceeds the
        // best squared distance (it and every later entry are strictly
        // farther, so ties are still all seen).
        const int cx = (int)qx >> LC_GRID_SHIFT, cy = (int)qy >> LC_GRID_SHIFT;
        const int4 *blk = reinterpret_cast<const int4 *>(g.cand_blk) + 8 * (size_t)(cy * g.ncx + cx);
        int4 h4[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) h4[u] = __ldg(blk + u);
        const int start = h4[0].x, cnt = h4[0].y;
        if (cnt >= 0) {
            const int x0 = cx << LC_GRID_SHIFT, y0 = cy << LC_GRID_SHIFT;
            const float qxf = (float)qx, qyf = (float)qy;
            const int head[32] = {h4[0].z, h4[0].w, h4[1].x, h4[1].y, h4[1].z, h4[1].w, h4[2].x, h4[2].y,
                                  h4[2].z, h4[2].w, h4[3].x, h4[3].y, h4[3].z, h4[3].w, h4[4].x, h4[4].y,
                                  h4[4].z, h4[4].w, h4[5].x, h4[5].y, h4[5].z, h4[5].w, h4[6].x, h4[6].y,
                                  h4[6].z, h4[6].w, h4[7].x, h4[7].y, h4[7].z, h4[7].w, -1, -1};
            // long lists: put every line of the tail in flight now (L1
            // prefetch, no registers), so the batches below mostly hit L1
            // instead of paying one L2 round trip per 128 B line in turn
            if (cnt > LC_CAND_HEAD) {
                const uintptr_t l0 = reinterpret_cast<uintptr_t>(g.cand_pts + start + LC_CAND_HEAD - 2) & ~uintptr_t(127);
                const uintptr_t l1 = reinterpret_cast<uintptr_t>(g.cand_pts + start + cnt - 1);
                for (uintptr_t l = l0; l <= l1; l += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(l));
            }
            bool stop = false;
            nn_batch16(head, min(cnt, 16), x0, y0, qx, qy, qxf, qyf, best, bk, stop);
            if (!stop && cnt > 16) nn_batch16(head + 16, min(cnt, LC_CAND_HEAD) - 16, x0, y0, qx, qy, qxf, qyf, best, bk, stop);
#ifdef LC_NN_STATS
            int scanned = min(cnt, stop ? 16 : LC_CAND_HEAD);
#endif
            // the tail, 16 keys (4 x 128-bit loads) at a time; it restarts
            // at the aligned index 28 (re-visiting two head keys is harmless)
            const int4 *cp = reinterpret_cast<const int4 *>(g.cand_pts + start);
            for (int k = LC_CAND_HEAD - 2; k < cnt && !stop; k += 16) {
#ifdef LC_NN_STATS
                scanned += min(16, cnt - k);
#endif
                int4 e4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    e4[u] = k + 4 * u < cnt ? __ldg(cp + (k >> 2) + u) : make_int4(-1, -1, -1, -1);
                const int e[16] = {e4[0].x, e4[0].y, e4[0].z, e4[0].w, e4[1].x, e4[1].y, e4[1].z, e4[1].w,
                                   e4[2].x, e4[2].y, e4[2].z, e4[2].w, e4[3].x, e4[3].y, e4[3].z, e4[3].w};
                nn_batch16(e, min(16, cnt - k), x0, y0, qx, qy, qxf, qyf, best, bk, stop);
            }
#ifdef LC_NN_STATS
            atomicAdd(&g_nn_stats[0], 1ull);
            atomicAdd(&g_nn_stats[1], (unsigned long long)scanned);
            atomicMax(&g_nn_stats[8], (unsigned long long)scanned);
            atomicMax(&g_nn_stats[9], (unsigned long long)cnt);
            atomicAdd(&g_nn_stats[10 + min(5, scanned / 64)], 1ull);
            if (hint >= 0) atomicAdd(&g_nn_stats[3], 1ull);
#endif
            d2out = best;
            return bk;
        }
    }
#ifdef LC_NN_STATS
    atomicAdd(&g_nn_stats[2], 1ull);
#endif
    if (g.quad) {
        nn_quadtree(g, qx, qy, best, bk);
        d2out = best;
        return bk;
    }
    for (int k = 0; k < g.K; ++k) nn_consider(g, k, qx, qy, best, bk);
    d2out = best;
    return bk;
}

// ---- per-cell candidate lists (built once per mask) ----------------------
// squared farthest / nearest distance from cell c's square to point p
__device__ __forceinline__ double cell_far2(int cx, int cy, int2 p) {
    const double x0 = (double)(cx * LC_GRID_CELL), y0 = (double)(cy * LC_GRID_CELL);
    const double x1 = x0 + LC_GRID_CELL, y1 = y0 + LC_GRID_CELL;
    const double dx = fmax(fabs(p.x - x0), fabs(p.x - x1)), dy = fmax(fabs(p.y - y0), fabs(p.y - y1));
    return dx * dx + dy * dy;
}
__device__ __forceinline__ int cell_near2_int(int cx, int cy, int2 p) {
    const int x0 = cx * LC_GRID_CELL, y0 = cy * LC_GRID_CELL;
    const int x1 = x0 + LC_GRID_CELL, y1 = y0 + LC_GRID_CELL;
    const int dx = p.x < x0 ? x0 - p.x : (p.x > x1 ? p.x - x1 : 0);
    const int dy = p.y < y0 ? y0 - p.y : (p.y > y1 ? p.y - y1 : 0);
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

// Bounded exact query: the squared distance to the nearest site when some
// site lies within R of (qx, qy), else +inf.  Only the cells overlapping the
// square of half-side R around the query are scanned (any site within R
// lies in one of them), so no search structure beyond the cell buckets is
// needed.  Threshold tests of the reference (rim distance <= 1.5 px,
// thickness probes >= 6 px) are decided exactly by it.
__device__ inline double nn_within2(const NnGridDev &g, double qx, double qy, double R) {
    double best = LC_INF;
    if (!(isfinite(qx) && isfinite(qy))) return best;
    const int cx0 = max(0, (int)floor((qx - R) / LC_GRID_CELL));
    const int cx1 = min(g.ncx - 1, (int)floor((qx + R) / LC_GRID_CELL));
    const int cy0 = max(0, (int)floor((qy - R) / LC_GRID_CELL));
    const int cy1 = min(g.ncy - 1, (int)floor((qy + R) / LC_GRID_CELL));
    for (int cy = cy0; cy <= cy1; ++cy)
        for (int cx = cx0; cx <= cx1; ++cx) {
            const int c = cy * g.ncx + cx;
            const int k0 = g.cell_start[c], k1 = g.cell_start[c + 1];
            for (int k = k0; k < k1; ++k) {
                const int2 p = g.pts[g.cell_pts[k]];
                const double dx = qx - (double)p.x, dy = qy - (double)p.y;
                best = fmin(best, dx * dx + dy * dy);
            }
        }
    return best <= R * R ? best : LC_INF;
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
    if (k == 0x7fffffff) { r.dist = LC_INF; r.vx = r.vy = 0.0; r.clamped = true; return r; }
    if (hint) *hint = k;
    const double d = sqrt(d2);
    const int2 p = site_xy(k);
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

// the sample's cell: top-left pixel (x0, y0), fractions, flags
struct Bilin {
    int x0, y0;
    double fx, fy;
    bool clamped, inx, iny;
};

__device__ __forceinline__ Bilin bilinear_cell(int W, int H, double x, double y) {
    Bilin b;
    b.clamped = (x < 0) || (x > W - 1) || (y < 0) || (y > H - 1);
    const double xc = fmin(fmax(x, 0.0), (double)(W - 1));
    const double yc = fmin(fmax(y, 0.0), (double)(H - 1));
    b.x0 = min((int)floor(xc), W - 2);
    b.y0 = min((int)floor(yc), H - 2);
    b.fx = xc - b.x0;
    b.fy = yc - b.y0;
    b.inx = (x >= 0) && (x <= W - 1);
    b.iny = (y >= 0) && (y <= H - 1);
    return b;
}

// value + gradient of one channel from the cell's four corner values
__device__ __forceinline__ void bilinear_mix(const Bilin &b, double c00, double c01, double c10, double c11,
                                             double &val, double &gx, double &gy) {
    const double fx = b.fx, fy = b.fy;
    const double top = c00 * (1 - fx) + c01 * fx;
    const double bot = c10 * (1 - fx) + c11 * fx;
    val = top * (1 - fy) + bot * fy;
    gx = b.inx ? (c01 - c00) * (1 - fy) + (c11 - c10) * fy : 0.0;
    gy = b.iny ? bot - top : 0.0;
}

__device__ __forceinline__ bool bilinear3(const double *img, int W, int H, double x, double y,
                                          double val[3], double gx[3], double gy[3]) {
    const Bilin b = bilinear_cell(W, H, x, y);
    const double *p00 = img + ((size_t)b.y0 * W + b.x0) * 3;
    const double *p10 = p00 + (size_t)W * 3;
    for (int c = 0; c < 3; ++c) bilinear_mix(b, p00[c], p00[3 + c], p10[c], p10[3 + c], val[c], gx[c], gy[c]);
    return b.clamped;
}

// One pixel of a blur-pyramid level computed from the raw frame with the
// fused pyramid kernel's arithmetic (pyr_level, lc_setup.cu: vertical pass
// over clamped rows, then horizontal over clamped columns, centre tap first,
// symmetric pairs outermost inward) -- bit-identical to the stored level.
// tp: the level's taps, centre at tp[h].
static __device__ __noinline__ double blur_at(const double *img, int W, int H, const double *tp, int h, int y, int x,
                                       int ch) {
    auto vert = [&](int xx) -> double {
        xx = min(max(xx, 0), W - 1);
        double acc = img[((size_t)y * W + xx) * 3 + ch] * tp[h];
        for (int j = h; j >= 1; --j) {
            const int ya = max(y - j, 0), yb = min(y + j, H - 1);
            acc = acc + (img[((size_t)ya * W + xx) * 3 + ch] + img[((size_t)yb * W + xx) * 3 + ch]) * tp[h + j];
        }
        return acc;
    };
    double acc = vert(x) * tp[h];
    for (int j = h; j >= 1; --j) acc = acc + (vert(x - j) + vert(x + j)) * tp[h + j];
    return acc;
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
// np.linalg.inv of one 3x3 block (LAPACK getrf + getrs on the identity):
// LU with partial pivoting (first maximal |pivot|), the multipliers scaled
// by the pivot's reciprocal (dgetf2), then forward / back substitution per
// identity column.  Agrees with numpy to ~1e-11 relative even on blocks of
// condition 1e7, where the adjugate formula is off by 1e-5 (the photometric
// blocks are nearly rank-deficient).  false when a pivot is exactly zero
// (np.linalg.inv raises; the caller switches to pinv).
__device__ inline bool lu_inv3(const double m[9], double o[9]) {
    double a[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) a[i][j] = m[3 * i + j];
    int piv[3] = {0, 1, 2};
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
        int p = k;
        double best = fabs(a[k][k]);
        for (int i = k + 1; i < 3; ++i)
            if (fabs(a[i][k]) > best) { best = fabs(a[i][k]); p = i; }
        if (p != k) {
            for (int j = 0; j < 3; ++j) { const double t = a[k][j]; a[k][j] = a[p][j]; a[p][j] = t; }
            const int t = piv[k]; piv[k] = piv[p]; piv[p] = t;
        }
        if (a[k][k] == 0.0) { ok = false; continue; }
        const double r = 1.0 / a[k][k];
        for (int i = k + 1; i < 3; ++i) a[i][k] *= r;
        for (int i = k + 1; i < 3; ++i)
            for (int j = k + 1; j < 3; ++j) a[i][j] -= a[i][k] * a[k][j];
    }
    if (!ok || !(isfinite(a[0][0]) && isfinite(a[1][1]) && isfinite(a[2][2]))) return false;
    for (int j = 0; j < 3; ++j) {
        double b[3];
        for (int i = 0; i < 3; ++i) b[i] = piv[i] == j ? 1.0 : 0.0;
        for (int i = 1; i < 3; ++i)
            for (int k = 0; k < i; ++k) b[i] -= a[i][k] * b[k];
        for (int i = 2; i >= 0; --i) {
            for (int k = i + 1; k < 3; ++k) b[i] -= a[i][k] * b[k];
            b[i] /= a[i][i];
        }
        for (int i = 0; i < 3; ++i) o[3 * i + j] = b[i];
    }
    return true;
}

// Eigen-decomposition of a symmetric 3x3 (full storage m[9], row-major) by
// cyclic Jacobi rotations: m = V diag(lam) V^T, eigenvectors in V's columns.
__device__ inline void sym3_eig(const double m_in[9], double lam[3], double V[9]) {
    double a[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            a[i][j] = m_in[3 * i + j];
            V[3 * i + j] = i == j ? 1.0 : 0.0;
        }
    for (int sweep = 0; sweep < 50; ++sweep) {
        const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
        const double dia = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
        if (off == 0.0 || off <= 1e-36 * dia) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                if (a[p][q] == 0.0) continue;
                const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {   // a <- a G (columns p, q)
                    const double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {   // a <- G^T a (rows p, q)
                    const double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {   // V <- V G
                    const double vkp = V[3 * k + p], vkq = V[3 * k + q];
                    V[3 * k + p] = c * vkp - s * vkq;
                    V[3 * k + q] = s * vkp + c * vkq;
                }
            }
    }
    for (int i = 0; i < 3; ++i) lam[i] = a[i][i];
}

// Moore-Penrose pseudo-inverse of a 3x3 block (np.linalg.pinv, rcond 1e-15:
// singular values <= 1e-15 * max are dropped).  The reference switches every
// Jacobi block to pinv once np.linalg.inv hits an exactly singular block
// (solvers.py:110-114).  Symmetric blocks (every normal-system diagonal) use
// their eigen-decomposition (s = |lam|, pinv = sum v v^T / lam); general ones
// the eigen-decomposition of A^T A (pinv = sum v (A v)^T / s^2).
__device__ inline void pinv3(const double a[9], double o[9]) {
    const bool sym = a[1] == a[3] && a[2] == a[6] && a[5] == a[7];
    double B[9];
    if (sym)
        for (int k = 0; k < 9; ++k) B[k] = a[k];
    else
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) B[3 * i + j] = a[i] * a[j] + a[3 + i] * a[3 + j] + a[6 + i] * a[6 + j];
    double lam[3], V[9];
    sym3_eig(B, lam, V);
    double sv[3], smax = 0.0;
    for (int k = 0; k < 3; ++k) {
        sv[k] = sym ? fabs(lam[k]) : sqrt(fmax(lam[k], 0.0));
        smax = fmax(smax, sv[k]);
    }
    const double cut = 1e-15 * smax;
    for (int k = 0; k < 9; ++k) o[k] = 0.0;
    for (int k = 0; k < 3; ++k) {
        if (!(sv[k] > cut)) continue;
        const double v0 = V[k], v1 = V[3 + k], v2 = V[6 + k];
        double u0, u1, u2, sc;
        if (sym) { u0 = v0; u1 = v1; u2 = v2; sc = 1.0 / lam[k]; }
        else {
            u0 = a[0] * v0 + a[1] * v1 + a[2] * v2;
            u1 = a[3] * v0 + a[4] * v1 + a[5] * v2;
            u2 = a[6] * v0 + a[7] * v1 + a[8] * v2;
            sc = 1.0 / lam[k];
        }
        o[0] += sc * v0 * u0; o[1] += sc * v0 * u1; o[2] += sc * v0 * u2;
        o[3] += sc * v1 * u0; o[4] += sc * v1 * u1; o[5] += sc * v1 * u2;
        o[6] += sc * v2 * u0; o[7] += sc * v2 * u1; o[8] += sc * v2 * u2;
    }
}
__device__ __forceinline__ void sym3_pinv(const double s[6], double o[6]) {
    const double a[9] = {s[0], s[1], s[2], s[1], s[3], s[4], s[2], s[4], s[5]};
    double f[9];
    pinv3(a, f);
    o[0] = f[0]; o[1] = 0.5 * (f[1] + f[3]); o[2] = 0.5 * (f[2] + f[6]);
    o[3] = f[4]; o[4] = 0.5 * (f[5] + f[7]); o[5] = f[8];
}

__device__ __forceinline__ V3 sym3_mul(const double s[6], V3 v) {
    return V3{s[0] * v.x + s[1] * v.y + s[2] * v.z, s[1] * v.x + s[3] * v.y + s[4] * v.z,
              s[2] * v.x + s[4] * v.y + s[5] * v.z};
}
