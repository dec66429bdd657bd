/*
 * ORACLE (test infrastructure only; never linked into the product).
 *
 * Plain-C restatement of the reference's two numba kernels:
 *   - sequential depth-buffered triangle rasterizer
 *       reference pkg/src/montrack/rasterizer.py:18-68 (_raster_core)
 *   - exact squared Euclidean distance transform (column sweeps, then the
 *     lower envelope of parabolas per row)
 *       reference pkg/src/montrack/imageproc.py:52-115 (_edt_squared)
 *
 * Arithmetic is fp64 in the reference's operation order; build with
 * -ffp-contract=off so a*b+c is never fused (numba without fastmath does
 * not fuse either).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

/* mode 0: depth only, 1: + barycentric attributes, 2: + max-barycentric id */
void oracle_raster(int h, int w, const double *pix, const double *depth,
                   const int64_t *tris, int64_t n_tris,
                   const double *attrs, int n_attr, const int64_t *ids,
                   double *zbuf, double *abuf, int64_t *ibuf, int mode)
{
    for (int64_t t = 0; t < n_tris; ++t) {
        const int64_t a = tris[3 * t], b = tris[3 * t + 1], c = tris[3 * t + 2];
        if (depth[a] <= 0.0 || depth[b] <= 0.0 || depth[c] <= 0.0)
            continue;
        const double ax = pix[2 * a], ay = pix[2 * a + 1];
        const double bx = pix[2 * b], by = pix[2 * b + 1];
        const double cx = pix[2 * c], cy = pix[2 * c + 1];
        const double area = (bx - ax) * (cy - ay) - (cx - ax) * (by - ay);
        if (area > -1e-12 && area < 1e-12)
            continue;
        double lo_x = fmin(ax, fmin(bx, cx)), hi_x = fmax(ax, fmax(bx, cx));
        double lo_y = fmin(ay, fmin(by, cy)), hi_y = fmax(ay, fmax(by, cy));
        long x0 = (long)floor(lo_x), x1 = (long)ceil(hi_x);
        long y0 = (long)floor(lo_y), y1 = (long)ceil(hi_y);
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > w - 1) x1 = w - 1;
        if (y1 > h - 1) y1 = h - 1;
        const double inv = 1.0 / area;
        for (long py = y0; py <= y1; ++py) {
            const double fy = (double)py;
            for (long px = x0; px <= x1; ++px) {
                const double fx = (double)px;
                const double l0 = ((bx - fx) * (cy - fy) - (cx - fx) * (by - fy)) * inv;
                const double l1 = ((fx - ax) * (cy - ay) - (cx - ax) * (fy - ay)) * inv;
                const double l2 = 1.0 - l0 - l1;
                if (l0 < 0.0 || l1 < 0.0 || l2 < 0.0)
                    continue;
                const double z = l0 * depth[a] + l1 * depth[b] + l2 * depth[c];
                const long pi = py * (long)w + px;
                if (!(z < zbuf[pi]))
                    continue;
                zbuf[pi] = z;
                if (mode == 1) {
                    for (int k = 0; k < n_attr; ++k)
                        abuf[pi * n_attr + k] = l0 * attrs[a * n_attr + k]
                                              + l1 * attrs[b * n_attr + k]
                                              + l2 * attrs[c * n_attr + k];
                } else if (mode == 2) {
                    int64_t pick;
                    if (l0 >= l1 && l0 >= l2) pick = ids[a];
                    else if (l1 >= l2) pick = ids[b];
                    else pick = ids[c];
                    ibuf[pi] = pick;
                }
            }
        }
    }
}

#define EDT_INF 1e18

/* out[y,x] = squared distance to the nearest nonzero feature pixel
 * (EDT_INF when the image has no feature). */
void oracle_edt_squared(int h, int w, const uint8_t *feature, double *out)
{
    double *col = (double *)malloc(sizeof(double) * (size_t)h * w);
    /* vertical pass: distance along each column to the nearest feature */
    for (int x = 0; x < w; ++x) {
        double run = EDT_INF;
        for (int y = 0; y < h; ++y) {
            if (feature[(size_t)y * w + x]) run = 0.0;
            else if (run < EDT_INF) run += 1.0;
            col[(size_t)y * w + x] = run;
        }
        run = EDT_INF;
        for (int y = h - 1; y >= 0; --y) {
            if (feature[(size_t)y * w + x]) run = 0.0;
            else if (run < EDT_INF) run += 1.0;
            if (run < col[(size_t)y * w + x]) col[(size_t)y * w + x] = run;
        }
    }
    for (size_t i = 0; i < (size_t)h * w; ++i)
        if (col[i] < EDT_INF) col[i] = col[i] * col[i];

    /* horizontal pass: lower envelope of parabolas f(q) + (x-q)^2 */
    int *site = (int *)malloc(sizeof(int) * w);
    double *bound = (double *)malloc(sizeof(double) * (w + 1));
    for (int y = 0; y < h; ++y) {
        const double *f = col + (size_t)y * w;
        int top = -1;
        for (int q = 0; q < w; ++q) {
            if (f[q] >= EDT_INF) continue;
            double s = 0.0;
            while (top >= 0) {
                const int v = site[top];
                s = ((f[q] + (double)q * q) - (f[v] + (double)v * v)) / (2.0 * (q - v));
                if (s <= bound[top]) --top;
                else break;
            }
            if (top < 0) {
                top = 0;
                site[0] = q;
                bound[0] = -EDT_INF;
                bound[1] = EDT_INF;
            } else {
                ++top;
                site[top] = q;
                bound[top] = s;
                bound[top + 1] = EDT_INF;
            }
        }
        double *o = out + (size_t)y * w;
        if (top < 0) {
            for (int x = 0; x < w; ++x) o[x] = EDT_INF;
            continue;
        }
        int k = 0;
        for (int x = 0; x < w; ++x) {
            while (bound[k + 1] < x) ++k;
            const double dx = (double)(x - site[k]);
            o[x] = dx * dx + f[site[k]];
        }
    }
    free(site);
    free(bound);
    free(col);
}
