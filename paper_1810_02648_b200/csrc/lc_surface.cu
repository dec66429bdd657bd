// Stage II: per-vertex non-rigid Gauss-Newton, one persistent CTA per stream.
//
// Reference: NonrigidProblem.evaluate / normal_system (nonrigid_stage.py:
// 189-304), pcg_solve (solvers.py:104-145), solve_nonrigid (:372-403) and
// snap_vertices (:417-500).
//
// The normal system is kept in compact matrix-free form:
//   diag_i  = Jp_i^T Jp_i + g_i g_i^T + sum_{e ni i} (a_e I + b_e d_e d_e^T) + (cv^2+ca^2) I
//   A_ij    = -(a_e I + b_e d_e d_e^T)           for every mesh edge e = {i, j}
// with a_e = cs_fwd^2 + cs_rev^2 and b_e = ce_fwd^2 + ce_rev^2 per-config
// constants and d_e the current unit edge direction.  Every CTA-wide sum is a
// fixed-order tree (deterministic); there are no atomics.
#include <cstdlib>
#include "lc_pose.cuh"
#include "lc_team.cuh"

namespace {

// 256 threads x 128 registers, 2 CTAs per SM: two streams' teams share each
// SM, so one team's barrier waits hide behind the other's work (measured
// +2.5% frames/s over 512 x 1 at the bench's 16 streams)
#ifndef LC_SURF_NT
#define LC_SURF_NT 256
#endif
// resident CTAs per SM the register budget is sized for
#ifndef LC_SURF_MINB
#define LC_SURF_MINB 2
#endif
constexpr int NT = LC_SURF_NT;

struct SurfCtx {
    const SurfJob *J;
    NnGridDev obs;
    ActorDev A;
    CamDev cam;
    EdgeConstDev ec;
    SurfHyperDev hp;
    int H, W, P, B, N, E;
    int lo, hi, p0, p1, b0, b1;   // own_ranges(): this CTA's vertices, visible rows, boundary rows
    bool has_prev;
    bool sil_on;
    double *red;
};

// one pyramid level as bilinear3 samples it: the stored level where its
// tile was computed (the pyramid's region of interest), else the same bits
// blurred on demand from the raw frame
struct LevelSrc {
    const double *lvl;
    const uint8_t *flags;   // null: every tile computed
    const double *raw;
    const double *taps;
    int half, tiles_x;
};

__device__ __forceinline__ LevelSrc level_src(const SurfCtx &c, int level) {
    LevelSrc L;
    L.lvl = c.J->pyr + (size_t)level * c.H * c.W * 3;
    L.flags = c.J->pyr_tile;
    L.raw = c.J->image;
    L.taps = c.hp.taps + 32 * level;
    L.half = c.hp.half[level];
    L.tiles_x = (c.W + LC_PYR_TILE - 1) / LC_PYR_TILE;
    return L;
}

// the sample's four pixels lie in computed tiles
__device__ __forceinline__ bool level_stored(const LevelSrc &L, int W, int H, double x, double y) {
    if (!L.flags) return true;
    const Bilin b = bilinear_cell(W, H, x, y);
    const int tx0 = b.x0 / LC_PYR_TILE, tx1 = (b.x0 + 1) / LC_PYR_TILE;
    const int ty0 = b.y0 / LC_PYR_TILE, ty1 = (b.y0 + 1) / LC_PYR_TILE;
    return L.flags[ty0 * L.tiles_x + tx0] && L.flags[ty0 * L.tiles_x + tx1] && L.flags[ty1 * L.tiles_x + tx0] &&
           L.flags[ty1 * L.tiles_x + tx1];
}

__device__ __forceinline__ bool bilinear3_src(const LevelSrc &L, int W, int H, double x, double y, double val[3],
                                              double gx[3], double gy[3]) {
    if (!L.flags) return bilinear3(L.lvl, W, H, x, y, val, gx, gy);
    const Bilin b = bilinear_cell(W, H, x, y);
    const int tx0 = b.x0 / LC_PYR_TILE, tx1 = (b.x0 + 1) / LC_PYR_TILE;
    const int ty0 = b.y0 / LC_PYR_TILE, ty1 = (b.y0 + 1) / LC_PYR_TILE;
    const bool stored = L.flags[ty0 * L.tiles_x + tx0] && L.flags[ty0 * L.tiles_x + tx1] &&
                        L.flags[ty1 * L.tiles_x + tx0] && L.flags[ty1 * L.tiles_x + tx1];
    if (stored) return bilinear3(L.lvl, W, H, x, y, val, gx, gy);
    for (int ch = 0; ch < 3; ++ch) {
        const double c00 = blur_at(L.raw, W, H, L.taps, L.half, b.y0, b.x0, ch);
        const double c01 = blur_at(L.raw, W, H, L.taps, L.half, b.y0, b.x0 + 1, ch);
        const double c10 = blur_at(L.raw, W, H, L.taps, L.half, b.y0 + 1, b.x0, ch);
        const double c11 = blur_at(L.raw, W, H, L.taps, L.half, b.y0 + 1, b.x0 + 1, ch);
        bilinear_mix(b, c00, c01, c10, c11, val[ch], gx[ch], gy[ch]);
    }
    return b.clamped;
}

// photometric row of visible vertex i at position p (nonrigid_stage.py:196-213)
struct PhotoRow { double r[3], J[3][3]; bool behind, pruned; };

// Returns false (o untouched) when `lazy` and the sample falls outside the
// pyramid's computed tiles: the row is then unknown but >= 0 (see
// surf_energy_trials).
__device__ __forceinline__ bool photo_row(const SurfCtx &c, const LevelSrc &img, int i, V3 p,
                                          bool with_jac, PhotoRow &o, bool lazy = false) {
    double px, py;
    const bool ok = project(c.cam, p, px, py);
    if (lazy && !level_stored(img, c.W, c.H, px, py)) return false;
    double val[3], gx[3], gy[3];
    const bool cl = bilinear3_src(img, c.W, c.H, px, py, val, gx, gy);
    const double *col = c.A.colors + 3 * (size_t)i;
    const double d0 = val[0] - col[0], d1 = val[1] - col[1], d2 = val[2] - col[2];
    const bool prune = sqrt(d0 * d0 + d1 * d1 + d2 * d2) > c.hp.tau;
    o.pruned = prune && ok && !cl;
    o.behind = !ok;
    const double w = sqrt(c.hp.w_photo) * ((ok && !cl && !prune) ? 1.0 : 0.0);
    o.r[0] = d0 * w; o.r[1] = d1 * w; o.r[2] = d2 * w;
    if (with_jac) {
        double a0, a2, b1, b2;
        proj_jac(c.cam, p, a0, a2, b1, b2);
        for (int ch = 0; ch < 3; ++ch) {
            o.J[ch][0] = (gx[ch] * a0 + gy[ch] * 0.0) * w;
            o.J[ch][1] = (gx[ch] * 0.0 + gy[ch] * b1) * w;
            o.J[ch][2] = (gx[ch] * a2 + gy[ch] * b2) * w;
        }
    }
    return true;
}

// silhouette row of boundary slot b (nonrigid_stage.py:215-233)
struct SilRow { double r, g[3]; bool behind; };

__device__ __forceinline__ void sil_row(const SurfCtx &c, int b, V3 p, bool with_jac, SilRow &o) {
    const SurfJob &J = *c.J;
    double px, py;
    const bool ok = project(c.cam, p, px, py);
    o.behind = !ok;
    if (!J.enabled[b]) {   // weight 0 (rim / part gating): the residual row is zero, no query needed
        o.r = 0.0;
        o.g[0] = o.g[1] = o.g[2] = 0.0;
        return;
    }
    const NnResult nn = field_nearest(c.obs, px, py, J.nn_hint ? J.nn_hint + b : nullptr);
    double val, gx, gy;
    field_residual(nn, val, gx, gy);
    const double w = sqrt(c.hp.w_sil) * ((ok && !nn.clamped && J.enabled[b]) ? 1.0 : 0.0);
    o.r = val * w;
    if (with_jac) {
        double a0, a2, b1, b2;
        proj_jac(c.cam, p, a0, a2, b1, b2);
        const double sign = J.directional ? side_sign(c.obs, nn, px, py, J.n2d[2 * b], J.n2d[2 * b + 1]) : 1.0;
        const double sc = w * sign;
        o.g[0] = (gx * a0 + gy * 0.0) * sc;
        o.g[1] = (gx * 0.0 + gy * b1) * sc;
        o.g[2] = (gx * a2 + gy * b2) * sc;
    }
}

// The edge's smooth + edge energies, both directed halves together:
// |(u c_f)|^2 + |(u c_r)|^2 = alpha |u|^2 with alpha = c_f^2 + c_r^2 (and
// beta for the length term) -- the reference's terms up to fp64 rounding.
// The assembly (e0) and the line-search trials (e1) use this same formula,
// so a zero step reproduces e0 exactly and is accepted (e1 <= e0) as in the
// reference.
__device__ __forceinline__ void edge_energy(const SurfCtx &c, int e, V3 u, double len_err, double &es,
                                            double &ee) {
    es = c.ec.alpha[e] * ((u.x * u.x + u.y * u.y) + u.z * u.z);
    ee = c.ec.beta[e] * (len_err * len_err);
}

// One mesh edge seen from one of its endpoints i (slot of i's adjacency):
// the reference's per-edge quantities (nonrigid_stage.py:235-255) with the
// edge oriented src -> dst exactly as the reference forms them, so both
// endpoints compute the same bits.
struct SlotEdge { V3 u, d, g; double len_err; bool degenerate; };

__device__ __forceinline__ void slot_edge(const SurfCtx &c, int e, bool src, V3 vi, V3 vsi, V3 vj, V3 vsj,
                                          double al, double be, SlotEdge &q) {
    const V3 ev = src ? vi - vj : vj - vi;
    const V3 sd = src ? vsi - vsj : vsj - vsi;
    q.u = ev - sd;
    const double len = norm3(ev);
    q.degenerate = len < 1e-9;
    if (q.degenerate) q.d = ld3(c.A.rest_dir + 3 * (size_t)e);
    else {
        const double l = fmax(len, 1e-300);
        q.d = v3(ev.x / l, ev.y / l, ev.z / l);
    }
    q.len_err = len - c.A.rest_len[e];
    q.g = al * q.u + be * (q.len_err * q.d);
}

// The team's work partition, shared by the assembly and the line-search
// trials so that both sum every energy term in the same order (a zero step
// reproduces e0 exactly and is accepted, as in the reference): CTA r owns
// the vertex chunk [lo, hi) (the PCG's chunk too), the visible rows
// [p0, p1) and boundary rows [b0, b1) of its vertices (both lists are in
// ascending vertex order), and every edge at its src endpoint's slot.
// Everything the assembly writes for a vertex is written by the vertex's
// own CTA, so its phases are separated by CTA barriers only.
__device__ __forceinline__ int lower_bound_ids(const int *ids, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (ids[m] < key) lo = m + 1;
        else hi = m;
    }
    return lo;
}

template <typename T>
__device__ __forceinline__ void own_ranges(SurfCtx &c) {
    const int chunk = (c.N + T::ctas - 1) / T::ctas;
    c.lo = min(c.N, T::rank() * chunk);
    c.hi = min(c.N, c.lo + chunk);
    const SurfJob &J = *c.J;
    c.p0 = J.vis ? lower_bound_ids(J.vis, c.P, c.lo) : 0;
    c.p1 = J.vis ? lower_bound_ids(J.vis, c.P, c.hi) : 0;
    c.b0 = J.bidx ? lower_bound_ids(J.bidx, c.B, c.lo) : 0;
    c.b1 = J.bidx ? lower_bound_ids(J.bidx, c.B, c.hi) : 0;
}

// energies of nt <= 4 line-search trials v + step * sc0 * 0.5^h at once (h < nt;
// sc0 a power of two, so every product is exact):
// each element's trials are evaluated back to back (their gathers and
// nearest-contour queries overlap), one team reduction for all 24 sums
constexpr int kSurfTrials = 4;
//
// Unless `exact`, a photometric row whose sample falls outside the blur
// pyramid's computed tiles (a wild trial step) is not evaluated: it adds 0
// and is counted in unk[h].  All energy terms are >= 0 and fp addition of
// non-negative values is monotone, so such a trial's sum is a lower bound of
// its exact energy: if it already exceeds e0 the trial is rejected exactly
// as the reference rejects it (rejected trials' energies are not reported);
// otherwise the caller re-evaluates the batch with `exact`.
template <typename T>
__device__ void surf_energy_trials(const SurfCtx &c, int level, const double *v, const double *step, int nt,
                                   double sc0, bool exact, double en[kSurfTrials][6], double unk[kSurfTrials]) {
    const SurfJob &J = *c.J;
    double acc[kSurfTrials * 7];
    for (int k = 0; k < kSurfTrials * 7; ++k) acc[k] = 0.0;
    const LevelSrc img = level_src(c, level);
    if (J.enable_photo)
        for (int k = c.p0 + (int)threadIdx.x; k < c.p1; k += NT) {
            const int i = J.vis[k];
            const V3 vi = ld3(v + 3 * (size_t)i), si = ld3(step + 3 * (size_t)i);
            double sc = sc0;
#pragma unroll
            for (int h = 0; h < kSurfTrials; ++h, sc *= 0.5) {
                if (h >= nt) break;
                PhotoRow o;
                if (photo_row(c, img, i, vi + sc * si, false, o, !exact))
                    acc[6 * h] += o.r[0] * o.r[0] + o.r[1] * o.r[1] + o.r[2] * o.r[2];
                else
                    acc[kSurfTrials * 6 + h] += 1.0;
            }
        }
    if (c.sil_on)
        for (int b = c.b0 + (int)threadIdx.x; b < c.b1; b += NT) {
            const int i = J.bidx[b];
            const V3 vi = ld3(v + 3 * (size_t)i), si = ld3(step + 3 * (size_t)i);
            double sc = sc0;
#pragma unroll
            for (int h = 0; h < kSurfTrials; ++h, sc *= 0.5) {
                if (h >= nt) break;
                SilRow o;
                sil_row(c, b, vi + sc * si, false, o);
                acc[6 * h + 1] += o.r * o.r;
            }
        }
    // (the next edge's endpoint ids are loaded one iteration ahead, so each
    // edge costs one dependent round trip: its vertex gathers)
    const int2 *edges2 = reinterpret_cast<const int2 *>(c.A.edges);
    int2 ab_next = T::tid() < c.E ? edges2[T::tid()] : make_int2(0, 0);
    for (int e = T::tid(); e < c.E; e += T::size) {
        // one load of the endpoints, their steps and V^S per edge for every
        // trial; energies only (the unit direction is not needed here)
        const int a = ab_next.x, b = ab_next.y;
        if (e + T::size < c.E) ab_next = edges2[e + T::size];
        const V3 va = ld3(v + 3 * (size_t)a), vb = ld3(v + 3 * (size_t)b);
        const V3 sa = ld3(step + 3 * (size_t)a), sb = ld3(step + 3 * (size_t)b);
        const V3 sd = ld3(J.vs + 3 * (size_t)a) - ld3(J.vs + 3 * (size_t)b);
        const double rl = c.A.rest_len[e];
        double sc = sc0;
#pragma unroll
        for (int h = 0; h < kSurfTrials; ++h, sc *= 0.5) {
            if (h >= nt) break;
            const V3 ev = (va + sc * sa) - (vb + sc * sb);
            double es, ee;
            edge_energy(c, e, ev - sd, norm3(ev) - rl, es, ee);
            acc[6 * h + 2] += es;
            acc[6 * h + 3] += ee;
        }
    }
    const double cv = sqrt(c.hp.w_vel), ca = sqrt(c.hp.w_acc);
    if (c.has_prev)
        for (int i = c.lo + (int)threadIdx.x; i < c.hi; i += NT) {
            const V3 vi = ld3(v + 3 * (size_t)i), si = ld3(step + 3 * (size_t)i);
            const V3 q1 = ld3(J.prev + 3 * (size_t)i);
            const V3 q2 = J.prev2 ? ld3(J.prev2 + 3 * (size_t)i) : q1;
            double sc = sc0;
#pragma unroll
            for (int h = 0; h < kSurfTrials; ++h, sc *= 0.5) {
                if (h >= nt) break;
                const V3 p = vi + sc * si;
                const V3 vr = (p - q1) * cv;
                const V3 ar = ((p - 2.0 * q1) + q2) * ca;
                acc[6 * h + 4] += vr.x * vr.x + vr.y * vr.y + vr.z * vr.z;
                acc[6 * h + 5] += ar.x * ar.x + ar.y * ar.y + ar.z * ar.z;
            }
        }
    // (the trials only read: v and the step were ordered by the team barrier
    // before this phase, and the caller's next global writes come after a
    // full barrier)
    T::template sums_light<kSurfTrials * 7>(acc, c.red);
    for (int h = 0; h < kSurfTrials; ++h) {
        for (int k = 0; k < 6; ++k) en[h][k] = acc[6 * h + k];
        unk[h] = acc[kSurfTrials * 6 + h];
    }
}

__device__ __forceinline__ double total_energy(const double en[6], bool has_prev) {
    double t = ((en[0] + en[1]) + en[2]) + en[3];
    if (has_prev) t = (t + en[4]) + en[5];
    return t;
}

// GN evaluation with the normal system (diag, minv, rhs, and the edge
// directions of every ELL slot / CSR-tail edge the matvec reads); returns
// energies + counters.  One edge-parallel pass evaluates every edge once
// (balanced over the team) and scatters its direction and signed gradient
// to the ELL slots of both endpoints; after that single team barrier the
// rest is owner-computes (see own_ranges): the CTA's photometric and
// silhouette rows, then its vertices' full blocks, separated by CTA
// barriers only, and one light team reduction at the end.
template <typename T>
__device__ void surf_assemble(const SurfCtx &c, int level, const double *v, double en[6],
                              int counts[3], int fine = -1) {
    const SurfJob &J = *c.J;
    auto fst = [&](int k) {
        if (fine >= 0 && J.phase && T::tid() == 0) J.phase[fine + k] = gtimer();
    };
    const double cv = sqrt(c.hp.w_vel), ca = sqrt(c.hp.w_acc);
    // 6 energies, pruned, behind, singular blocks, degenerate directed edges
    double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    // E: every edge once -- energies, direction, signed gradient into its
    // ELL slots at both endpoints (CSR tails: per edge, edir / eg)
    const size_t LN = (size_t)LC_ELL * c.N;
    const int2 *edges2 = reinterpret_cast<const int2 *>(c.A.edges);
    int2 ab_next = T::tid() < c.E ? edges2[T::tid()] : make_int2(0, 0);   // (one edge ahead)
    for (int e = T::tid(); e < c.E; e += T::size) {
        const int a = ab_next.x, b = ab_next.y;
        if (e + T::size < c.E) ab_next = edges2[e + T::size];
        const double al = c.ec.alpha[e], be = c.ec.beta[e];
        SlotEdge q;
        slot_edge(c, e, true, ld3(v + 3 * (size_t)a), ld3(J.vs + 3 * (size_t)a), ld3(v + 3 * (size_t)b),
                  ld3(J.vs + 3 * (size_t)b), al, be, q);
        double es, ee;
        edge_energy(c, e, q.u, q.len_err, es, ee);
        acc[2] += es;
        acc[3] += ee;
        acc[9] += q.degenerate ? 2.0 : 0.0;
        const int ps = c.A.epos[2 * e], pd = c.A.epos[2 * e + 1];
        if (ps >= 0) {   // the src side subtracts g
            J.ell_d[ps] = q.d.x; J.ell_d[LN + ps] = q.d.y; J.ell_d[2 * LN + ps] = q.d.z;
            J.ell_g[ps] = -q.g.x; J.ell_g[LN + ps] = -q.g.y; J.ell_g[2 * LN + ps] = -q.g.z;
        }
        if (pd >= 0) {
            J.ell_d[pd] = q.d.x; J.ell_d[LN + pd] = q.d.y; J.ell_d[2 * LN + pd] = q.d.z;
            J.ell_g[pd] = q.g.x; J.ell_g[LN + pd] = q.g.y; J.ell_g[2 * LN + pd] = q.g.z;
        }
        if (ps < 0 || pd < 0) {   // in a pole vertex's CSR tail
            st3(J.edir + 3 * (size_t)e, q.d);
            st3(J.eg + 3 * (size_t)e, q.g);
        }
    }
    // R0: clear the data blocks of the CTA's vertices
    for (int i = c.lo + (int)threadIdx.x; i < c.hi; i += NT) {
        double *dg = J.diag + 6 * (size_t)i;
        for (int k = 0; k < 6; ++k) dg[k] = 0.0;
        st3(J.rhs + 3 * (size_t)i, v3(0, 0, 0));
    }
    T::sync();   // the only team barrier before the reduction: slots written by any CTA
    fst(0);
    // R1: photometric data blocks (visible ids are unique)
    const LevelSrc img = level_src(c, level);
    if (J.enable_photo)
        for (int k = c.p0 + (int)threadIdx.x; k < c.p1; k += NT) {
            const int i = J.vis[k];
            PhotoRow o;
            photo_row(c, img, i, ld3(v + 3 * (size_t)i), true, o);
            acc[0] += o.r[0] * o.r[0] + o.r[1] * o.r[1] + o.r[2] * o.r[2];
            acc[6] += o.pruned ? 1.0 : 0.0;
            acc[7] += o.behind ? 1.0 : 0.0;
            double *dg = J.diag + 6 * (size_t)i;
            const int map[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
            for (int m = 0; m < 6; ++m) {
                const int a = map[m][0], b = map[m][1];
                dg[m] = o.J[0][a] * o.J[0][b] + o.J[1][a] * o.J[1][b] + o.J[2][a] * o.J[2][b];
            }
            double *rh = J.rhs + 3 * (size_t)i;
            for (int a = 0; a < 3; ++a)
                rh[a] = -(o.J[0][a] * o.r[0] + o.J[1][a] * o.r[1] + o.J[2][a] * o.r[2]);
        }
    __syncthreads();
    fst(1);
    // R2: silhouette rank-1 blocks (boundary ids are unique)
    if (c.sil_on)
        for (int b = c.b0 + (int)threadIdx.x; b < c.b1; b += NT) {
            const int i = J.bidx[b];
            SilRow o;
            sil_row(c, b, ld3(v + 3 * (size_t)i), true, o);
            acc[1] += o.r * o.r;
            acc[7] += o.behind ? 1.0 : 0.0;
            double *dg = J.diag + 6 * (size_t)i;
            dg[0] += o.g[0] * o.g[0]; dg[1] += o.g[0] * o.g[1]; dg[2] += o.g[0] * o.g[2];
            dg[3] += o.g[1] * o.g[1]; dg[4] += o.g[1] * o.g[2]; dg[5] += o.g[2] * o.g[2];
            double *rh = J.rhs + 3 * (size_t)i;
            rh[0] += -o.g[0] * o.r; rh[1] += -o.g[1] * o.r; rh[2] += -o.g[2] * o.r;
        }
    __syncthreads();
    fst(2);
    // R3: full diagonal blocks, rhs, Jacobi preconditioner, temporal
    // energies of the CTA's vertices; incident edges in the reference's
    // order: ELL slots (coalesced, independent loads), then the CSR tail
    for (int i = c.lo + (int)threadIdx.x; i < c.hi; i += NT) {
        double dg[6];
        for (int k = 0; k < 6; ++k) dg[k] = J.diag[6 * (size_t)i + k];
        V3 rh = ld3(J.rhs + 3 * (size_t)i);
        const int cnt = c.A.ell_cnt[i];
#pragma unroll
        for (int k = 0; k < LC_ELL; ++k) {
            if (k >= cnt) continue;
            const size_t pos = (size_t)k * c.N + i;
            const V3 d = v3(J.ell_d[pos], J.ell_d[LN + pos], J.ell_d[2 * LN + pos]);
            const double al = c.ec.ell_a[pos], be = c.ec.ell_b[pos];
            dg[0] += al + be * (d.x * d.x); dg[1] += be * (d.x * d.y); dg[2] += be * (d.x * d.z);
            dg[3] += al + be * (d.y * d.y); dg[4] += be * (d.y * d.z); dg[5] += al + be * (d.z * d.z);
            rh = rh + v3(J.ell_g[pos], J.ell_g[LN + pos], J.ell_g[2 * LN + pos]);
        }
        if (cnt > LC_ELL)
            for (int k = c.A.adj_ptr[i] + LC_ELL; k < c.A.adj_ptr[i + 1]; ++k) {
                const int e = c.A.adj_edge[k];
                const V3 d = ld3(J.edir + 3 * (size_t)e);
                const double al = c.ec.alpha[e], be = c.ec.beta[e];
                dg[0] += al + be * (d.x * d.x); dg[1] += be * (d.x * d.y); dg[2] += be * (d.x * d.z);
                dg[3] += al + be * (d.y * d.y); dg[4] += be * (d.y * d.z); dg[5] += al + be * (d.z * d.z);
                const V3 g = ld3(J.eg + 3 * (size_t)e);
                rh = (c.A.edges[2 * e] == i) ? rh - g : rh + g;
            }
        if (c.has_prev) {
            const double cc = cv * cv + ca * ca;
            dg[0] += cc; dg[3] += cc; dg[5] += cc;
            const V3 p = ld3(v + 3 * (size_t)i);
            const V3 q1 = ld3(J.prev + 3 * (size_t)i);
            const V3 q2 = J.prev2 ? ld3(J.prev2 + 3 * (size_t)i) : q1;
            const V3 vr = (p - q1) * cv;
            const V3 ar = ((p - 2.0 * q1) + q2) * ca;
            acc[4] += vr.x * vr.x + vr.y * vr.y + vr.z * vr.z;
            acc[5] += ar.x * ar.x + ar.y * ar.y + ar.z * ar.z;
            rh = rh - (cv * vr + ca * ar);
        }
        for (int k = 0; k < 6; ++k) J.diag[6 * (size_t)i + k] = dg[k];
        st3(J.rhs + 3 * (size_t)i, rh);
        // M^-1 = np.linalg.inv of the full block (LU; not symmetrised, as numpy)
        const double full[9] = {dg[0], dg[1], dg[2], dg[1], dg[3], dg[4], dg[2], dg[4], dg[5]};
        double mi[9];
        if (!lu_inv3(full, mi)) {
            acc[8] += 1.0;
            for (int k = 0; k < 9; ++k) mi[k] = 0.0;
        }
        for (int k = 0; k < 9; ++k) J.minv[9 * (size_t)i + k] = mi[k];
    }
    fst(3);
    // R1-R3 write only the CTA's own vertices, which the PCG reads from the
    // same CTA: the energies are the only team exchange left
    T::template sums_light<10>(acc, c.red);
    fst(4);
    // np.linalg.inv raised on an exactly singular block: the reference
    // pseudo-inverts every block (solvers.py:110-114)
    if (acc[8] > 0.0) {
        for (int i = c.lo + (int)threadIdx.x; i < c.hi; i += NT) {
            const double *dg = J.diag + 6 * (size_t)i;
            const double full[9] = {dg[0], dg[1], dg[2], dg[1], dg[3], dg[4], dg[2], dg[4], dg[5]};
            pinv3(full, J.minv + 9 * (size_t)i);
        }
        __syncthreads();
    }
    for (int k = 0; k < 6; ++k) en[k] = acc[k];
    counts[0] = (int)acc[6];
    counts[1] = (int)acc[9];
    counts[2] = (int)acc[7];
}

// Block-Jacobi PCG from zero, best-residual iterate (solvers.py:104-145).
//
// Team layout: CTA r of the team owns the contiguous vertex chunk
// [r*chunk, min(N, (r+1)*chunk)); thread t owns chunk vertices t, t+NT, ...
// for the whole solve.  The vectors a vertex's owner alone touches (p, Ap)
// and the one its neighbours gather (z) live in the owner's shared memory
// (pcg_mode 2; mode 1: z only, p / Ap in global scratch; mode 0: all in
// global scratch, for chunks too large for shared memory).  Mesh vertices
// are numbered ring by ring, so almost every neighbour z_j is a local
// shared-memory load; the few across a chunk border come over DSMEM.
//
// Each iteration needs exactly two team barriers, both inside the two
// reductions the algorithm requires anyway:
//   A: Az = A z (gathering z_j), p = z + beta p, Ap = Az + beta Ap,
//      sums p.Ap, p.p                                   -> barrier 1 (alpha)
//   B: x += alpha p, r -= alpha Ap, z = M^-1 r,
//      sums r.z, r.r                                    -> barrier 2 (beta;
//      also publishes the new z to the neighbours' next phase A)
// i.e. A p_k is formed as A z_k + beta A p_{k-1} (the same vector; fp64
// rounding order only) so the updated p never has to be exchanged.  The
// best iterate (smallest ||r||, strict) is copied from x by its owner one
// phase later, when the reduction has decided it.
template <typename T>
__device__ bool surf_pcg(const SurfCtx &c, int iters, double *sm, int mode, int fine = -1) {
    const SurfJob &J = *c.J;
    auto fst = [&](int k) {
        if (fine >= 0 && J.phase && T::tid() == 0) J.phase[fine + k] = gtimer();
    };
    fst(0);
    const int N = c.N;
    const int chunk = (N + T::ctas - 1) / T::ctas;
    const int lo = T::rank() * chunk, hi = min(N, lo + chunk);
    // own-vertex storage: zs / ps / aps indexed by (i - off)
    const bool z_sm = mode >= 1;
    // mode 3: z plus the chunk's ELL neighbour ids and counts in shared
    // memory, so the matvec's dependent chain (count -> neighbour id -> z_j)
    // never leaves the SM; the per-slot coefficients stream from L2 as
    // independent loads (the kernel prologue fills the ids once per solve)
    const bool idx_sm = mode == 3;
    double *zs = z_sm ? sm : J.z;
    double *ps = mode == 2 ? sm + 3 * (size_t)chunk : J.p;
    double *aps = mode == 2 ? sm + 6 * (size_t)chunk : J.ap;
    int *nbr_s = reinterpret_cast<int *>(sm + 3 * (size_t)chunk);   // [LC_ELL][chunk] (mode 3)
    int *cnt_s = nbr_s + (size_t)LC_ELL * chunk;                      // [chunk]
    const int zoff = z_sm ? lo : 0, poff = mode == 2 ? lo : 0;
    const double *__restrict__ diag = J.diag;
    const double *__restrict__ minv = J.minv;
    const double *__restrict__ rhs = J.rhs;
    const int *__restrict__ ell_nbr = c.A.ell_nbr;
    const int *__restrict__ ell_cnt = c.A.ell_cnt;
    const double *__restrict__ ell_d = J.ell_d;
    const double *__restrict__ ell_a = c.ec.ell_a;
    const double *__restrict__ ell_b = c.ec.ell_b;
    double *__restrict__ X = J.x;
    double *__restrict__ R = J.r;
    double *__restrict__ BEST = J.best;
    const size_t LN = (size_t)LC_ELL * N;
    // z_j of any vertex: own chunk from local shared memory, another CTA's
    // chunk over DSMEM, or global scratch (mode 0)
    auto zload = [&](int j) -> V3 {
        if (!z_sm) return ld3(zs + 3 * (size_t)j);
        if (j >= lo && j < hi) return ld3(zs + 3 * (size_t)(j - lo));
        if constexpr (T::ctas == 1) {
            return v3(0, 0, 0);   // unreachable: one CTA owns every vertex
        } else {
            const int owner = j / chunk;
            const double *q = cg::this_cluster().map_shared_rank(zs, owner) + 3 * (size_t)(j - owner * chunk);
            return v3(q[0], q[1], q[2]);
        }
    };
    // mode 3: the prologue stored each slot's neighbour as (owner CTA << 20 |
    // index in the owner's chunk), so the gather is one branch-free load
    // through the cluster's shared window (own CTA included): the 8 slots'
    // loads issue back to back
    auto zload_packed = [&](int q) -> V3 {
        const double *base;
        if constexpr (T::ctas == 1) base = zs;
        else base = cg::this_cluster().map_shared_rank(zs, (unsigned)q >> 20);
        const double *p = base + 3 * (size_t)(q & 0xFFFFF);
        return v3(p[0], p[1], p[2]);
    };
    double part[2] = {0, 0};
    for (int i = lo + (int)threadIdx.x; i < hi; i += NT) {
        const V3 r = ld3(rhs + 3 * (size_t)i);
        const V3 z = mat_vec(minv + 9 * (size_t)i, r);
        st3(X + 3 * (size_t)i, v3(0, 0, 0));
        st3(BEST + 3 * (size_t)i, v3(0, 0, 0));
        st3(R + 3 * (size_t)i, r);
        st3(zs + 3 * (size_t)(i - zoff), z);
        part[0] += r.x * z.x + r.y * z.y + r.z * z.z;
        part[1] += r.x * r.x + r.y * r.y + r.z * r.z;
    }
    // with z in shared memory every exchange inside the PCG is shared-memory
    // only (x, r, best, p, Ap are owner-only), so its reductions are the
    // light mbarrier handshake; mode 0 publishes z through global memory
    auto team_sums2 = [&](double (&v2)[2]) {
        if (z_sm) T::template sums_light<2>(v2, c.red);
        else T::template sums<2>(v2, c.red);
    };
    team_sums2(part);   // (also publishes z)
    fst(1);
    double rz = part[0];
    double best_norm = sqrt(part[1]);
    bool breakdown = false, pend_best = false;
    double beta = 0.0;
    // CSR tails of the few high-degree vertices (mesh poles, degree up to
    // ~50): one warp per vertex, lanes over the tail edges, into the
    // assembly's per-edge gradient buffer (consumed before the PCG starts)
    double *tail_y = J.eg;
    for (int it = 0; it < iters; ++it) {
        // ---- A: Az, p, Ap
        if (c.A.n_heavy > 0) {
            const int w = (int)threadIdx.x >> 5, lane = (int)threadIdx.x & 31;
            for (int h = w; h < c.A.n_heavy; h += NT / 32) {
                const int i = c.A.heavy[h];
                if (i < lo || i >= hi) continue;
                V3 acc = v3(0, 0, 0);
                for (int k = c.A.adj_ptr[i] + LC_ELL + lane; k < c.A.adj_ptr[i + 1]; k += 32) {
                    const int e = c.A.adj_edge[k];
                    const V3 zj = zload(c.A.adj_nbr[k]);
                    const V3 d = ld3(J.edir + 3 * (size_t)e);
                    acc = acc + (c.ec.alpha[e] * zj + (c.ec.beta[e] * dot3(d, zj)) * d);
                }
                for (int o = 16; o > 0; o >>= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
                }
                if (lane == 0) st3(tail_y + 3 * (size_t)h, acc);
            }
            __syncthreads();
        }
        double s1[2] = {0, 0};
        for (int i = lo + (int)threadIdx.x; i < hi; i += NT) {
            const V3 zi = ld3(zs + 3 * (size_t)(i - zoff));
            V3 y = sym3_mul(diag + 6 * (size_t)i, zi);
            const int cnt = idx_sm ? cnt_s[i - lo] : ell_cnt[i];
#pragma unroll
            for (int k = 0; k < LC_ELL; ++k) {
                if (k >= cnt) continue;
                const size_t pos = (size_t)k * N + i;
                const V3 zj = idx_sm ? zload_packed(nbr_s[(size_t)k * chunk + (i - lo)]) : zload(ell_nbr[pos]);
                const V3 d = v3(ell_d[pos], ell_d[LN + pos], ell_d[2 * LN + pos]);
                y = y - (ell_a[pos] * zj + (ell_b[pos] * dot3(d, zj)) * d);
            }
            if (cnt > LC_ELL) y = y - ld3(tail_y + 3 * (size_t)c.A.heavy_id[i]);
            V3 p = zi, ap = y;
            if (it > 0) {
                p = zi + beta * ld3(ps + 3 * (size_t)(i - poff));
                ap = y + beta * ld3(aps + 3 * (size_t)(i - poff));
            }
            st3(ps + 3 * (size_t)(i - poff), p);
            st3(aps + 3 * (size_t)(i - poff), ap);
            s1[0] += p.x * ap.x + p.y * ap.y + p.z * ap.z;
            s1[1] += p.x * p.x + p.y * p.y + p.z * p.z;
        }
        if (it == 0) fst(2);
        team_sums2(s1);
        if (it == 0) fst(3);
        const double pap = s1[0];
        if (pap <= 1e-14 * fmax(s1[1], 1e-300)) { breakdown = true; break; }
        const double alpha = rz / pap;
        // ---- B: x, r, z
        double s2[2] = {0, 0};
        for (int i = lo + (int)threadIdx.x; i < hi; i += NT) {
            V3 x = ld3(X + 3 * (size_t)i);
            if (pend_best) st3(BEST + 3 * (size_t)i, x);
            x = x + alpha * ld3(ps + 3 * (size_t)(i - poff));
            const V3 r = ld3(R + 3 * (size_t)i) - alpha * ld3(aps + 3 * (size_t)(i - poff));
            const V3 z = mat_vec(minv + 9 * (size_t)i, r);
            st3(X + 3 * (size_t)i, x);
            st3(R + 3 * (size_t)i, r);
            st3(zs + 3 * (size_t)(i - zoff), z);
            s2[0] += r.x * z.x + r.y * z.y + r.z * z.z;
            s2[1] += r.x * r.x + r.y * r.y + r.z * r.z;
        }
        if (it == 0) fst(4);
        team_sums2(s2);
        if (it == 0) fst(5);
        const double nrm = sqrt(s2[1]);
        pend_best = nrm < best_norm;
        if (pend_best) best_norm = nrm;
        const bool stop = rz <= 0.0;
        beta = stop ? 0.0 : s2[0] / rz;
        if (it == 0) fst(6);
        if (stop) { breakdown = true; break; }
        rz = s2[0];
    }
    if (pend_best)
        for (int i = lo + (int)threadIdx.x; i < hi; i += NT) st3(BEST + 3 * (size_t)i, ld3(X + 3 * (size_t)i));
    T::sync();   // the best iterate of every chunk, for the line search
    return breakdown;
}

// silhouette snapping (snap_vertices, nonrigid_stage.py:417-500)
template <typename T>
__device__ void surf_snap(const SurfCtx &c, double *v) {
    const SurfJob &J = *c.J;
    const SurfHyperDev &hp = c.hp;
    auto fst = [&](int k) {
        if (J.phase && T::tid() == 0) J.phase[24 + k] = gtimer();
    };
    fst(0);
    double cnt[4] = {0, 0, 0, 0};  // walked, reached, stuck, moved
    for (int i = T::tid(); i < c.N; i += T::size) {
        st3(J.off0 + 3 * (size_t)i, v3(0, 0, 0));
        J.hold[i] = 0;
    }
    T::sync();
    fst(1);
    // One thread per boundary vertex, so a 4-CTA team covers its ~700
    // boundary vertices in one round.  A walk step tries step, step/2,
    // step/4 along the gradient in order and takes the first trial that
    // lowers the interface distance (the sequential search); most steps take
    // the first trial, so a step is usually one query.  The accepted
    // trial's query is the next step's gradient query (same point, same
    // exact answer).  The loop is warp-uniform (finished walks idle).
    {
        constexpr int QPT = T::size;
        for (int b0 = 0; b0 < c.B; b0 += QPT) {
            const int b = b0 + T::tid();
            const bool valid = b < c.B;
            int i = 0;
            V3 p = v3(0, 0, 0);
            bool en = false;
            double px = 0.0, py = 0.0;
            int hint = -1;
            NnResult g{LC_INF, 0.0, 0.0, true};
            double sign = 1.0, val = 0.0;
            if (valid) {
                i = J.bidx[b];
                J.hold[i] = 1;
                p = ld3(v + 3 * (size_t)i);
                const bool ok = project(c.cam, p, px, py);
                en = J.enabled[b] && ok;
                if (en) {   // (a disabled row is neither walked nor counted)
                    hint = J.nn_hint ? J.nn_hint[b] : -1;
                    g = field_nearest(c.obs, px, py, &hint);
                    sign = side_sign(c.obs, g, px, py, J.n2d[2 * b], J.n2d[2 * b + 1]);
                    val = field_interface(g);
                }
            }
            double qx = px, qy = py;
            bool active = valid && en && val > hp.snap_band;
            bool stuck = false;
#ifdef LC_NN_STATS
            const long long w0 = clock64();
            int nsteps = 0;
#endif
            for (int s = 0; s < hp.snap_max_steps; ++s) {
                if (!__any_sync(0xffffffffu, active)) break;
#ifdef LC_NN_STATS
                nsteps += active ? 1 : 0;
#endif
                if (!active) continue;
                const double gn = sqrt(g.vx * g.vx + g.vy * g.vy);
                const bool good = gn > 1e-9;
                const double gd = fmax(gn, 1e-300);
                const double dx = (-sign * g.vx) / gd, dy = (-sign * g.vy) / gd;
                bool hit = false;
                if (good) {
                    double step = hp.snap_step;   // step * 0.5^h (exact halvings)
                    for (int h = 0; h < 3; ++h) {
                        const double tx = qx + step * dx, ty = qy + step * dy;
                        int th = hint;
                        const NnResult t = field_nearest(c.obs, tx, ty, &th);
                        const double tv = field_interface(t);
                        if (tv < val) {
                            qx = tx; qy = ty;
                            val = tv;
                            g = t;
                            hint = th;
                            hit = true;
                            break;
                        }
                        step *= 0.5;
                    }
                }
                if (!hit) {
                    stuck = true;
                    active = false;
                }
                active = active && val > hp.snap_band;
            }
#ifdef LC_NN_STATS
            if (valid) {
                const unsigned long long cyc = (unsigned long long)(clock64() - w0);
                const unsigned long long prev = atomicMax(&g_nn_stats[4], cyc);
                if (cyc > prev) g_nn_stats[5] = (unsigned long long)nsteps;
                atomicMax(&g_nn_stats[6], (unsigned long long)nsteps);
                atomicAdd(&g_nn_stats[7], (unsigned long long)nsteps);
            }
#endif
            if (valid) {
                cnt[0] += en ? 1.0 : 0.0;
                cnt[1] += (en && val <= hp.snap_band) ? 1.0 : 0.0;
                cnt[2] += (stuck && en) ? 1.0 : 0.0;
                if (en) {
                    const double z = p.z;
                    const V3 landed = v3((qx - c.cam.cx) * z / c.cam.fx, (qy - c.cam.cy) * z / c.cam.fy, z);
                    st3(J.off0 + 3 * (size_t)i, landed - p);
                }
            }
        }
    }
    T::sync();
    fst(2);
    // two uniform-Laplacian diffusion steps with the boundary held
    double *src = J.off0, *dst = J.off1;
    for (int round = 0; round < 2; ++round) {
        for (int i = T::tid(); i < c.N; i += T::size) {
            if (J.hold[i]) { st3(dst + 3 * (size_t)i, ld3(src + 3 * (size_t)i)); continue; }
            V3 a = v3(0, 0, 0);
            const int cnt = c.A.ell_cnt[i];
#pragma unroll
            for (int k = 0; k < LC_ELL; ++k) {
                if (k >= cnt) continue;
                a = a + ld3(src + 3 * (size_t)c.A.ell_nbr[(size_t)k * c.N + i]);
            }
            if (cnt > LC_ELL)
                for (int k = c.A.adj_ptr[i] + LC_ELL; k < c.A.adj_ptr[i + 1]; ++k)
                    a = a + ld3(src + 3 * (size_t)c.A.adj_nbr[k]);
            const double dg = (double)c.A.degrees[i];
            st3(dst + 3 * (size_t)i, v3(a.x / dg, a.y / dg, a.z / dg));
        }
        T::sync();
    fst(3);
        double *t = src; src = dst; dst = t;
    }
    for (int i = T::tid(); i < c.N; i += T::size) {
        const V3 o = ld3(src + 3 * (size_t)i);
        st3(v + 3 * (size_t)i, ld3(v + 3 * (size_t)i) + o);
        cnt[3] += (o.x != 0.0 || o.y != 0.0 || o.z != 0.0) ? 1.0 : 0.0;
    }
    T::template sums<4>(cnt, c.red);
    if (T::tid() == 0 && J.report) {
        J.report->snapped = 1;
        J.report->snap_walked = (int)cnt[0];
        J.report->snap_reached = (int)cnt[1];
        J.report->snap_stuck = (int)cnt[2];
        J.report->snap_moved = (int)cnt[3];
    }
    T::sync();
    fst(4);
}

template <typename T>
__device__ __forceinline__ void stamp(const SurfJob &J, int &k) {
    if (J.phase && T::tid() == 0 && k < LC_NPHASE) J.phase[k] = gtimer();
    ++k;
}

}  // namespace

template <int CS>
__global__ void __launch_bounds__(NT, LC_SURF_MINB) k_surface_solve_t(JobArg<SurfJob> jobs, ActorDev A, CamDev cam,
                                                           EdgeConstDev ec, SurfHyperDev hp, int H,
                                                           int W, int pcg_mode) {
    extern __shared__ __align__(16) double pcg_sm[];   // surf_pcg's own-chunk vectors (pcg_mode >= 1)
    lc_pdl_wait();
    using T = Team<CS, NT>;
    // this stream's descriptor, from the parameter bank into shared memory
    __shared__ SurfJob sJ;
    if (threadIdx.x == 0) sJ = jobs[T::stream()];
    __syncthreads();
    const SurfJob &J = sJ;
    if (!J.active) return;
    __shared__ double red[T::red_doubles];
    T::init_red(red);
    __syncthreads();
    SurfCtx c;
    c.J = &J;
    c.obs = J.obs;
    c.obs.K = J.obs_K ? *J.obs_K : 0;
    c.A = A;
    c.cam = cam;
    c.ec = ec;
    c.hp = hp;
    c.H = H;
    c.W = W;
    c.P = J.P ? *J.P : 0;
    c.B = J.B ? *J.B : 0;
    c.N = A.N;
    c.E = A.E;
    c.has_prev = J.prev != nullptr;
    c.red = red;
    const bool has_field = J.has_field && c.obs.K > 0;
    c.sil_on = J.enable_sil && has_field;
    own_ranges<T>(c);
    if (pcg_mode == 3) {   // surf_pcg's ELL ids of the CTA's chunk, once per solve (read by their owner thread)
        const int chunk = (c.N + CS - 1) / CS;
        int *nbr_s = reinterpret_cast<int *>(pcg_sm + 3 * (size_t)chunk);
        int *cnt_s = nbr_s + (size_t)LC_ELL * chunk;
        for (int i = c.lo + (int)threadIdx.x; i < c.hi; i += NT) {
            cnt_s[i - c.lo] = A.ell_cnt[i];
            for (int k = 0; k < LC_ELL; ++k) {
                const int j = A.ell_nbr[(size_t)k * c.N + i], owner = j / chunk;
                nbr_s[(size_t)k * chunk + (i - c.lo)] = (owner << 20) | (j - owner * chunk);
            }
        }
    }
    double *v = J.v;
    for (int i = T::tid(); i < c.N * 3; i += T::size) v[i] = J.v0[i];
    if (J.nn_hint)
        for (int b = T::tid(); b < c.B; b += T::size) J.nn_hint[b] = -1;
    T::sync();
    lc_nonrigid_report *rep = J.report;
    int ph = 0;
    stamp<T>(J, ph);
    if (J.do_solve) {
        const int levels = min(hp.gn, hp.n_levels);
        int tot[3] = {0, 0, 0};
        for (int it = 0; it < hp.gn; ++it) {
            const int level = min(it, levels - 1);
            double en[6];
            int counts[3];
            surf_assemble<T>(c, level, v, en, counts, it == 1 ? 16 : -1);
            stamp<T>(J, ph);
            for (int k = 0; k < 3; ++k) tot[k] += counts[k];
            const bool breakdown = surf_pcg<T>(c, hp.pcg, pcg_sm, pcg_mode, it == 1 ? 40 : -1);
            stamp<T>(J, ph);
            const double e0 = total_energy(en, c.has_prev);
            // halving line search (nonrigid_stage.py:386-399): the first
            // trial v + best * 0.5^h (h <= max_halvings) with e1 <= e0 is
            // taken, else the step is rejected.  Trials are evaluated up to
            // four at a time (exact halvings: the sequential search's bits).
            int halv = 0;
            bool rejected = false;
            double e1 = e0;
            double base_sc = 1.0;
            // (first batch: hp.first_trials trials -- the full step alone by
            // default -- then hp.next_trials at a time; see fill_surf_hyper)
            for (int base = 0, nt = hp.first_trials;; base += nt, nt = hp.next_trials) {
                nt = min(nt, hp.max_halvings + 1 - base);
                double et[kSurfTrials][6], unk[kSurfTrials];
                surf_energy_trials<T>(c, level, v, J.best, nt, base_sc, false, et, unk);
                {   // a trial with unevaluated rows and a lower bound <= e0 before
                    // the first exact accept: evaluate the batch exactly
                    bool undecided = false;
                    for (int h = 0; h < nt; ++h) {
                        const bool le = total_energy(et[h], c.has_prev) <= e0;
                        if (le && unk[h] > 0.0) { undecided = true; break; }
                        if (le) break;
                    }
                    if (undecided) surf_energy_trials<T>(c, level, v, J.best, nt, base_sc, true, et, unk);
                }
                int hit = -1;
                double sc = base_sc, hit_sc = 0.0;
                for (int h = 0; h < nt; ++h, sc *= 0.5) {
                    const double eh = total_energy(et[h], c.has_prev);
                    if (eh <= e0) { hit = h; e1 = eh; hit_sc = sc; break; }
                }
                if (hit >= 0) {
                    for (int i = T::tid(); i < c.N * 3; i += T::size) v[i] = v[i] + hit_sc * J.best[i];
                    T::sync();
                    halv = base + hit;
                    break;
                }
                if (base + nt > hp.max_halvings) { halv = hp.max_halvings; rejected = true; e1 = e0; break; }
                // later batches start at step * 0.5^base: a power of two,
                // so sc * step has the bits of the reference's repeated
                // in-place halvings (no rescaling pass, no team barrier)
                for (int h = 0; h < nt; ++h) base_sc *= 0.5;
            }
            stamp<T>(J, ph);
            if (T::tid() == 0 && J.counters) {
                J.counters[1] += 1;
                J.counters[2] += hp.pcg;
                J.counters[3] += halv + 1;
            }
            if (T::tid() == 0 && rep && it < LC_MAX_LOG) {
                rep->level[it] = level;
                rep->energy_before[it] = e0;
                rep->energy_after[it] = e1;
                for (int k = 0; k < 6; ++k) rep->terms[it][k] = en[k];
                rep->halvings[it] = halv;
                rep->rejected[it] = rejected;
                rep->pcg_breakdown[it] = breakdown;
            }
        }
        if (T::tid() == 0 && J.counters) {
            J.counters[0] += 1;
            J.counters[4] += c.P;
            J.counters[5] += c.B;
            J.counters[6] += c.obs.K;
        }
        if (T::tid() == 0 && rep) {
            rep->n_iterations = hp.gn;
            rep->pruned = tot[0];
            rep->degenerate_edges = tot[1];
            rep->behind_camera = tot[2];
            rep->has_temporal = c.has_prev;
            rep->n_visible = c.P;
            rep->n_boundary = c.B;
        }
    }
    if (J.do_snap && has_field && c.B > 0) surf_snap<T>(c, v);
    stamp<T>(J, ph);
    // no CTA exits while a peer may still read its shared memory (DSMEM)
    T::sync();
}

template __global__ void k_surface_solve_t<1>(JobArg<SurfJob>, ActorDev, CamDev, EdgeConstDev, SurfHyperDev, int, int, int);
template __global__ void k_surface_solve_t<2>(JobArg<SurfJob>, ActorDev, CamDev, EdgeConstDev, SurfHyperDev, int, int, int);
template __global__ void k_surface_solve_t<4>(JobArg<SurfJob>, ActorDev, CamDev, EdgeConstDev, SurfHyperDev, int, int, int);
template __global__ void k_surface_solve_t<8>(JobArg<SurfJob>, ActorDev, CamDev, EdgeConstDev, SurfHyperDev, int, int, int);
template __global__ void k_surface_solve_t<16>(JobArg<SurfJob>, ActorDev, CamDev, EdgeConstDev, SurfHyperDev, int, int, int);

int surface_block_threads() { return NT; }

// surf_pcg's shared-memory mode for a team of `cs` CTAs over N vertices and
// the dynamic shared memory it needs (per vertex of the CTA's chunk):
//   3 = z + the ELL neighbour ids and counts (60 B),
//   2 = z, p, Ap (72 B), 1 = z only (24 B), 0 = none (all in global scratch).
// The default is the highest mode whose buffer leaves two CTAs per SM
// (<= 100 KB); LIVECAP_PCG_MODE selects one explicitly (measurement sweeps;
// falls back to 0 when it does not fit).
int surface_pcg_mode(int N, int cs, size_t *smem_bytes) {
    const size_t chunk = ((size_t)N + cs - 1) / cs;
    const size_t per[4] = {0, 24, 72, 24 + 4 * LC_ELL + 4};
    const size_t budget = 100 * 1024;
    static const int env = [] {
        const char *v = getenv("LIVECAP_PCG_MODE");
        return v ? atoi(v) : -1;
    }();
    int mode = 0;
    if (env >= 0 && env <= 3) mode = per[env] * chunk <= budget ? env : 0;
    else if (per[3] * chunk <= budget) mode = 3;
    else if (per[1] * chunk <= budget) mode = 1;
    *smem_bytes = per[mode] * chunk;
    return mode;
}

#ifdef LC_NN_STATS
extern "C" int lc_debug_nn_stats_surface(unsigned long long *o, int reset) {
    cudaMemcpyFromSymbol(o, g_nn_stats, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_nn_stats, z, sizeof z);
    }
    return 0;
}
#endif
