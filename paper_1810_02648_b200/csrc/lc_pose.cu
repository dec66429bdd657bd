// Stage I: skeletal pose Gauss-Newton, one persistent CTA per stream.
//
// Reference: PoseProblem.evaluate (pose_stage.py:319-404) and solve_pose
// (pose_stage.py:429-459).  Per evaluation: FK on one warp, the joint /
// dual-quaternion Jacobian tables in shared memory, residual rows computed
// NT at a time into a shared chunk, and J^T J / J^T F accumulated from the
// chunk by 27 register-tiled tasks (21 upper 6x6 tiles + 6 rhs strips) per
// row group.  The 36x36 system is solved in shared memory (lc_qr.cuh); the
// halving line search re-evaluates energies only.  No host round trip.
#include "livecap.h"
#include "lc_kernels.cuh"
#include "lc_qr.cuh"
#include "lc_pose.cuh"
#include "lc_team.cuh"

namespace {

constexpr int NT = 256;
constexpr int G = NT / 32;  // row groups for the J^T J accumulation
#ifdef LC_POSE_JTJ_NOFMA    // (comparison build: unfused products and sums)
#define LC_JTJ_MAD(a, b, c) ((c) + (a) * (b))
#else
#define LC_JTJ_MAD(a, b, c) fma((a), (b), (c))
#endif

struct PoseSmem {
    SkelDev sk;
    FkState f;
    QrSmemT<LC_NP> qr;
    double A[LC_NP * LC_NP];
    double rhs[LC_NP];
    double x[LC_NP], xt[LC_NP], step[LC_NP];
    double red[Team<1, NT>::red_doubles];
    double pix[LC_MAXJ + 4][2];
    int okz[LC_MAXJ + 4];
    // nonzero DQ Jacobian columns per joint: 0..5 (root) + 6+k for the DOFs k
    // that move the joint's frame (skinning.py:269-300)
    unsigned char jcol[LC_MAXJ][LC_NP];
    int jcnt[LC_MAXJ];
};

// one evaluation point: FK state, parameters and joint/marker projections
struct PoseView {
    FkState *f;
    double *xt;
    double (*pix)[2];
    int *okz;
};

// line-search trial points evaluated together (aliases the Jacobian tables,
// which only the with-Jacobian evaluation uses)
constexpr int kTrials = 4;
struct TrialSmem {
    FkState f[kTrials];
    double xt[kTrials][LC_NP];
    double pix[kTrials][LC_MAXJ + 4][2];
    int okz[kTrials][LC_MAXJ + 4];
};

struct PoseCtx {
    const PoseJob *J;
    PoseSmem *s;
    double *jp;    // (J+4)*3*36
    double *dqj;   // J*8*36
    double *rows;  // NT*37
    int B, n2, n3, nt, R;
    CamDev cam;
    ActorDev A;
    NnGridDev obs;
};

// one residual row; writes the 36 Jacobian entries to `jr` when non-null.
// Returns F and sets `term` (0 2d, 1 3d, 2 sil, 3 temporal, 4 anatomic).
__device__ double pose_row(const PoseCtx &c, const PoseView &pv, int r, double *jr, int &term, int &behind) {
    const PoseSmem &s = *c.s;
    const SkelDev &sk = s.sk;
    const FkState &f = *pv.f;
    const PoseJob &J = *c.J;
    const PoseHyperDev &hp = J.hp;
    const int nj = sk.J;
    behind = 0;
    if (r < c.n2) {                                      // 2D detections
        term = 0;
        const int n = r >> 1, comp = r & 1;
        const double lam = n < nj ? hp.l2d : hp.l2d * hp.face;
        const double w2 = (sqrt(lam) * (J.v2d[n] ? 1.0 : 0.0)) * (pv.okz[n] ? 1.0 : 0.0);
        const double F = (pv.pix[n][comp] - J.j2d[2 * n + comp]) * w2;
        behind = comp == 0 && !pv.okz[n];   // each joint / marker once (pose_stage.py:334)
        if (jr) {
            const V3 p = n < nj ? ld3(f.pos[n]) : ld3(f.markers[n - nj]);
            double a0, a2, b1, b2;
            proj_jac(c.cam, p, a0, a2, b1, b2);
            const double d0 = comp == 0 ? a0 : 0.0, d1 = comp == 0 ? 0.0 : b1, d2 = comp == 0 ? a2 : b2;
            const double *jn = c.jp + (size_t)n * 3 * LC_NP;
            for (int q = 0; q < LC_NP; ++q)
                jr[q] = (d0 * jn[q] + d1 * jn[LC_NP + q] + d2 * jn[2 * LC_NP + q]) * w2;
        }
        return F;
    }
    r -= c.n2;
    if (r < c.n3) {                                      // 3D detections
        term = 1;
        const int i = r / 3, comp = r % 3;
        const double w3 = sqrt(hp.l3d) * (J.v3d[i] ? 1.0 : 0.0);
        const double F = ((f.pos[i][comp] - J.j3d[3 * i + comp]) - pv.xt[33 + comp]) * w3;
        if (jr) {
            const double *jn = c.jp + ((size_t)i * 3 + comp) * LC_NP;
            for (int q = 0; q < LC_NP; ++q) jr[q] = (jn[q] - (q == 33 + comp ? 1.0 : 0.0)) * w3;
        }
        return F;
    }
    r -= c.n3;
    if (r < c.B) {                                       // silhouette
        term = 2;
        const int b = r;
        const int v = J.cidx[b];
        const V3 rest = J.crest ? ld3(J.crest + 3 * (size_t)b) : ld3(J.drest + 3 * (size_t)v);
        Blend Bl;
        struct SmemDq {
            const FkState *f;
            __device__ double operator()(int j, int k) const { return f->dq[j][k]; }
        };
        dq_blend(c.A.skin_idx + 4 * v, c.A.skin_w + 4 * v, c.A.dominant[v], SmemDq{&f}, Bl);
        Q4 cr;
        const V3 sp = dq_apply(Bl, rest, cr);
        double px, py;
        const bool cok = project(c.cam, sp, px, py);
        behind = !cok;
        if (J.enabled && !J.enabled[b]) {   // weight 0 (rim / part gating): a zero row, no query needed
            if (jr)
                for (int q = 0; q < LC_NP; ++q) jr[q] = 0.0;
            return 0.0;
        }
        NnResult nn;
        double val = 0.0, gx = 0.0, gy = 0.0;
        nn = field_nearest(c.obs, px, py, J.nn_hint ? J.nn_hint + b : nullptr);
        field_residual(nn, val, gx, gy);
        bool ok = cok && !nn.clamped;
        if (J.enabled) ok = ok && J.enabled[b];
        const double ws = sqrt(hp.lsil) * (ok ? 1.0 : 0.0);
        const double F = val * ws;
        if (jr) {
            double a0, a2, b1, b2;
            proj_jac(c.cam, sp, a0, a2, b1, b2);
            const V3 g3 = v3(gx * a0, gy * b1, gx * a2 + gy * b2);
            double dv[3][8];
            dq_dtransform(Bl, rest, dv);
            double h[8];
            for (int k = 0; k < 8; ++k) h[k] = g3.x * dv[0][k] + g3.y * dv[1][k] + g3.z * dv[2][k];
            const double sign = J.directional ? side_sign(c.obs, nn, px, py, J.n2d[2 * b], J.n2d[2 * b + 1]) : 1.0;
            const double sc = ws * sign;
            for (int q = 0; q < LC_NP; ++q) jr[q] = 0.0;
            // only the parameters that move the joint's frame have nonzero DQ
            // Jacobian columns (root rotation / translation and the DOFs of
            // its ancestors and itself, s.jcol): the other columns stay 0
            if (Bl.degenerate) {
                const double *t = c.dqj + (size_t)Bl.dom * 8 * LC_NP;
                const unsigned char *cols = s.jcol[Bl.dom];
                for (int m = 0; m < s.jcnt[Bl.dom]; ++m) {
                    const int q = cols[m];
                    double a = 0.0;
                    for (int k = 0; k < 8; ++k) a += h[k] * t[k * LC_NP + q];
                    jr[q] = a;
                }
            } else {
                for (int sl = 0; sl < 4; ++sl) {
                    const double cf = Bl.coef[sl];
                    if (cf == 0.0) continue;
                    const double *t = c.dqj + (size_t)Bl.js[sl] * 8 * LC_NP;
                    const unsigned char *cols = s.jcol[Bl.js[sl]];
                    for (int m = 0; m < s.jcnt[Bl.js[sl]]; ++m) {
                        const int q = cols[m];
                        double a = 0.0;
                        for (int k = 0; k < 8; ++k) a += h[k] * t[k * LC_NP + q];
                        jr[q] += cf * a;
                    }
                }
            }
            for (int q = 0; q < LC_NP; ++q) jr[q] *= sc;
        }
        return F;
    }
    r -= c.B;
    if (r < c.nt) {                                      // temporal
        term = 3;
        const int i = r / 3, comp = r % 3;
        const double wt = sqrt(hp.ltemp * hp.tw[i]);
        const double F = (f.pos[i][comp] - J.prev_pos[3 * i + comp]) * wt;
        if (jr) {
            const double *jn = c.jp + ((size_t)i * 3 + comp) * LC_NP;
            for (int q = 0; q < LC_NP; ++q) jr[q] = jn[q] * wt;
        }
        return F;
    }
    r -= c.nt;                                           // anatomic (27 rows)
    term = 4;
    const double th = pv.xt[6 + r];
    const bool hi = th > sk.tmax[r], lo = th < sk.tmin[r];
    const double wa = sqrt(hp.lanat);
    const double F = wa * ((hi ? th - sk.tmax[r] : 0.0) + (lo ? sk.tmin[r] - th : 0.0));
    if (jr) {
        for (int q = 0; q < LC_NP; ++q) jr[q] = 0.0;
        jr[6 + r] = wa * ((hi ? 1.0 : 0.0) - (lo ? 1.0 : 0.0));
    }
    return F;
}

// evaluate at s.xt; with_jac fills s.A / s.rhs.  Returns the total energy,
// per-term energies in terms[5], behind-camera count.  Rows are split over
// the team's CTAs; every CTA ends with the same totals.
template <typename T>
__device__ double pose_eval(PoseCtx &c, bool with_jac, double terms[5], int &behind_out, int fine = -1,
                            bool fk_valid = false) {
    PoseSmem &s = *c.s;
    auto fst = [&](int k) {
        if (fine >= 0 && c.J->phase && T::tid() == 0) c.J->phase[fine + k] = gtimer();
    };
    fst(0);
    const SkelDev &sk = s.sk;
    const int nj = sk.J;
    const PoseView pv{&s.f, s.xt, s.pix, s.okz};
    // s.f already holds the FK of this point when it is the previous line
    // search's accepted trial (or the unchanged point of a rejected step)
    if (!fk_valid && threadIdx.x < 32) fk_warp(sk, s.xt, s.f);
    __syncthreads();
    fst(1);
    // projections of joints + markers
    for (int n = threadIdx.x; n < nj + 4; n += NT) {
        const V3 p = n < nj ? ld3(s.f.pos[n]) : ld3(s.f.markers[n - nj]);
        double px, py;
        s.okz[n] = project(c.cam, p, px, py);
        s.pix[n][0] = px;
        s.pix[n][1] = py;
    }
    if (with_jac) {
        // joint/marker position Jacobian (J+4, 3, 36)
        const int npos = (nj + 4) * 3 * LC_NP;
        for (int e = threadIdx.x; e < npos; e += NT) {
            const int q = e % LC_NP, comp = (e / LC_NP) % 3, pt = e / (3 * LC_NP);
            double val;
            if (q >= 3 && q < 6) val = (q - 3 == comp) ? 1.0 : 0.0;
            else if (q >= 33) val = 0.0;
            else {
                const V3 sp = joint_spin(sk, s.f, pt, q < 3 ? q : q - 3);
                val = comp == 0 ? sp.x : (comp == 1 ? sp.y : sp.z);
            }
            c.jp[e] = val;
        }
        // dual-quaternion Jacobian (J, 8, 36)
        for (int e = threadIdx.x; e < nj * LC_NP; e += NT) {
            const int j = e / LC_NP, q = e % LC_NP;
            double o[8];
            if (q >= 3 && q < 6) {
                const Q4 d = dq_trans(s.f, j, q - 3);
                o[0] = o[1] = o[2] = o[3] = 0.0;
                o[4] = d.w; o[5] = d.x; o[6] = d.y; o[7] = d.z;
            } else if (q >= 33) {
                for (int k = 0; k < 8; ++k) o[k] = 0.0;
            } else {
                dq_spin(sk, s.f, j, q < 3 ? q : q - 3, o);
            }
            for (int k = 0; k < 8; ++k) c.dqj[((size_t)j * 8 + k) * LC_NP + q] = o[k];
        }
    }
    __syncthreads();
    fst(2);

    double acc[5] = {0, 0, 0, 0, 0};
    double total = 0.0;
    int behind = 0;
    // J^T J tiles: task = tid / G (27 tasks), group = tid % G
    const int task = threadIdx.x / G, grp = threadIdx.x % G;
    double tile[36];
#pragma unroll
    for (int k = 0; k < 36; ++k) tile[k] = 0.0;
    int ta = 0, tb = 0;
    bool is_rhs = false;
    if (task < 21) {
        int t = task;
        for (ta = 0; ta < 6; ++ta) {
            if (t < 6 - ta) { tb = ta + t; break; }
            t -= 6 - ta;
        }
    } else if (task < 27) {
        is_rhs = true;
        ta = task - 21;
    }
    for (int r0 = T::rank() * NT; r0 < c.R; r0 += T::size) {
        const int r = r0 + threadIdx.x;
        if (r < c.R) {
            int term, bh;
            double *jr = with_jac ? c.rows + (size_t)threadIdx.x * 37 : nullptr;
            const double F = pose_row(c, pv, r, jr, term, bh);
            if (jr) jr[36] = F;
            acc[term] += F * F;
            behind += bh;
        }
        if (with_jac) {
            __syncthreads();
            if (r0 == T::rank() * NT) fst(6);   // first chunk's rows done (fine timer)
            const int nr = min(NT, c.R - r0);
            if (task < 27) {
                for (int rr = grp; rr < nr; rr += G) {
                    const double *row = c.rows + (size_t)rr * 37;
                    // (FMA: the reference forms J^T J / J^T F with BLAS, which
                    // fuses; SURVEY Appendix B allows it in this accumulation)
                    if (is_rhs) {
                        const double F = row[36];
#pragma unroll
                        for (int i = 0; i < 6; ++i) tile[i] = LC_JTJ_MAD(row[6 * ta + i], F, tile[i]);
                    } else {
                        double a[6], b[6];
#pragma unroll
                        for (int i = 0; i < 6; ++i) { a[i] = row[6 * ta + i]; b[i] = row[6 * tb + i]; }
#pragma unroll
                        for (int i = 0; i < 6; ++i)
#pragma unroll
                            for (int j = 0; j < 6; ++j) tile[6 * i + j] = LC_JTJ_MAD(a[i], b[j], tile[6 * i + j]);
                    }
                }
            }
            __syncthreads();
        }
    }
    fst(3);
    // total energy = sum of F^2 over all rows (pose_stage.py:279-281)
    {
        double v8[8] = {acc[0], acc[1], acc[2], acc[3], acc[4], (double)behind, 0.0, 0.0};
        T::template sums_light<8>(v8, s.red);   // (the phases exchange shared memory only)
        for (int k = 0; k < 5; ++k) terms[k] = v8[k];
        behind_out = (int)v8[5];
        total = (((v8[0] + v8[1]) + v8[2]) + v8[3]) + v8[4];
    }
    fst(4);
    if (with_jac) {
        // partial tiles -> shared (reuse the row chunk), then reduce over groups
        double *part = c.rows;
        const int per_group = 21 * 36 + 6 * 6;
        if (task < 27) {
            double *dst = part + (size_t)grp * per_group + (is_rhs ? 21 * 36 + 6 * ta : 36 * task);
            const int cnt = is_rhs ? 6 : 36;
#pragma unroll
            for (int k = 0; k < 36; ++k)
                if (k < cnt) dst[k] = tile[k];
        }
        __syncthreads();
        // groups -> this CTA's partial, then the team total in rank order
        double *cta_part = part + (size_t)G * per_group;
        double *team_tot = cta_part + per_group;
        for (int e = threadIdx.x; e < per_group; e += NT) {
            double sum = part[e];
            for (int g = 1; g < G; ++g) sum += part[(size_t)g * per_group + e];
            cta_part[e] = sum;
        }
        __syncthreads();
        T::sum_arrays_light(cta_part, team_tot, per_group, s.red);
        for (int e = threadIdx.x; e < per_group; e += NT) {
            const double sum = team_tot[e];
            if (e < 21 * 36) {
                int t = e / 36, k = e % 36, a = 0, b = 0;
                for (a = 0; a < 6; ++a) {
                    if (t < 6 - a) { b = a + t; break; }
                    t -= 6 - a;
                }
                const int i = 6 * a + k / 6, j = 6 * b + k % 6;
                s.A[i * LC_NP + j] = sum;
                s.A[j * LC_NP + i] = sum;
            } else {
                const int i = e - 21 * 36;
                s.rhs[i] = -sum;
            }
        }
        __syncthreads();
    }
    fst(5);
    return total;
}

// Energies of nt line-search trial points at once (ts.xt[h], h < nt): FK on
// warp h, then the nt*R residual rows spread over the team, one team
// reduction of the nt x 5 term sums.  e[h] is summed in the same term order
// as the single-point evaluation (pose_stage.py:279-281).
template <typename T>
__device__ void pose_trials(PoseCtx &c, TrialSmem &ts, int nt, double e[kTrials], int fine = -1) {
    PoseSmem &s = *c.s;
    auto fst = [&](int k) {
        if (fine >= 0 && c.J->phase && T::tid() == 0) c.J->phase[fine + k] = gtimer();
    };
    fst(0);
    const SkelDev &sk = s.sk;
    const int nj = sk.J;
    const int w = threadIdx.x >> 5;
    if (w < nt) fk_warp(sk, ts.xt[w], ts.f[w]);
    __syncthreads();
    fst(1);
    for (int k = threadIdx.x; k < nt * (nj + 4); k += NT) {
        const int h = k / (nj + 4), n = k - h * (nj + 4);
        const V3 p = n < nj ? ld3(ts.f[h].pos[n]) : ld3(ts.f[h].markers[n - nj]);
        double px, py;
        ts.okz[h][n] = project(c.cam, p, px, py);
        ts.pix[h][n][0] = px;
        ts.pix[h][n][1] = py;
    }
    __syncthreads();
    fst(2);
    double acc[kTrials * 5];
    for (int k = 0; k < kTrials * 5; ++k) acc[k] = 0.0;
    for (int rr = T::tid(); rr < nt * c.R; rr += T::size) {
        const int h = rr / c.R, r = rr - h * c.R;
        const PoseView pv{&ts.f[h], ts.xt[h], ts.pix[h], ts.okz[h]};
        int term, bh;
        const double F = pose_row(c, pv, r, nullptr, term, bh);
        const double f2 = F * F;
        const int slot = h * 5 + term;
#pragma unroll
        for (int k = 0; k < kTrials * 5; ++k)
            if (k == slot) acc[k] += f2;
    }
    fst(3);
    T::template sums_light<kTrials * 5>(acc, s.red);
    fst(4);
    for (int h = 0; h < kTrials; ++h)
        e[h] = (((acc[5 * h] + acc[5 * h + 1]) + acc[5 * h + 2]) + acc[5 * h + 3]) + acc[5 * h + 4];
}

}  // namespace

template <int CS>
__global__ void __launch_bounds__(NT, 1) k_pose_solve_t(JobArg<PoseJob> jobs, const SkelDev *skg,
                                                        ActorDev A, CamDev cam) {
    lc_pdl_wait();
    using T = Team<CS, NT>;
    __shared__ PoseJob sJ;   // this stream's descriptor, parameter bank -> shared memory
    if (threadIdx.x == 0) sJ = jobs[T::stream()];
    __syncthreads();
    const PoseJob &J = sJ;
    if (!J.active) return;
    extern __shared__ __align__(16) unsigned char dsm[];
    PoseSmem &s = *reinterpret_cast<PoseSmem *>(dsm);
    double *tail = reinterpret_cast<double *>(dsm + ((sizeof(PoseSmem) + 15) & ~size_t(15)));
    T::init_red(s.red);
    {
        const int *src = reinterpret_cast<const int *>(skg);
        int *dst = reinterpret_cast<int *>(&s.sk);
        for (int i = threadIdx.x; i < (int)(sizeof(SkelDev) / sizeof(int)); i += NT) dst[i] = src[i];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < s.sk.J; j += NT) {
        int n = 0;
        for (int q = 0; q < 6; ++q) s.jcol[j][n++] = (unsigned char)q;
        for (int k = 0; k < LC_NDOF; ++k)
            if ((s.sk.moves_frame[k] >> j) & 1u) s.jcol[j][n++] = (unsigned char)(6 + k);
        s.jcnt[j] = n;
    }
    __syncthreads();
    PoseCtx c;
    c.J = &J;
    c.s = &s;
    c.cam = cam;
    c.A = A;
    const int nj = s.sk.J;
    c.jp = tail;
    c.dqj = c.jp + (size_t)(nj + 4) * 3 * LC_NP;
    c.rows = c.dqj + (size_t)nj * 8 * LC_NP;
    c.obs = J.obs;
    c.obs.K = J.obs_K ? *J.obs_K : 0;
    c.B = (J.has_field && c.obs.K > 0 && J.B) ? *J.B : 0;
    c.n2 = 2 * (nj + 4);
    c.n3 = 3 * nj;
    c.nt = J.prev_pos ? 3 * nj : 0;
    c.R = c.n2 + c.n3 + c.B + c.nt + 27;
    for (int i = threadIdx.x; i < LC_NP; i += NT) s.x[i] = J.x0[i];
    if (J.nn_hint)
        for (int b = T::tid(); b < c.B; b += T::size) J.nn_hint[b] = -1;
    T::sync();

    lc_pose_report *rep = J.report;
    int log0 = J.log_offset;
    int ph = 0;
    auto stamp = [&]() {
        if (J.phase && T::tid() == 0 && ph < LC_NPHASE) J.phase[ph] = gtimer();
        ++ph;
    };
    stamp();
    int behind_total = 0, gimbal = 0;
    bool fk_valid = false;   // s.f holds FK(s.x) (block-uniform)
    for (int it = 0; it < J.hp.gn; ++it) {
        for (int i = threadIdx.x; i < LC_NP; i += NT) s.xt[i] = s.x[i];
        __syncthreads();
        double terms[5];
        int behind;
        const double e0 = pose_eval<T>(c, true, terms, behind, it == 1 ? 32 : -1, fk_valid);
        stamp();
        behind_total += behind;
        gimbal |= s.f.gimbal;
        double damping;
        const bool damped = dense_solve_block<NT>(s.qr, s.A, s.rhs, LC_NP, damping);
        for (int i = threadIdx.x; i < LC_NP; i += NT) s.step[i] = s.qr.x[i];
        __syncthreads();
        stamp();
        // halving line search (pose_stage.py:441-453): accept the first
        // trial step * 0.5^h with e1 <= e0, h <= max_halvings, else reject.
        // Trials are evaluated kTrials at a time; halving is exact, so every
        // trial point has the bits of the sequential search.
        TrialSmem &ts = *reinterpret_cast<TrialSmem *>(c.jp);
        int halv = 0;
        bool rejected = false;
        double e1 = e0;
        // (the full step is accepted in nearly every GN step, so the first
        // batch is J.hp.first_trials trials -- the full step alone by default)
        for (int base = 0, nb = J.hp.first_trials;; base += nb, nb = kTrials) {
            const int nt = min(nb, J.hp.max_halvings + 1 - base);
            for (int i = threadIdx.x; i < LC_NP; i += NT) {
                double st = s.step[i];
                for (int h = 0; h < nt; ++h) {
                    ts.xt[h][i] = s.x[i] + st;
                    st = 0.5 * st;
                }
            }
            __syncthreads();
            double et[kTrials];
            pose_trials<T>(c, ts, nt, et, (it == 1 && base == 0) ? 40 : -1);
            int hit = -1;
            for (int h = 0; h < nt; ++h)
                if (et[h] <= e0) { hit = h; break; }
            const bool last = base + nt > J.hp.max_halvings;
            const int nh = hit >= 0 ? hit : (last ? nt - 1 : nt);   // halvings applied to s.step
            for (int i = threadIdx.x; i < LC_NP; i += NT) {
                double st = s.step[i];
                for (int h = 0; h < nh; ++h) st = 0.5 * st;
                s.step[i] = st;
                if (hit >= 0) s.x[i] = ts.xt[hit][i];
            }
            if (hit >= 0) {   // the accepted trial's FK is FK(new x): keep it for the next evaluation
                const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&ts.f[hit]);
                unsigned long long *dst = reinterpret_cast<unsigned long long *>(&s.f);
                for (int i = threadIdx.x; i < (int)(sizeof(FkState) / 8); i += NT) dst[i] = src[i];
            }
            __syncthreads();
            if (hit >= 0) { halv = base + hit; e1 = et[hit]; break; }
            if (last) { halv = J.hp.max_halvings; rejected = true; e1 = e0; break; }
        }
        fk_valid = true;   // accepted: copied from the trial; rejected: s.f is still FK(s.x)
        stamp();
        if (T::tid() == 0 && rep) {
            const int k = log0 + it;
            if (k < LC_MAX_LOG) {
                rep->energy_before[k] = e0;
                rep->energy_after[k] = e1;
                double sn = 0.0;
                for (int i = 0; i < LC_NP; ++i) sn += s.step[i] * s.step[i];
                rep->step_norm[k] = sqrt(sn);
                for (int t = 0; t < 5; ++t) rep->terms[k][t] = terms[t];
                rep->halvings[k] = halv;
                rep->rejected[k] = rejected;
                rep->damped[k] = damped;
            }
        }
        __syncthreads();
    }
    if (T::rank() == 0) {
        for (int i = threadIdx.x; i < LC_NP; i += NT) J.x_out[i] = s.x[i];
        // s.f = FK(s.x) after every GN step (the accepted trial's FK, or the
        // unchanged point's): Stage II skins from it instead of a k_fk launch
        if (J.fk_out && J.hp.gn > 0) {
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&s.f);
            unsigned long long *dst = reinterpret_cast<unsigned long long *>(J.fk_out);
            for (int i = threadIdx.x; i < (int)(sizeof(FkState) / 8); i += NT) dst[i] = src[i];
        }
    }
    if (T::tid() == 0 && rep) {
        rep->n_iterations = log0 + J.hp.gn;
        rep->behind_camera += behind_total;
        rep->gimbal = rep->gimbal || gimbal;
        rep->n_contour = c.B;
        rep->has_temporal = J.prev_pos != nullptr;
    }
    // peers may still be reading this CTA's shared memory (the last team
    // reduction reads every rank's partials over DSMEM): no CTA may exit first
    T::sync();
}

template __global__ void k_pose_solve_t<1>(JobArg<PoseJob>, const SkelDev *, ActorDev, CamDev);
template __global__ void k_pose_solve_t<2>(JobArg<PoseJob>, const SkelDev *, ActorDev, CamDev);
template __global__ void k_pose_solve_t<4>(JobArg<PoseJob>, const SkelDev *, ActorDev, CamDev);
template __global__ void k_pose_solve_t<8>(JobArg<PoseJob>, const SkelDev *, ActorDev, CamDev);
template __global__ void k_pose_solve_t<16>(JobArg<PoseJob>, const SkelDev *, ActorDev, CamDev);

size_t pose_smem_bytes(int n_joints) {
    const size_t head = (sizeof(PoseSmem) + 15) & ~size_t(15);
    size_t tables = (size_t)(n_joints + 4) * 3 * LC_NP + (size_t)n_joints * 8 * LC_NP;
    const size_t trial = (sizeof(TrialSmem) + sizeof(double) - 1) / sizeof(double);
    if (tables < trial) tables = trial;
    const size_t rows = (size_t)NT * 37;
    return head + (tables + rows) * sizeof(double);
}

int pose_block_threads() { return NT; }

#ifdef LC_NN_STATS
extern "C" int lc_debug_nn_stats_pose(unsigned long long *o, int reset) {
    cudaMemcpyFromSymbol(o, g_nn_stats, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_nn_stats, z, sizeof z);
    }
    return 0;
}
#endif
