// Forward kinematics, joint Jacobians and dual-quaternion skinning (device).
//
// Reference: skinning.py:171-398.  FK runs on one warp per stream: the 30
// sin/cos pairs in parallel, then the joint tree level by level (joints at
// the same depth are independent), then markers and per-joint dual
// quaternions in parallel.
#pragma once
#include "lc_device.cuh"

struct FkState {
    double rot[LC_MAXJ][9];
    double pos[LC_MAXJ][3];
    double markers[4][3];
    double axes[LC_NROT][3];
    double piv[LC_NROT][3];
    double trans[LC_MAXJ][3];
    double dq[LC_MAXJ][8];
    double cs[LC_NROT][2];
    int gimbal;
};

// rotation about a unit axis (skinning.py:171-179)
__device__ __forceinline__ void axis_rot(const double *ax, double c, double s, double *m) {
    const double x = ax[0], y = ax[1], z = ax[2], k = 1.0 - c;
    m[0] = c + x * x * k;     m[1] = x * y * k - z * s; m[2] = x * z * k + y * s;
    m[3] = y * x * k + z * s; m[4] = c + y * y * k;     m[5] = y * z * k - x * s;
    m[6] = z * x * k - y * s; m[7] = z * y * k + x * s; m[8] = c + z * z * k;
}

// Shepperd's largest-pivot branch (skinning.py:115-141)
__device__ __forceinline__ Q4 rot_to_quat(const double *m) {
    const double tr = m[0] + m[4] + m[8];
    const double mx = fmax(m[0], fmax(m[4], m[8]));
    if (tr > mx) {
        const double s = sqrt(tr + 1.0) * 2.0;
        return Q4{0.25 * s, (m[7] - m[5]) / s, (m[2] - m[6]) / s, (m[3] - m[1]) / s};
    }
    if (m[0] >= m[4] && m[0] >= m[8]) {
        const double s = sqrt(1.0 + m[0] - m[4] - m[8]) * 2.0;
        return Q4{(m[7] - m[5]) / s, 0.25 * s, (m[1] + m[3]) / s, (m[2] + m[6]) / s};
    }
    if (m[4] >= m[8]) {
        const double s = sqrt(1.0 + m[4] - m[0] - m[8]) * 2.0;
        return Q4{(m[2] - m[6]) / s, (m[1] + m[3]) / s, 0.25 * s, (m[5] + m[7]) / s};
    }
    const double s = sqrt(1.0 + m[8] - m[0] - m[4]) * 2.0;
    return Q4{(m[3] - m[1]) / s, (m[2] + m[6]) / s, (m[5] + m[7]) / s, 0.25 * s};
}

// Executed by all 32 lanes of one warp (forward_kinematics, skinning.py:206-246).
__device__ inline void fk_warp(const SkelDev &sk, const double *x, FkState &f) {
    const int lane = threadIdx.x & 31;
    if (lane < LC_NROT) {
        const double ang = lane < 3 ? x[lane] : x[6 + lane - 3];
        f.cs[lane][0] = cos(ang);
        f.cs[lane][1] = sin(ang);
    }
    __syncwarp();
    if (lane == 0) {
        const double ex[3] = {1, 0, 0}, ey[3] = {0, 1, 0}, ez[3] = {0, 0, 1};
        double rx[9], ry[9], rz[9], rxy[9];
        axis_rot(ex, f.cs[0][0], f.cs[0][1], rx);
        axis_rot(ey, f.cs[1][0], f.cs[1][1], ry);
        axis_rot(ez, f.cs[2][0], f.cs[2][1], rz);
        mat_mul(rx, ry, rxy);
        mat_mul(rxy, rz, f.rot[0]);
        const V3 pel = v3(x[3] + sk.off[0][0], x[4] + sk.off[0][1], x[5] + sk.off[0][2]);
        st3(f.pos[0], pel);
        st3(f.axes[0], v3(1, 0, 0));
        st3(f.axes[1], mat_vec(rx, v3(0, 1, 0)));
        st3(f.axes[2], mat_vec(rxy, v3(0, 0, 1)));
        for (int a = 0; a < 3; ++a) st3(f.piv[a], pel);
        f.gimbal = fabs(f.cs[1][0]) < 1e-6;
    }
    __syncwarp();
    for (int L = 1; L < sk.n_tree_levels; ++L) {
        const int s = sk.level_start[L], e = sk.level_start[L + 1];
        if (lane < e - s) {
            const int i = sk.level_joint[s + lane];
            const int p = sk.parents[i];
            const V3 pi = mat_vec(f.rot[p], ld3(sk.off[i])) + ld3(f.pos[p]);
            st3(f.pos[i], pi);
            double r[9], t[9], m[9];
            for (int q = 0; q < 9; ++q) r[q] = f.rot[p][q];
            for (int d = sk.dof_start[i]; d < sk.dof_start[i + 1]; ++d) {
                const int k = sk.dof_list[d];
                st3(f.axes[3 + k], mat_vec(r, ld3(sk.dof_axes[k])));
                st3(f.piv[3 + k], pi);
                axis_rot(sk.dof_axes[k], f.cs[3 + k][0], f.cs[3 + k][1], m);
                mat_mul(r, m, t);
                for (int q = 0; q < 9; ++q) r[q] = t[q];
            }
            for (int q = 0; q < 9; ++q) f.rot[i][q] = r[q];
        }
        __syncwarp();
    }
    if (lane < 4) {
        const double *R = f.rot[sk.head];
        const double *o = sk.marker[lane];
        for (int i = 0; i < 3; ++i)
            f.markers[lane][i] = (o[0] * R[3 * i] + o[1] * R[3 * i + 1] + o[2] * R[3 * i + 2])
                                 + f.pos[sk.head][i];
    }
    if (lane < sk.J) {
        const int j = lane;
        const V3 tr = ld3(f.pos[j]) - mat_vec(f.rot[j], ld3(sk.rest[j]));
        st3(f.trans[j], tr);
        const Q4 qr = rot_to_quat(f.rot[j]);
        const Q4 qd0 = qmul(Q4{0.0, tr.x, tr.y, tr.z}, qr);
        const double d[8] = {qr.w, qr.x, qr.y, qr.z, 0.5 * qd0.w, 0.5 * qd0.x, 0.5 * qd0.y,
                             0.5 * qd0.z};
        for (int q = 0; q < 8; ++q) f.dq[j][q] = d[q];
    }
    __syncwarp();
}

// rotational parameter a (0..29) -> column of the 36-vector
__device__ __forceinline__ int rot_col(int a) { return a < 3 ? a : a + 3; }

// d(point)/d(x) entry for joint/marker `pt`, component c, rotational param a
// (joint_position_jacobian, skinning.py:249-266)
__device__ __forceinline__ V3 joint_spin(const SkelDev &sk, const FkState &f, int pt, int a) {
    bool reach = true;
    if (a >= 3) {
        const int k = a - 3;
        reach = pt < sk.J ? ((sk.moves_pos[k] >> pt) & 1u) : ((sk.moves_frame[k] >> sk.head) & 1u);
    }
    if (!reach) return v3(0, 0, 0);
    const V3 p = pt < sk.J ? ld3(f.pos[pt]) : ld3(f.markers[pt - sk.J]);
    return cross3(ld3(f.axes[a]), p - ld3(f.piv[a]));
}

// d(dq_j)/d(x) for rotational param a (joint_dq_jacobian, skinning.py:269-300)
__device__ __forceinline__ void dq_spin(const SkelDev &sk, const FkState &f, int j, int a,
                                        double out[8]) {
    const bool reach = a < 3 || ((sk.moves_frame[a - 3] >> j) & 1u);
    if (!reach) { for (int q = 0; q < 8; ++q) out[q] = 0.0; return; }
    const Q4 qr{f.dq[j][0], f.dq[j][1], f.dq[j][2], f.dq[j][3]};
    const V3 ax = ld3(f.axes[a]);
    const Q4 r0 = qmul(Q4{0.0, ax.x, ax.y, ax.z}, qr);
    const Q4 dqr{0.5 * r0.w, 0.5 * r0.x, 0.5 * r0.y, 0.5 * r0.z};
    const V3 tr = ld3(f.trans[j]);
    const V3 td = cross3(ax, tr - ld3(f.piv[a]));
    const Q4 p1 = qmul(Q4{0.0, td.x, td.y, td.z}, qr);
    const Q4 p2 = qmul(Q4{0.0, tr.x, tr.y, tr.z}, dqr);
    out[0] = dqr.w; out[1] = dqr.x; out[2] = dqr.y; out[3] = dqr.z;
    out[4] = 0.5 * (p1.w + p2.w); out[5] = 0.5 * (p1.x + p2.x);
    out[6] = 0.5 * (p1.y + p2.y); out[7] = 0.5 * (p1.z + p2.z);
}

// dual part of d(dq_j)/d(root translation axis ax)
__device__ __forceinline__ Q4 dq_trans(const FkState &f, int j, int ax) {
    const Q4 qr{f.dq[j][0], f.dq[j][1], f.dq[j][2], f.dq[j][3]};
    const Q4 e{0.0, ax == 0 ? 1.0 : 0.0, ax == 1 ? 1.0 : 0.0, ax == 2 ? 1.0 : 0.0};
    const Q4 r = qmul(e, qr);
    return Q4{0.5 * r.w, 0.5 * r.x, 0.5 * r.y, 0.5 * r.z};
}

// ---------------------------------------------------------------------------
// dual-quaternion blend (skinning.py:314-329)

struct Blend {
    double b[8];
    double a;
    double coef[4];
    int js[4];
    int dom;
    bool degenerate;
};

template <typename DQ>
__device__ __forceinline__ void dq_blend(const int *idx4, const double *w4, int dom,
                                         const DQ &dq, Blend &B) {
    B.dom = dom;
    const double d0 = dq(dom, 0), d1 = dq(dom, 1), d2 = dq(dom, 2), d3 = dq(dom, 3);
    for (int s = 0; s < 4; ++s) {
        const int j = idx4[s] < 0 ? 0 : idx4[s];
        B.js[s] = j;
        const double dot = dq(j, 0) * d0 + dq(j, 1) * d1 + dq(j, 2) * d2 + dq(j, 3) * d3;
        B.coef[s] = w4[s] * (dot < 0.0 ? -1.0 : 1.0);
    }
    for (int k = 0; k < 8; ++k) {
        double acc = B.coef[0] * dq(B.js[0], k);
        for (int s = 1; s < 4; ++s) acc = acc + B.coef[s] * dq(B.js[s], k);
        B.b[k] = acc;
    }
    B.a = sqrt(B.b[0] * B.b[0] + B.b[1] * B.b[1] + B.b[2] * B.b[2] + B.b[3] * B.b[3]);
    B.degenerate = B.a < 1e-8;
    if (B.degenerate) {
        for (int k = 0; k < 8; ++k) B.b[k] = dq(dom, k);
        B.a = sqrt(B.b[0] * B.b[0] + B.b[1] * B.b[1] + B.b[2] * B.b[2] + B.b[3] * B.b[3]);
    }
}

// normalized transform of a rest point (dq_transform_points, skinning.py:371-375)
__device__ __forceinline__ V3 dq_apply(const Blend &B, V3 rest, Q4 &cr_out) {
    const Q4 cr{B.b[0] / B.a, B.b[1] / B.a, B.b[2] / B.a, B.b[3] / B.a};
    const Q4 cd{B.b[4] / B.a, B.b[5] / B.a, B.b[6] / B.a, B.b[7] / B.a};
    const Q4 t = qmul(cd, qconj(cr));
    cr_out = cr;
    return qrot(cr, rest) + v3(2.0 * t.x, 2.0 * t.y, 2.0 * t.z);
}

// (3,8) derivative of the normalized transform w.r.t. the blend
// (_transform_jacobian_wrt_blend, skinning.py:332-368)
__device__ inline void dq_dtransform(const Blend &B, V3 r, double J[3][8]) {
    const double a = B.a;
    const double cr[4] = {B.b[0] / a, B.b[1] / a, B.b[2] / a, B.b[3] / a};
    const double cd[4] = {B.b[4] / a, B.b[5] / a, B.b[6] / a, B.b[7] / a};
    const double w = cr[0];
    const V3 u = v3(cr[1], cr[2], cr[3]);
    const double rv[3] = {r.x, r.y, r.z}, uu[3] = {u.x, u.y, u.z};
    const double uv = u.x * r.x + u.y * r.y + u.z * r.z;
    double drot[3][4];
    const V3 c0 = cross3(u, r);
    drot[0][0] = 2.0 * (w * r.x + c0.x);
    drot[1][0] = 2.0 * (w * r.y + c0.y);
    drot[2][0] = 2.0 * (w * r.z + c0.z);
    const double skew[3][3] = {{0.0, -r.z, r.y}, {r.z, 0.0, -r.x}, {-r.y, r.x, 0.0}};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            drot[i][1 + j] = 2.0 * (uu[i] * rv[j] - rv[i] * uu[j] + uv * (i == j ? 1.0 : 0.0)
                                    - w * skew[i][j]);
    // rblk = 2 * Right(conj(cr))[1:, :], lblk = 2 * (Left(cd) * [1,-1,-1,-1])[1:, :]
    const double cw = cr[0], cx = cr[1], cy = cr[2], cz = cr[3];
    const double rblk[3][4] = {{2.0 * -cx, 2.0 * cw, 2.0 * -cz, 2.0 * cy},
                               {2.0 * -cy, 2.0 * cz, 2.0 * cw, 2.0 * -cx},
                               {2.0 * -cz, 2.0 * -cy, 2.0 * cx, 2.0 * cw}};
    const double dw = cd[0], dx = cd[1], dy = cd[2], dz = cd[3];
    const double lblk[3][4] = {{2.0 * dx, 2.0 * -dw, 2.0 * dz, 2.0 * -dy},
                               {2.0 * dy, 2.0 * -dz, 2.0 * -dw, 2.0 * dx},
                               {2.0 * dz, 2.0 * dy, 2.0 * -dx, 2.0 * -dw}};
    double proj[4][4], dcd[4][4];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            proj[i][j] = ((i == j ? 1.0 : 0.0) - cr[i] * cr[j]) / a;
            dcd[i][j] = -(cd[i] * cr[j]) / a;
        }
    for (int i = 0; i < 3; ++i) {
        for (int k = 0; k < 4; ++k) {
            double s1 = (drot[i][0] + lblk[i][0]) * proj[0][k];
            for (int j = 1; j < 4; ++j) s1 = s1 + (drot[i][j] + lblk[i][j]) * proj[j][k];
            double s2 = rblk[i][0] * dcd[0][k];
            for (int j = 1; j < 4; ++j) s2 = s2 + rblk[i][j] * dcd[j][k];
            J[i][k] = s1 + s2;
            J[i][4 + k] = rblk[i][k] / a;
        }
    }
}
