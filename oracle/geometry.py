"""ORACLE (test infrastructure only): camera, quaternions, FK, DQ skinning.

Restates reference `camera.py:45-83`, `skinning.py:85-398` in numpy.
"""

from __future__ import annotations

import numpy as np

GIMBAL_EPS = 1e-6          # skinning.py:29
DEGENERATE_BLEND_EPS = 1e-8  # skinning.py:30


# ---------------------------------------------------------------------------
# camera (camera.py:45-83)

def project(cam, pts):
    """(pix (...,2), valid (...)); rows with z <= 1e-9 are zeroed."""
    pts = np.asarray(pts, dtype=np.float64)
    z = pts[..., 2]
    ok = z > 1e-9
    zs = np.where(ok, z, 1.0)
    pix = np.empty(pts.shape[:-1] + (2,))
    pix[..., 0] = cam.fx * pts[..., 0] / zs + cam.cx
    pix[..., 1] = cam.fy * pts[..., 1] / zs + cam.cy
    pix[~ok] = 0.0
    return pix, ok


def projection_jac(cam, pts):
    """(...,2,3) d(pix)/d(point); zero rows when z <= 1e-9."""
    pts = np.asarray(pts, dtype=np.float64)
    z = pts[..., 2]
    ok = z > 1e-9
    zs = np.where(ok, z, 1.0)
    out = np.zeros(pts.shape[:-1] + (2, 3))
    out[..., 0, 0] = cam.fx / zs
    out[..., 0, 2] = -cam.fx * pts[..., 0] / (zs * zs)
    out[..., 1, 1] = cam.fy / zs
    out[..., 1, 2] = -cam.fy * pts[..., 1] / (zs * zs)
    out[~ok] = 0.0
    return out, ok


# ---------------------------------------------------------------------------
# quaternions (w, x, y, z)  (skinning.py:85-165)

def qmul(a, b):
    aw, ax, ay, az = np.moveaxis(a, -1, 0)
    bw, bx, by, bz = np.moveaxis(b, -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw], axis=-1)


def qconj(q):
    out = np.array(q, dtype=np.float64, copy=True)
    out[..., 1:] *= -1.0
    return out


def qrot(q, v):
    u = q[..., 1:]
    t = 2.0 * np.cross(u, v)
    return v + q[..., 0:1] * t + np.cross(u, t)


def as_pure(v):
    out = np.zeros(v.shape[:-1] + (4,))
    out[..., 1:] = v
    return out


def rotmat_to_quat(m):
    """Shepperd's largest-pivot branch (skinning.py:115-141), one matrix."""
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    if tr > max(m[0, 0], m[1, 1], m[2, 2]):
        s = np.sqrt(tr + 1.0) * 2.0
        return np.array([0.25 * s, (m[2, 1] - m[1, 2]) / s,
                         (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s])
    if m[0, 0] >= m[1, 1] and m[0, 0] >= m[2, 2]:
        s = np.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2.0
        return np.array([(m[2, 1] - m[1, 2]) / s, 0.25 * s,
                         (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s])
    if m[1, 1] >= m[2, 2]:
        s = np.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2.0
        return np.array([(m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s,
                         0.25 * s, (m[1, 2] + m[2, 1]) / s])
    s = np.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2.0
    return np.array([(m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s,
                     (m[1, 2] + m[2, 1]) / s, 0.25 * s])


def _left(p):
    w, x, y, z = np.moveaxis(p, -1, 0)
    return np.stack([np.stack([w, -x, -y, -z], -1), np.stack([x, w, -z, y], -1),
                     np.stack([y, z, w, -x], -1), np.stack([z, -y, x, w], -1)], -2)


def _right(q):
    w, x, y, z = np.moveaxis(q, -1, 0)
    return np.stack([np.stack([w, -x, -y, -z], -1), np.stack([x, w, z, -y], -1),
                     np.stack([y, -z, w, x], -1), np.stack([z, y, -x, w], -1)], -2)


# ---------------------------------------------------------------------------
# forward kinematics (skinning.py:171-300)

def axis_angle_matrix(axis, angle):
    c, s = np.cos(angle), np.sin(angle)
    x, y, z = axis
    k = 1.0 - c
    return np.array([[c + x * x * k, x * y * k - z * s, x * z * k + y * s],
                     [y * x * k + z * s, c + y * y * k, y * z * k - x * s],
                     [z * x * k - y * s, z * y * k + x * s, c + z * z * k]])


_E = np.eye(3)


class Fk:
    """rot (J,3,3), pos (J,3), markers (4,3), axes/pivots (30,3), dqs (J,8)."""

    def __init__(self, sk, x):
        x = np.asarray(x, dtype=np.float64)
        j = sk.n_joints
        rot = np.empty((j, 3, 3))
        pos = np.empty((j, 3))
        axes = np.zeros((30, 3))
        piv = np.zeros((30, 3))
        ra = x[0:3]
        rx = axis_angle_matrix(_E[0], ra[0])
        ry = axis_angle_matrix(_E[1], ra[1])
        rz = axis_angle_matrix(_E[2], ra[2])
        rot[0] = rx @ ry @ rz
        pos[0] = x[3:6] + sk.local_offsets[0]
        axes[0] = _E[0]
        axes[1] = rx @ _E[1]
        axes[2] = rx @ ry @ _E[2]
        piv[0:3] = pos[0]
        self.gimbal = bool(abs(np.cos(ra[1])) < GIMBAL_EPS)
        theta = x[6:33]
        per_joint = [[] for _ in range(j)]
        for k, jk in enumerate(sk.dof_joint):
            per_joint[jk].append(k)
        for i in range(1, j):
            p = sk.parents[i]
            pos[i] = rot[p] @ sk.local_offsets[i] + pos[p]
            r = rot[p]
            for k in per_joint[i]:
                axes[3 + k] = r @ sk.dof_axes[k]
                piv[3 + k] = pos[i]
                r = r @ axis_angle_matrix(sk.dof_axes[k], theta[k])
            rot[i] = r
        h = sk.head_index
        self.markers = sk.marker_offsets @ rot[h].T + pos[h]
        self.trans = pos - np.einsum("jik,jk->ji", rot, sk.rest_positions())
        qr = np.stack([rotmat_to_quat(m) for m in rot])
        qd = 0.5 * qmul(as_pure(self.trans), qr)
        self.rot, self.pos, self.axes, self.pivots = rot, pos, axes, piv
        self.dqs = np.concatenate([qr, qd], axis=-1)


def joint_jacobian(sk, fk):
    """(J+4,3,36) d(joints, markers)/dx  (skinning.py:249-266)."""
    j = sk.n_joints
    pts = np.concatenate([fk.pos, fk.markers])
    lever = pts[None] - fk.pivots[:, None]
    spin = np.cross(fk.axes[:, None, :], lever)
    reach = np.ones((30, j + 4), dtype=bool)
    reach[3:, :j] = sk.dof_moves_position
    reach[3:, j:] = sk.dof_moves_frame[:, sk.head_index][:, None]
    spin = spin * reach[:, :, None]
    out = np.zeros((j + 4, 3, 36))
    out[:, :, 0:3] = np.moveaxis(spin[0:3], 0, 2)
    out[:, :, 6:33] = np.moveaxis(spin[3:], 0, 2)
    out[:, :, 3:6] = np.eye(3)
    return out


def dq_jacobian(sk, fk):
    """(J,8,36) d(joint dual quaternions)/dx  (skinning.py:269-300)."""
    j = sk.n_joints
    qr = fk.dqs[:, :4]
    reach = np.ones((30, j), dtype=bool)
    reach[3:] = sk.dof_moves_frame
    dqr = 0.5 * qmul(as_pure(fk.axes)[:, None, :], qr[None])
    tdot = np.cross(fk.axes[:, None, :], fk.trans[None] - fk.pivots[:, None, :])
    dqd = 0.5 * (qmul(as_pure(tdot), qr[None]) + qmul(as_pure(fk.trans)[None], dqr))
    dqr = dqr * reach[:, :, None]
    dqd = dqd * reach[:, :, None]
    out = np.zeros((j, 8, 36))
    out[:, 0:4, 0:3] = np.moveaxis(dqr[0:3], 0, 2)
    out[:, 4:8, 0:3] = np.moveaxis(dqd[0:3], 0, 2)
    out[:, 0:4, 6:33] = np.moveaxis(dqr[3:], 0, 2)
    out[:, 4:8, 6:33] = np.moveaxis(dqd[3:], 0, 2)
    for a in range(3):
        out[:, 4:8, 3 + a] = 0.5 * qmul(as_pure(_E[a])[None], qr)
    return out


# ---------------------------------------------------------------------------
# dual-quaternion skinning (skinning.py:314-398)

def _blend(skin, dqs, subset):
    idx = skin.indices if subset is None else skin.indices[subset]
    w = skin.weights if subset is None else skin.weights[subset]
    dom = skin.dominant if subset is None else skin.dominant[subset]
    safe = np.where(idx < 0, 0, idx)
    g = dqs[safe]
    dots = np.einsum("msk,mk->ms", g[:, :, :4], dqs[dom, :4])
    coef = w * np.where(dots < 0.0, -1.0, 1.0)
    b = np.einsum("ms,msk->mk", coef, g)
    a = np.linalg.norm(b[:, :4], axis=1)
    deg = a < DEGENERATE_BLEND_EPS
    if deg.any():
        b[deg] = dqs[dom[deg]]
        a[deg] = np.linalg.norm(b[deg, :4], axis=1)
    return b, a, coef, safe, dom, deg


def _dtransform_dblend(b, a, rest):
    m = b.shape[0]
    cr = b[:, :4] / a[:, None]
    cd = b[:, 4:] / a[:, None]
    w, u = cr[:, 0], cr[:, 1:]
    uv = np.einsum("mi,mi->m", u, rest)
    drot = np.empty((m, 3, 4))
    drot[:, :, 0] = 2.0 * (w[:, None] * rest + np.cross(u, rest))
    skew = np.zeros((m, 3, 3))
    skew[:, 0, 1], skew[:, 0, 2] = -rest[:, 2], rest[:, 1]
    skew[:, 1, 0], skew[:, 1, 2] = rest[:, 2], -rest[:, 0]
    skew[:, 2, 0], skew[:, 2, 1] = -rest[:, 1], rest[:, 0]
    drot[:, :, 1:] = 2.0 * (np.einsum("mi,mj->mij", u, rest) - np.einsum("mi,mj->mij", rest, u)
                            + uv[:, None, None] * np.eye(3)[None] - w[:, None, None] * skew)
    flip = np.array([1.0, -1.0, -1.0, -1.0])
    rblk = 2.0 * _right(qconj(cr))[:, 1:, :]
    lblk = 2.0 * (_left(cd) * flip[None, None, :])[:, 1:, :]
    proj = (np.eye(4)[None] - np.einsum("mi,mj->mij", cr, cr)) / a[:, None, None]
    dcd = -np.einsum("mi,mj->mij", cd, cr) / a[:, None, None]
    dv_dbr = np.einsum("mij,mjk->mik", drot + lblk, proj) + np.einsum("mij,mjk->mik", rblk, dcd)
    return np.concatenate([dv_dbr, rblk / a[:, None, None]], axis=2)


def skin(rest, skin_w, dqs, dqj=None, subset=None):
    """(positions (M,3), rotations (M,4), jac (M,3,36)|None, degenerate)."""
    rest = np.asarray(rest, dtype=np.float64)
    b, a, coef, safe, dom, deg = _blend(skin_w, dqs, subset)
    cr = b[:, :4] / a[:, None]
    cd = b[:, 4:] / a[:, None]
    trans = 2.0 * qmul(cd, qconj(cr))[:, 1:]
    pos = qrot(cr, rest) + trans
    jac = None
    if dqj is not None:
        db = np.einsum("ms,mskp->mkp", coef, dqj[safe])
        if deg.any():
            db[deg] = dqj[dom[deg]]
        jac = np.einsum("mik,mkp->mip", _dtransform_dblend(b, a, rest), db)
    return pos, cr, jac, deg
