"""ORACLE (test infrastructure only): Stage I skeletal pose Gauss-Newton.

Restates reference `pose_stage.py:92-459`: detection conditioning,
constant-velocity init, occluding-contour extraction, contour side signs,
outer-rim filter, the stacked residual / Jacobian of the pose energy and the
halving Gauss-Newton loop.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import Fk, dq_jacobian, joint_jacobian, project, projection_jac, skin
from .imaging import DistanceField, render_depth
from .linsolve import dense_solve

VISIBILITY_DEPTH_TOL = 0.01  # pose_stage.py:34


def rescale_detections(j3d, sk, valid3d=None):
    """Bone-length rescale, root outward (pose_stage.py:92-116)."""
    j3d = np.asarray(j3d, dtype=np.float64)
    rest = sk.rest_positions()
    bone = sk.bone_lengths()
    out = np.zeros_like(j3d)
    out[0] = j3d[0]
    fallback = []
    for i in range(1, sk.n_joints):
        p = sk.parents[i]
        d = j3d[i] - j3d[p]
        n = np.linalg.norm(d)
        if not (n > 1e-9 and (valid3d is None or (valid3d[i] and valid3d[p]))):
            d = rest[i] - rest[p]
            n = np.linalg.norm(d)
            fallback.append(i)
        out[i] = out[p] + bone[i] * d / n
    return out, fallback


def extrapolate(x1, x2, sk):
    """2 x1 - x2 with theta clamped (pose_stage.py:119-127); vectors in, vector out."""
    x = np.array(x1, dtype=np.float64) if x2 is None else 2.0 * np.asarray(x1) - np.asarray(x2)
    x = x.copy()
    x[6:33] = sk.clamp_theta(x[6:33])
    return x


def vertex_normals(verts, tris):
    """Area-weighted, add.at in slot order (pose_stage.py:139-148)."""
    p = verts[tris]
    tn = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
    out = np.zeros_like(verts)
    for k in range(3):
        np.add.at(out, tris[:, k], tn)
    nrm = np.linalg.norm(out, axis=1)
    nrm[nrm < 1e-12] = 1.0
    return out / nrm[:, None]


def contour_vertices(verts, mesh, cam, zbuf=None):
    """(indices ascending, normals2d)  (pose_stage.py:151-191)."""
    tris = mesh.triangles
    p = verts[tris]
    tn = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
    front = np.einsum("ti,ti->t", tn, p.mean(axis=1)) < 0.0
    ta, tb = mesh.edge_tris[:, 0], mesh.edge_tris[:, 1]
    sil = np.where(tb < 0, front[ta], front[ta] != front[np.maximum(tb, 0)])
    cand = np.unique(mesh.edges[sil])
    if cand.size == 0:
        return cand, np.zeros((0, 2))
    if zbuf is None:
        zbuf = render_depth(cam, verts, tris)
    pix, ok = project(cam, verts[cand])
    z = verts[cand, 2]
    xi = np.clip(np.round(pix[:, 0]).astype(int), 0, cam.width - 1)
    yi = np.clip(np.round(pix[:, 1]).astype(int), 0, cam.height - 1)
    inimg = ((pix[:, 0] >= -0.5) & (pix[:, 0] <= cam.width - 0.5)
             & (pix[:, 1] >= -0.5) & (pix[:, 1] <= cam.height - 0.5))
    cand = cand[ok & inimg & (z <= zbuf[yi, xi] + VISIBILITY_DEPTH_TOL * z)]
    n3 = vertex_normals(verts, tris)[cand]
    jac, _ = projection_jac(cam, verts[cand])
    n2 = np.einsum("bij,bj->bi", jac, n3)
    nn = np.linalg.norm(n2, axis=1)
    good = nn > 1e-12
    n2[good] /= nn[good, None]
    n2[~good] = 0.0
    return cand, n2


def side_signs(field, normals2d, pix):
    """b = -1 iff inside the mask and n . (-dir) < 0  (pose_stage.py:194-215)."""
    z = -field.side_direction(pix)
    flip = np.einsum("bi,bi->b", normals2d, -z) < 0.0
    return np.where(field.inside(pix), np.where(flip, -1.0, 1.0), 1.0)


def outer_rim(verts, idx, cam, zbuf, min_thickness=12.0, max_distance=1.5):
    """Rim keep mask (pose_stage.py:218-264)."""
    mask = np.isfinite(zbuf)
    if idx.size == 0 or not mask.any():
        return np.zeros(idx.shape[0], dtype=bool)
    pix, ok = project(cam, verts[idx])
    own = DistanceField(mask)
    d, c = own.sample_value(pix)
    keep = ok & ~c & (d <= max_distance)
    if min_thickness > 0.0 and keep.any():
        rmax = int(np.ceil(min_thickness / 2.0)) + 2
        ang = np.linspace(0.0, 2.0 * np.pi, 16, endpoint=False)
        offs = (np.stack([np.cos(ang), np.sin(ang)], axis=1)[:, None, :]
                * np.arange(1, rmax + 1, dtype=np.float64)[None, :, None])
        probe = (pix[None, None, :, :] + offs[:, :, None, :]).reshape(-1, 2)
        pd, _ = own.sample_value(probe)
        deep = np.where(own.inside(probe), pd, 0.0).reshape(-1, len(pix)).max(axis=0)
        keep &= 2.0 * deep >= min_thickness
    return keep


@dataclass
class PoseProblem:
    skeleton: object
    skinning: object
    camera: object
    detections: object           # joints3d already rescaled
    field: DistanceField | None
    contour_idx: np.ndarray
    normals2d: np.ndarray
    contour_rest: np.ndarray     # (B,3)
    hyper: object
    prev_positions: np.ndarray | None = None
    directional: bool = True
    enabled: np.ndarray | None = None

    def __post_init__(self):
        j = self.skeleton.n_joints
        b = len(self.contour_idx)
        nt = 3 * j if self.prev_positions is not None else 0
        sizes = [("detection2d", 2 * (j + 4)), ("detection3d", 3 * j), ("silhouette", b),
                 ("temporal", nt), ("anatomic", 27)]
        self.blocks, at = {}, 0
        for name, n in sizes:
            self.blocks[name] = slice(at, at + n)
            at += n
        self.n_rows = at
        self.tw = np.array([self.hyper.temporal_group_weights[g]
                            for g in self.skeleton.temporal_groups])
        self.l2d = np.full(j + 4, self.hyper.lambda_2d)
        self.l2d[j:] *= self.hyper.face_weight


def pose_evaluate(pb: PoseProblem, x, with_jac=True):
    """(F, J|None, energies, behind, gimbal)  (pose_stage.py:319-404)."""
    sk, cam, hp = pb.skeleton, pb.camera, pb.hyper
    j = sk.n_joints
    x = np.asarray(x, dtype=np.float64)
    fk = Fk(sk, x)
    jp = joint_jacobian(sk, fk) if with_jac else None
    F = np.zeros(pb.n_rows)
    J = np.zeros((pb.n_rows, 36)) if with_jac else None
    behind = 0

    pts = np.concatenate([fk.pos, fk.markers])
    pix, okz = project(cam, pts)
    behind += int(np.sum(~okz))
    dpi, _ = projection_jac(cam, pts)
    s = pb.blocks["detection2d"]
    w2 = np.sqrt(pb.l2d) * pb.detections.valid2d * okz
    F[s] = ((pix - pb.detections.joints2d) * w2[:, None]).reshape(-1)
    if with_jac:
        J[s] = (np.einsum("nij,njp->nip", dpi, jp) * w2[:, None, None]).reshape(-1, 36)

    s = pb.blocks["detection3d"]
    w3 = np.sqrt(hp.lambda_3d) * pb.detections.valid3d
    F[s] = ((fk.pos - pb.detections.joints3d - x[33:36]) * w3[:, None]).reshape(-1)
    if with_jac:
        j3 = jp[:j].copy()
        j3[:, :, 33:36] -= np.eye(3)
        J[s] = (j3 * w3[:, None, None]).reshape(-1, 36)

    s = pb.blocks["silhouette"]
    if len(pb.contour_idx) and pb.field is not None:
        dqj = dq_jacobian(sk, fk) if with_jac else None
        spos, _, sjac, _ = skin(pb.contour_rest, pb.skinning, fk.dqs, dqj, subset=pb.contour_idx)
        cpix, cok = project(cam, spos)
        behind += int(np.sum(~cok))
        val, grad, clamped = pb.field.sample_residual(cpix)
        ok = cok & ~clamped
        if pb.enabled is not None:
            ok = ok & pb.enabled
        ws = np.sqrt(hp.lambda_sil) * ok
        F[s] = val * ws
        if with_jac:
            cdpi, _ = projection_jac(cam, spos)
            rows = np.einsum("bi,bij,bjp->bp", grad, cdpi, sjac)
            sign = side_signs(pb.field, pb.normals2d, cpix) if pb.directional else 1.0
            J[s] = rows * (ws * sign)[:, None]

    if pb.prev_positions is not None:
        s = pb.blocks["temporal"]
        wt = np.sqrt(hp.lambda_temporal * pb.tw)
        F[s] = ((fk.pos - pb.prev_positions) * wt[:, None]).reshape(-1)
        if with_jac:
            J[s] = (jp[:j] * wt[:, None, None]).reshape(-1, 36)

    s = pb.blocks["anatomic"]
    th = x[6:33]
    hi = th > sk.theta_max
    lo = th < sk.theta_min
    wa = np.sqrt(hp.lambda_anatomic)
    F[s] = wa * (np.where(hi, th - sk.theta_max, 0.0) + np.where(lo, sk.theta_min - th, 0.0))
    if with_jac:
        J[s.start + np.arange(27), 6 + np.arange(27)] = wa * (hi.astype(float) - lo.astype(float))
    energies = {k: float(np.sum(F[sl] ** 2)) for k, sl in pb.blocks.items()}
    return F, J, energies, behind, fk.gimbal


def solve_pose(pb: PoseProblem, x0):
    """Halving GN (pose_stage.py:429-459). Returns (x, logs, behind, gimbal);
    logs are dicts with energy_before/after, terms, step_norm, halvings, rejected, damped."""
    x = np.array(x0, dtype=np.float64, copy=True)
    logs, behind, gimbal = [], 0, False
    for _ in range(pb.hyper.gn_iterations):
        F, J, terms, bh, gb = pose_evaluate(pb, x)
        behind += bh
        gimbal = gimbal or gb
        a = J.T @ J
        a = 0.5 * (a + a.T)
        delta, damped, _ = dense_solve(a, -(J.T @ F))
        e0 = float(np.sum(F ** 2))
        halv, rej, step = 0, False, delta
        while True:
            F1 = pose_evaluate(pb, x + step, with_jac=False)[0]
            e1 = float(np.sum(F1 ** 2))
            if e1 <= e0:
                x = x + step
                break
            if halv >= pb.hyper.max_halvings:
                rej, e1 = True, e0
                break
            step = 0.5 * step
            halv += 1
        logs.append(dict(energy_before=e0, energy_after=e1, terms=terms,
                         step_norm=float(np.linalg.norm(step)), halvings=halv,
                         rejected=rej, damped=damped))
    return x, logs, behind, gimbal
