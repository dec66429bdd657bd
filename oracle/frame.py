"""ORACLE (test infrastructure only): per-frame glue and sequence recursion.

Restates reference `pipeline.py:156-302,378-397`: preprocessing, detection
conditioning, Stage I rounds (frame-0 cold start), Stage II setup (visibility,
contour, rim filter, part mask gating), solve, snapping, displacement warp
and the `TrackState` update.  Sequence drivers beyond the sequential loop are
out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from paper_1810_02648_b200.actor import _class_weight_array
from paper_1810_02648_b200.config import FrameDetections

from .geometry import Fk, project, qconj, qrot, skin
from .imaging import DistanceField, gaussian_pyramid, render_depth
from .posefit import PoseProblem, contour_vertices, extrapolate, outer_rim, rescale_detections, solve_pose
from .surface import SurfaceProblem, part_label_mask, snap, solve_surface, visible_vertices

POSE_CONTOUR_MIN_RIGIDITY = 2.0  # pipeline.py:45


@dataclass
class Prepared:
    field: DistanceField | None
    pyramid: list
    detections: FrameDetections


@dataclass
class State:
    """Vectors instead of PoseParams: x_prev (36,), x_prev2, joints_prev (J,3),
    disp_rest (N,3), v_prev (N,3), v_prev2."""
    x_prev: np.ndarray | None = None
    x_prev2: np.ndarray | None = None
    joints_prev: np.ndarray | None = None
    disp_rest: np.ndarray | None = None
    v_prev: np.ndarray | None = None
    v_prev2: np.ndarray | None = None


def prepare(image, mask, det, actor, config):
    """preprocess_frame + condition_detections (pipeline.py:156-170)."""
    fld = DistanceField(mask) if np.any(mask) else None
    pyr = gaussian_pyramid(image, config.nonrigid.pyramid_kernels)
    j3, _ = rescale_detections(det.joints3d, actor.skeleton, det.valid3d)
    return Prepared(fld, pyr, FrameDetections(det.joints2d, j3, det.valid2d, det.valid3d))


def stage1(prep, actor, cam, config, st: State, drest, trace=None):
    """pipeline.py:173-224. Returns (x, logs)."""
    sk, sw, mesh = actor.skeleton, actor.skinning, actor.mesh
    hyper = config.pose
    if config.mode == "detections_only":
        hyper = replace(hyper, lambda_sil=0.0)
    if st.x_prev is None:
        x = np.zeros(36)
        rounds = [{"lambda_2d": 0.0, "lambda_sil": 0.0}, {"lambda_sil": 0.0}]
        rounds += [{}] * max(1, config.frame0_rounds - len(rounds))
        hyper = replace(hyper, gn_iterations=hyper.gn_iterations * config.frame0_iteration_scale)
        prev_pos = None
    else:
        x = extrapolate(st.x_prev, st.x_prev2, sk)
        rounds = [{}]
        prev_pos = st.joints_prev
    rigid = _class_weight_array(mesh.vertex_labels)
    logs = []
    for ov in rounds:
        hp = replace(hyper, **ov) if ov else hyper
        fk = Fk(sk, x)
        model = skin(drest, sw, fk.dqs)[0]
        zbuf = render_depth(cam, model, mesh.triangles)
        cidx, n2 = contour_vertices(model, mesh, cam, zbuf)
        rim = outer_rim(model, cidx, cam, zbuf)
        rim &= rigid[cidx] >= POSE_CONTOUR_MIN_RIGIDITY
        pb = PoseProblem(sk, sw, cam, prep.detections, prep.field, cidx, n2, drest[cidx], hp,
                         prev_positions=prev_pos, directional=config.directional, enabled=rim)
        if trace is not None:
            trace.append(("pose_round", dict(x0=x.copy(), contour=cidx.copy(), rim=rim.copy())))
        x, lg, _, _ = solve_pose(pb, x)
        logs.extend(lg)
    return x, logs


def stage2_problem(prep, actor, cam, config, st: State, x, drest):
    """Stage II setup (pipeline.py:227-255). Returns (problem, v_init, V^S, rot)."""
    mesh, sk, sw = actor.mesh, actor.skeleton, actor.skinning
    fk = Fk(sk, x)
    vs, rot, _, _ = skin(mesh.rest_vertices, sw, fk.dqs)
    v_init = skin(drest, sw, fk.dqs)[0]
    zbuf = render_depth(cam, v_init, mesh.triangles)
    visible = np.flatnonzero(visible_vertices(v_init, mesh, cam, zbuf))
    bidx, n2 = contour_vertices(v_init, mesh, cam, zbuf)
    enabled = outer_rim(v_init, bidx, cam, zbuf, min_thickness=0.0)
    if config.enable_part_mask and len(bidx):
        labels, vparts = part_label_mask(v_init, mesh, sw, sk, cam, config.nonrigid.part_dilation)
        pix, ok = project(cam, v_init[bidx])
        xi = np.clip(np.round(pix[:, 0]).astype(int), 0, cam.width - 1)
        yi = np.clip(np.round(pix[:, 1]).astype(int), 0, cam.height - 1)
        at = labels[yi, xi]
        enabled &= ok & ((at == 0) | (at == vparts[bidx]))
    pb = SurfaceProblem(mesh, cam, config.nonrigid, vs, prep.pyramid, prep.field, visible, bidx,
                        n2, enabled, prev=st.v_prev, prev2=st.v_prev2,
                        directional=config.directional)
    return pb, v_init, vs, rot


def solve_frame(prep, actor, cam, config, st: State, trace=None):
    """pipeline.py:263-302. Returns (x, v, V^S, new_state, pose_logs, surf_logs)."""
    mesh = actor.mesh
    n = mesh.n_vertices
    disp = st.disp_rest if st.disp_rest is not None else np.zeros((n, 3))
    drest = mesh.rest_vertices + disp
    x, plogs = stage1(prep, actor, cam, config, st, drest, trace)
    slogs = None
    if config.mode == "full":
        pb, v_init, vs, rot = stage2_problem(prep, actor, cam, config, st, x, drest)
        if trace is not None:
            trace.append(("surface_problem", dict(problem=pb, v_init=v_init.copy())))
        v, slogs, _ = solve_surface(pb, v_init)
        if config.enable_snapping:
            v, _ = snap(v, pb)
        delta = v - vs
        new_disp = qrot(qconj(rot), delta) if config.enable_warping else delta
    else:
        fk = Fk(actor.skeleton, x)
        vs = skin(mesh.rest_vertices, actor.skinning, fk.dqs)[0]
        v = vs
        new_disp = np.zeros((n, 3))
    fk = Fk(actor.skeleton, x)
    new = State(x_prev=x, x_prev2=st.x_prev, joints_prev=fk.pos, disp_rest=new_disp,
                v_prev=v, v_prev2=st.v_prev)
    return x, v, vs, new, plogs, slogs


def run_sequence(images, masks, dets, actor, cam, config):
    """Sequential driver (pipeline.py:378-397): per-frame (x, v)."""
    st = State()
    out = []
    for img, msk, det in zip(images, masks, dets):
        prep = prepare(img, msk, det, actor, config)
        x, v, _, st, _, _ = solve_frame(prep, actor, cam, config, st)
        out.append((x, v))
    return out
