"""Stage-level parity: solve_pose / solve_nonrigid / snap_vertices on the GPU
against the oracle on identical problems (per call).

Tolerances (BASELINE.json north_star): per-iteration energy rel. err <= 1e-4,
final vertices <= 1e-4 of the bounding-box diagonal, identical decision
traces (halvings / rejected / damped / breakdown)."""

import numpy as np
import pytest

from helpers import bbox_diag, scene

pytestmark = pytest.mark.gpu
ETOL = 1e-4


def _pose_problems(actor, cam, frames, directional):
    """Stage I problems of frame 0 (3 rounds) and a teacher-forced frame 1."""
    from oracle import frame as OF
    from oracle import posefit as OP
    from paper_1810_02648_b200.config import SequenceConfig
    cfg = SequenceConfig(directional=directional)
    out = []
    st = OF.State()
    for fr in frames[:2]:
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        trace = []
        OF.stage1(prep, actor, cam, cfg, st, actor.mesh.rest_vertices + (0 if st.disp_rest is None else st.disp_rest), trace)
        out.append((prep, trace, st))
        _, _, _, st, _, _ = OF.solve_frame(prep, actor, cam, cfg, st)
    return out, cfg


def _check_pose_logs(rep, logs):
    assert len(rep.iterations) == len(logs)
    for g, o in zip(rep.iterations, logs):
        assert g.halvings == o["halvings"] and g.rejected == o["rejected"] and g.damped == o["damped"]
        assert abs(g.energy_before - o["energy_before"]) <= ETOL * max(o["energy_before"], 1e-12)
        assert abs(g.energy_after - o["energy_after"]) <= ETOL * max(o["energy_after"], 1e-12)


@pytest.mark.parametrize("directional", [False, True])
def test_solve_pose_matches_oracle(directional):
    from dataclasses import replace
    from oracle import posefit as OP
    from oracle.frame import POSE_CONTOUR_MIN_RIGIDITY
    from oracle.geometry import Fk, skin
    from oracle.imaging import render_depth
    from paper_1810_02648_b200.actor import _class_weight_array
    from paper_1810_02648_b200.config import ContourVertexSet, PoseParams
    from paper_1810_02648_b200.imageproc import DistanceField
    from paper_1810_02648_b200.pose_stage import PoseProblem, solve_pose
    actor, cam, frames = scene("small", 128, 2)
    cfg_rounds = [dict(lambda_2d=0.0, lambda_sil=0.0), dict(lambda_sil=0.0), {}]
    from paper_1810_02648_b200.config import PoseHyperparams
    hyper0 = PoseHyperparams()
    x = np.zeros(36)
    from oracle import frame as OF
    from paper_1810_02648_b200.config import SequenceConfig
    prep = OF.prepare(frames[0].image, frames[0].mask, frames[0].detections, actor,
                      SequenceConfig(directional=directional))
    gfield = DistanceField(frames[0].mask)
    rig = _class_weight_array(actor.mesh.vertex_labels)
    for over in cfg_rounds:
        hp = replace(hyper0, gn_iterations=12, **over)
        fk = Fk(actor.skeleton, x)
        model = skin(actor.mesh.rest_vertices, actor.skinning, fk.dqs)[0]
        zb = render_depth(cam, model, actor.mesh.triangles)
        idx, n2 = OP.contour_vertices(model, actor.mesh, cam, zb)
        rim = OP.outer_rim(model, idx, cam, zb) & (rig[idx] >= POSE_CONTOUR_MIN_RIGIDITY)
        opb = OP.PoseProblem(actor.skeleton, actor.skinning, cam, prep.detections, prep.field, idx, n2,
                             actor.mesh.rest_vertices[idx], hp, directional=directional, enabled=rim)
        xo, logs, _, _ = OP.solve_pose(opb, x)
        gpb = PoseProblem(actor.skeleton, actor.skinning, cam, prep.detections, gfield,
                          ContourVertexSet(idx, n2), actor.mesh.rest_vertices[idx], hp,
                          directional=directional, contour_enabled=rim)
        xg, rep = solve_pose(gpb, PoseParams.from_vector(x))
        _check_pose_logs(rep, logs)
        assert np.abs(xg.to_vector() - xo).max() <= 1e-6 * max(1.0, np.abs(xo).max())
        x = xo


def _surface(actor, cam, frames, directional, frame=1):
    """Stage II problem of a teacher-forced frame."""
    from oracle import frame as OF
    from paper_1810_02648_b200.config import SequenceConfig
    cfg = SequenceConfig(directional=directional)
    st = OF.State()
    for fr in frames[:frame]:
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        _, _, _, st, _, _ = OF.solve_frame(prep, actor, cam, cfg, st)
    fr = frames[frame]
    prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
    disp = st.disp_rest if st.disp_rest is not None else 0.0
    drest = actor.mesh.rest_vertices + disp
    x, _ = OF.stage1(prep, actor, cam, cfg, st, drest)
    pb, v_init, vs, rot = OF.stage2_problem(prep, actor, cam, cfg, st, x, drest)
    return pb, v_init


def _mirror(pb, actor):
    from paper_1810_02648_b200.config import ContourVertexSet
    from paper_1810_02648_b200.imageproc import DistanceField
    from paper_1810_02648_b200.nonrigid_stage import NonrigidProblem
    return NonrigidProblem(actor.mesh, pb.camera, pb.hyper, pb.skinned, pb.pyramid,
                           DistanceField(pb.field.mask), pb.visible,
                           ContourVertexSet(pb.boundary_idx, pb.normals2d), pb.enabled,
                           pb.prev, pb.prev2, pb.directional)


@pytest.mark.parametrize("preset,res,frame", [("small", 128, 0), ("small", 128, 1), ("standard", 256, 1)])
def test_solve_nonrigid_matches_oracle(preset, res, frame):
    from oracle import surface as OS
    from paper_1810_02648_b200.nonrigid_stage import solve_nonrigid
    actor, cam, frames = scene(preset, res, frame + 1)
    pb, v_init = _surface(actor, cam, frames, directional=False, frame=frame)
    vo, logs, tot = OS.solve_surface(pb, v_init)
    vg, rep = solve_nonrigid(_mirror(pb, actor), v_init)
    assert len(rep.iterations) == len(logs)
    for g, o in zip(rep.iterations, logs):
        assert g.level == o["level"]
        assert g.halvings == o["halvings"] and g.rejected == o["rejected"]
        assert g.pcg_breakdown == o["pcg_breakdown"]
        assert abs(g.energy_before - o["energy_before"]) <= ETOL * o["energy_before"]
        assert abs(g.energy_after - o["energy_after"]) <= ETOL * o["energy_after"]
        for k, val in o["terms"].items():
            assert abs(g.terms[k] - val) <= ETOL * max(o["energy_before"], 1e-12), k
    assert rep.pruned == tot["pruned"] and rep.behind_camera == tot["behind_camera"]
    assert np.abs(vg - vo).max() <= 1e-4 * bbox_diag(actor)


def test_snap_matches_oracle():
    from oracle import surface as OS
    from paper_1810_02648_b200.nonrigid_stage import snap_vertices
    actor, cam, frames = scene("small", 128, 2)
    pb, v_init = _surface(actor, cam, frames, directional=False, frame=1)
    vo, info = OS.snap(v_init, pb)
    vg, ginfo = snap_vertices(v_init, _mirror(pb, actor))
    assert (ginfo.walked, ginfo.reached, ginfo.stuck) == (info["walked"], info["reached"], info["stuck"])
    assert np.abs(vg - vo).max() <= 1e-9 * bbox_diag(actor)
