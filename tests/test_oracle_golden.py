"""CPU: pin the oracle (and the restated input generator) to golden fixtures
produced by running the real reference (tools/make_golden.py).  The oracle
must reproduce the reference bit for bit on these scenes."""

import os

import numpy as np
import pytest

from helpers import posing

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name), allow_pickle=False))


def gen(preset, res, n, seed):
    from oracle import imaging as OI
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.camera import suggest_camera
    actor = S.build_actor(preset, with_skirt=True)
    cam = suggest_camera(res, res)
    frames = S.generate_sequence(actor, cam, S.default_script(n, noise=S.NoiseParams(seed=seed)),
                                 OI.render_attributes, posing)
    return actor, cam, frames


def check_digest(g, frames):
    assert np.array_equal(g["img_sum"], [f.image.sum() for f in frames])
    assert np.array_equal(g["img_sq"], [(f.image ** 2).sum() for f in frames])
    assert np.array_equal(g["mask_count"], [f.mask.sum() for f in frames])
    assert np.array_equal(g["j2d"], np.stack([f.detections.joints2d for f in frames]))
    assert np.array_equal(g["j3d"], np.stack([f.detections.joints3d for f in frames]))


@pytest.mark.parametrize("name", ["ref_frames_small128_dir1.npz", "ref_frames_small128_dir0.npz",
                                  "ref_frames_standard256_dir0.npz"])
def test_oracle_sequence_bit_exact(name):
    from oracle import frame as OF
    from paper_1810_02648_b200.config import SequenceConfig
    g = load(name)
    preset, res, n, directional, seed = g["meta"]
    actor, cam, frames = gen(preset, int(res), int(n), int(seed))
    check_digest(g, frames)
    cfg = SequenceConfig(directional=bool(int(directional)))
    st = OF.State()
    for k, fr in enumerate(frames):
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        x, v, vs, st, plogs, slogs = OF.solve_frame(prep, actor, cam, cfg, st)
        assert np.array_equal(x, g["poses"][k])
        assert np.array_equal(v, g["vertices"][k])
        assert np.array_equal(vs, g["skinned"][k])
        assert np.array_equal([o["energy_before"] for o in plogs], g["pose_e0"][k][:len(plogs)])
        assert np.array_equal([o["halvings"] for o in slogs], g["nr_halv"][k])
        assert np.array_equal([o["energy_before"] for o in slogs], g["nr_e0"][k])


def test_oracle_kernels_bit_exact():
    from oracle import geometry as OG, imaging as OI, linsolve as OL, posefit as OP, surface as OS
    from paper_1810_02648_b200.actor import joint_body_parts
    from paper_1810_02648_b200.config import FrameDetections, PoseHyperparams, NonrigidHyperparams
    g = load("ref_kernels_small128.npz")
    actor, cam, frames = gen("small", 128, 2, 3)
    check_digest(g, frames)
    fr = frames[1]
    mesh, sk, sw = actor.mesh, actor.skeleton, actor.skinning
    assert np.array_equal(mesh.edges, g["edges"]) and np.array_equal(mesh.edge_tris, g["edge_tris"])
    assert np.array_equal(mesh.directed_weights, g["directed_weights"])
    assert np.array_equal(sw.dominant, g["dominant"])
    assert np.array_equal(joint_body_parts(sk), g["body_parts"])
    x = g["fk_x"]
    fk = OG.Fk(sk, x)
    assert np.array_equal(fk.pos, g["fk_pos"]) and np.array_equal(fk.markers, g["fk_markers"])
    assert np.array_equal(fk.dqs, g["fk_dqs"])
    assert np.array_equal(OG.joint_jacobian(sk, fk), g["fk_jp"])
    sub = g["skin_sub"]
    p, r, jac, _ = OG.skin(mesh.rest_vertices[sub], sw, fk.dqs, OG.dq_jacobian(sk, fk), subset=sub)
    assert np.array_equal(p, g["skin_pos"]) and np.array_equal(r, g["skin_rot"])
    assert np.array_equal(jac, g["skin_jac"])
    v = fr.gt_vertices
    zb = OI.render_depth(cam, v, mesh.triangles)
    assert np.array_equal(zb, g["zbuf"])
    ids, _ = OI.render_vertex_ids(cam, v, mesh.triangles, joint_body_parts(sk)[sw.dominant], background=0)
    assert np.array_equal(ids, g["part_ids"])
    labels, _ = OS.part_label_mask(v, mesh, sw, sk, cam, 10)
    assert np.array_equal(labels, g["part_labels"])
    idx, n2 = OP.contour_vertices(v, mesh, cam)
    assert np.array_equal(idx, g["contour_idx"]) and np.array_equal(n2, g["contour_n2d"])
    assert np.array_equal(OP.outer_rim(v, idx, cam, zb), g["rim_stage1"])
    assert np.array_equal(OP.outer_rim(v, idx, cam, zb, min_thickness=0.0), g["rim_stage2"])
    assert np.array_equal(np.flatnonzero(OS.visible_vertices(v, mesh, cam, zb)), g["visible"])
    df = OI.DistanceField(fr.mask)
    q = g["dt_q"]
    assert np.array_equal(df.sample_value(q)[0], g["dt_val"])
    res, grad, _ = df.sample_residual(q)
    assert np.array_equal(res, g["dt_res"]) and np.array_equal(grad, g["dt_grad"])
    assert np.array_equal(df.inside(q), g["dt_inside"])
    assert np.array_equal(OI.euclidean_dt(fr.mask), g["edt"])
    pyr = OI.gaussian_pyramid(fr.image, (15, 9, 3))
    assert np.array_equal([p.sum() for p in pyr], g["pyr_sum"])
    assert np.array_equal(np.stack([p[40:48, 50:58] for p in pyr]), g["pyr_samples"])
    j3, _ = OP.rescale_detections(fr.detections.joints3d, sk, fr.detections.valid3d)
    assert np.array_equal(j3, g["rescaled_j3d"])
    # Stage II system / PCG / solve / snap on the reference's problem
    import dataclasses
    hyper = NonrigidHyperparams()
    pyr_pb = OI.gaussian_pyramid(fr.image, hyper.pyramid_kernels)
    pb = OS.SurfaceProblem(mesh, cam, hyper, g["nr_skinned"], pyr_pb, OI.DistanceField(fr.mask), g["visible"],
                           g["contour_idx"], g["contour_n2d"], np.ones(len(g["contour_idx"]), bool),
                           prev=v + 0.001, prev2=v - 0.001, directional=False)
    ev = OS.surface_evaluate(pb, g["nr_v0"], 1)
    assert np.array_equal([ev["energies"][k] for k in ("photo", "silhouette", "smooth", "edge", "velocity",
                                                       "acceleration")], g["nr_energy_terms"])
    xo, done, brk, norms = OL.pcg(*OS.normal_system(pb, ev), 4)
    assert np.array_equal(xo, g["pcg_delta"]) and np.array_equal(norms, g["pcg_norms"])
    vo, logs, _ = OS.solve_surface(pb, g["nr_v0"])
    assert np.array_equal(vo, g["nr_solve_v"])
    assert np.array_equal([[o["energy_before"], o["energy_after"], o["halvings"]] for o in logs], g["nr_solve_e"])
    vs, info = OS.snap(vo, pb)
    assert np.array_equal(vs, g["snap_v"])
    assert [info["walked"], info["reached"], info["stuck"]] == list(g["snap_info"])
    det = FrameDetections(fr.detections.joints2d, j3, fr.detections.valid2d, fr.detections.valid3d)
    pp = OP.PoseProblem(sk, sw, cam, det, OI.DistanceField(fr.mask), idx, n2, mesh.rest_vertices[idx],
                        PoseHyperparams(), prev_positions=fk.pos + 0.01, directional=False)
    F, J, _, _, _ = OP.pose_evaluate(pp, x)
    assert np.array_equal(F, g["pose_F"]) and np.array_equal(J, g["pose_J"])
    a = J.T @ J
    a = 0.5 * (a + a.T)
    d, damped, _ = OL.dense_solve(a, -(J.T @ F))
    assert np.array_equal(d, g["dense_x"]) and damped == bool(g["dense_damped"])
    xs, plogs, _, _ = OP.solve_pose(pp, x)
    assert np.array_equal(xs, g["pose_solve_x"])
    assert np.array_equal([[o["energy_before"], o["energy_after"], o["halvings"]] for o in plogs], g["pose_solve_e"])
