"""Generate golden fixtures by running the REAL reference (`montrack`).

Run in the build container only (the reference is not on the GPU box):
  PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py [--bench]
Writes tests/golden/*.npz.  The fixtures hold small outputs plus input
checksums; inputs are regenerated from seeds by the restated generator
(`paper_1810_02648_b200.synthetic`, pinned by those checksums).
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden")


def _inputs_digest(frames):
    return dict(
        img_sum=np.array([f.image.sum() for f in frames]),
        img_sq=np.array([(f.image ** 2).sum() for f in frames]),
        mask_count=np.array([f.mask.sum() for f in frames]),
        j2d=np.stack([f.detections.joints2d for f in frames]),
        j3d=np.stack([f.detections.joints3d for f in frames]),
    )


def frames_fixture(preset, res, n, directional, seed=0):
    import montrack.actors as A
    from montrack.pipeline import SequenceConfig, SequenceInputs, run_sequence
    from montrack.synthetic import NoiseParams, default_script, generate_synthetic_sequence
    actor = A.build_actor(preset, with_skirt=True)
    cam = A.suggest_camera(res, res)
    seq = generate_synthetic_sequence(actor, cam, default_script(n, noise=NoiseParams(seed=seed)))
    inp = SequenceInputs(actor, cam, [f.image for f in seq.frames], [f.mask for f in seq.frames],
                         [f.detections for f in seq.frames])
    r = run_sequence(inp, SequenceConfig(directional=directional))
    out = _inputs_digest(seq.frames)
    out["poses"] = np.stack([fr.pose.to_vector() for fr in r.frames])
    out["vertices"] = np.stack([fr.vertices for fr in r.frames])
    out["skinned"] = np.stack([fr.skinned for fr in r.frames])
    pe = [[it.energy_before for it in fr.pose_report.iterations] for fr in r.frames]
    pa = [[it.energy_after for it in fr.pose_report.iterations] for fr in r.frames]
    ph = [[it.halvings for it in fr.pose_report.iterations] for fr in r.frames]
    width = max(len(x) for x in pe)
    pad = lambda rows, fill: np.array([x + [fill] * (width - len(x)) for x in rows])  # noqa: E731
    out["pose_e0"], out["pose_e1"], out["pose_halv"] = pad(pe, np.nan), pad(pa, np.nan), pad(ph, -1)
    out["nr_e0"] = np.array([[it.energy_before for it in fr.nonrigid_report.iterations] for fr in r.frames])
    out["nr_e1"] = np.array([[it.energy_after for it in fr.nonrigid_report.iterations] for fr in r.frames])
    out["nr_halv"] = np.array([[it.halvings for it in fr.nonrigid_report.iterations] for fr in r.frames])
    out["nr_terms"] = np.array([[[it.terms.get(k, 0.0) for k in ("photo", "silhouette", "smooth", "edge",
                                                                   "velocity", "acceleration")]
                                 for it in fr.nonrigid_report.iterations] for fr in r.frames])
    out["meta"] = np.array([preset, str(res), str(n), str(int(directional)), str(seed)])
    return out


# the survey's runtime presets, registered without editing the reference
RUNTIME_PRESETS = {
    "x5k": dict(segs=26, limb_rings=11, torso_rings=16, head=(16, 26), skirt=(26, 80)),
    "x20k": dict(segs=48, limb_rings=22, torso_rings=30, head=(32, 48), skirt=(50, 150)),
}


def _rows_digest(v):
    """A compact, order-sensitive digest of a (F, N, 3) vertex stack: per-frame
    sums, sums of squares, and every 97th row."""
    return dict(sum=v.sum(axis=(1, 2)), sq=(v ** 2).sum(axis=(1, 2)), rows=v[:, ::97].copy())


def frames_digest_fixture(preset, res, n, directional, seed=0, gn=None, pcg=None):
    """Like frames_fixture for the bench-sized scenes, with vertex digests in
    place of full vertex stacks (x20k @1024: 0.46 MB per frame)."""
    import dataclasses

    import montrack.actors as A
    from montrack.pipeline import SequenceConfig, SequenceInputs, run_sequence
    from montrack.synthetic import NoiseParams, default_script, generate_synthetic_sequence
    A._PRESETS.update(RUNTIME_PRESETS)
    actor = A.build_actor(preset, with_skirt=True)
    cam = A.suggest_camera(res, res)
    seq = generate_synthetic_sequence(actor, cam, default_script(n, noise=NoiseParams(sigma2d=1.0, sigma3d=0.008,
                                                                                      seed=seed)))
    inp = SequenceInputs(actor, cam, [f.image for f in seq.frames], [f.mask for f in seq.frames],
                         [f.detections for f in seq.frames])
    cfg = SequenceConfig(directional=directional)
    if gn is not None or pcg is not None:
        nr = cfg.nonrigid
        cfg = dataclasses.replace(cfg, nonrigid=dataclasses.replace(
            nr, gn_iterations=gn if gn is not None else nr.gn_iterations,
            pcg_iterations=pcg if pcg is not None else nr.pcg_iterations))
    r = run_sequence(inp, cfg, pipelined=False)
    out = _inputs_digest(seq.frames)
    out["poses"] = np.stack([fr.pose.to_vector() for fr in r.frames])
    for k, v in _rows_digest(np.stack([fr.vertices for fr in r.frames])).items():
        out["v_" + k] = v
    pe = [[it.energy_before for it in fr.pose_report.iterations] for fr in r.frames]
    pa = [[it.energy_after for it in fr.pose_report.iterations] for fr in r.frames]
    ph = [[it.halvings for it in fr.pose_report.iterations] for fr in r.frames]
    width = max(len(x) for x in pe)
    pad = lambda rows, fill: np.array([x + [fill] * (width - len(x)) for x in rows])  # noqa: E731
    out["pose_e0"], out["pose_e1"], out["pose_halv"] = pad(pe, np.nan), pad(pa, np.nan), pad(ph, -1)
    out["nr_e0"] = np.array([[it.energy_before for it in fr.nonrigid_report.iterations] for fr in r.frames])
    out["nr_e1"] = np.array([[it.energy_after for it in fr.nonrigid_report.iterations] for fr in r.frames])
    out["nr_halv"] = np.array([[it.halvings for it in fr.nonrigid_report.iterations] for fr in r.frames])
    out["meta"] = np.array([preset, str(res), str(n), str(int(directional)), str(seed), str(gn), str(pcg)])
    return out


def kernels_fixture():
    """Reference outputs of the individual hot-path functions on one scene."""
    import montrack.actors as A
    from montrack import imageproc as I, nonrigid_stage as NS, pose_stage as PS
    from montrack import rasterizer as R, skinning as SK, solvers as SV
    from montrack.pipeline import SequenceConfig, condition_detections, preprocess_frame
    from montrack.synthetic import NoiseParams, default_script, generate_synthetic_sequence
    actor = A.build_actor("small", with_skirt=True)
    cam = A.suggest_camera(128, 128)
    seq = generate_synthetic_sequence(actor, cam, default_script(2, noise=NoiseParams(seed=3)))
    fr = seq.frames[1]
    mesh, sk, sw = actor.mesh, actor.skeleton, actor.skinning
    out = _inputs_digest(seq.frames)
    out["edges"] = mesh.edges
    out["edge_tris"] = mesh.edge_tris
    out["directed_weights"] = mesh.directed_weights
    out["dominant"] = sw.dominant
    out["body_parts"] = NS.body_parts(sk)
    rng = np.random.default_rng(11)
    x = fr.pose.to_vector() + rng.uniform(-0.05, 0.05, 36)
    fk = SK.forward_kinematics(sk, SK.PoseParams.from_vector(x))
    out["fk_x"], out["fk_pos"], out["fk_markers"], out["fk_dqs"] = x, fk.positions, fk.marker_positions, fk.joint_dqs
    out["fk_jp"] = SK.joint_position_jacobian(sk, fk)
    dqj = SK.joint_dq_jacobian(sk, fk)
    sub = np.arange(0, mesh.n_vertices, 5)
    sres = SK.skin_points(mesh.rest_vertices[sub], sw, fk.joint_dqs, dqj, subset=sub)
    out["skin_sub"], out["skin_pos"], out["skin_rot"], out["skin_jac"] = sub, sres.positions, sres.rotations, sres.jacobian
    v = fr.gt_vertices
    out["zbuf"] = R.render_depth(cam, v, mesh.triangles)
    ids, _ = R.render_vertex_ids(cam, v, mesh.triangles, NS.body_parts(sk)[sw.dominant], background=0)
    out["part_ids"] = ids
    labels, vparts = NS.build_body_part_mask(v, mesh, sw, sk, cam, 10)
    out["part_labels"] = labels
    c = PS.extract_contour_vertices(v, mesh, cam)
    out["contour_idx"], out["contour_n2d"] = c.indices, c.normals2d
    out["rim_stage1"] = PS.outer_rim_mask(v, c.indices, cam, out["zbuf"])
    out["rim_stage2"] = PS.outer_rim_mask(v, c.indices, cam, out["zbuf"], min_thickness=0.0)
    out["visible"] = np.flatnonzero(NS.visible_vertices(v, mesh, cam, out["zbuf"]))
    df = I.DistanceField(fr.mask)
    q = rng.uniform(-20, 150, (2000, 2))
    out["dt_q"] = q
    out["dt_val"], _ = df.sample_value(q)
    res, grad, _ = df.sample_residual(q)
    out["dt_res"], out["dt_grad"] = res, grad
    out["dt_inside"] = df.inside(q)
    out["edt"] = I.euclidean_dt(fr.mask)
    pyr = I.gaussian_pyramid(fr.image, (15, 9, 3))
    out["pyr_sum"] = np.array([p.sum() for p in pyr])
    out["pyr_samples"] = np.stack([p[40:48, 50:58] for p in pyr])
    cfg = SequenceConfig(directional=False)
    pre = preprocess_frame(1, fr.image, fr.mask, cfg)
    cond = condition_detections(pre, fr.detections, actor)
    out["rescaled_j3d"] = cond.detections.joints3d
    # Stage II system + PCG at the ground-truth-ish state
    vs_rest = SK.skin_points(mesh.rest_vertices, sw, fk.joint_dqs).positions
    out["nr_skinned"] = vs_rest
    prob = NS.NonrigidProblem(mesh, cam, cfg.nonrigid, vs_rest, pre.pyramid, pre.dt_field,
                              out["visible"], c, np.ones(len(c.indices), bool), prev=v + 0.001,
                              prev2=v - 0.001, directional=False)
    v0 = v + 0.003 * rng.standard_normal(v.shape)
    ev = prob.evaluate(v0, 1)
    system = prob.normal_system(ev)
    delta, info = SV.pcg_solve(system, 4)
    out["nr_v0"], out["nr_energy_terms"] = v0, np.array([ev.energies[k] for k in
                                                        ("photo", "silhouette", "smooth", "edge", "velocity", "acceleration")])
    out["pcg_delta"], out["pcg_norms"] = delta, np.array(info.residual_norms)
    vnr, rep = NS.solve_nonrigid(prob, v0)
    out["nr_solve_v"] = vnr
    out["nr_solve_e"] = np.array([[it.energy_before, it.energy_after, it.halvings] for it in rep.iterations])
    vs, sinfo = NS.snap_vertices(vnr, prob)
    out["snap_v"], out["snap_info"] = vs, np.array([sinfo.walked, sinfo.reached, sinfo.stuck])
    # dense solve on the Stage I normal matrix at x
    det = cond.detections
    pprob = PS.PoseProblem(sk, sw, cam, det, pre.dt_field, c, mesh.rest_vertices[c.indices],
                           cfg.pose, prev_positions=fk.positions + 0.01, directional=False)
    pev = pprob.evaluate(x)
    a = pev.jacobian.T @ pev.jacobian
    a = 0.5 * (a + a.T)
    d, dinfo = SV.dense_solve(SV.DenseNormalSystem(a, -(pev.jacobian.T @ pev.residuals)))
    out["pose_F"], out["pose_J"], out["dense_x"], out["dense_damped"] = pev.residuals, pev.jacobian, d, np.array(dinfo.damped)
    xs, prep_ = PS.solve_pose(pprob, SK.PoseParams.from_vector(x))
    out["pose_solve_x"] = xs.to_vector()
    out["pose_solve_e"] = np.array([[it.energy_before, it.energy_after, it.halvings] for it in prep_.iterations])
    return out


def main_bench():
    """The bench's own workloads: x5k @1024, seed 0,
    directional=False, frames 0-24; cfg4 x20k @1024, 4 GN x 8 PCG, frames 0-2."""
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "ref_digest_x5k1024_dir0.npz"),
                        **frames_digest_fixture("x5k", 1024, 25, False))
    np.savez_compressed(os.path.join(OUT, "ref_digest_x20k1024_cfg4.npz"),
                        **frames_digest_fixture("x20k", 1024, 3, False, gn=4, pcg=8))


def main():
    if "--bench" in sys.argv:
        return main_bench()
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "ref_frames_small128_dir1.npz"), **frames_fixture("small", 128, 4, True))
    np.savez_compressed(os.path.join(OUT, "ref_frames_small128_dir0.npz"), **frames_fixture("small", 128, 4, False))
    np.savez_compressed(os.path.join(OUT, "ref_frames_standard256_dir0.npz"),
                        **frames_fixture("standard", 256, 3, False))
    np.savez_compressed(os.path.join(OUT, "ref_kernels_small128.npz"), **kernels_fixture())
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
