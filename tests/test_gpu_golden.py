"""GPU path against golden fixtures produced by the real reference
(tools/make_golden.py).  Tolerances per BASELINE.json north_star."""

import numpy as np
import pytest

from helpers import bbox_diag
from test_oracle_golden import check_digest, gen, load

pytestmark = pytest.mark.gpu


def golden_state(actor, g, k):
    """TrackState entering frame k, rebuilt from the reference's outputs of
    frames k-1, k-2 (pipeline.py:281-299): teacher forcing."""
    from oracle.geometry import Fk, qconj, qrot, skin
    from paper_1810_02648_b200.config import TrackState
    if k == 0:
        return TrackState()
    x1 = g["poses"][k - 1]
    fk = Fk(actor.skeleton, x1)
    _, rot, _, _ = skin(actor.mesh.rest_vertices, actor.skinning, fk.dqs)
    disp = qrot(qconj(rot), g["vertices"][k - 1] - g["skinned"][k - 1])
    return TrackState(x1, g["poses"][k - 2] if k >= 2 else None, fk.pos, disp, g["vertices"][k - 1],
                      g["vertices"][k - 2] if k >= 2 else None)


@pytest.mark.parametrize("name", ["ref_frames_small128_dir0.npz", "ref_frames_standard256_dir0.npz",
                                  "ref_frames_small128_dir1.npz"])
def test_tracker_against_reference_sequence(name):
    """Every frame teacher-forced from the reference's own previous outputs."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    g = load(name)
    preset, res, n, directional, seed = g["meta"]
    directional = bool(int(directional))
    actor, cam, frames = gen(preset, int(res), int(n), int(seed))
    check_digest(g, frames)
    tr = Tracker(actor, cam, SequenceConfig(directional=directional), 1)
    diag = bbox_diag(actor)
    # default-directional frames >= 2 fail the oracle's own self-jitter screen
    # (SURVEY.md §8c); compare them only when directional is off
    last = len(frames) if not directional else 2
    for k, fr in enumerate(frames[:last]):
        tr.set_state(0, golden_state(actor, g, k))
        tr.set_frame(0, fr.image, fr.mask, fr.detections)
        tr.step()
        x, v, vs, rep = tr.result(0)
        assert np.abs(v - g["vertices"][k]).max() <= 1e-4 * diag, k
        e0 = [rep.nonrigid.energy_before[i] for i in range(rep.nonrigid.n_iterations)]
        assert np.allclose(e0, g["nr_e0"][k], rtol=1e-4), k
        assert [rep.nonrigid.halvings[i] for i in range(rep.nonrigid.n_iterations)] == list(g["nr_halv"][k])
        pe = [rep.pose.energy_before[i] for i in range(rep.pose.n_iterations)]
        assert np.allclose(pe, g["pose_e0"][k][:len(pe)], rtol=1e-4), k
        assert [rep.pose.halvings[i] for i in range(rep.pose.n_iterations)] == \
            list(g["pose_halv"][k][:len(pe)]), k


def test_free_running_first_frames_match_reference():
    """Free-running (no state injection): the frames before the recursion's
    amplification of fp64 reordering noise (frames 0-1) match the reference."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    g = load("ref_frames_small128_dir0.npz")
    actor, cam, frames = gen("small", 128, 4, 0)
    tr = Tracker(actor, cam, SequenceConfig(directional=False), 1)
    for k, fr in enumerate(frames[:2]):
        tr.set_frame(0, fr.image, fr.mask, fr.detections)
        tr.step()
        _, v, _, _ = tr.result(0)
        assert np.abs(v - g["vertices"][k]).max() <= 1e-4 * bbox_diag(actor), k


def test_kernels_against_reference():
    from paper_1810_02648_b200 import imageproc as G, skinning as SKG
    from paper_1810_02648_b200.pose_stage import extract_contour_vertices
    from paper_1810_02648_b200.solvers import DenseNormalSystem, dense_solve
    g = load("ref_kernels_small128.npz")
    actor, cam, frames = gen("small", 128, 2, 3)
    fr = frames[1]
    mesh = actor.mesh
    v = fr.gt_vertices
    assert np.array_equal(G.render_depth(cam, v, mesh.triangles), g["zbuf"])
    c = extract_contour_vertices(v, actor, cam)
    assert np.array_equal(c.indices, g["contour_idx"])
    assert np.allclose(c.normals2d, g["contour_n2d"], atol=1e-12)
    df = G.DistanceField(fr.mask)
    assert np.array_equal(df.sample_value(g["dt_q"])[0], g["dt_val"])
    res, grad, _ = df.sample_residual(g["dt_q"])
    assert np.array_equal(res, g["dt_res"]) and np.array_equal(grad, g["dt_grad"])
    assert np.array_equal(df.inside(g["dt_q"]), g["dt_inside"])
    pyr = G.gaussian_pyramid(fr.image, (15, 9, 3))
    assert np.array_equal(np.stack([p[40:48, 50:58] for p in pyr]), g["pyr_samples"])
    fk = SKG.forward_kinematics(actor, g["fk_x"])
    assert np.allclose(fk.joint_dqs, g["fk_dqs"], atol=1e-13)
    sub = g["skin_sub"]
    s = SKG.skin_points(actor, g["fk_x"], mesh.rest_vertices[sub], subset=sub, with_jacobian=True)
    assert np.allclose(s.positions, g["skin_pos"], atol=1e-13)
    assert np.allclose(s.jacobian, g["skin_jac"], atol=1e-11)
    J, F = g["pose_J"], g["pose_F"]
    a = J.T @ J
    a = 0.5 * (a + a.T)
    d, info = dense_solve(DenseNormalSystem(a, -(J.T @ F)))
    assert np.allclose(d, g["dense_x"], rtol=1e-8, atol=1e-10 * np.abs(g["dense_x"]).max())
