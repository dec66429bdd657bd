"""§8f rows: post-processing (smooth_trajectory, iou, frame latencies) and the
reference's on-disk formats.  CPU tests pin the oracle and the readers /
writers against fixtures made by the real reference (tools/make_golden_post.py);
GPU tests check the device kernels and drivers against the same fixtures."""

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _post():
    return np.load(os.path.join(GOLD, "ref_post.npz"))


# ---------------------------------------------------------------- CPU ---------

def test_oracle_smoothing_matches_reference():
    from oracle import post as OP
    g = _post()
    assert np.array_equal(OP.smooth_trajectory(g["vals"], (0.15, 0.7, 0.15)), g["s3"])
    assert np.array_equal(OP.smooth_trajectory(g["vals"], (0.1, 0.2, 0.4, 0.2, 0.1)), g["s5"])
    assert np.array_equal(OP.smooth_trajectory(g["vals1"]), g["s1"])
    with pytest.raises(ValueError):
        OP.smooth_trajectory(g["vals"], (0.5, 0.5))


def test_oracle_iou_matches_reference():
    from oracle import post as OP
    g = _post()
    assert np.array_equal(np.array([OP.iou(a, b) for a, b in zip(g["ma"], g["mb"])]), g["ious"])


def test_reference_latency_contract():
    """sequential emits in the ingest slot, pipelined two slots later."""
    g = _post()
    assert (g["lat_seq"] == 0).all() and (g["lat_pip"] == 2).all()


def test_load_reference_written_sequence():
    from paper_1810_02648_b200 import io
    g = np.load(os.path.join(GOLD, "ref_seq_tiny.npz"))
    inp = io.load_sequence_inputs(os.path.join(GOLD, "seq_tiny"))
    m = inp.actor.mesh
    assert np.array_equal(m.rest_vertices, g["rest"]) and np.array_equal(m.triangles, g["tris"])
    assert np.array_equal(m.vertex_colors, g["colors"]) and np.array_equal(m.vertex_labels, g["labels"])
    sk = inp.actor.skeleton
    assert np.array_equal(sk.parents, g["parents"]) and np.array_equal(sk.local_offsets, g["offsets"])
    assert np.array_equal(sk.dof_axes, g["dof_axes"]) and np.array_equal(sk.theta_min, g["tmin"])
    assert np.array_equal(inp.actor.skinning.indices, g["skin_idx"])
    assert np.array_equal(inp.actor.skinning.weights, g["skin_w"])
    c = inp.camera
    assert np.array_equal([c.fx, c.fy, c.cx, c.cy, c.width, c.height], g["cam"])
    assert np.array_equal(np.stack(inp.images), g["images"])
    assert np.array_equal(np.stack(inp.masks), g["masks"])
    assert np.array_equal(np.stack([d.joints2d for d in inp.detections]), g["j2d"])
    assert np.array_equal(np.stack([d.valid3d for d in inp.detections]), g["v3d"])
    u8 = io.load_sequence_inputs(os.path.join(GOLD, "seq_tiny"), as_uint8=True)
    assert u8.images[0].dtype == np.uint8
    assert np.array_equal(np.stack(u8.images).astype(np.float64) / 255.0, g["images"])


def test_writers_round_trip(tmp_path):
    """our writers -> our readers (both naming schemes of the actor, F9)."""
    from paper_1810_02648_b200 import io
    inp = io.load_sequence_inputs(os.path.join(GOLD, "seq_tiny"))
    io.save_sequence(tmp_path, inp.actor, inp.camera, inp.images, inp.masks, inp.detections)
    back = io.load_sequence_inputs(tmp_path)          # actor.obj / .skel / .skin names
    assert np.array_equal(back.actor.mesh.rest_vertices, inp.actor.mesh.rest_vertices)
    assert np.array_equal(back.actor.skinning.weights, inp.actor.skinning.weights)
    assert np.array_equal(np.stack(back.masks), np.stack(inp.masks))
    # colours are quantised to bytes by the writer: a second round trip is exact
    io.save_sequence(tmp_path / "b", back.actor, back.camera, back.images, back.masks, back.detections)
    again = io.load_sequence_inputs(tmp_path / "b")
    assert np.array_equal(np.stack(again.images), np.stack(back.images))
    traj = [np.arange(36) * 0.1 + k for k in range(3)]
    io.save_pose_trajectory(tmp_path / "p.txt", traj)
    assert np.allclose([p.to_vector() for p in io.load_pose_trajectory(tmp_path / "p.txt")], traj, atol=1e-11)


# ---------------------------------------------------------------- GPU ---------

@pytest.mark.gpu
def test_device_smoothing_bit_exact():
    from paper_1810_02648_b200.postprocess import smooth_trajectory
    g = _post()
    assert np.array_equal(smooth_trajectory(g["vals"], (0.15, 0.7, 0.15)), g["s3"])
    assert np.array_equal(smooth_trajectory(g["vals"], (0.1, 0.2, 0.4, 0.2, 0.1)), g["s5"])
    assert np.array_equal(smooth_trajectory(g["vals1"]), g["s1"])


@pytest.mark.gpu
def test_device_iou():
    from paper_1810_02648_b200.postprocess import iou_batch
    g = _post()
    assert np.array_equal(iou_batch(g["ma"], g["mb"]), g["ious"])


@pytest.mark.gpu
def test_sequence_drivers_events_and_smoothing(tmp_path):
    from paper_1810_02648_b200 import io
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.pipeline import frame_latencies, run_sequence
    from oracle import post as OP
    g = _post()
    inp = io.load_sequence_inputs(os.path.join(GOLD, "seq_tiny"))
    cfg = SequenceConfig(directional=False)
    a = run_sequence(inp, cfg, pipelined=False)
    b = run_sequence(inp, cfg, pipelined=True)
    ev = lambda r: np.array([[e["slot"], e["event"] == "emit", e["frame"]] for e in r.events])
    assert np.array_equal(ev(a), g["ev_seq"]) and np.array_equal(ev(b), g["ev_pip"])
    assert list(frame_latencies(b.events).values()) == [2, 2, 2]
    assert np.array_equal(a.poses, b.poses) and np.array_equal(a.vertices, b.vertices)
    assert np.array_equal(a.poses_smoothed, OP.smooth_trajectory(a.poses))
    assert np.array_equal(a.vertices_smoothed, OP.smooth_trajectory(a.vertices))
    io.save_results(tmp_path, b)
    assert (tmp_path / "report.json").exists() and (tmp_path / "surfaces.npz").exists()


@pytest.mark.gpu
def test_uint8_upload_path_identical():
    """uint8 frames (converted on the device with / 255.0) solve exactly like
    the same frames given as float64 (img / 255.0 on the host)."""
    from paper_1810_02648_b200 import io
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.pipeline import run_sequence
    f64 = io.load_sequence_inputs(os.path.join(GOLD, "seq_tiny"))
    u8 = io.load_sequence_inputs(os.path.join(GOLD, "seq_tiny"), as_uint8=True)
    cfg = SequenceConfig(directional=False)
    a = run_sequence(f64, cfg)
    b = run_sequence(u8, cfg)
    assert np.array_equal(a.poses, b.poses) and np.array_equal(a.vertices, b.vertices)
