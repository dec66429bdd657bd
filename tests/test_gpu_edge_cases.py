"""Edge cases of the hot path against the oracle and the reference SPEC's
known answers (SPEC.md "Operations" examples and error rules).

* contour_pixels / euclidean_dt / metric_iou known answers, and their error
  rules (empty mask -> empty contour, `euclidean_dt` raises, two empty masks
  -> IoU 1.0 flagged);
* extract_contour_vertices on a single triangle (boundary edges count);
* whole frames teacher-forced through the tracker where the input degenerates:
  an empty observed mask (the subject left the frame: pipeline.py:158-161
  builds no distance field, pose_stage.py:360 / nonrigid_stage.py:219,431 skip
  the silhouette rows and snapping), a mask covering the whole frame (the
  contour is the image border), all 2D / all 3D detections invalid and a
  ragged validity pattern (rescale_detections' fallback, pipeline.py:165-170).
Every frame: identical decision traces, energies within 1e-4, vertices within
1e-4 of the bbox diagonal (helpers.check_frame_strict).
"""

import numpy as np
import pytest

from helpers import bbox_diag, check_frame_strict, oracle_state_to_mirror, scene

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- known answers

def test_contour_known_answers():
    """SPEC contour_pixels: single pixel, 3x3 block (8 border pixels, the
    centre not), full frame (the outer ring); an empty mask has no field."""
    from oracle.imaging import contour_mask
    from paper_1810_02648_b200.imageproc import DistanceField
    m = np.zeros((16, 16), dtype=bool)
    m[4, 7] = True
    f = DistanceField(m)
    assert f.n_contour == 1 and f.dt[4, 7] == 0.0
    m = np.zeros((16, 16), dtype=bool)
    m[5:8, 5:8] = True
    f = DistanceField(m)
    assert f.n_contour == 8
    assert f.dt[6, 6] == 1.0 and (f.dt[contour_mask(m)] == 0.0).all()
    m = np.ones((9, 13), dtype=bool)
    f = DistanceField(m)
    assert f.n_contour == 2 * (9 + 13) - 4
    assert f.dt[4, 6] == 4.0
    # the reference's DistanceField computes euclidean_dt on construction
    # (imageproc.py:180-182), which rejects a mask without contour
    with pytest.raises(ValueError, match="distance transform undefined"):
        DistanceField(np.zeros((8, 8), dtype=bool))


def test_edt_known_answers_and_empty_mask_error():
    """SPEC euclidean_dt: one contour pixel at (5,5) -> DT(8,9) = 5 (the
    3-4-5 triangle), 0 on every contour pixel; an empty mask raises
    (imageproc.py:121-123)."""
    from paper_1810_02648_b200.imageproc import euclidean_dt
    m = np.zeros((20, 20), dtype=bool)
    m[5, 5] = True
    dt = euclidean_dt(m)
    assert dt[8, 9] == 5.0 and dt[9, 8] == 5.0 and dt[5, 5] == 0.0
    yy, xx = np.mgrid[0:20, 0:20]
    assert np.array_equal(dt, np.sqrt((yy - 5.0) ** 2 + (xx - 5.0) ** 2))
    with pytest.raises(ValueError, match="distance transform undefined"):
        euclidean_dt(np.zeros((12, 12), dtype=bool))


def test_iou_known_answers():
    """SPEC metric_iou: identical -> 1.0, disjoint -> 0.0, both empty -> 1.0
    flagged, shape mismatch rejected (metrics.py:8-23)."""
    from paper_1810_02648_b200.metrics import iou
    rng = np.random.default_rng(5)
    a = rng.random((33, 47)) < 0.4
    assert iou(a, a) == 1.0
    assert iou(a, ~a) == 0.0
    assert iou(np.zeros((6, 6)), np.zeros((6, 6)), return_empty_flag=True) == (1.0, True)
    b = rng.random((33, 47)) < 0.4
    want = float(np.float64((a & b).sum()) / np.float64((a | b).sum()))
    assert iou(a, b, return_empty_flag=True) == (want, False)
    with pytest.raises(ValueError):
        iou(a, a[:, :-1])


@pytest.mark.parametrize("winding,n_contour", [((0, 2, 1), 3), ((0, 1, 2), 0)])
def test_single_triangle_contour(winding, n_contour):
    """SPEC extract_contour_vertices: a single front-facing triangle has all
    three vertices on the contour (its edges are boundary edges); seen from
    the back it has none.  Indices and image-plane normals match the oracle."""
    from oracle.posefit import contour_vertices
    from paper_1810_02648_b200.actor import TemplateMesh
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.pose_stage import extract_contour_vertices
    cam = suggest_camera(128, 128)
    v = np.array([[-0.3, -0.2, 2.5], [0.3, -0.2, 2.5], [0.0, 0.35, 2.5]])
    mesh = TemplateMesh(v, np.array([winding]), np.full((3, 3), 0.5), np.ones(3, dtype=np.int64))
    c = extract_contour_vertices(v, mesh, cam)
    idx, n2 = contour_vertices(v, mesh, cam)
    assert len(idx) == n_contour
    assert np.array_equal(c.indices, idx)
    assert np.allclose(c.normals2d, n2, atol=1e-12)


# ------------------------------------------------------------- degenerate frames

def _teacher_forced(frames, actor, cam, cfg):
    from oracle import frame as OF
    from paper_1810_02648_b200.device import Tracker
    tr = Tracker(actor, cam, cfg, 1)
    st = OF.State()
    diag = bbox_diag(actor)
    try:
        for fr in frames:
            prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
            tr.set_state(0, oracle_state_to_mirror(st))
            tr.set_frame(0, fr.image, fr.mask, fr.detections)
            tr.step()
            xo, vo, vso, st_new, plogs, slogs = OF.solve_frame(prep, actor, cam, cfg, st)
            x, v, vs, rep = tr.result(0)
            check_frame_strict(rep, plogs, slogs, v, vo, diag, f"frame {fr.index}")
            assert np.abs(x - xo).max() <= 1e-6, fr.index
            st = st_new
    finally:
        tr.close()


def _with(fr, mask=None, det=None):
    import copy
    g = copy.copy(fr)
    if mask is not None:
        g.mask = mask
    if det is not None:
        g.detections = det
    return g


def _det(d, valid2d=None, valid3d=None):
    from paper_1810_02648_b200.config import FrameDetections
    return FrameDetections(d.joints2d.copy(), d.joints3d.copy(),
                           d.valid2d.copy() if valid2d is None else valid2d,
                           d.valid3d.copy() if valid3d is None else valid3d)


@pytest.mark.parametrize("empty_frames", [(1,), (0, 1)])
def test_empty_observed_mask(empty_frames):
    """No foreground in the observed mask: no distance field, so neither
    stage has silhouette rows and Stage II does not snap; the next frame's
    recursion continues from those results."""
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene("small", 128, 3)
    frames = [_with(fr, mask=np.zeros_like(fr.mask)) if fr.index in empty_frames else fr for fr in frames]
    _teacher_forced(frames, actor, cam, SequenceConfig(directional=False))


def test_mask_covering_the_frame():
    """Foreground everywhere: the contour is the image's outer ring (SPEC
    contour_pixels, border counts as background)."""
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene("small", 128, 3)
    frames = [_with(fr, mask=np.ones_like(fr.mask)) if fr.index == 1 else fr for fr in frames]
    _teacher_forced(frames, actor, cam, SequenceConfig(directional=False))


def test_invalid_detections():
    """Frame 1: every 2D detection invalid; frame 2: every 3D detection
    invalid (each bone's rescale falls back); frame 3: a ragged half of each."""
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene("small", 128, 4)
    rng = np.random.default_rng(11)
    out = []
    for fr in frames:
        d = fr.detections
        if fr.index == 1:
            fr = _with(fr, det=_det(d, valid2d=np.zeros_like(d.valid2d)))
        elif fr.index == 2:
            fr = _with(fr, det=_det(d, valid3d=np.zeros_like(d.valid3d)))
        elif fr.index == 3:
            fr = _with(fr, det=_det(d, valid2d=d.valid2d & (rng.random(d.valid2d.shape) < 0.5),
                                    valid3d=d.valid3d & (rng.random(d.valid3d.shape) < 0.5)))
        out.append(fr)
    _teacher_forced(out, actor, cam, SequenceConfig(directional=False))


def test_empty_mask_directional_and_pose_only():
    """The empty-mask frame under the reference's default directional rows
    and in pose-only mode (frames 0-1: the directional config's stable
    frames)."""
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene("small", 128, 2)
    frames = [_with(fr, mask=np.zeros_like(fr.mask)) if fr.index == 1 else fr for fr in frames]
    _teacher_forced(frames, actor, cam, SequenceConfig())
    _teacher_forced(frames, actor, cam, SequenceConfig(directional=False, mode="pose_only"))


@pytest.mark.parametrize("shift", [2.45, 2.6])
def test_subject_partly_behind_the_camera(shift):
    """Frame 1 starts from previous poses moved `shift` m towards the camera,
    so the extrapolated model straddles the image plane: joints, markers and
    contour vertices behind the camera drop their rows (pose_stage.py:330-365)
    and are counted in the reports (pose_stage.py:435, nonrigid_stage.py:383),
    the counts equal to the oracle's."""
    import oracle.frame as OF
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene("small", 128, 3)
    cfg = SequenceConfig(directional=False)
    counts = {}
    real_pose, real_surface = OF.solve_pose, OF.solve_surface

    def pose_counted(pb, x):
        r = real_pose(pb, x)
        counts["pose"] = counts.get("pose", 0) + r[2]
        return r

    def surface_counted(pb, v):
        r = real_surface(pb, v)
        counts["surface"] = counts.get("surface", 0) + r[2]["behind_camera"]
        return r

    tr = Tracker(actor, cam, cfg, 1)
    st = OF.State()
    diag = bbox_diag(actor)
    behind = 0
    try:
        OF.solve_pose, OF.solve_surface = pose_counted, surface_counted
        for fr in frames:
            if fr.index == 1:
                for x in (st.x_prev, st.x_prev2):
                    if x is not None:
                        x[5] -= shift
            prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
            tr.set_state(0, oracle_state_to_mirror(st))
            tr.set_frame(0, fr.image, fr.mask, fr.detections)
            tr.step()
            counts.clear()
            xo, vo, vso, st_new, plogs, slogs = OF.solve_frame(prep, actor, cam, cfg, st)
            x, v, vs, rep = tr.result(0)
            check_frame_strict(rep, plogs, slogs, v, vo, diag, f"frame {fr.index}")
            assert rep.pose.behind_camera == counts.get("pose", 0), (fr.index, rep.pose.behind_camera, counts)
            assert rep.nonrigid.behind_camera == counts.get("surface", 0), (fr.index, counts)
            behind += rep.pose.behind_camera
            st = st_new
    finally:
        OF.solve_pose, OF.solve_surface = real_pose, real_surface
        tr.close()
    assert behind > 0, "the shifted frames must exercise the behind-camera rows"
