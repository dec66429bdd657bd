"""The drop-in against the REAL reference.

`montrack` is installed unmodified into baseline/_ref by the recipe in
DESIGN.md (pip --no-index --target baseline/_ref, git-ignored; it travels to
the GPU box).  `install(montrack, level)` rebinds the reference's consumer
names; the reference's own `run_sequence` then drives the device path.  Each
level is compared with the uninstalled reference run on the same inputs:
frames 0-1 within the parity bar (later frames of a free-running recursion
are chaotic), the GPU kernels must actually run, and uninstall
restores the reference.  Skipped when baseline/_ref is absent.
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def montrack():
    if not os.path.isdir(os.path.join(REF, "montrack")):
        pytest.skip("reference not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import montrack as M
    import montrack.pipeline  # noqa: F401
    return M


@pytest.fixture(scope="module")
def ref_run(montrack):
    import montrack.actors as A
    from montrack.pipeline import SequenceConfig, SequenceInputs, run_sequence
    from montrack.synthetic import NoiseParams, default_script, generate_synthetic_sequence
    actor = A.build_actor("small", with_skirt=True)
    cam = A.suggest_camera(128, 128)
    seq = generate_synthetic_sequence(actor, cam, default_script(3, noise=NoiseParams(seed=5)))
    inputs = SequenceInputs(actor, cam, [f.image for f in seq.frames], [f.mask for f in seq.frames],
                            [f.detections for f in seq.frames])
    cfg = SequenceConfig(directional=False)
    res = run_sequence(inputs, cfg, pipelined=False)
    return inputs, cfg, res


@pytest.mark.parametrize("level", ["solvers", "stages", "frame"])
@pytest.mark.parametrize("pipelined", [False, True])
def test_install_levels_match_reference(montrack, ref_run, level, pipelined):
    import paper_1810_02648_b200 as lc
    from montrack import pipeline as RP
    from paper_1810_02648_b200 import _lib
    inputs, cfg, ref = ref_run
    orig = (RP.solve_frame, RP.solve_pose, montrack.nonrigid_stage.pcg_solve)
    n0 = _lib.process_launches()   # the pipelined driver solves on worker threads (own contexts)
    uninstall = lc.install(montrack, level=level)
    try:
        assert montrack.nonrigid_stage.pcg_solve is not orig[2]
        got = RP.run_sequence(inputs, cfg, pipelined=pipelined)
    finally:
        uninstall()
    assert (RP.solve_frame, RP.solve_pose, montrack.nonrigid_stage.pcg_solve) == orig
    assert _lib.process_launches() > n0, "the device path did not run"
    diag = float(np.linalg.norm(np.ptp(inputs.actor.mesh.rest_vertices, axis=0)))
    assert got.vertices.shape == ref.vertices.shape and got.poses.shape == ref.poses.shape
    for f in range(2):
        err = np.abs(got.vertices[f] - ref.vertices[f]).max() / diag
        assert err <= 1e-4, (level, f, err)
        assert np.abs(got.poses[f] - ref.poses[f]).max() <= 1e-5, (level, f)
    # the reference's reports come back in the reference's own types
    fr = got.frames[1]
    assert type(fr.pose_report).__module__.startswith(("montrack", "paper_1810_02648_b200"))
    assert len(fr.pose_report.iterations) == len(ref.frames[1].pose_report.iterations)
    if fr.nonrigid_report is not None:
        assert [it.halvings for it in fr.nonrigid_report.iterations] == \
               [it.halvings for it in ref.frames[1].nonrigid_report.iterations]
    # later frames: same tracking quality (free-running recursion)
    assert np.abs(got.vertices[2] - ref.vertices[2]).max() / diag <= 1e-2


def test_reference_pose_params_accepted_by_tracker(montrack, ref_run):
    """Tracker.set_state takes the reference's own TrackState / PoseParams."""
    from montrack.pipeline import TrackState
    from montrack.skinning import PoseParams
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    inputs, _, ref = ref_run
    tr = Tracker(inputs.actor, inputs.camera, SequenceConfig(directional=False), 1)
    st = TrackState(pose_prev=PoseParams.from_vector(ref.poses[0]), pose_prev2=None,
                    joints_prev=None, disp_rest=None, v_prev=ref.vertices[0], v_prev2=None)
    with pytest.raises(ValueError):
        tr.set_state(0, st)            # joints_prev is required with pose_prev (pipeline.py:268)
    from montrack.skinning import forward_kinematics
    st.joints_prev = forward_kinematics(inputs.actor.skeleton, st.pose_prev).positions
    tr.set_state(0, st)
    back = tr.get_state(0)
    assert np.array_equal(back.pose_prev.to_vector(), ref.poses[0])
    tr.close()


def test_tracker_cache_is_bounded(montrack, ref_run):
    from paper_1810_02648_b200 import pipeline as PL
    inputs, cfg, _ = ref_run
    from paper_1810_02648_b200.config import SequenceConfig
    for rounds in (1, 2, 3):
        for d in (False, True):
            PL._tracker_for(inputs.actor, inputs.camera, SequenceConfig(directional=d, frame0_rounds=rounds))
    assert len(PL._trackers) <= PL.TRACKER_CACHE
