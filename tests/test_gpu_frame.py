"""Frame-level parity of the batched device tracker (solve_frame,
pipeline.py:263-302) against the oracle, teacher-forced per frame: every
frame starts from the oracle's TrackState (the free-running
tracker is chaotic, so only per-call / teacher-forced parity is defined)."""

import numpy as np
import pytest
import torch

from helpers import bbox_diag, scene

pytestmark = pytest.mark.gpu


def _oracle_state_to_mirror(st):
    from paper_1810_02648_b200.config import TrackState
    return TrackState(st.x_prev, st.x_prev2, st.joints_prev, st.disp_rest, st.v_prev, st.v_prev2)


def _run(preset, res, n, directional, mode="full", streams=1):
    from oracle import frame as OF
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene(preset, res, n)
    cfg = SequenceConfig(directional=directional, mode=mode)
    tr = Tracker(actor, cam, cfg, streams)
    st = OF.State()
    diag = bbox_diag(actor)
    errs = []
    for fr in frames:
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        for s in range(streams):
            tr.set_state(s, _oracle_state_to_mirror(st))
            tr.set_frame(s, fr.image, fr.mask, fr.detections)
        tr.step()
        xo, vo, vso, st_new, plogs, slogs = OF.solve_frame(prep, actor, cam, cfg, st)
        for s in range(streams):
            x, v, vs, rep = tr.result(s)
            errs.append((fr.index, s, np.abs(x - xo).max(), np.abs(v - vo).max() / diag))
            assert rep.pose.n_iterations == len(plogs)
            for k, o in enumerate(plogs):
                assert rep.pose.halvings[k] == o["halvings"], (fr.index, k)
                assert rep.pose.rejected[k] == o["rejected"], (fr.index, k)
            if mode == "full":
                for k, o in enumerate(slogs):
                    assert rep.nonrigid.halvings[k] == o["halvings"], (fr.index, k)
                    e = rep.nonrigid.energy_before[k]
                    assert abs(e - o["energy_before"]) <= 1e-4 * o["energy_before"]
            assert np.abs(v - vo).max() <= 1e-4 * diag, (fr.index, s, errs[-1])
        st = st_new
    return errs


@pytest.mark.parametrize("preset,res", [("small", 128), ("standard", 256)])
def test_tracker_teacher_forced(preset, res):
    _run(preset, res, 3, directional=False)


def test_tracker_pose_only():
    _run("small", 128, 3, directional=False, mode="pose_only")


def test_tracker_directional_stable_frames():
    # frames 0 and 1 are stable under the self-jitter screen
    _run("small", 128, 2, directional=True)


def test_tracker_batched_streams_identical():
    errs = _run("small", 128, 2, directional=False, streams=3)
    by_frame = {}
    for f, s, dx, dv in errs:
        by_frame.setdefault(f, []).append(dv)
    for f, v in by_frame.items():
        assert max(v) == min(v), "streams fed identical inputs must agree exactly"


@pytest.mark.slow
def test_tracker_x5k_frame0():
    _run("x5k", 1024, 2, directional=False)


def test_pipelined_equals_sequential():
    """run_sequence_pipelined's 2-slot schedule (pipeline.py:432-499): frame
    f+1 is queued (uploaded + preprocessed on the auxiliary stream) before
    frame f is solved.  The solves are the same, so results are bit-identical."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.pipeline import SequenceInputs, run_sequence
    actor, cam, frames = scene("standard", 256, 4)
    inputs = SequenceInputs(actor, cam, [f.image for f in frames], [f.mask for f in frames],
                            [f.detections for f in frames])
    cfg = SequenceConfig(directional=False)
    a = run_sequence(inputs, cfg, pipelined=False)
    b = run_sequence(inputs, cfg, pipelined=True)
    assert b.pipelined and not a.pipelined
    assert np.array_equal(a.poses, b.poses)
    assert np.array_equal(a.vertices, b.vertices)


def test_queue_depth_is_three():
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene("small", 128, 4)
    tr = Tracker(actor, cam, SequenceConfig(directional=False), 1)
    with pytest.raises(Exception):
        tr.step()                       # nothing queued
    for f in range(3):
        tr.set_frame(0, frames[f].image, frames[f].mask, frames[f].detections)
    with pytest.raises(ValueError):
        tr.set_frame(0, frames[3].image, frames[3].mask, frames[3].detections)
    tr.step()
    tr.set_frame(0, frames[3].image, frames[3].mask, frames[3].detections)
    for _ in range(3):
        tr.step()
    with pytest.raises(Exception):
        tr.step()
    tr.close()


def test_stage_pipeline_gpu_pair_matches_single_tracker():
    """§8e: Stage I and Stage II on a GPU pair (here both on cuda:0, each
    stage tracker on its own CUDA stream; the handoffs are the same peer
    copies) give exactly the single-device tracker's results."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import StagePipeline, Tracker
    actor, cam, frames = scene("standard", 256, 3)
    cfg = SequenceConfig(directional=False)
    S = 4
    ref = Tracker(actor, cam, cfg, S)
    pipe = StagePipeline(actor, cam, cfg, S, pose_device=0, surface_device=0, groups=2)
    for fr in frames:
        for s in range(S):
            ref.set_frame(s, fr.image, fr.mask, fr.detections)
            pipe.set_frame(s, fr.image, fr.mask, fr.detections)
        ref.step()
        pipe.step()
        pipe.synchronize()
        for s in range(S):
            x0, v0, _, _ = ref.result(s)
            x1, v1, _, _ = pipe.result(s)
            assert np.array_equal(x0, x1) and np.array_equal(v0, v1), (fr.index, s)
    pipe.close()
    ref.close()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_stage_pipeline_two_devices_matches_single_tracker():
    """§8e on two real devices: Stage I on cuda:0, Stage II on cuda:1, the
    handoffs are cudaMemcpyPeerAsync between the devices."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import StagePipeline, Tracker
    actor, cam, frames = scene("small", 128, 3)
    cfg = SequenceConfig(directional=False)
    S = 2
    ref = Tracker(actor, cam, cfg, S)
    pipe = StagePipeline(actor, cam, cfg, S, pose_device=0, surface_device=1, groups=2)
    for fr in frames:
        for s in range(S):
            ref.set_frame(s, fr.image, fr.mask, fr.detections)
            pipe.set_frame(s, fr.image, fr.mask, fr.detections)
        ref.step()
        pipe.step()
        pipe.synchronize()
        for s in range(S):
            x0, v0, _, _ = ref.result(s)
            x1, v1, _, _ = pipe.result(s)
            assert np.array_equal(x0, x1) and np.array_equal(v0, v1), (fr.index, s)
    pipe.close()
    ref.close()


def test_stage_two_refuses_frame_without_image():
    """A frame queued mask-only (the Stage-I tracker's ingest) solves Stage I;
    Stage II on it fails loudly instead of reading a stale pyramid."""
    from paper_1810_02648_b200 import _lib as L
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene("small", 128, 2)
    tr = Tracker(actor, cam, SequenceConfig(directional=False), 1)
    tr.set_frame(0, None, frames[0].mask, frames[0].detections)
    L.check(tr.ctx.lib.lc_tracker_step_stage(tr.handle, 1))
    tr.set_frame(0, None, frames[1].mask, frames[1].detections)
    with pytest.raises(ValueError, match="image"):
        L.check(tr.ctx.lib.lc_tracker_step_stage(tr.handle, 2))
    tr.close()


@pytest.mark.parametrize("preset,res", [("standard", 256), ("x5k", 1024)])
def test_pyramid_region_of_interest_bit_identical(preset, res):
    """The blur pyramid is computed only near the observed silhouette; the
    photometric samples outside that region are blurred on demand from the
    raw frame with the same arithmetic.  Every margin -- every tile (-1), no
    tile (-2: every sample on the on-demand path), 0 and the default --
    gives bit-identical tracker results."""
    from paper_1810_02648_b200 import _lib as L
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene(preset, res, 3)
    cfg = SequenceConfig(directional=False)
    out = {}
    for margin in (-1, -2, 0, None):
        ctx = L.Context(0)
        if margin is not None:
            ctx.set_pyramid_margin(margin)
        tr = Tracker(actor, cam, cfg, 1, ctx=ctx)
        res_ = []
        for fr in frames:
            tr.set_frame(0, fr.image, fr.mask, fr.detections)
            tr.step()
            x, v, _, _ = tr.result(0)
            res_.append((x, v))
        tr.close()
        ctx.close()
        out[margin] = res_
    for margin in (-2, 0, None):
        for (x0, v0), (x1, v1) in zip(out[-1], out[margin]):
            assert np.array_equal(x0, x1) and np.array_equal(v0, v1), margin


def test_batch_tracker_groups_identical():
    """Streams split over concurrently stepped groups (own contexts / CUDA
    streams) give exactly the single tracker's results."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import BatchTracker, Tracker
    actor, cam, frames = scene("small", 128, 3)
    cfg = SequenceConfig(directional=False)
    ref = Tracker(actor, cam, cfg, 5)
    bt = BatchTracker(actor, cam, cfg, 5, groups=3)
    assert bt.sizes == [2, 2, 1]
    for fr in frames:
        for s in range(5):
            ref.set_frame(s, fr.image, fr.mask, fr.detections)
            bt.set_frame(s, fr.image, fr.mask, fr.detections)
        ref.step()
        bt.step()
        for s in range(5):
            x0, v0, _, _ = ref.result(s)
            x1, v1, _, _ = bt.result(s)
            assert np.array_equal(x0, x1) and np.array_equal(v0, v1)
    bt.close()
    ref.close()


@pytest.mark.parametrize("on_device", [False, True])
def test_graph_mode_bit_identical(on_device):
    """CUDA-graph mode (lc_tracker_set_graph): steady-state steps replay a
    captured graph per frame-queue phase; results equal the eager tracker's
    bit for bit, and the graphs are actually replayed."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene("standard", 256, 9)
    cfg = SequenceConfig(directional=False)
    S = 2
    imgs = [torch.from_numpy(fr.image).cuda() for fr in frames]
    msks = [torch.from_numpy(fr.mask.astype(np.uint8)).cuda() for fr in frames]
    out = []
    for graph in (False, True):
        tr = Tracker(actor, cam, cfg, S)
        tr.set_graph(graph)

        def q(f):
            for s in range(S):
                if on_device:
                    tr.set_frame(s, imgs[f].data_ptr(), msks[f].data_ptr(), frames[f].detections, on_device=True)
                else:
                    tr.set_frame(s, frames[f].image, frames[f].mask, frames[f].detections)
        res = []
        q(0)
        q(1)
        for f in range(len(frames)):
            if f + 2 < len(frames):
                q(f + 2)
            tr.step()
            res.append([tr.result(s)[:2] for s in range(S)])
        if graph:
            n_graphs, replays = tr.graph_stats()
            assert n_graphs >= 1 and replays >= 3, (n_graphs, replays)
        tr.close()
        out.append(res)
    for a, b in zip(*out):
        for (x0, v0), (x1, v1) in zip(a, b):
            assert np.array_equal(x0, x1) and np.array_equal(v0, v1)
