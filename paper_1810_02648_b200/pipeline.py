"""Drop-in per-frame entry points (reference pipeline.py:89-302,378-397).

`solve_frame(cond, actor, camera, config, state)` runs the complete frame --
preprocessing, detection conditioning, Stage I, Stage II, snapping, warp --
on the GPU and returns the reference's `(FrameResult, TrackState)`.  The
CPU-side `preprocess_frame` / `condition_detections` only package their
inputs: the blur pyramid, contour grid and bone-length rescaling are computed
on the device inside `solve_frame`.

`run_sequence` is the sequential driver over the same call.  For throughput
over many independent streams use `device.Tracker` directly (batched).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np

from .config import (FrameDetections, FrameResult, PoseParams, SequenceConfig, TrackState)
from .device import Tracker, nonrigid_report_from_c, pose_report_from_c


@dataclass
class SequenceInputs:
    actor: object
    camera: object
    images: list
    masks: list
    detections: list

    @property
    def n_frames(self) -> int:
        return len(self.images)


@dataclass
class PreprocessedFrame:
    index: int
    image: np.ndarray
    mask: np.ndarray
    dt_field: object | None = None   # computed on the device inside solve_frame
    pyramid: list = field(default_factory=list)


@dataclass
class ConditionedFrame:
    pre: PreprocessedFrame
    detections: FrameDetections      # raw; rescaled on the device
    rescale_fallbacks: int = 0


def preprocess_frame(index, image, mask, config=None) -> PreprocessedFrame:
    return PreprocessedFrame(index, np.asarray(image, dtype=np.float64), np.asarray(mask, dtype=bool))


def condition_detections(pre, det, actor=None) -> ConditionedFrame:
    return ConditionedFrame(pre, det)


_trackers: dict = {}
TRACKER_CACHE = 2   # single-stream drop-in trackers kept alive (LRU); evicted ones are closed


def _tracker_for(actor, camera, config) -> Tracker:
    key = (id(actor), id(getattr(actor, "mesh", None)), camera.fx, camera.fy, camera.cx, camera.cy,
           camera.width, camera.height, repr(config))
    t = _trackers.pop(key, None)
    if t is not None and t[0] is not actor:
        t[1].close()
        t = None
    if t is None:
        t = (actor, Tracker(actor, camera, config, 1))
    _trackers[key] = t                       # most recently used last
    while len(_trackers) > TRACKER_CACHE:
        _trackers.pop(next(iter(_trackers)))[1].close()
    return t[1]


def solve_frame(cond, actor, camera, config, state):
    """Stage I + Stage II for one frame; returns (FrameResult, TrackState)."""
    config = SequenceConfig.from_reference(config) if config is not None else SequenceConfig()
    pre = cond.pre
    tr = _tracker_for(actor, camera, config)
    tr.set_state(0, state)
    raw = getattr(cond, "raw_detections", None) or cond.detections
    tr.set_frame(0, pre.image, pre.mask, raw)
    t0 = time.perf_counter()
    tr.step()
    x, v, vs, rep = tr.result(0)
    elapsed = time.perf_counter() - t0
    new_state = tr.get_state(0)
    pose_rep = pose_report_from_c(rep.pose)
    nr_rep = nonrigid_report_from_c(rep.nonrigid) if config.mode == "full" else None
    result = FrameResult(pre.index, PoseParams.from_vector(x), v, vs, pose_rep, nr_rep,
                         {"solve": elapsed})
    return result, new_state


@dataclass
class SequenceResult:
    """Reference `pipeline.py:328-343`."""
    config: SequenceConfig
    frames: list                      # FrameResult
    poses: np.ndarray                 # (F,36) raw
    vertices: np.ndarray              # (F,N,3) raw
    poses_smoothed: np.ndarray
    vertices_smoothed: np.ndarray
    events: list                      # slot-ordered ingest/emit records
    timings: dict
    pipelined: bool

    @property
    def fps(self) -> float:
        total = self.timings.get("total", 0.0)
        return len(self.frames) / total if total > 0 else float("inf")


def _prepare_actor(actor, config: SequenceConfig):
    """Reference `pipeline.py:346-354`: uniform material weight override."""
    from .actor import Actor
    actor = Actor.from_reference(actor)
    if config.uniform_material_weight is None:
        return actor
    mesh = replace(actor.mesh)
    s = float(config.uniform_material_weight)
    mesh.edge_weights = np.full(len(mesh.edges), s)
    mesh.directed_weights = np.full(2 * len(mesh.edges), s)
    return type(actor)(mesh, actor.skeleton, actor.skinning)


def _finalize(config, results, events, t_total, pipelined) -> SequenceResult:
    """Reference `pipeline.py:357-375`; the smoothing runs on the device."""
    from .postprocess import smooth_trajectory
    poses = np.stack([r.pose.to_vector() for r in results])
    vertices = np.stack([r.vertices for r in results])
    if config.smooth_output and len(results) > 1:
        poses_s = smooth_trajectory(poses, config.smoothing_stencil)
        vertices_s = smooth_trajectory(vertices, config.smoothing_stencil)
    else:
        poses_s = poses.copy()
        vertices_s = vertices.copy()
    stage_sums = {"preprocess": 0.0, "condition": 0.0, "pose": 0.0, "nonrigid": 0.0}
    for r in results:
        for k, v in r.timings.items():
            stage_sums[k] = stage_sums.get(k, 0.0) + v
    stage_sums["total"] = t_total
    return SequenceResult(config, results, poses, vertices, poses_s, vertices_s, events, stage_sums, pipelined)


def frame_latencies(events: list) -> dict:
    """Frame index -> emit slot minus ingest slot (reference `pipeline.py:503-507`)."""
    ingest, emit = {}, {}
    for e in events:
        (ingest if e["event"] == "ingest" else emit)[e["frame"]] = e["slot"]
    return {f: emit[f] - ingest[f] for f in sorted(emit)}


def run_sequence(inputs, config=None, pipelined=False) -> SequenceResult:
    """Sequence drivers (reference `pipeline.py:378-515`); the track state
    stays on the device.

    pipelined=False is run_sequence_sequential: frame f is ingested,
    preprocessed and solved in slot f.  pipelined=True is
    run_sequence_pipelined's slot schedule: frame f is ingested in slot f and
    emitted in slot f+2.  On the device that is the tracker's frame queue:
    slot s queues frame s (its upload and, once the next frame is queued
    behind it, its preprocessing overlap the solves of frames s-2 and s-1)
    and solves frame s-2.  The solves are the same in both drivers, so their
    results are identical (pipelined == sequential) and the events /
    latencies match the reference's.
    """
    config = SequenceConfig.from_reference(config) if config is not None else SequenceConfig()
    actor = _prepare_actor(inputs.actor, config)
    tr = Tracker(actor, inputs.camera, config, 1)
    frames, events = [], []
    n = inputs.n_frames

    def queue(f):
        tr.set_frame(0, inputs.images[f], inputs.masks[f], inputs.detections[f])

    def emit(f, slot, t0):
        tr.step()
        x, v, vs, rep = tr.result(0)
        frames.append(FrameResult(f, PoseParams.from_vector(x), v, vs, pose_report_from_c(rep.pose),
                                  nonrigid_report_from_c(rep.nonrigid) if config.mode == "full" else None,
                                  {"solve": time.perf_counter() - t0}))
        events.append({"slot": slot, "event": "emit", "frame": f})

    t_start = time.perf_counter()
    if pipelined:
        for slot in range(n + 2):
            t0 = time.perf_counter()
            if slot < n:
                events.append({"slot": slot, "event": "ingest", "frame": slot})
                queue(slot)
            if 0 <= slot - 2 < n:
                emit(slot - 2, slot, t0)
    else:
        for f in range(n):
            t0 = time.perf_counter()
            events.append({"slot": f, "event": "ingest", "frame": f})
            queue(f)
            emit(f, f, t0)
    total = time.perf_counter() - t_start
    tr.close()
    return _finalize(config, frames, events, total, pipelined)
