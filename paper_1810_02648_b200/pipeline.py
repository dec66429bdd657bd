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
from dataclasses import dataclass, field

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


def _tracker_for(actor, camera, config) -> Tracker:
    key = (id(actor), id(getattr(actor, "mesh", None)), camera.fx, camera.fy, camera.cx, camera.cy,
           camera.width, camera.height, repr(config))
    t = _trackers.get(key)
    if t is None or t[0] is not actor:
        t = (actor, Tracker(actor, camera, config, 1))
        _trackers[key] = t
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
    config: SequenceConfig
    frames: list
    poses: np.ndarray
    vertices: np.ndarray
    timings: dict
    pipelined: bool = False

    @property
    def fps(self) -> float:
        total = self.timings.get("total", 0.0)
        return len(self.frames) / total if total > 0 else float("inf")


def run_sequence(inputs, config=None, pipelined=False) -> SequenceResult:
    """Sequence drivers (pipeline.py:378-515); the track state stays on the device.

    pipelined=False is run_sequence_sequential: frame f is uploaded,
    preprocessed and solved before frame f+1 is touched.  pipelined=True is
    run_sequence_pipelined's 2-slot schedule: frame f+1 is queued before
    frame f is solved, so its upload and preprocessing (pyramid, observed
    contour grid) overlap frame f's solve.  The solves themselves are the
    same, so both drivers return identical results (pipelined == sequential).
    """
    config = SequenceConfig.from_reference(config) if config is not None else SequenceConfig()
    tr = Tracker(inputs.actor, inputs.camera, config, 1)
    frames = []
    n = inputs.n_frames

    def queue(f):
        tr.set_frame(0, inputs.images[f], inputs.masks[f], inputs.detections[f])

    t0 = time.perf_counter()
    if pipelined and n:
        queue(0)
    for f in range(n):
        if not pipelined:
            queue(f)
        elif f + 1 < n:
            queue(f + 1)
        tr.step()
        x, v, vs, rep = tr.result(0)
        frames.append(FrameResult(f, PoseParams.from_vector(x), v, vs, pose_report_from_c(rep.pose),
                                  nonrigid_report_from_c(rep.nonrigid) if config.mode == "full" else None,
                                  {}))
    total = time.perf_counter() - t0
    tr.close()
    return SequenceResult(config, frames, np.stack([r.pose.to_vector() for r in frames]),
                          np.stack([r.vertices for r in frames]), {"total": total}, pipelined)
