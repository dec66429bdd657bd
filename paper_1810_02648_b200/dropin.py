"""Drop-in installation into the reference package (`montrack`).

The reference imports its solvers with `from X import f`, so the names to
rebind live in the *consumer* modules:

  level "solvers": montrack.nonrigid_stage.pcg_solve  (nonrigid_stage.py:26)
                   montrack.pose_stage.dense_solve    (pose_stage.py:24)
  level "stages":  + montrack.pipeline.solve_pose / solve_nonrigid / snap_vertices
                     (pipeline.py:26-33)
  level "frame":   + montrack.pipeline.preprocess_frame / condition_detections /
                     solve_frame (pipeline.py:156-302): the whole per-frame
                     solve runs on the GPU, `run_sequence` keeps its drivers.

`install(montrack)` returns an `uninstall()` callable restoring the originals.
"""

from __future__ import annotations

import importlib


def _mods(pkg):
    name = pkg.__name__ if hasattr(pkg, "__name__") else str(pkg)
    get = lambda m: importlib.import_module(f"{name}.{m}")  # noqa: E731
    return get("pipeline"), get("pose_stage"), get("nonrigid_stage")


def install(pkg, level: str = "frame"):
    from . import nonrigid_stage as NR
    from . import pipeline as PL
    from . import pose_stage as PS
    from . import solvers as SV
    if level not in ("solvers", "stages", "frame"):
        raise ValueError("level must be 'solvers', 'stages' or 'frame'")
    pipeline, pose_stage, nonrigid_stage = _mods(pkg)
    saved = []

    def bind(mod, name, fn):
        saved.append((mod, name, getattr(mod, name)))
        setattr(mod, name, fn)

    bind(nonrigid_stage, "pcg_solve", SV.pcg_solve)
    bind(pose_stage, "dense_solve", SV.dense_solve)
    if level in ("stages", "frame"):
        bind(pipeline, "solve_pose", PS.solve_pose)
        bind(pipeline, "solve_nonrigid", NR.solve_nonrigid)
        bind(pipeline, "snap_vertices", NR.snap_vertices)
    if level == "frame":
        bind(pipeline, "preprocess_frame", PL.preprocess_frame)
        bind(pipeline, "condition_detections", PL.condition_detections)
        bind(pipeline, "solve_frame", PL.solve_frame)

    def uninstall():
        for mod, name, fn in reversed(saved):
            setattr(mod, name, fn)
    return uninstall
