"""B200-native LiveCap pose + non-rigid Gauss-Newton hot path.

A drop-in for the reference package's (`montrack`) per-frame solver path:
`solve_frame`, `solve_pose`, `solve_nonrigid`, `snap_vertices`, `pcg_solve`,
`dense_solve`, `DistanceField`, `gaussian_pyramid`, skinning and rasterizer
primitives -- all computed by hand-written sm_100a kernels in
`liblivecap.so` (C-ABI: include/livecap.h), called through ctypes.
`Tracker` batches S independent capture streams per kernel launch.
"""

from .actor import Actor, Skeleton, SkinningWeights, TemplateMesh, class_weight
from .camera import CameraIntrinsics, suggest_camera
from .config import (ContourVertexSet, FrameDetections, NonrigidHyperparams, PoseHyperparams,
                     PoseParams, SequenceConfig, TrackState)

__version__ = "0.1.0"

_LAZY = {
    "Tracker": ".device", "DeviceActor": ".device",
    "solve_frame": ".pipeline", "run_sequence": ".pipeline", "preprocess_frame": ".pipeline",
    "condition_detections": ".pipeline", "SequenceInputs": ".pipeline",
    "solve_pose": ".pose_stage", "PoseProblem": ".pose_stage",
    "extract_contour_vertices": ".pose_stage",
    "solve_nonrigid": ".nonrigid_stage", "snap_vertices": ".nonrigid_stage",
    "NonrigidProblem": ".nonrigid_stage",
    "pcg_solve": ".solvers", "dense_solve": ".solvers", "BlockSparseSystem": ".solvers",
    "DenseNormalSystem": ".solvers",
    "DistanceField": ".imageproc", "gaussian_pyramid": ".imageproc", "render_depth": ".imageproc",
    "render_attributes": ".imageproc", "render_vertex_ids": ".imageproc",
    "forward_kinematics": ".skinning", "skin_points": ".skinning",
    "install": ".dropin",
    "mean_vertex_error": ".metrics", "aligned_joint_error": ".metrics", "umeyama_alignment": ".metrics",
    "sequence_errors": ".metrics", "iou": ".metrics", "evaluate_tracking": ".evaluation",
}


def __getattr__(name):
    if name in _LAZY:
        import importlib
        mod = importlib.import_module(_LAZY[name], __name__)
        return getattr(mod, name)
    raise AttributeError(name)
