"""Configuration, pose parameters, detections, reports and tracker state.

Plain containers mirroring the reference's public dataclasses so a caller of
`montrack` finds the same fields: `PoseHyperparams` (`pose_stage.py:37-48`),
`NonrigidHyperparams` (`nonrigid_stage.py:33-49`), `SequenceConfig`
(`pipeline.py:48-86`), `PoseParams` (`skinning.py:33-65`), `FrameDetections`
(`pose_stage.py:51-64`), the per-iteration logs / stage reports
(`pose_stage.py:407-426`, `nonrigid_stage.py:352-369,409-414`,
`solvers.py:35-38,97-101`) and `TrackState` / `FrameResult`
(`pipeline.py:135-153`).
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, field, fields

import numpy as np

N_POSE_PARAMS = 36
MODES = ("full", "pose_only", "detections_only")

TEMPORAL_GROUP_WEIGHTS = {"torso": 2.5, "head": 2.5, "shoulder": 2.0,
                          "elbow": 1.5, "knee": 1.5, "hand": 1.0, "foot": 1.0}


@dataclass
class PoseHyperparams:
    lambda_2d: float = 460.0
    lambda_3d: float = 28.0
    lambda_sil: float = 200.0
    lambda_temporal: float = 1.5
    lambda_anatomic: float = 1.0e6
    face_weight: float = 0.326
    temporal_group_weights: dict = field(default_factory=lambda: dict(TEMPORAL_GROUP_WEIGHTS))
    gn_iterations: int = 6
    max_halvings: int = 3


@dataclass
class NonrigidHyperparams:
    w_photo: float = 10000.0
    w_sil: float = 600.0
    w_smooth: float = 10.0
    w_edge: float = 30.0
    w_velocity: float = 0.25
    w_acceleration: float = 0.1
    tau_color: float = 0.3
    gn_iterations: int = 3
    pcg_iterations: int = 4
    max_halvings: int = 3
    pyramid_kernels: tuple = (15, 9, 3)
    part_dilation: int = 10
    snap_step: float = 0.5
    snap_max_steps: int = 30
    snap_band: float = 0.25


@dataclass
class SequenceConfig:
    mode: str = "full"
    directional: bool = True
    enable_warping: bool = True
    enable_part_mask: bool = True
    enable_snapping: bool = True
    smooth_output: bool = True
    smoothing_stencil: tuple = (0.15, 0.7, 0.15)
    uniform_material_weight: float | None = None
    frame0_rounds: int = 3
    frame0_iteration_scale: int = 2
    pose: PoseHyperparams = field(default_factory=PoseHyperparams)
    nonrigid: NonrigidHyperparams = field(default_factory=NonrigidHyperparams)

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, rec: dict) -> "SequenceConfig":
        rec = dict(rec)
        unknown = set(rec) - {f.name for f in fields(cls)}
        if unknown:
            raise ValueError(f"unknown config keys: {sorted(unknown)}")
        if isinstance(rec.get("pose"), dict):
            rec["pose"] = PoseHyperparams(**rec["pose"])
        if isinstance(rec.get("nonrigid"), dict):
            rec["nonrigid"] = NonrigidHyperparams(**rec["nonrigid"])
        if "smoothing_stencil" in rec:
            rec["smoothing_stencil"] = tuple(rec["smoothing_stencil"])
        if isinstance(rec.get("nonrigid"), NonrigidHyperparams):
            rec["nonrigid"].pyramid_kernels = tuple(rec["nonrigid"].pyramid_kernels)
        return cls(**rec)

    @classmethod
    def from_reference(cls, ref) -> "SequenceConfig":
        if isinstance(ref, cls):
            return ref
        d = asdict(ref)
        return cls.from_dict(d)


@dataclass
class PoseParams:
    root_rotation: np.ndarray
    root_translation: np.ndarray
    theta: np.ndarray
    aux_translation: np.ndarray

    def __post_init__(self):
        self.root_rotation = np.asarray(self.root_rotation, dtype=np.float64)
        self.root_translation = np.asarray(self.root_translation, dtype=np.float64)
        self.theta = np.asarray(self.theta, dtype=np.float64)
        self.aux_translation = np.asarray(self.aux_translation, dtype=np.float64)
        if self.theta.shape != (27,):
            raise ValueError(f"expected 27 joint angles, got {self.theta.shape}")

    @classmethod
    def zero(cls) -> "PoseParams":
        return cls(np.zeros(3), np.zeros(3), np.zeros(27), np.zeros(3))

    @classmethod
    def from_vector(cls, x) -> "PoseParams":
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (N_POSE_PARAMS,):
            raise ValueError(f"pose vector must have {N_POSE_PARAMS} entries")
        return cls(x[0:3].copy(), x[3:6].copy(), x[6:33].copy(), x[33:36].copy())

    def to_vector(self) -> np.ndarray:
        return np.concatenate([self.root_rotation, self.root_translation,
                               self.theta, self.aux_translation])

    def copy(self) -> "PoseParams":
        return PoseParams.from_vector(self.to_vector())


@dataclass
class FrameDetections:
    joints2d: np.ndarray  # (J+4,2)
    joints3d: np.ndarray  # (J,3) root-relative
    valid2d: np.ndarray   # (J+4,)
    valid3d: np.ndarray   # (J,)

    def __post_init__(self):
        self.joints2d = np.asarray(self.joints2d, dtype=np.float64)
        self.joints3d = np.asarray(self.joints3d, dtype=np.float64)
        self.valid2d = np.asarray(self.valid2d, dtype=bool)
        self.valid3d = np.asarray(self.valid3d, dtype=bool)
        if self.joints2d.shape[0] != self.joints3d.shape[0] + 4:
            raise ValueError("2D detections must cover the joints plus 4 landmarks")


@dataclass
class ContourVertexSet:
    indices: np.ndarray    # (B,) ascending vertex ids
    normals2d: np.ndarray  # (B,2)


# ---------------------------------------------------------------------------
# reports (numeric events are flags, never exceptions)

@dataclass
class DenseSolveInfo:
    damped: bool = False
    damping: float = 0.0


@dataclass
class PcgInfo:
    iterations: int = 0
    breakdown: bool = False
    residual_norms: list = field(default_factory=list)


@dataclass
class PoseIterationLog:
    energy_before: float
    energy_after: float
    terms: dict
    step_norm: float
    halvings: int
    rejected: bool
    damped: bool


@dataclass
class PoseStageReport:
    iterations: list = field(default_factory=list)
    behind_camera: int = 0
    gimbal: bool = False

    @property
    def final_energy(self) -> float:
        return self.iterations[-1].energy_after if self.iterations else float("nan")


@dataclass
class NonrigidIterationLog:
    level: int
    energy_before: float
    energy_after: float
    terms: dict
    halvings: int
    rejected: bool
    pcg_breakdown: bool


@dataclass
class SnapInfo:
    walked: int = 0
    reached: int = 0
    stuck: int = 0
    moved_vertices: np.ndarray | None = None


@dataclass
class NonrigidStageReport:
    iterations: list = field(default_factory=list)
    pruned: int = 0
    degenerate_edges: int = 0
    behind_camera: int = 0
    snap: SnapInfo | None = None


@dataclass
class TrackState:
    pose_prev: PoseParams | None = None
    pose_prev2: PoseParams | None = None
    joints_prev: np.ndarray | None = None
    disp_rest: np.ndarray | None = None
    v_prev: np.ndarray | None = None
    v_prev2: np.ndarray | None = None


@dataclass
class FrameResult:
    index: int
    pose: PoseParams
    vertices: np.ndarray
    skinned: np.ndarray
    pose_report: object
    nonrigid_report: object | None
    timings: dict


POSE_TERM_NAMES = ("detection2d", "detection3d", "silhouette", "temporal", "anatomic")
NONRIGID_TERM_NAMES = ("photo", "silhouette", "smooth", "edge", "velocity", "acceleration")
