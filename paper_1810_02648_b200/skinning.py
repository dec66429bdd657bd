"""Forward kinematics and dual-quaternion skinning on the GPU
(reference skinning.py:206-398).

The device keeps the skeleton with the uploaded actor, so these take the
actor (or a (skeleton, skinning) pair) instead of the bare skeleton.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .config import PoseParams
from .device import DeviceActor


@dataclass
class FkResult:
    rotations: np.ndarray         # (J,3,3)
    positions: np.ndarray         # (J,3)
    marker_positions: np.ndarray  # (4,3)
    joint_dqs: np.ndarray         # (J,8)
    gimbal: bool


@dataclass
class SkinResult:
    positions: np.ndarray
    rotations: np.ndarray
    jacobian: np.ndarray | None


def _dev(actor_or_parts, ctx):
    if isinstance(actor_or_parts, tuple):
        return DeviceActor.for_pose(actor_or_parts[0], actor_or_parts[1], ctx)
    return DeviceActor.get(actor_or_parts, ctx)


def forward_kinematics(actor, pose, ctx: L.Context | None = None) -> FkResult:
    ctx = ctx or L.default_context()
    dev = _dev(actor, ctx)
    x = L.f64c(pose.to_vector() if isinstance(pose, PoseParams) or hasattr(pose, "to_vector") else pose)
    J = dev.n_joints
    rot, pos, mk, dq = np.empty((J, 3, 3)), np.empty((J, 3)), np.empty((4, 3)), np.empty((J, 8))
    g = C.c_int32()
    L.check(ctx.lib.lc_forward_kinematics(ctx.handle, dev.handle, L.ptr(x), L.ptr(rot), L.ptr(pos), L.ptr(mk),
                                          L.ptr(dq), C.byref(g)))
    return FkResult(rot, pos, mk, dq, bool(g.value))


def skin_points(actor, pose, rest_points, subset=None, with_jacobian=False,
                ctx: L.Context | None = None) -> SkinResult:
    """Skin rest points at `pose`; `subset` gives the skinning rows of the
    (already gathered) rest points, as in the reference."""
    ctx = ctx or L.default_context()
    dev = _dev(actor, ctx)
    x = L.f64c(pose.to_vector() if hasattr(pose, "to_vector") else pose)
    r = L.f64c(rest_points)
    m = len(r)
    sub = None if subset is None else L.i64c(subset)
    pos, rot = np.empty((m, 3)), np.empty((m, 4))
    jac = np.empty((m, 3, 36)) if with_jacobian else None
    L.check(ctx.lib.lc_skin_points(ctx.handle, dev.handle, L.ptr(x), m, L.ptr(r), L.ptr(sub), L.ptr(pos),
                                   L.ptr(rot), L.ptr(jac)))
    return SkinResult(pos, rot, jac)
