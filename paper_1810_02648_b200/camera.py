"""Pinhole intrinsics container (reference `camera.py:20-33`).

Projection itself runs on the device (`csrc/lc_device.cuh: project`); this
module only validates and carries the six numbers across the C-ABI.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class CameraIntrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if self.fx <= 0.0 or self.fy <= 0.0:
            raise ValueError(f"focal lengths must be positive, got fx={self.fx} fy={self.fy}")
        if self.width <= 0 or self.height <= 0:
            raise ValueError(f"image size must be positive, got {self.width}x{self.height}")

    @classmethod
    def from_reference(cls, cam) -> "CameraIntrinsics":
        if isinstance(cam, cls):
            return cam
        return cls(float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                   int(cam.width), int(cam.height))


def suggest_camera(width: int = 256, height: int = 256, depth: float = 2.5,
                   span: float = 2.1) -> CameraIntrinsics:
    """Intrinsics framing a `span`-metre body at `depth` (reference `actors.py:307-312`)."""
    f = 0.78 * height * depth / span
    return CameraIntrinsics(f, f, (width - 1) / 2.0, (height - 1) / 2.0, width, height)
