"""Shared scene builders for the parity tests (oracle = checker only)."""

from __future__ import annotations

import numpy as np

from paper_1810_02648_b200 import synthetic as S
from paper_1810_02648_b200.camera import suggest_camera


def posing(actor, pose, rest):
    from oracle import geometry as OG
    fk = OG.Fk(actor.skeleton, pose.to_vector())
    return OG.skin(rest, actor.skinning, fk.dqs)[0], fk.pos, fk.markers


def scene(preset="small", res=128, n_frames=3, seed=0, with_skirt=True):
    from oracle import imaging as OI
    actor = S.build_actor(preset, with_skirt=with_skirt)
    cam = suggest_camera(res, res)
    frames = S.generate_sequence(actor, cam, S.default_script(n_frames, noise=S.NoiseParams(seed=seed)),
                                 OI.render_attributes, posing)
    return actor, cam, frames


def bbox_diag(actor):
    return float(np.linalg.norm(np.ptp(actor.mesh.rest_vertices, axis=0)))


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return abs(a - b) / max(abs(b), 1e-300)
