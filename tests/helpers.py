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


def scene_bench(preset="x5k", res=1024, n_frames=25, seed=0):
    """The bench's stream `seed` (bench.make_stream_frames), rendered by the oracle."""
    from oracle import imaging as OI
    actor = S.build_actor(preset, with_skirt=True)
    cam = suggest_camera(res, res)
    script = S.default_script(n_frames, noise=S.NoiseParams(sigma2d=1.0, sigma3d=0.008, seed=seed))
    return actor, cam, S.generate_sequence(actor, cam, script, OI.render_attributes, posing)


def oracle_state_to_mirror(st):
    from paper_1810_02648_b200.config import TrackState
    return TrackState(st.x_prev, st.x_prev2, st.joints_prev, st.disp_rest, st.v_prev, st.v_prev2)


def check_pose_strict(P, plogs, tag, rtol=1e-4):
    """Stage I decision trace identical, energies within rtol."""
    assert P.n_iterations == len(plogs), (tag, P.n_iterations, len(plogs))
    for k, o in enumerate(plogs):
        assert P.halvings[k] == o["halvings"], (tag, "pose halvings", k)
        assert bool(P.rejected[k]) == bool(o["rejected"]), (tag, "pose rejected", k)
        assert bool(P.damped[k]) == bool(o["damped"]), (tag, "pose damped", k)
        for key in ("energy_before", "energy_after"):
            ref = o[key]
            got = getattr(P, key)[k]
            assert abs(got - ref) <= rtol * max(abs(ref), 1e-300), (tag, "pose", key, k, got, ref)


def check_surface_strict(R, slogs, v, vo, diag, tag, rtol=1e-4):
    """Stage II decision trace identical (halvings / rejected / PCG
    breakdown), per-iteration energies and energy terms within rtol, final
    vertices within rtol of the bbox diagonal."""
    if slogs is not None:
        assert R.n_iterations == len(slogs), (tag, R.n_iterations, len(slogs))
        names = ("photo", "silhouette", "smooth", "edge", "velocity", "acceleration")
        for k, o in enumerate(slogs):
            assert R.halvings[k] == o["halvings"], (tag, "surface halvings", k)
            assert bool(R.rejected[k]) == bool(o["rejected"]), (tag, "surface rejected", k)
            assert bool(R.pcg_breakdown[k]) == bool(o["pcg_breakdown"]), (tag, "pcg breakdown", k)
            for key in ("energy_before", "energy_after"):
                ref = o[key]
                got = getattr(R, key)[k]
                assert abs(got - ref) <= rtol * max(abs(ref), 1e-300), \
                    (tag, "surface", key, k, got, ref, [R.terms[k][j] for j in range(6)], o["terms"])
            for j, nm in enumerate(names):
                ref = o["terms"].get(nm, 0.0)
                assert abs(R.terms[k][j] - ref) <= rtol * max(abs(ref), 1e-12 * o["energy_before"]), \
                    (tag, "term", nm, k, R.terms[k][j], ref)
    err = float(np.abs(v - vo).max()) / diag
    assert err <= rtol, (tag, "vertices / diag", err)
    return err


def check_frame_strict(rep, plogs, slogs, v, vo, diag, tag, rtol=1e-4):
    """Both stages of one teacher-forced frame (see the two checks above)."""
    check_pose_strict(rep.pose, plogs, tag, rtol)
    return check_surface_strict(rep.nonrigid, slogs, v, vo, diag, tag, rtol)
