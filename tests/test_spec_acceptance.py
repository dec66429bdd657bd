"""Known-answer / acceptance criteria of the reference's SPEC
(SPEC.md "ACCEPTANCE CRITERIA") that concern the hot path, run against the
device implementation:

  2. EDT exactness: euclidean_dt equals the brute-force nearest-contour
     distance on 100 random 64x64 masks (to 1e-9; here exactly).
  3. Skinning sanity: single-joint-weight vertices reproduce the joint's
     rigid transform to 1e-10; the DQ blend of two same-axis rotations
     matches the half-angle formula to 1e-8.
  5. Solver equivalence: tests/test_gpu_stages.py (PCG-200 vs direct solve).
 10. Pipelined == sequential, 2-frame latency: tests/test_gpu_frame.py,
     tests/test_post_io.py.
 12. Hyperparameter fidelity: the default SequenceConfig and Table 1 equal
     the reference's own (golden from tools/make_golden_config.py).

Criterion 4 (pose recovery from a 5-degree perturbation to 1e-3 rad) is not
met by the reference itself on its synthetic actor (the oracle, which is
bit-identical to it, ends 0.1-0.8 rad away after 6 GN steps), so
it is not a parity gate.  6-8 are whole-sequence ablation claims about the
algorithm, reported by tools/spec_ablations.py, not asserted.
"""

import json
import os

import numpy as np
import pytest

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_default_config_equals_reference():
    """Acceptance 12 (CPU)."""
    from paper_1810_02648_b200.actor import MATERIAL_CLASS_WEIGHTS
    from paper_1810_02648_b200.config import SequenceConfig
    ref = json.load(open(os.path.join(G, "ref_config.json")))
    mine = json.loads(json.dumps(SequenceConfig().to_dict(), default=list))
    assert mine == ref["config"]
    assert {str(k): v for k, v in MATERIAL_CLASS_WEIGHTS.items()} == ref["material_class_weights"]


def _blob_mask(rng, n=64):
    from scipy.ndimage import gaussian_filter
    f = gaussian_filter(rng.standard_normal((n, n)), sigma=rng.uniform(2, 6))
    return f > np.quantile(f, rng.uniform(0.3, 0.9))


def _brute_dt(mask):
    from oracle.imaging import contour_mask
    pts = np.argwhere(contour_mask(mask)).astype(np.float64)
    yy, xx = np.mgrid[0:mask.shape[0], 0:mask.shape[1]]
    q = np.stack([yy.ravel(), xx.ravel()], 1).astype(np.float64)
    d2 = ((q[:, None, :] - pts[None, :, :]) ** 2).sum(-1).min(1)
    return np.sqrt(d2).reshape(mask.shape)


@pytest.mark.gpu
def test_edt_exact_on_100_random_masks():
    """Acceptance 2."""
    from paper_1810_02648_b200.imageproc import euclidean_dt
    rng = np.random.default_rng(2)
    for t in range(100):
        m = _blob_mask(rng)
        if not m.any():
            continue
        got = euclidean_dt(m)
        assert np.abs(got - _brute_dt(m)).max() <= 1e-9, t


def _qrot(q, v):
    w, u = q[0], q[1:]
    t = 2.0 * np.cross(u, v)
    return v + w * t + np.cross(u, t)


@pytest.mark.gpu
def test_single_joint_vertices_are_rigid():
    """Acceptance 3a: a vertex weighted to one joint moves by that joint's
    rigid transform (rotation = the DQ's real part, translation
    2 q_d q_r^*), to 1e-10."""
    from helpers import scene
    from paper_1810_02648_b200.config import PoseParams
    from paper_1810_02648_b200.skinning import forward_kinematics, skin_points
    actor, _, frames = scene("small", 128, 2)
    sw = actor.skinning
    single = np.flatnonzero((sw.weights[:, 0] == 1.0) & (sw.weights[:, 1:] == 0).all(1))
    assert len(single) > 50
    rng = np.random.default_rng(3)
    for fr in frames:
        x = fr.pose.to_vector() + rng.uniform(-0.2, 0.2, 36)
        fk = forward_kinematics(actor, PoseParams.from_vector(x))
        rest = actor.mesh.rest_vertices[single]
        got = skin_points(actor, PoseParams.from_vector(x), rest, subset=single).positions
        for k, i in enumerate(single):
            dq = fk.joint_dqs[sw.indices[i, 0]]
            qr, qd = dq[:4], dq[4:]
            # 2 q_d q_r^* (vector part)
            w1, v1 = qd[0], qd[1:]
            w2, v2 = qr[0], -qr[1:]
            t = 2.0 * (w1 * v2 + w2 * v1 + np.cross(v1, v2))
            ref = _qrot(qr, rest[k]) + t
            assert np.abs(got[k] - ref).max() <= 1e-10, (i, got[k], ref)


@pytest.mark.gpu
def test_dq_blend_of_same_axis_rotations_half_angle():
    """Acceptance 3b: spine and chest both rotate about x (parent chain with
    axis-aligned rest frames), so a w : 1-w blend of their quaternions is a
    rotation about x by phi with tan(phi/2) = (w sin(A/2) + (1-w) sin(B/2)) /
    (w cos(A/2) + (1-w) cos(B/2)), A = theta_spine, B = theta_spine +
    theta_chest; checked to 1e-8 on the device's blended rotations."""
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.actor import SkinningWeights
    from paper_1810_02648_b200.config import PoseParams
    from paper_1810_02648_b200.skinning import skin_points
    sk = S.default_skeleton()
    names = list(sk.joint_names)
    js, jc = names.index("spine"), names.index("chest")
    dof = [(names[int(j)], tuple(np.round(a, 6))) for j, a in zip(sk.dof_joint, sk.dof_axes)]
    ks, kc = dof.index(("spine", (1.0, 0.0, 0.0))), dof.index(("chest", (1.0, 0.0, 0.0)))
    ws = np.linspace(0.05, 0.95, 19)
    idx = np.full((len(ws), 4), -1)
    w4 = np.zeros((len(ws), 4))
    idx[:, 0], idx[:, 1] = js, jc
    w4[:, 0], w4[:, 1] = ws, 1.0 - ws
    skin = SkinningWeights(idx, w4)
    rest = np.zeros((len(ws), 3)) + [0.05, -0.2, 2.5]
    for a, b in ((0.3, 0.2), (-0.4, 0.25), (0.1, -0.45)):
        x = np.zeros(36)
        x[6 + ks], x[6 + kc] = a, b
        rot = skin_points((sk, skin), PoseParams.from_vector(x), rest, subset=np.arange(len(ws))).rotations
        A, B = a, a + b
        phi = 2.0 * np.arctan2(ws * np.sin(A / 2) + (1 - ws) * np.sin(B / 2),
                               ws * np.cos(A / 2) + (1 - ws) * np.cos(B / 2))
        q = rot * np.sign(rot[:, :1])
        assert np.abs(q[:, 2:]).max() <= 1e-12                      # about x only
        assert np.abs(2.0 * np.arctan2(q[:, 1], q[:, 0]) - phi).max() <= 1e-8, (a, b)
