"""Bit-exact parity of the tracker's index / set work:
contour vertices, the Stage I and Stage II rim filters, the part-label
gating and the visible set, computed by the tracker's own kernels
(`lc_surface_sets`, the same launches `run_frame` makes).

* against the reference's own outputs (ref_kernels_small128.npz keys
  contour_idx, rim_stage1, rim_stage2, part_labels, visible);
* against the oracle on the Stage II starting surfaces (v_init) the tracker
  itself produced on small, standard and x5k@1024 frames (the sets the
  surface solve actually consumed, read back with lc_tracker_inspect).

Reference: pose_stage.py:139-264, nonrigid_stage.py:87-128, pipeline.py:211,236-249.
"""

import numpy as np
import pytest

from helpers import scene, scene_bench
from test_oracle_golden import check_digest, gen, load

pytestmark = pytest.mark.gpu


def _oracle_sets(v, actor, cam, dilation=10):
    from oracle import frame as OF
    from oracle.imaging import render_depth
    from oracle.posefit import contour_vertices, outer_rim
    from oracle.surface import part_label_mask, visible_vertices
    from oracle.geometry import project
    from paper_1810_02648_b200.actor import _class_weight_array
    mesh = actor.mesh
    zbuf = render_depth(cam, v, mesh.triangles)
    idx, n2 = contour_vertices(v, mesh, cam, zbuf)
    rim1 = outer_rim(v, idx, cam, zbuf) & (_class_weight_array(mesh.vertex_labels)[idx] >= OF.POSE_CONTOUR_MIN_RIGIDITY)
    rim2 = outer_rim(v, idx, cam, zbuf, min_thickness=0.0)
    labels, vparts = part_label_mask(v, mesh, actor.skinning, actor.skeleton, cam, dilation)
    en = rim2.copy()
    if len(idx):
        pix, ok = project(cam, v[idx])
        xi = np.clip(np.round(pix[:, 0]).astype(int), 0, cam.width - 1)
        yi = np.clip(np.round(pix[:, 1]).astype(int), 0, cam.height - 1)
        at = labels[yi, xi]
        en &= ok & ((at == 0) | (at == vparts[idx]))
    vis = np.flatnonzero(visible_vertices(v, mesh, cam, zbuf))
    return dict(contour=idx, normals2d=n2, rim1=rim1, rim2=rim2, enabled=en, visible=vis, labels=labels)


def _device_sets(v, actor, cam, labels=False):
    from paper_1810_02648_b200.pose_stage import tracker_sets
    s1 = tracker_sets(v, actor, cam, stage=1)
    s2 = tracker_sets(v, actor, cam, stage=2, part_gate=False)
    s3 = tracker_sets(v, actor, cam, stage=2, part_gate=True, with_labels=labels)
    assert np.array_equal(s1["contour"], s2["contour"]) and np.array_equal(s2["contour"], s3["contour"])
    out = dict(contour=s3["contour"], normals2d=s3["normals2d"], rim1=s1["keep"], rim2=s2["keep"],
               enabled=s3["keep"], visible=s3["visible"])
    if labels:
        out["labels"] = s3["labels"]
    return out


def test_sets_against_reference_golden():
    from oracle.posefit import contour_vertices  # noqa: F401  (oracle import check)
    from paper_1810_02648_b200.actor import _class_weight_array
    g = load("ref_kernels_small128.npz")
    actor, cam, frames = gen("small", 128, 2, 3)
    check_digest(g, frames)
    v = frames[1].gt_vertices
    d = _device_sets(v, actor, cam, labels=True)
    assert np.array_equal(d["contour"], g["contour_idx"])
    rig = _class_weight_array(actor.mesh.vertex_labels)[g["contour_idx"]] >= 2.0
    assert np.array_equal(d["rim1"], g["rim_stage1"] & rig)
    assert np.array_equal(d["rim2"], g["rim_stage2"])
    assert np.array_equal(d["labels"], g["part_labels"])
    assert np.array_equal(d["visible"], g["visible"])
    assert np.abs(d["normals2d"] - g["contour_n2d"]).max() <= 1e-12


def _compare(d, o, tag):
    for k in ("contour", "rim1", "rim2", "enabled", "visible"):
        assert np.array_equal(d[k], o[k]), (tag, k, len(d[k]), len(o[k]))
    assert np.abs(d["normals2d"] - o["normals2d"]).max(initial=0.0) <= 1e-12, tag
    if "labels" in d:
        assert np.array_equal(d["labels"], o["labels"]), tag


@pytest.mark.parametrize("preset,res,n,labels", [("small", 128, 3, True), ("standard", 256, 3, True),
                                                 ("x5k", 1024, 3, False)])
def test_sets_on_tracker_surfaces(preset, res, n, labels):
    """The sets for the Stage II starting surface the tracker produced
    (lc_tracker_inspect v_init), and the tracker's own consumed sets."""
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = (scene(preset, res, n) if preset != "x5k" else scene_bench(preset, res, n))
    tr = Tracker(actor, cam, SequenceConfig(directional=False), 1)
    for fr in frames:
        tr.set_frame(0, fr.image, fr.mask, fr.detections)
        tr.step()
        ins = tr.inspect(0)
        o = _oracle_sets(ins["v_init"], actor, cam)
        d = _device_sets(ins["v_init"], actor, cam, labels=labels)
        _compare(d, o, (preset, fr.index))
        # what the surface solve consumed in the tracker
        assert np.array_equal(ins["boundary"], o["contour"]), (preset, fr.index)
        assert np.array_equal(ins["enabled"], o["enabled"]), (preset, fr.index)
        assert np.array_equal(ins["visible"], o["visible"]), (preset, fr.index)
    tr.close()
