"""Evaluation row: metrics.py / evaluation.py.

CPU: the oracle restatement reproduces the reference-made goldens
(tools/make_golden_eval.py) bit for bit.  GPU: the device metrics
(csrc/lc_eval.cu) reproduce them — mean_vertex_error bit-exact, the Umeyama
alignment within 1e-12 (a Jacobi SVD in place of LAPACK's) — and
evaluate_tracking on the reference-written seq_tiny capture and results.
"""

import json
import os

import numpy as np
import pytest

from oracle import post as OP

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _g():
    return np.load(os.path.join(G, "ref_metrics.npz"))


def test_oracle_metrics_match_reference():
    g = _g()
    for k in range(4):
        p, q, idx = g[f"mve_pred{k}"], g[f"mve_gt{k}"], g[f"mve_idx{k}"]
        assert OP.mean_vertex_error(p, q) == float(g[f"mve_c{k}"])
        assert OP.mean_vertex_error(p, q, center=False) == float(g[f"mve_nc{k}"])
        assert OP.mean_vertex_error(p, q, indices=idx) == float(g[f"mve_ci{k}"])
    for k in range(6):
        for ws in (0, 1):
            sc, R, t = OP.umeyama(g[f"um_src{k}"], g[f"um_dst{k}"], bool(ws))
            assert sc == float(g[f"um_scale{k}_{ws}"])
            assert np.array_equal(R, g[f"um_rot{k}_{ws}"]) and np.array_equal(t, g[f"um_t{k}_{ws}"])
            assert OP.aligned_joint_error(g[f"um_src{k}"], g[f"um_dst{k}"], bool(ws)) == float(g[f"um_err{k}_{ws}"])
    labels = g["se_labels"]
    ci = {f"class{c}": np.flatnonzero(labels == c) for c in np.unique(labels)}
    assert OP.sequence_errors(g["se_pred"], g["se_gt"], ci) == json.loads(str(g["se_json"]))


@pytest.mark.gpu
def test_device_vertex_error_bit_exact():
    from paper_1810_02648_b200 import metrics as M
    g = _g()
    for k in range(4):
        p, q, idx = g[f"mve_pred{k}"], g[f"mve_gt{k}"], g[f"mve_idx{k}"]
        assert M.mean_vertex_error(p, q) == float(g[f"mve_c{k}"])
        assert M.mean_vertex_error(p, q, center=False) == float(g[f"mve_nc{k}"])
        assert M.mean_vertex_error(p, q, indices=idx) == float(g[f"mve_ci{k}"])
    labels = g["se_labels"]
    ci = {f"class{c}": np.flatnonzero(labels == c) for c in np.unique(labels)}
    assert M.sequence_errors(g["se_pred"], g["se_gt"], ci) == json.loads(str(g["se_json"]))
    with pytest.raises(ValueError):
        M.mean_vertex_error(np.zeros((4, 3)), np.zeros((5, 3)))


@pytest.mark.gpu
def test_device_umeyama_matches_reference():
    from paper_1810_02648_b200 import metrics as M
    g = _g()
    for k in range(6):
        for ws in (0, 1):
            src, dst = g[f"um_src{k}"], g[f"um_dst{k}"]
            sc, R, t = M.umeyama_alignment(src, dst, bool(ws))
            assert abs(sc - float(g[f"um_scale{k}_{ws}"])) <= 1e-12 * max(1.0, abs(sc)), (k, ws)
            assert np.abs(R - g[f"um_rot{k}_{ws}"]).max() <= 1e-12, (k, ws)
            assert np.abs(t - g[f"um_t{k}_{ws}"]).max() <= 1e-11, (k, ws)
            assert abs(np.linalg.det(R) - 1.0) < 1e-12
            e = M.aligned_joint_error(src, dst, bool(ws))
            assert abs(e - float(g[f"um_err{k}_{ws}"])) <= 1e-12 * max(1.0, e), (k, ws)
    # batched == per frame
    src = np.stack([g[f"um_src{k}"] for k in range(4)])
    dst = np.stack([g[f"um_dst{k}"] for k in range(4)])
    eb = M.aligned_joint_error_batch(src, dst)
    assert np.array_equal(eb, [M.aligned_joint_error(s, d) for s, d in zip(src, dst)])
    with pytest.raises(ValueError):
        M.umeyama_alignment(np.zeros((2, 3)), np.zeros((2, 3)))


@pytest.mark.gpu
def test_evaluate_tracking_matches_reference():
    from paper_1810_02648_b200.evaluation import evaluate_tracking
    g = np.load(os.path.join(G, "ref_eval_tiny.npz"))
    for key, sm in (("smoothed", True), ("raw", False)):
        ref = json.loads(str(g[key]))
        got = evaluate_tracking(os.path.join(G, "seq_tiny"), os.path.join(G, "seq_tiny_result"), use_smoothed=sm)
        assert got["n_frames"] == ref["n_frames"]
        assert got["vertex_error_per_frame"] == ref["vertex_error_per_frame"]   # bit-exact
        for k in ref:
            if k.startswith("vertex_error") and k != "vertex_error_per_frame":
                assert got[k] == ref[k], k
        assert got["mean_iou"] == ref["mean_iou"]                               # bit-exact raster + counts
        assert abs(got["joint_error"] - ref["joint_error"]) <= 1e-12 * max(1.0, ref["joint_error"])
