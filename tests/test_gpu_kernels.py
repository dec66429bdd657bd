"""GPU kernel parity against the CPU oracle (which is bit-identical to the
reference, see test_oracle_golden.py).  Bit-exact where the domain is
integer / index / fixed-order arithmetic; fp64 tolerances elsewhere."""

import numpy as np
import pytest

from helpers import bbox_diag, scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small():
    return scene("small", 128, 2)


def test_dense_solve_matches_oracle(ctx):
    from oracle.linsolve import dense_solve as odense
    from paper_1810_02648_b200.solvers import DenseNormalSystem, dense_solve
    rng = np.random.default_rng(1)
    for trial in range(5):
        J = rng.standard_normal((80, 36))
        a = J.T @ J
        b = rng.standard_normal(36)
        x, info = dense_solve(DenseNormalSystem(a, b))
        xo, damped, _ = odense(a, b)
        assert not info.damped and not damped
        assert np.allclose(x, xo, rtol=1e-9, atol=1e-12)
    # rank deficient: two identical columns -> damping path (solvers.py:48-54)
    J = rng.standard_normal((80, 36))
    J[:, 5] = J[:, 4]
    a = J.T @ J
    b = rng.standard_normal(36)
    x, info = dense_solve(DenseNormalSystem(a, b))
    xo, damped, lam = odense(a, b)
    assert info.damped and damped
    assert info.damping == pytest.approx(lam, rel=1e-14)
    assert np.allclose(x, xo, rtol=1e-7, atol=1e-9)


def test_dense_solve_rejects_nonfinite():
    from paper_1810_02648_b200.solvers import DenseNormalSystem
    with pytest.raises(ValueError):
        DenseNormalSystem(np.full((3, 3), np.nan), np.zeros(3))


def _surface_problem(actor, cam, frames, directional=False):
    from paper_1810_02648_b200.config import SequenceConfig
    from oracle import frame as OF
    cfg = SequenceConfig(directional=directional)
    prep = OF.prepare(frames[0].image, frames[0].mask, frames[0].detections, actor, cfg)
    st = OF.State()
    x, _ = OF.stage1(prep, actor, cam, cfg, st, actor.mesh.rest_vertices)
    pb, v_init, vs, rot = OF.stage2_problem(prep, actor, cam, cfg, st, x, actor.mesh.rest_vertices)
    return pb, v_init, cfg, prep


def test_pcg_bsr_matches_oracle(small):
    from oracle import surface as OS
    from oracle.linsolve import pcg
    from paper_1810_02648_b200.solvers import BlockSparseSystem, pcg_solve
    actor, cam, frames = small
    pb, v_init, _, _ = _surface_problem(actor, cam, frames)
    ev = OS.surface_evaluate(pb, v_init, 0)
    diag, off, rows, cols, rhs = OS.normal_system(pb, ev)
    for iters in (1, 4, 12):
        x, info = pcg_solve(BlockSparseSystem(diag, off, rows, cols, rhs), iters)
        xo, done, brk, norms = pcg(diag, off, rows, cols, rhs, iters)
        assert info.iterations == done and info.breakdown == brk
        assert np.allclose(info.residual_norms, norms, rtol=1e-6)
        assert np.abs(x - xo).max() <= 1e-6 * max(np.abs(xo).max(), 1e-300)


def test_pcg_bsr_random_spd_converges():
    """SPEC acceptance #5: 200 iterations match a direct solve (N=200)."""
    from paper_1810_02648_b200.solvers import BlockSparseSystem, pcg_solve
    rng = np.random.default_rng(7)
    n = 200
    rows, cols = [], []
    for i in range(n):
        for j in rng.choice(n, 4, replace=False):
            if i != j:
                rows += [i, j]
                cols += [j, i]
    pairs = sorted(set(zip(rows, cols)))
    rows = np.array([p[0] for p in pairs])
    cols = np.array([p[1] for p in pairs])
    A = np.zeros((3 * n, 3 * n))
    off = np.zeros((len(rows), 3, 3))
    done = {}
    for k, (i, j) in enumerate(zip(rows, cols)):
        if (j, i) in done:
            off[k] = off[done[(j, i)]].T
        else:
            off[k] = 0.1 * rng.standard_normal((3, 3))
            done[(i, j)] = k
        A[3 * i:3 * i + 3, 3 * j:3 * j + 3] += off[k]
    diag = np.zeros((n, 3, 3))
    for i in range(n):
        m = rng.standard_normal((3, 3))
        diag[i] = m @ m.T + 5.0 * np.eye(3)
        A[3 * i:3 * i + 3, 3 * i:3 * i + 3] += diag[i]
    rhs = rng.standard_normal((n, 3))
    x, info = pcg_solve(BlockSparseSystem(diag, off, rows, cols, rhs), 60)
    xd = np.linalg.solve(A, rhs.ravel()).reshape(n, 3)
    assert np.linalg.norm(A @ x.ravel() - rhs.ravel()) <= 1e-6 * np.linalg.norm(rhs)
    assert np.allclose(x, xd, atol=1e-6)


def test_render_bit_exact(small):
    from oracle import imaging as OI
    from paper_1810_02648_b200 import imageproc as G
    actor, cam, frames = small
    v = frames[1].gt_vertices
    tris = actor.mesh.triangles
    assert np.array_equal(G.render_depth(cam, v, tris), OI.render_depth(cam, v, tris))
    ga, gz = G.render_attributes(cam, v, tris, actor.mesh.vertex_colors)
    oa, oz = OI.render_attributes(cam, v, tris, actor.mesh.vertex_colors)
    assert np.array_equal(gz, oz) and np.array_equal(ga, oa)
    ids = np.arange(len(v)) % 7 + 1
    gi, _ = G.render_vertex_ids(cam, v, tris, ids, background=0)
    oi, _ = OI.render_vertex_ids(cam, v, tris, ids, background=0)
    assert np.array_equal(gi, oi)


def test_render_large_exact():
    from oracle import imaging as OI
    from paper_1810_02648_b200 import imageproc as G
    actor, cam, frames = scene("x5k", 1024, 1)
    v = frames[0].gt_vertices
    assert np.array_equal(G.render_depth(cam, v, actor.mesh.triangles),
                          OI.render_depth(cam, v, actor.mesh.triangles))


def test_pyramid_bit_exact(small):
    from oracle import imaging as OI
    from paper_1810_02648_b200 import imageproc as G
    actor, cam, frames = small
    img = frames[0].image
    odd = np.random.default_rng(5).random((45, 77, 3))   # non-multiple-of-tile shape
    for a, b in zip(G.gaussian_pyramid(odd, (15, 9, 3)), OI.gaussian_pyramid(odd, (15, 9, 3))):
        assert np.array_equal(a, b)
    for ks in ((15, 9, 3), (5, 21), (1, 7, 13, 15)):
        gp = G.gaussian_pyramid(img, ks)
        op = OI.gaussian_pyramid(img, ks)
        for a, b in zip(gp, op):
            assert np.array_equal(a, b)
    # the bench's frame size: interior tiles take the 16-byte load path
    big = np.random.default_rng(6).random((1024, 1024, 3))
    for a, b in zip(G.gaussian_pyramid(big, (15, 9, 3)), OI.gaussian_pyramid(big, (15, 9, 3))):
        assert np.array_equal(a, b)


def test_distance_field_matches_ckdtree(small):
    from oracle import imaging as OI
    from paper_1810_02648_b200 import imageproc as G
    actor, cam, frames = small
    mask = frames[0].mask
    g, o = G.DistanceField(mask), OI.DistanceField(mask)
    assert g.n_contour == len(o.points)
    rng = np.random.default_rng(3)
    q = np.concatenate([rng.uniform(-40, 170, (4000, 2)), rng.uniform(30, 90, (4000, 2)),
                        [[np.nan, 3.0], [1e6, -1e6]]])
    gd, gc = g.sample_value(q)
    od, oc = o.sample_value(q)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gd, od)
    gr, gg, _ = g.sample_residual(q)
    orr, og, _ = o.sample_residual(q)
    assert np.array_equal(gr, orr) and np.array_equal(gg, og)
    assert np.array_equal(g.inside(q[:-2]), o.inside(q[:-2]))
    assert np.array_equal(g.sample_interface(q)[0], o.sample_interface(q)[0])


def test_skinning_and_fk_match_oracle(small):
    from oracle import geometry as OG
    from paper_1810_02648_b200 import skinning as G
    actor, cam, frames = small
    x = frames[1].pose.to_vector() + np.random.default_rng(0).uniform(-0.05, 0.05, 36)
    fk = G.forward_kinematics(actor, x)
    ofk = OG.Fk(actor.skeleton, x)
    assert np.allclose(fk.positions, ofk.pos, rtol=0, atol=1e-13)
    assert np.allclose(fk.marker_positions, ofk.markers, rtol=0, atol=1e-13)
    assert np.allclose(fk.joint_dqs, ofk.dqs, rtol=0, atol=1e-13)
    rest = actor.mesh.rest_vertices
    sk = G.skin_points(actor, x, rest)
    p, r, _, _ = OG.skin(rest, actor.skinning, ofk.dqs)
    assert np.allclose(sk.positions, p, atol=1e-13) and np.allclose(sk.rotations, r, atol=1e-13)
    sub = np.arange(0, len(rest), 7)
    sj = G.skin_points(actor, x, rest[sub], subset=sub, with_jacobian=True)
    p, _, jac, _ = OG.skin(rest[sub], actor.skinning, ofk.dqs, OG.dq_jacobian(actor.skeleton, ofk), subset=sub)
    assert np.allclose(sj.positions, p, atol=1e-13)
    assert np.allclose(sj.jacobian, jac, atol=1e-11)


def test_contour_vertices_match_oracle(small):
    from oracle.posefit import contour_vertices
    from paper_1810_02648_b200.pose_stage import extract_contour_vertices
    actor, cam, frames = small
    for fr in frames:
        c = extract_contour_vertices(fr.gt_vertices, actor, cam)
        idx, n2 = contour_vertices(fr.gt_vertices, actor.mesh, cam)
        assert np.array_equal(c.indices, idx)
        assert np.allclose(c.normals2d, n2, atol=1e-12)


def test_edt_bit_exact():
    """a9: DistanceField.dt / euclidean_dt / _edt_squared (imageproc.py:52-124,
    182) on the device, bit-identical to the reference's golden and to the
    oracle's C restatement (random features, rows without any feature)."""
    from oracle import imaging as OI
    from paper_1810_02648_b200.imageproc import DistanceField, edt_squared, euclidean_dt
    from test_oracle_golden import check_digest, gen, load
    g = load("ref_kernels_small128.npz")
    _, _, frames = gen("small", 128, 2, 3)
    check_digest(g, frames)
    assert np.array_equal(euclidean_dt(frames[1].mask), g["edt"])
    assert np.array_equal(DistanceField(frames[1].mask).dt, g["edt"])
    rng = np.random.default_rng(7)
    for shape, p in (((37, 53), 0.02), ((128, 96), 0.001), ((64, 64), 0.3), ((1, 17), 0.2)):
        feat = rng.random(shape) < p
        feat[shape[0] // 2] = False            # a featureless row
        assert np.array_equal(edt_squared(feat), OI.edt_squared(feat)), shape
