"""ORACLE (test infrastructure only): Stage II per-vertex non-rigid registration.

Restates reference `nonrigid_stage.py:87-500`: visibility, body-part label
mask, the residual blocks and their explicit 3x3-block normal system, the
coarse-to-fine halving GN loop with PCG, and silhouette snapping.  Also
provides the compact matrix-free form of the same normal system
 used to check the device operator.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_1810_02648_b200.actor import TORSO_PART, joint_body_parts

from .geometry import project, projection_jac
from .imaging import DistanceField, edt_squared, render_depth, render_vertex_ids, sample_bilinear
from .linsolve import pcg
from .posefit import side_signs


def visible_vertices(verts, mesh, cam, zbuf=None):
    """Depth-test with a 1%-of-depth tolerance (nonrigid_stage.py:87-99)."""
    if zbuf is None:
        zbuf = render_depth(cam, verts, mesh.triangles)
    pix, ok = project(cam, verts)
    xi = np.clip(np.round(pix[:, 0]).astype(int), 0, cam.width - 1)
    yi = np.clip(np.round(pix[:, 1]).astype(int), 0, cam.height - 1)
    inimg = ((pix[:, 0] >= -0.5) & (pix[:, 0] <= cam.width - 0.5)
             & (pix[:, 1] >= -0.5) & (pix[:, 1] <= cam.height - 0.5))
    z = verts[:, 2]
    return ok & inimg & (z <= zbuf[yi, xi] + 0.01 * z)


def part_label_mask(verts, mesh, skin_w, sk, cam, dilation=10):
    """(labels (H,W), vertex_parts (N,))  (nonrigid_stage.py:102-128)."""
    vparts = joint_body_parts(sk)[skin_w.dominant]
    ibuf, _ = render_vertex_ids(cam, verts, mesh.triangles, vparts, background=0)
    out = ibuf.copy()
    bg = ibuf == 0
    present = [p for p in np.unique(ibuf) if p > 0]
    if present:
        d = np.stack([np.sqrt(edt_squared(ibuf == p)) for p in present])
        near = np.argmin(d, axis=0)
        grow = bg & (d.min(axis=0) <= dilation)
        out[grow] = np.array(present)[near[grow]]
        if TORSO_PART in present:
            out[bg & (d[present.index(TORSO_PART)] <= dilation)] = TORSO_PART
    return out, vparts


@dataclass
class SurfaceProblem:
    mesh: object
    camera: object
    hyper: object
    skinned: np.ndarray
    pyramid: list
    field: DistanceField | None
    visible: np.ndarray
    boundary_idx: np.ndarray
    normals2d: np.ndarray
    enabled: np.ndarray
    prev: np.ndarray | None = None
    prev2: np.ndarray | None = None
    directional: bool = True
    enable_photo: bool = True
    enable_sil: bool = True

    def __post_init__(self):
        m = self.mesh
        e = len(m.edges)
        rl = m.rest_edge_lengths()
        self.dir_rest = np.concatenate([rl, rl])
        self.rev = np.concatenate([np.arange(e, 2 * e), np.arange(0, e)])
        deg = m.degrees[m.edge_src].astype(np.float64)
        self.c_smooth = np.sqrt(self.hyper.w_smooth * m.directed_weights / deg)
        self.c_edge = np.sqrt(self.hyper.w_edge * m.directed_weights / deg)
        self.skinned_diff = self.skinned[m.edge_src] - self.skinned[m.edge_dst]


def surface_evaluate(pb: SurfaceProblem, v, level):
    """Residual blocks (nonrigid_stage.py:189-268).  Returns a dict."""
    m, hp, cam = pb.mesh, pb.hyper, pb.camera
    en = {}
    behind = 0
    P = len(pb.visible)
    pr, pj, pruned = np.zeros((P, 3)), np.zeros((P, 3, 3)), 0
    if P and pb.enable_photo:
        pos = v[pb.visible]
        pix, ok = project(cam, pos)
        behind += int(np.sum(~ok))
        val, grad, cl = sample_bilinear(pb.pyramid[level], pix)
        diff = val - m.vertex_colors[pb.visible]
        prune = np.linalg.norm(diff, axis=1) > hp.tau_color
        pruned = int(np.sum(prune & ok & ~cl))
        w = np.sqrt(hp.w_photo) * (ok & ~cl & ~prune)
        pr = diff * w[:, None]
        dpi, _ = projection_jac(cam, pos)
        pj = np.einsum("pcd,pdk->pck", grad, dpi) * w[:, None, None]
    en["photo"] = float(np.sum(pr ** 2))

    B = len(pb.boundary_idx)
    sr, sg = np.zeros(B), np.zeros((B, 3))
    if B and pb.enable_sil and pb.field is not None:
        pos = v[pb.boundary_idx]
        pix, ok = project(cam, pos)
        behind += int(np.sum(~ok))
        val, grad, cl = pb.field.sample_residual(pix)
        w = np.sqrt(hp.w_sil) * (ok & ~cl & pb.enabled)
        sr = val * w
        sign = side_signs(pb.field, pb.normals2d, pix) if pb.directional else 1.0
        dpi, _ = projection_jac(cam, pos)
        sg = np.einsum("bd,bdk->bk", grad, dpi) * (w * sign)[:, None]
    en["silhouette"] = float(np.sum(sr ** 2))

    ev = v[m.edge_src] - v[m.edge_dst]
    smooth_r = (ev - pb.skinned_diff) * pb.c_smooth[:, None]
    en["smooth"] = float(np.sum(smooth_r ** 2))
    ln = np.linalg.norm(ev, axis=1)
    deg = ln < 1e-9
    rd = m.rest_vertices[m.edge_src] - m.rest_vertices[m.edge_dst]
    edir = np.where(deg[:, None], rd / np.linalg.norm(rd, axis=1)[:, None],
                    ev / np.maximum(ln, 1e-300)[:, None])
    edge_r = (ln - pb.dir_rest) * pb.c_edge
    en["edge"] = float(np.sum(edge_r ** 2))

    vel_r = acc_r = None
    cv, ca = np.sqrt(hp.w_velocity), np.sqrt(hp.w_acceleration)
    if pb.prev is not None:
        vel_r = (v - pb.prev) * cv
        en["velocity"] = float(np.sum(vel_r ** 2))
        p2 = pb.prev if pb.prev2 is None else pb.prev2
        acc_r = (v - 2.0 * pb.prev + p2) * ca
        en["acceleration"] = float(np.sum(acc_r ** 2))
    return dict(photo_r=pr, photo_j=pj, sil_r=sr, sil_g=sg, smooth_r=smooth_r,
                edge_r=edge_r, edge_dir=edir, vel_r=vel_r, acc_r=acc_r, cv=cv, ca=ca,
                energies=en, energy=float(sum(en.values())), pruned=pruned,
                degenerate=int(np.sum(deg)), behind=behind)


def normal_system(pb: SurfaceProblem, ev):
    """Explicit block system (diag, off, rows, cols, rhs)  (nonrigid_stage.py:270-304)."""
    m = pb.mesh
    n = m.n_vertices
    diag = np.zeros((n, 3, 3))
    rhs = np.zeros((n, 3))
    if len(pb.visible):
        np.add.at(diag, pb.visible, np.einsum("pci,pcj->pij", ev["photo_j"], ev["photo_j"]))
        np.add.at(rhs, pb.visible, -np.einsum("pci,pc->pi", ev["photo_j"], ev["photo_r"]))
    if len(pb.boundary_idx):
        np.add.at(diag, pb.boundary_idx, np.einsum("bi,bj->bij", ev["sil_g"], ev["sil_g"]))
        np.add.at(rhs, pb.boundary_idx, -ev["sil_g"] * ev["sil_r"][:, None])
    src, dst = m.edge_src, m.edge_dst
    s2, e2 = pb.c_smooth ** 2, pb.c_edge ** 2
    I = np.eye(3)
    dd = np.einsum("mi,mj->mij", ev["edge_dir"], ev["edge_dir"])
    blk = s2[:, None, None] * I + e2[:, None, None] * dd
    np.add.at(diag, src, blk)
    np.add.at(diag, dst, blk)
    off = -((s2 + s2[pb.rev])[:, None, None] * I
            + (e2[:, None, None] * dd + e2[pb.rev][:, None, None] * dd[pb.rev]))
    js = pb.c_smooth[:, None] * ev["smooth_r"]
    je = ev["edge_dir"] * (pb.c_edge * ev["edge_r"])[:, None]
    np.add.at(rhs, src, -(js + je))
    np.add.at(rhs, dst, js + je)
    if ev["vel_r"] is not None:
        diag += (ev["cv"] ** 2 + ev["ca"] ** 2) * I
        rhs -= ev["cv"] * ev["vel_r"] + ev["ca"] * ev["acc_r"]
    return diag, off, src, dst, rhs


def solve_surface(pb: SurfaceProblem, v0):
    """Coarse-to-fine halving GN (nonrigid_stage.py:372-403).
    Returns (v, logs, totals) with logs as dicts."""
    hp = pb.hyper
    v = np.array(v0, dtype=np.float64, copy=True)
    logs = []
    tot = dict(pruned=0, degenerate_edges=0, behind_camera=0)
    top = min(hp.gn_iterations, len(pb.pyramid))
    for it in range(hp.gn_iterations):
        level = min(it, top - 1)
        ev = surface_evaluate(pb, v, level)
        tot["pruned"] += ev["pruned"]
        tot["degenerate_edges"] += ev["degenerate"]
        tot["behind_camera"] += ev["behind"]
        delta, _, breakdown, _ = pcg(*normal_system(pb, ev), hp.pcg_iterations)
        e0 = ev["energy"]
        halv, rej, step = 0, False, delta
        while True:
            e1 = surface_evaluate(pb, v + step, level)["energy"]
            if e1 <= e0:
                v = v + step
                break
            if halv >= hp.max_halvings:
                rej, e1 = True, e0
                break
            step = 0.5 * step
            halv += 1
        logs.append(dict(level=level, energy_before=e0, energy_after=e1,
                         terms=ev["energies"], halvings=halv, rejected=rej,
                         pcg_breakdown=breakdown))
    return v, logs, tot


def snap(v, pb: SurfaceProblem):
    """Boundary walk onto the interface + 2 Laplacian diffusion steps
    (nonrigid_stage.py:417-500).  Returns (v_out, info dict)."""
    hp, f, cam, idx = pb.hyper, pb.field, pb.camera, pb.boundary_idx
    info = dict(walked=0, reached=0, stuck=0, moved_vertices=None)
    if f is None or len(idx) == 0:
        return v.copy(), info
    pix, ok = project(cam, v[idx])
    en = pb.enabled & ok
    sign = side_signs(f, pb.normals2d, pix)
    val, _ = f.sample_interface(pix)
    pos = pix.copy()
    active = en & (val > hp.snap_band)
    info["walked"] = int(np.sum(en))
    stuck = np.zeros(len(idx), dtype=bool)
    for _ in range(hp.snap_max_steps):
        if not active.any():
            break
        ai = np.flatnonzero(active)
        g, _ = f.sample_gradient(pos[ai])
        gn = np.linalg.norm(g, axis=1)
        good = gn > 1e-9
        dirn = -sign[ai, None] * g / np.maximum(gn, 1e-300)[:, None]
        step = hp.snap_step
        cur = val[ai]
        npos, nval = pos[ai].copy(), cur.copy()
        pending = good.copy()
        for _ in range(3):
            if not pending.any():
                break
            trial = pos[ai] + step * dirn
            tv, _ = f.sample_interface(trial)
            better = pending & (tv < cur)
            npos[better] = trial[better]
            nval[better] = tv[better]
            pending &= ~better
            step *= 0.5
        moved = ~pending & good
        pos[ai[moved]] = npos[moved]
        val[ai[moved]] = nval[moved]
        bad = ai[pending | ~good]
        stuck[bad] = True
        active[bad] = False
        active[ai] &= val[ai] > hp.snap_band
    info["reached"] = int(np.sum(en & (val <= hp.snap_band)))
    info["stuck"] = int(np.sum(stuck & en))
    out = v.copy()
    off = np.zeros_like(v)
    sn = np.flatnonzero(en)
    z = v[idx[sn], 2]
    landed = np.stack([(pos[sn, 0] - cam.cx) * z / cam.fx,
                       (pos[sn, 1] - cam.cy) * z / cam.fy, z], axis=1)
    off[idx[sn]] = landed - v[idx[sn]]
    m = pb.mesh
    hold = np.zeros(len(v), dtype=bool)
    hold[idx] = True
    o = off
    for _ in range(2):
        acc = np.zeros_like(o)
        np.add.at(acc, m.edge_src, o[m.edge_dst])
        acc /= m.degrees[:, None]
        o = np.where(hold[:, None], o, acc)
    out += o
    info["moved_vertices"] = np.flatnonzero(np.any(o != 0.0, axis=1))
    return out, info


def compact_operator(pb: SurfaceProblem, ev):
    """The same normal system in compact form: per-vertex symmetric data block
    + (c_v^2 + c_a^2) I, and per undirected edge (alpha, beta, d) with
    A_ij = -(alpha I + beta d d^T).  For tests only."""
    m = pb.mesh
    e = len(m.edges)
    n = m.n_vertices
    s2, e2 = pb.c_smooth ** 2, pb.c_edge ** 2
    alpha = s2[:e] + s2[e:]
    beta = e2[:e] + e2[e:]
    d = ev["edge_dir"][:e]
    # the reverse edge's direction is exactly -d (or the negated rest
    # direction when degenerate), so d d^T is shared by both halves
    data = np.zeros((n, 3, 3))
    np.add.at(data, pb.visible, np.einsum("pci,pcj->pij", ev["photo_j"], ev["photo_j"]))
    np.add.at(data, pb.boundary_idx, np.einsum("bi,bj->bij", ev["sil_g"], ev["sil_g"]))
    return data, alpha, beta, d
