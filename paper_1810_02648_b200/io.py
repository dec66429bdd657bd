"""On-disk formats of the reference (§8f: real-data ingest and result output).

Restates the reference readers / writers so a capture directory written by
the reference (or its synthetic generator) feeds the device tracker, and
results are written in the reference's layout:

* mesh: OBJ (`v` / `f` rows, 1-based) + `<obj>.attrs` sidecar of `r g b class`
  rows (template.py:262-291);
* skeleton: `joint` / `dof` / `marker` rows (template.py:293-340);
* skinning: `<vertex> <joint name> <weight>` rows, <= 4 per vertex (:342-366);
* calibration: one line `fx fy cx cy width height` (camera.py:94-106);
* detections: JSONL with joints2d / joints3d / valid2d / valid3d (pose_stage.py:67-89);
* pose trajectories: one 36-vector per line, `%.12g` (skinning.py:68-79);
* frames: `frames/frame_%04d_color.png` (RGB / 255) and `_mask.png` (gray >= 128)
  (imageproc.py:288-304);
* results: poses.txt, poses_smoothed.txt, surfaces.npz, report.json (pipeline.py:518-546).

The reference's sequence reader looks for `actor_template.obj`,
`actor_skeleton.txt` and `actor_skinning.txt` while its writer produces
`actor.obj`, `actor.skel` and `actor.skin`; `load_sequence_inputs`
accepts either set.  Colour frames can be kept as uint8 (`as_uint8=True`):
the tracker then uploads 1 byte per channel and converts on the device with
the reference's exact `/ 255.0`.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .actor import Actor, Skeleton, SkinningWeights, TemplateMesh
from .camera import CameraIntrinsics
from .config import FrameDetections, PoseParams


def _rows(path):
    for line in Path(path).read_text().splitlines():
        parts = line.split()
        if parts and not parts[0].startswith("#"):
            yield parts


# ---- mesh / skeleton / skinning ----------------------------------------------------

def load_mesh(path) -> TemplateMesh:
    path = Path(path)
    verts, tris = [], []
    for parts in _rows(path):
        if parts[0] == "v":
            verts.append([float(x) for x in parts[1:4]])
        elif parts[0] == "f":
            tris.append([int(tok.split("/")[0]) - 1 for tok in parts[1:4]])
    side = path.with_suffix(path.suffix + ".attrs")
    if not side.exists():
        raise FileNotFoundError(f"missing vertex attribute sidecar {side}")
    attrs = np.loadtxt(side, ndmin=2)
    if attrs.shape != (len(verts), 4):
        raise ValueError(f"sidecar {side} must hold {len(verts)} 'r g b class' rows")
    return TemplateMesh(np.array(verts), np.array(tris, dtype=np.int64), attrs[:, :3],
                        attrs[:, 3].astype(np.int64))


def save_mesh(path, mesh: TemplateMesh) -> None:
    path = Path(path)
    out = [f"v {x:.9g} {y:.9g} {z:.9g}" for x, y, z in mesh.rest_vertices]
    out += [f"f {a + 1} {b + 1} {c + 1}" for a, b, c in mesh.triangles]
    path.write_text("\n".join(out) + "\n")
    np.savetxt(path.with_suffix(path.suffix + ".attrs"),
               np.column_stack([mesh.vertex_colors, mesh.vertex_labels]), fmt="%.9g %.9g %.9g %d")


def load_skeleton(path) -> Skeleton:
    names, parents, offsets, groups = [], [], [], []
    dof_joint, dof_axes, tmin, tmax, mnames, moffs = [], [], [], [], [], []
    for parts in _rows(path):
        kind = parts[0]
        if kind == "joint":
            names.append(parts[1])
            parents.append(-1 if parts[2] == "-" else names.index(parts[2]))
            offsets.append([float(v) for v in parts[3:6]])
            groups.append(parts[6])
        elif kind == "dof":
            dof_joint.append(names.index(parts[1]))
            dof_axes.append([float(v) for v in parts[2:5]])
            tmin.append(float(parts[5]))
            tmax.append(float(parts[6]))
        elif kind == "marker":
            mnames.append(parts[1])
            moffs.append([float(v) for v in parts[2:5]])
        else:
            raise ValueError(f"unknown skeleton row kind '{kind}'")
    return Skeleton(names, np.array(parents), np.array(offsets), np.array(dof_joint), np.array(dof_axes),
                    np.array(tmin), np.array(tmax), mnames, np.array(moffs), groups)


def save_skeleton(path, sk: Skeleton) -> None:
    out = ["# joint <name> <parent|-> <ox> <oy> <oz> <temporal_group>",
           "# dof rows define the joint-angle order; detections follow joint order then marker order"]
    for i, name in enumerate(sk.joint_names):
        parent = "-" if sk.parents[i] < 0 else sk.joint_names[sk.parents[i]]
        o = sk.local_offsets[i]
        out.append(f"joint {name} {parent} {o[0]:.9g} {o[1]:.9g} {o[2]:.9g} {sk.temporal_groups[i]}")
    for k in range(len(sk.dof_joint)):
        a = sk.dof_axes[k]
        out.append(f"dof {sk.joint_names[sk.dof_joint[k]]} {a[0]:.9g} {a[1]:.9g} {a[2]:.9g} "
                   f"{sk.theta_min[k]:.9g} {sk.theta_max[k]:.9g}")
    for name, o in zip(sk.marker_names, sk.marker_offsets):
        out.append(f"marker {name} {o[0]:.9g} {o[1]:.9g} {o[2]:.9g}")
    Path(path).write_text("\n".join(out) + "\n")


def load_skinning(path, skeleton: Skeleton, n_vertices: int) -> SkinningWeights:
    idx = np.full((n_vertices, 4), -1, dtype=np.int64)
    w = np.zeros((n_vertices, 4))
    cnt = np.zeros(n_vertices, dtype=np.int64)
    for parts in _rows(path):
        v, j = int(parts[0]), skeleton.joint_names.index(parts[1])
        if cnt[v] >= 4:
            raise ValueError(f"vertex {v} has more than 4 skinning influences")
        idx[v, cnt[v]] = j
        w[v, cnt[v]] = float(parts[2])
        cnt[v] += 1
    return SkinningWeights(idx, w)


def save_skinning(path, sk: SkinningWeights, skeleton: Skeleton) -> None:
    out = [f"{v} {skeleton.joint_names[j]} {w:.9g}"
           for v in range(sk.indices.shape[0]) for j, w in zip(sk.indices[v], sk.weights[v]) if j >= 0 and w > 0]
    Path(path).write_text("\n".join(out) + "\n")


def load_actor(template_file, skeleton_file, skinning_file) -> Actor:
    mesh = load_mesh(template_file)
    sk = load_skeleton(skeleton_file)
    return Actor(mesh, sk, load_skinning(skinning_file, sk, mesh.n_vertices))


def save_actor(directory, actor: Actor, stem: str = "actor"):
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    paths = d / f"{stem}.obj", d / f"{stem}.skel", d / f"{stem}.skin"
    save_mesh(paths[0], actor.mesh)
    save_skeleton(paths[1], actor.skeleton)
    save_skinning(paths[2], actor.skinning, actor.skeleton)
    return paths


# ---- camera / detections / poses -------------------------------------------------------

def load_calibration(path) -> CameraIntrinsics:
    f = Path(path).read_text().split()
    if len(f) != 6:
        raise ValueError(f"calibration file {path} must hold 6 values, got {len(f)}")
    return CameraIntrinsics(float(f[0]), float(f[1]), float(f[2]), float(f[3]), int(f[4]), int(f[5]))


def save_calibration(path, cam) -> None:
    Path(path).write_text(f"{cam.fx} {cam.fy} {cam.cx} {cam.cy} {cam.width} {cam.height}\n")


def load_detections(path) -> list:
    out = []
    for line in Path(path).read_text().splitlines():
        if line.strip():
            r = json.loads(line)
            out.append(FrameDetections(np.array(r["joints2d"]), np.array(r["joints3d"]),
                                       np.array(r["valid2d"]), np.array(r["valid3d"])))
    return out


def save_detections(path, detections) -> None:
    out = [json.dumps({"frame": i, "joints2d": d.joints2d.tolist(), "joints3d": d.joints3d.tolist(),
                       "valid2d": np.asarray(d.valid2d).astype(int).tolist(),
                       "valid3d": np.asarray(d.valid3d).astype(int).tolist()})
           for i, d in enumerate(detections)]
    Path(path).write_text("\n".join(out) + "\n")


def load_pose_trajectory(path) -> list:
    return [PoseParams.from_vector(np.array([float(v) for v in line.split()]))
            for line in Path(path).read_text().splitlines() if line.strip()]


def save_pose_trajectory(path, poses) -> None:
    vecs = [p.to_vector() if hasattr(p, "to_vector") else np.asarray(p) for p in poses]
    Path(path).write_text("\n".join(" ".join(f"{v:.12g}" for v in x) for x in vecs) + "\n")


# ---- frames ------------------------------------------------------------------------------

def load_mask(path) -> np.ndarray:
    from PIL import Image
    return np.asarray(Image.open(path).convert("L")) >= 128


def save_mask(path, mask) -> None:
    from PIL import Image
    Image.fromarray(np.where(mask, 255, 0).astype(np.uint8), mode="L").save(path)


def load_color(path, as_uint8: bool = False) -> np.ndarray:
    """RGB / 255 in float64 (imageproc.py:297-299); `as_uint8` keeps the raw
    bytes for the tracker's uint8 upload path (same values after its / 255)."""
    from PIL import Image
    img = np.asarray(Image.open(path).convert("RGB"))
    return np.ascontiguousarray(img) if as_uint8 else img.astype(np.float64) / 255.0


def save_color(path, image) -> None:
    from PIL import Image
    img = np.clip(np.asarray(image) * 255.0 + 0.5, 0, 255).astype(np.uint8)
    Image.fromarray(img, mode="RGB").save(path)


# ---- sequences ---------------------------------------------------------------------------

def _actor_files(d: Path):
    for names in (("actor_template.obj", "actor_skeleton.txt", "actor_skinning.txt"),
                  ("actor.obj", "actor.skel", "actor.skin")):
        paths = [d / n for n in names]
        if all(p.exists() for p in paths):
            return paths
    raise FileNotFoundError(f"no actor files in {d} (actor_template.obj/... or actor.obj/...)")


def load_sequence_inputs(seq_dir, as_uint8: bool = False):
    """Reference pipeline.py:102-113 (either actor file naming, see F9)."""
    from .pipeline import SequenceInputs
    d = Path(seq_dir)
    actor = load_actor(*_actor_files(d))
    camera = load_calibration(d / "camera.txt")
    dets = load_detections(d / "detections.jsonl")
    images = [load_color(d / "frames" / f"frame_{f:04d}_color.png", as_uint8) for f in range(len(dets))]
    masks = [load_mask(d / "frames" / f"frame_{f:04d}_mask.png") for f in range(len(dets))]
    return SequenceInputs(actor, camera, images, masks, dets)


def save_sequence(out_dir, actor, camera, images, masks, detections, poses=None) -> None:
    """The generator's directory layout (synthetic.py:206-222, frames + inputs)."""
    out = Path(out_dir)
    (out / "frames").mkdir(parents=True, exist_ok=True)
    save_actor(out, actor, "actor")
    save_calibration(out / "camera.txt", camera)
    save_detections(out / "detections.jsonl", detections)
    if poses is not None:
        save_pose_trajectory(out / "poses_gt.txt", poses)
    for f, (img, m) in enumerate(zip(images, masks)):
        save_color(out / "frames" / f"frame_{f:04d}_color.png", img)
        save_mask(out / "frames" / f"frame_{f:04d}_mask.png", m)


def _jsonable(x):
    if isinstance(x, dict):
        return {k: _jsonable(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [_jsonable(v) for v in x]
    if isinstance(x, np.ndarray):
        return x.tolist()
    if isinstance(x, np.generic):
        return x.item()
    return x


def save_results(out_dir, result, inputs=None) -> None:
    """Reference pipeline.py:518-546."""
    from .pipeline import frame_latencies
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    save_pose_trajectory(out / "poses.txt", list(result.poses))
    save_pose_trajectory(out / "poses_smoothed.txt", list(result.poses_smoothed))
    np.savez_compressed(out / "surfaces.npz", vertices=result.vertices, vertices_smoothed=result.vertices_smoothed)
    rep = {
        "n_frames": len(result.frames),
        "pipelined": result.pipelined,
        "fps": result.fps,
        "timings": result.timings,
        "events": result.events,
        "latencies": frame_latencies(result.events),
        "config": _jsonable(result.config.to_dict()),
        "frames": [{
            "index": r.index,
            "pose_energy": r.pose_report.final_energy,
            "pose_iterations": len(r.pose_report.iterations),
            "nonrigid_energy": (r.nonrigid_report.iterations[-1].energy_after
                                if r.nonrigid_report and r.nonrigid_report.iterations else None),
            "timings": r.timings,
        } for r in result.frames],
    }
    (out / "report.json").write_text(json.dumps(rep, indent=2) + "\n")
