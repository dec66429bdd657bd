"""Actor data layout: template mesh, skeleton, skinning weights, material classes.

Host-side containers only (no per-frame compute happens here).  Field names
and derived connectivity follow the reference's `montrack.template`
(`pkg/src/montrack/template.py:68-256`) so reference actors can be passed in
unchanged; `Actor.from_reference` adapts a `montrack.template.Actor`.

Derived connectivity is what the device tables are built from
(`paper_1810_02648_b200/device.py`):

* ``edges``          (E,2) undirected, i<j, lexicographically sorted
                     (reference `template.py:100-103`, `np.unique(axis=0)`)
* ``edge_src/dst``   (2E,) forward half then reversed half (`:104-105`)
* ``degrees``        out-degree per vertex in the directed list (`:106`)
* ``edge_tris``      (E,2) incident triangles in (triangle, local-edge) order,
                     -1 for an open boundary (`:116-123`)
* ``directed_weights`` s_ij = mean of the endpoint class weights (`:126-129`)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Table 1 of the paper: non-rigidity class -> rigidity weight
# (reference `template.py:24-32`).
MATERIAL_CLASS_WEIGHTS = {1: 1.0, 2: 2.0, 3: 2.5, 4: 3.0, 5: 50.0, 6: 100.0, 7: 200.0}


def class_weight(class_id: int) -> float:
    if int(class_id) not in MATERIAL_CLASS_WEIGHTS:
        raise ValueError(f"unknown non-rigidity class {class_id}")
    return MATERIAL_CLASS_WEIGHTS[int(class_id)]


def _class_weight_array(labels: np.ndarray) -> np.ndarray:
    lut = np.zeros(8)
    for k, w in MATERIAL_CLASS_WEIGHTS.items():
        lut[k] = w
    return lut[labels]


@dataclass
class TemplateMesh:
    rest_vertices: np.ndarray   # (N,3) f64
    triangles: np.ndarray       # (T,3) i64
    vertex_colors: np.ndarray   # (N,3) f64 in [0,1]
    vertex_labels: np.ndarray   # (N,) material class ids 1..7

    edges: np.ndarray = field(init=False)
    edge_src: np.ndarray = field(init=False)
    edge_dst: np.ndarray = field(init=False)
    degrees: np.ndarray = field(init=False)
    edge_tris: np.ndarray = field(init=False)
    edge_weights: np.ndarray = field(init=False)
    directed_weights: np.ndarray = field(init=False)

    def __post_init__(self):
        verts = np.asarray(self.rest_vertices, dtype=np.float64)
        tris = np.asarray(self.triangles, dtype=np.int64)
        n = verts.shape[0]
        if tris.size and (tris.min() < 0 or tris.max() >= n):
            raise ValueError("triangle index out of range")
        labels = np.asarray(self.vertex_labels, dtype=np.int64)
        bad = ~np.isin(labels, list(MATERIAL_CLASS_WEIGHTS))
        if bad.any():
            k = int(np.argmax(bad))
            raise ValueError(f"vertex {k} has invalid class {int(labels[k])}")
        self.rest_vertices = verts
        self.triangles = tris
        self.vertex_colors = np.asarray(self.vertex_colors, dtype=np.float64)
        self.vertex_labels = labels

        # undirected edge list: every triangle side, endpoints ordered, unique
        sides = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
        sides.sort(axis=1)
        edges = np.unique(sides, axis=0)
        self.edges = edges
        self.edge_src = np.concatenate([edges[:, 0], edges[:, 1]])
        self.edge_dst = np.concatenate([edges[:, 1], edges[:, 0]])
        self.degrees = np.bincount(self.edge_src, minlength=n)
        if (self.degrees < 2).any():
            raise ValueError(f"vertex {int(np.argmin(self.degrees))} has fewer than 2 neighbors")

        # incident triangles per edge, filled in (triangle, local side) order
        e_of_side = np.searchsorted(edges[:, 0] * n + edges[:, 1],
                                    sides[:, 0] * n + sides[:, 1])
        t_count = len(tris)
        side_tri = np.tile(np.arange(t_count), 3)
        side_local = np.repeat(np.arange(3), t_count)
        order = np.lexsort((side_local, side_tri))   # triangle-major, then side
        self.edge_tris = np.full((len(edges), 2), -1, dtype=np.int64)
        for s in order:
            e = e_of_side[s]
            slot = 0 if self.edge_tris[e, 0] < 0 else 1
            self.edge_tris[e, slot] = side_tri[s]
        self.refresh_edge_weights()

    def refresh_edge_weights(self):
        w = _class_weight_array(self.vertex_labels)
        self.edge_weights = 0.5 * (w[self.edges[:, 0]] + w[self.edges[:, 1]])
        self.directed_weights = np.concatenate([self.edge_weights, self.edge_weights])

    @property
    def n_vertices(self) -> int:
        return self.rest_vertices.shape[0]

    def rest_edge_lengths(self) -> np.ndarray:
        d = self.rest_vertices[self.edges[:, 0]] - self.rest_vertices[self.edges[:, 1]]
        return np.linalg.norm(d, axis=1)


@dataclass
class Skeleton:
    joint_names: list
    parents: np.ndarray        # (J,) root has -1, parents precede children
    local_offsets: np.ndarray  # (J,3)
    dof_joint: np.ndarray      # (27,)
    dof_axes: np.ndarray       # (27,3), normalised on construction
    theta_min: np.ndarray      # (27,)
    theta_max: np.ndarray      # (27,)
    marker_names: list
    marker_offsets: np.ndarray  # (4,3) in the head frame
    temporal_groups: list       # (J,)

    def __post_init__(self):
        self.parents = np.asarray(self.parents, dtype=np.int64)
        self.local_offsets = np.asarray(self.local_offsets, dtype=np.float64)
        self.dof_joint = np.asarray(self.dof_joint, dtype=np.int64)
        self.dof_axes = np.asarray(self.dof_axes, dtype=np.float64)
        self.theta_min = np.asarray(self.theta_min, dtype=np.float64)
        self.theta_max = np.asarray(self.theta_max, dtype=np.float64)
        self.marker_offsets = np.asarray(self.marker_offsets, dtype=np.float64)
        j = len(self.joint_names)
        if self.parents[0] != -1 or (self.parents[1:] < 0).any():
            raise ValueError("joint 0 must be the single root")
        if (self.parents[1:] >= np.arange(1, j)).any():
            raise ValueError("parents must precede children")
        if self.dof_joint.shape[0] != 27:
            raise ValueError(f"skeleton must expose 27 joint angles, got {self.dof_joint.shape[0]}")
        if (self.theta_min >= self.theta_max).any():
            raise ValueError("joint limits must satisfy min < max")
        lens = np.linalg.norm(self.dof_axes, axis=1)
        if (lens < 1e-9).any():
            raise ValueError("zero-length rotation axis")
        self.dof_axes = self.dof_axes / lens[:, None]
        if self.marker_offsets.shape != (4, 3):
            raise ValueError("exactly 4 face markers required")
        if "head" not in self.joint_names:
            raise ValueError("skeleton needs a joint named 'head' for face markers")
        self.head_index = self.joint_names.index("head")
        self.n_joints = j
        self.children = [[] for _ in range(j)]
        for c in range(1, j):
            self.children[self.parents[c]].append(c)
        anc = np.zeros((j, j), dtype=bool)          # anc[a, i]: a is i or above i
        for i in range(j):
            k = i
            while k != -1:
                anc[k, i] = True
                k = self.parents[k]
        self.ancestor_of = anc
        dj = self.dof_joint
        self.dof_moves_frame = anc[dj]
        self.dof_moves_position = anc[dj] & (np.arange(j)[None, :] != dj[:, None])

    @property
    def n_dofs(self) -> int:
        return self.dof_joint.shape[0]

    def bone_lengths(self) -> np.ndarray:
        return np.linalg.norm(self.local_offsets, axis=1)

    def rest_positions(self) -> np.ndarray:
        out = np.zeros((self.n_joints, 3))
        for i in range(self.n_joints):
            p = self.parents[i]
            out[i] = self.local_offsets[i] + (out[p] if p >= 0 else 0.0)
        return out

    def clamp_theta(self, theta: np.ndarray) -> np.ndarray:
        return np.clip(theta, self.theta_min, self.theta_max)


@dataclass
class SkinningWeights:
    indices: np.ndarray  # (N,4) joint ids, -1 padding
    weights: np.ndarray  # (N,4) rows sum to one

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.int64)
        self.weights = np.asarray(self.weights, dtype=np.float64)
        if self.indices.shape != self.weights.shape or self.indices.shape[1] != 4:
            raise ValueError("skinning arrays must be (N,4)")
        if (self.weights < -1e-12).any():
            raise ValueError("negative skinning weight")
        sums = self.weights.sum(axis=1)
        off = np.abs(sums - 1.0) > 1e-6
        if off.any():
            i = int(np.argmax(off))
            raise ValueError(f"skinning weights of vertex {i} sum to {sums[i]:.6f}, expected 1")
        if ((self.indices < 0) & (self.weights > 0)).any():
            raise ValueError("positive weight on padding slot")
        # first maximum wins (reference `template.py:242-243`)
        self.dominant = self.indices[np.arange(len(self.indices)),
                                     np.argmax(self.weights, axis=1)]


@dataclass
class Actor:
    mesh: TemplateMesh
    skeleton: Skeleton
    skinning: SkinningWeights

    def __post_init__(self):
        if (self.skinning.indices >= self.skeleton.n_joints).any():
            raise ValueError("skinning references a joint outside the skeleton")
        if self.skinning.indices.shape[0] != self.mesh.n_vertices:
            raise ValueError("skinning rows do not match mesh vertex count")

    @classmethod
    def from_reference(cls, ref_actor) -> "Actor":
        """Adapt a `montrack.template.Actor` (any object with the same fields)."""
        if isinstance(ref_actor, cls):
            return ref_actor
        m, s, w = ref_actor.mesh, ref_actor.skeleton, ref_actor.skinning
        mesh = TemplateMesh(m.rest_vertices, m.triangles, m.vertex_colors, m.vertex_labels)
        # keep caller-overridden material weights (uniform_material_weight)
        mesh.edge_weights = np.asarray(m.edge_weights, dtype=np.float64)
        mesh.directed_weights = np.asarray(m.directed_weights, dtype=np.float64)
        sk = Skeleton(list(s.joint_names), s.parents, s.local_offsets, s.dof_joint,
                      s.dof_axes, s.theta_min, s.theta_max, list(s.marker_names),
                      s.marker_offsets, list(s.temporal_groups))
        return cls(mesh, sk, SkinningWeights(w.indices, w.weights))


# ---------------------------------------------------------------------------
# body parts (reference `nonrigid_stage.py:55-84`): torso 1, head 2, limbs 3..

TORSO_PART = 1
HEAD_PART = 2


def joint_body_parts(skeleton: Skeleton) -> np.ndarray:
    j = skeleton.n_joints
    part = np.full(j, TORSO_PART, dtype=np.int64)

    def paint(root, pid):
        todo = [root]
        while todo:
            k = todo.pop()
            part[k] = pid
            todo.extend(skeleton.children[k])

    head = skeleton.head_index
    paint(head, HEAD_PART)
    nxt = HEAD_PART + 1
    on_head_chain = skeleton.ancestor_of[:, head]
    for i in range(j):
        if skeleton.parents[i] < 0 or part[i] != TORSO_PART:
            continue
        if not on_head_chain[i] and skeleton.temporal_groups[i] == "shoulder":
            paint(i, nxt)
            nxt += 1
    for i in range(j):
        if part[i] == TORSO_PART and skeleton.temporal_groups[i] == "knee":
            up = skeleton.parents[i]
            paint(up if part[up] == TORSO_PART else i, nxt)
            nxt += 1
    return part
