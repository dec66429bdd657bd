"""Device-resident actor tables, config conversion and the batched tracker.

`DeviceActor` uploads an actor once (reference layout, template.py:68-256);
`Tracker` runs `solve_frame` (pipeline.py:263-302) for S independent capture
streams per call, entirely on the GPU: preprocessing (pyramid, observed
contour grid), detection conditioning, Stage I rounds, Stage II setup, solve,
snapping and the TrackState update.  Only frame inputs go in and results come
out; state stays resident in HBM between frames.
"""

from __future__ import annotations

import ctypes as C
import sys

import numpy as np

from . import _lib as L
from .actor import Actor, joint_body_parts
from .config import (FrameDetections, NonrigidHyperparams, NonrigidIterationLog,
                     NonrigidStageReport, PoseHyperparams, PoseIterationLog, PoseParams,
                     PoseStageReport, SequenceConfig, SnapInfo, TEMPORAL_GROUP_WEIGHTS, MODES)

GROUP_NAMES = list(TEMPORAL_GROUP_WEIGHTS)


def _group_ids(skeleton) -> np.ndarray:
    ids = []
    for g in skeleton.temporal_groups:
        if g not in GROUP_NAMES:
            if len(GROUP_NAMES) >= 8:
                raise ValueError("at most 8 temporal groups are supported")
            GROUP_NAMES.append(g)
        ids.append(GROUP_NAMES.index(g))
    return np.asarray(ids, dtype=np.int32)


def pose_hyper_c(hp) -> L.PoseHyper:
    h = L.PoseHyper()
    h.lambda_2d, h.lambda_3d, h.lambda_sil = hp.lambda_2d, hp.lambda_3d, hp.lambda_sil
    h.lambda_temporal, h.lambda_anatomic, h.face_weight = (hp.lambda_temporal, hp.lambda_anatomic,
                                                           hp.face_weight)
    for name, w in hp.temporal_group_weights.items():
        if name not in GROUP_NAMES:
            if len(GROUP_NAMES) >= 8:
                raise ValueError("at most 8 temporal groups are supported")
            GROUP_NAMES.append(name)
        h.group_weights[GROUP_NAMES.index(name)] = float(w)
    h.gn_iterations, h.max_halvings = int(hp.gn_iterations), int(hp.max_halvings)
    if h.gn_iterations > L.LC_MAX_LOG:
        raise ValueError(f"at most {L.LC_MAX_LOG} Gauss-Newton iterations per solve")
    return h


def nonrigid_hyper_c(hp, n_levels=None) -> L.NonrigidHyper:
    h = L.NonrigidHyper()
    h.w_photo, h.w_sil, h.w_smooth, h.w_edge = hp.w_photo, hp.w_sil, hp.w_smooth, hp.w_edge
    h.w_velocity, h.w_acceleration, h.tau_color = hp.w_velocity, hp.w_acceleration, hp.tau_color
    h.gn_iterations, h.pcg_iterations, h.max_halvings = (int(hp.gn_iterations),
                                                         int(hp.pcg_iterations), int(hp.max_halvings))
    ks = tuple(hp.pyramid_kernels)
    if not 1 <= len(ks) <= 4:
        raise ValueError("1..4 pyramid levels are supported")
    for i, k in enumerate(ks):
        if k < 1 or k % 2 == 0:
            raise ValueError(f"kernel size must be odd and positive, got {k}")
        h.pyramid_kernels[i] = int(k)
        if k <= 32:
            for q, t in enumerate(L.gaussian_taps(int(k))):
                h.pyramid_taps[i][q] = float(t)
    h.n_levels = len(ks) if n_levels is None else int(n_levels)
    h.part_dilation = int(hp.part_dilation)
    h.snap_step, h.snap_max_steps, h.snap_band = hp.snap_step, int(hp.snap_max_steps), hp.snap_band
    if h.gn_iterations > L.LC_MAX_LOG:
        raise ValueError(f"at most {L.LC_MAX_LOG} Gauss-Newton iterations per solve")
    return h


def config_c(cfg: SequenceConfig) -> L.Config:
    c = L.Config()
    c.mode = MODES.index(cfg.mode)
    c.directional, c.enable_warping = int(cfg.directional), int(cfg.enable_warping)
    c.enable_part_mask, c.enable_snapping = int(cfg.enable_part_mask), int(cfg.enable_snapping)
    c.frame0_rounds, c.frame0_iteration_scale = int(cfg.frame0_rounds), int(cfg.frame0_iteration_scale)
    c.pose = pose_hyper_c(cfg.pose)
    c.nonrigid = nonrigid_hyper_c(cfg.nonrigid)
    # frame 0 logs every cold-start round's GN iterations in one report
    # (pipeline.py:182-195: 2 override rounds + max(1, rounds - 2) full ones)
    f0 = int(cfg.pose.gn_iterations) * int(cfg.frame0_iteration_scale) * (2 + max(1, int(cfg.frame0_rounds) - 2))
    if f0 > L.LC_MAX_LOG:
        raise ValueError(f"frame 0 would log {f0} pose GN iterations; at most {L.LC_MAX_LOG} are supported "
                         f"(gn_iterations * frame0_iteration_scale * cold-start rounds)")
    return c


def camera_c(cam) -> L.Camera:
    return L.Camera(float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                    int(cam.width), int(cam.height))


class _Mesh:
    """Placeholder mesh for skeleton-only device actors (the pose seam)."""

    def __init__(self, n):
        self.rest_vertices = np.zeros((n, 3))
        self.triangles = np.zeros((0, 3), dtype=np.int64)
        self.vertex_colors = np.zeros((n, 3))
        self.vertex_labels = np.full(n, 5, dtype=np.int64)
        self.edges = np.zeros((0, 2), dtype=np.int64)
        self.edge_tris = np.zeros((0, 2), dtype=np.int64)
        self.degrees = np.zeros(n, dtype=np.int64)
        self.directed_weights = np.zeros(0)
        self.n_vertices = n


class DeviceActor:
    """An actor's immutable device tables (shareable by every stream on a device).

    Built from a full actor, or from parts for the per-stage seams: a pose
    problem carries only skeleton + skinning, a non-rigid problem only the
    mesh; the missing part is filled with an inert placeholder.
    """

    _cache: dict = {}

    def __init__(self, mesh, skeleton, skinning, ctx: L.Context | None = None):
        self.ctx = ctx or L.default_context()
        m, sk = mesh, skeleton
        if skinning is None:
            idx = np.full((m.n_vertices, 4), -1, dtype=np.int64)
            idx[:, 0] = 0
            w = np.zeros((m.n_vertices, 4))
            w[:, 0] = 1.0
        else:
            idx, w = skinning.indices, skinning.weights
        keep = dict(
            rest=L.f64c(m.rest_vertices), tris=L.i64c(m.triangles), cols=L.f64c(m.vertex_colors),
            labels=L.i64c(m.vertex_labels), edges=L.i64c(m.edges), etris=L.i64c(m.edge_tris),
            deg=L.i64c(m.degrees), wdir=L.f64c(m.directed_weights), parents=L.i64c(sk.parents),
            offs=L.f64c(sk.local_offsets), dj=L.i64c(sk.dof_joint), dax=L.f64c(sk.dof_axes),
            tmin=L.f64c(sk.theta_min), tmax=L.f64c(sk.theta_max), mk=L.f64c(sk.marker_offsets),
            grp=_group_ids(sk), parts=np.ascontiguousarray(joint_body_parts(sk), dtype=np.int32),
            sidx=L.i64c(idx), sw=L.f64c(w))
        d = L.ActorDesc()
        d.n_vertices, d.n_triangles = m.n_vertices, len(m.triangles)
        d.n_edges, d.n_joints = len(m.edges), sk.n_joints
        d.rest_vertices, d.triangles = L.ptr(keep["rest"]), L.ptr(keep["tris"])
        d.vertex_colors, d.vertex_labels = L.ptr(keep["cols"]), L.ptr(keep["labels"])
        d.edges, d.edge_tris, d.degrees = L.ptr(keep["edges"]), L.ptr(keep["etris"]), L.ptr(keep["deg"])
        d.directed_weights = L.ptr(keep["wdir"])
        d.parents, d.local_offsets = L.ptr(keep["parents"]), L.ptr(keep["offs"])
        d.dof_joint, d.dof_axes = L.ptr(keep["dj"]), L.ptr(keep["dax"])
        d.theta_min, d.theta_max = L.ptr(keep["tmin"]), L.ptr(keep["tmax"])
        d.marker_offsets, d.head_index = L.ptr(keep["mk"]), sk.head_index
        d.temporal_group, d.joint_parts = L.ptr(keep["grp"]), L.ptr(keep["parts"])
        d.skin_indices, d.skin_weights = L.ptr(keep["sidx"]), L.ptr(keep["sw"])
        h = L.P()
        L.check(self.ctx.lib.lc_actor_upload(self.ctx.handle, C.byref(d), C.byref(h)))
        self.handle = h
        self.ctx.register(self)
        self.n_vertices = m.n_vertices
        self.n_joints = sk.n_joints

    CACHE_SIZE = 4   # uploaded actors kept per process (LRU; evicted ones are freed)

    @classmethod
    def _cached(cls, key, owner, build):
        hit = cls._cache.pop(key, None)
        if hit is not None and hit[0] is owner and hit[1].handle:   # (not freed with its context)
            cls._cache[key] = hit          # most recently used last
            return hit[1]
        dev = build()
        cls._cache[key] = (owner, dev)
        while len(cls._cache) > cls.CACHE_SIZE:
            # dropped from the cache; freed by __del__ once no Tracker holds it
            cls._cache.pop(next(iter(cls._cache)))
        return dev

    @classmethod
    def get(cls, actor, ctx: L.Context | None = None) -> "DeviceActor":
        """Full actor (mine or a reference `montrack.template.Actor`)."""
        ctx = ctx or L.default_context()
        key = ("actor", id(ctx), id(actor), id(actor.mesh), id(actor.mesh.directed_weights))
        return cls._cached(key, actor, lambda: cls(actor.mesh, actor.skeleton, actor.skinning, ctx))

    @classmethod
    def for_pose(cls, skeleton, skinning, ctx: L.Context | None = None) -> "DeviceActor":
        ctx = ctx or L.default_context()
        key = ("pose", id(ctx), id(skeleton), id(skinning))
        n = len(skinning.indices)
        return cls._cached(key, skinning, lambda: cls(_Mesh(n), skeleton, skinning, ctx))

    @classmethod
    def for_mesh(cls, mesh, ctx: L.Context | None = None) -> "DeviceActor":
        from .synthetic import default_skeleton
        ctx = ctx or L.default_context()
        key = ("mesh", id(ctx), id(mesh), id(mesh.directed_weights))
        return cls._cached(key, mesh, lambda: cls(mesh, default_skeleton(), None, ctx))

    def close(self):
        if getattr(self, "handle", None):
            if self.ctx.handle:   # (a closed context already freed it)
                self.ctx.lib.lc_actor_destroy(self.handle)
            self.handle = None

    def __del__(self, _finalizing=sys.is_finalizing):
        if _finalizing():   # the context may already be gone at interpreter exit
            return
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# report conversion (device structs -> reference dataclasses)

POSE_TERMS = ("detection2d", "detection3d", "silhouette", "temporal", "anatomic")
NR_TERMS = ("photo", "silhouette", "smooth", "edge", "velocity", "acceleration")


def pose_report_from_c(r: L.PoseReport, start: int = 0) -> PoseStageReport:
    rep = PoseStageReport(behind_camera=int(r.behind_camera), gimbal=bool(r.gimbal))
    for k in range(start, r.n_iterations):
        terms = {POSE_TERMS[t]: float(r.terms[k][t]) for t in range(5)}
        rep.iterations.append(PoseIterationLog(
            float(r.energy_before[k]), float(r.energy_after[k]), terms, float(r.step_norm[k]),
            int(r.halvings[k]), bool(r.rejected[k]), bool(r.damped[k])))
    return rep


def nonrigid_report_from_c(r: L.NonrigidReport) -> NonrigidStageReport:
    rep = NonrigidStageReport(pruned=int(r.pruned), degenerate_edges=int(r.degenerate_edges),
                              behind_camera=int(r.behind_camera))
    names = NR_TERMS if r.has_temporal else NR_TERMS[:4]
    for k in range(r.n_iterations):
        terms = {names[t]: float(r.terms[k][t]) for t in range(len(names))}
        rep.iterations.append(NonrigidIterationLog(
            int(r.level[k]), float(r.energy_before[k]), float(r.energy_after[k]), terms,
            int(r.halvings[k]), bool(r.rejected[k]), bool(r.pcg_breakdown[k])))
    if r.snapped:
        rep.snap = SnapInfo(int(r.snap_walked), int(r.snap_reached), int(r.snap_stuck))
    return rep


# ---------------------------------------------------------------------------
# batched multi-stream tracker

class Tracker:
    """S independent capture streams advanced one frame per `step()`.

    Mirrors the reference recursion `solve_frame` + `TrackState`
    (pipeline.py:135-142,263-302) per stream, with all streams batched into
    every kernel launch.  Inputs: per stream an (H,W,3) f64 image, an (H,W)
    bool mask and `FrameDetections` (host arrays, or device pointers with
    `on_device=True`).
    """

    def __init__(self, actor, camera, config: SequenceConfig | None = None, n_streams: int = 1,
                 ctx: L.Context | None = None):
        self.ctx = ctx or L.default_context()
        self.config = SequenceConfig.from_reference(config) if config is not None else SequenceConfig()
        self.dactor = DeviceActor.get(actor, self.ctx)
        self.camera = camera
        self.S = int(n_streams)
        self._cam = camera_c(camera)
        self._cfg = config_c(self.config)
        h = L.P()
        L.check(self.ctx.lib.lc_tracker_create(self.ctx.handle, self.dactor.handle, C.byref(self._cam),
                                               C.byref(self._cfg), self.S, C.byref(h)))
        self.handle = h
        self.ctx.register(self)
        self.N = self.dactor.n_vertices
        self.J = self.dactor.n_joints
        self._keep = []

    def set_frame(self, stream: int, image, mask, det: FrameDetections, on_device: bool = False):
        j2d = L.f64c(det.joints2d)
        j3d = L.f64c(det.joints3d)
        v2d = L.u8c(det.valid2d)
        v3d = L.u8c(det.valid3d)
        if j2d.shape != (self.J + 4, 2) or j3d.shape != (self.J, 3):
            raise ValueError("detections do not match the skeleton")
        d = L.Detections(L.ptr(j2d), L.ptr(j3d), L.ptr(v2d), L.ptr(v3d))
        u8 = False
        if on_device:
            img_p, mask_p = (None if image is None else int(image)), int(mask)
        else:
            H, W = self.camera.height, self.camera.width
            mask = L.u8c(mask)
            if image is not None:   # None: mask + detections only (a Stage-I-only tracker)
                u8 = isinstance(image, np.ndarray) and image.dtype == np.uint8
                image = np.ascontiguousarray(image) if u8 else L.f64c(image)
                if image.shape != (H, W, 3):
                    raise ValueError("image shape does not match the camera")
            if mask.shape != (H, W):
                raise ValueError("mask shape does not match the camera")
            img_p, mask_p = L.ptr(image), L.ptr(mask)
        fn = self.ctx.lib.lc_tracker_set_frame_u8 if u8 else self.ctx.lib.lc_tracker_set_frame
        L.check(fn(self.handle, stream, img_p, mask_p, C.byref(d), int(on_device)))

    def step(self):
        L.check(self.ctx.lib.lc_tracker_step(self.handle))

    def set_graph(self, on: bool = True):
        """Replay steady-state steps as captured CUDA graphs (lc_tracker_set_graph)."""
        L.check(self.ctx.lib.lc_tracker_set_graph(self.handle, int(bool(on))))

    def graph_stats(self):
        g, r = C.c_int64(), C.c_int64()
        L.check(self.ctx.lib.lc_tracker_graph_stats(self.handle, C.byref(g), C.byref(r)))
        return g.value, r.value

    def result(self, stream: int, with_report: bool = True):
        x = np.empty(36)
        v = np.empty((self.N, 3))
        vs = np.empty((self.N, 3))
        rep = L.FrameReport() if with_report else None
        L.check(self.ctx.lib.lc_tracker_get_result(self.handle, stream, L.ptr(x), L.ptr(v), L.ptr(vs),
                                                   C.byref(rep) if rep is not None else None))
        return x, v, vs, rep

    def result_async(self, stream: int, pose_out, verts_out):
        """Enqueue the D2H readout of the last stepped frame into caller
        buffers (pinned: fully asynchronous); valid once the context's stream
        passes this point.  Arguments are objects with a data pointer
        (numpy arrays, or torch tensors via .data_ptr())."""
        def p(a):
            if a is None:
                return None
            return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else L.ptr(a)
        L.check(self.ctx.lib.lc_tracker_get_result_async(self.handle, stream, p(pose_out), p(verts_out)))

    def set_state(self, stream: int, state):
        """Inject a TrackState (teacher forcing / resume)."""
        def arr(a, shape):
            if a is None:
                return None
            # this package's PoseParams or the reference's (duck-typed)
            a = L.f64c(a.to_vector() if hasattr(a, "to_vector") else a)
            if a.shape != shape:
                raise ValueError(f"state array has shape {a.shape}, expected {shape}")
            return a
        xs = [arr(state.pose_prev, (36,)), arr(state.pose_prev2, (36,)),
              arr(state.joints_prev, (self.J, 3)), arr(state.disp_rest, (self.N, 3)),
              arr(state.v_prev, (self.N, 3)), arr(state.v_prev2, (self.N, 3))]
        L.check(self.ctx.lib.lc_tracker_set_state(self.handle, stream, *[L.ptr(a) for a in xs]))

    def step_stage(self, stages: int):
        """1 = conditioning + Stage I, 2 = Stage II + state update, 3 = both
        (consumes the queued frame; see lc_tracker_step_stage)."""
        L.check(self.ctx.lib.lc_tracker_step_stage(self.handle, int(stages)))

    def set_pose(self, stream: int, pose):
        """The Stage I pose a following step_stage(2) solves Stage II from."""
        x = L.f64c(pose.to_vector() if hasattr(pose, "to_vector") else pose)
        if x.shape != (36,):
            raise ValueError("pose must have 36 parameters")
        L.check(self.ctx.lib.lc_tracker_set_pose(self.handle, stream, L.ptr(x)))

    def get_state(self, stream: int):
        from .config import TrackState
        flags = np.zeros(5, dtype=np.int32)
        x1, x2 = np.empty(36), np.empty(36)
        jp = np.empty((self.J, 3))
        dr, v1, v2 = np.empty((self.N, 3)), np.empty((self.N, 3)), np.empty((self.N, 3))
        L.check(self.ctx.lib.lc_tracker_get_state(self.handle, stream, L.ptr(flags), L.ptr(x1), L.ptr(x2),
                                                  L.ptr(jp), L.ptr(dr), L.ptr(v1), L.ptr(v2)))
        return TrackState(PoseParams.from_vector(x1) if flags[0] else None,
                          PoseParams.from_vector(x2) if flags[1] else None,
                          jp if flags[0] else None, dr if flags[2] else None,
                          v1 if flags[3] else None, v2 if flags[4] else None)

    def inspect(self, stream: int) -> dict:
        """Last Stage II setup of a stream: boundary ids, enabled flags, visible
        ids, normals2d, v_init, V^S (for parity tests)."""
        out = {}
        n = C.c_int64()
        cap = 3 * self.N
        for what, key in ((0, "boundary"), (1, "enabled"), (2, "visible")):
            buf = np.empty(cap, dtype=np.int64)
            L.check(self.ctx.lib.lc_tracker_inspect(self.handle, stream, what, L.ptr(buf), cap, C.byref(n)))
            out[key] = buf[:n.value].copy()
        out["enabled"] = out["enabled"].astype(bool)
        buf = np.empty(cap)
        L.check(self.ctx.lib.lc_tracker_inspect(self.handle, stream, 3, L.ptr(buf), cap, C.byref(n)))
        out["normals2d"] = buf[:2 * n.value].reshape(-1, 2).copy()
        for what, key in ((4, "v_init"), (5, "skinned")):
            buf = np.empty((self.N, 3))
            L.check(self.ctx.lib.lc_tracker_inspect(self.handle, stream, what, L.ptr(buf), cap, C.byref(n)))
            out[key] = buf
        return out

    def inspect_system(self, stream: int) -> dict:
        """The last Stage II GN step's compact normal system and PCG result:
        diag (N,6) symmetric (xx xy xz yy yz zz), minv (N,9), rhs (N,3), the best
        PCG iterate (N,3)."""
        out = {}
        n = C.c_int64()
        for what, key, w in ((6, "diag", 6), (7, "rhs", 3), (8, "best", 3), (9, "minv", 9)):
            buf = np.empty((self.N, w))
            L.check(self.ctx.lib.lc_tracker_inspect(self.handle, stream, what, L.ptr(buf), buf.size, C.byref(n)))
            out[key] = buf
        return out

    def phase_times(self, stream: int):
        """Device timestamps (ns, %globaltimer) of the last frame's solver
        phases: pose [start, per GN: eval, solve, line search], surface
        [start, per GN: assembly, PCG, line search, ..., snap]."""
        p = np.zeros(64, dtype=np.int64)
        q = np.zeros(64, dtype=np.int64)
        L.check(self.ctx.lib.lc_tracker_phase_times(self.handle, stream, L.ptr(p), L.ptr(q)))
        return p, q

    def counters(self, stream: int) -> np.ndarray:
        out = np.zeros(8, dtype=np.int64)
        L.check(self.ctx.lib.lc_tracker_counters(self.handle, stream, L.ptr(out)))
        return out

    def close(self):
        if self.handle:
            if self.ctx.handle:
                self.ctx.lib.lc_tracker_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StagePipeline:
    """The paper's pose -> non-rigid pipeline across a GPU pair.

    Stage I (conditioning, pose GN) of every stream runs on `pose_device`,
    Stage II (surface GN, PCG, snapping, warp) on `surface_device`.  Per frame
    the solved poses go pose -> surface device and the track state Stage I
    needs (x_prev, x_prev2, joints_prev, disp_rest) comes back, as peer copies
    over NVLink (lc_tracker_pipe).  Within one stream the stages are serial
    (frame t+1's Stage I needs frame t's surface), so the streams are split
    into `groups` groups on their own CUDA streams: while the surface device
    solves group g, the pose device solves group g+1.  The arithmetic is the
    single-device tracker's, so results are identical to it.
    """

    def __init__(self, actor, camera, config, n_streams: int, pose_device: int = 0, surface_device: int = 1,
                 groups: int = 2):
        if n_streams % groups:
            raise ValueError("n_streams must be a multiple of groups")
        self.groups = groups
        self.per = n_streams // groups
        self.ctx_a = [L.Context(pose_device) for _ in range(groups)]
        self.ctx_b = [L.Context(surface_device) for _ in range(groups)]
        self.A = [Tracker(actor, camera, config, self.per, ctx=c) for c in self.ctx_a]
        self.B = [Tracker(actor, camera, config, self.per, ctx=c) for c in self.ctx_b]

    def _where(self, stream):
        return divmod(stream, self.per)

    def set_frame(self, stream: int, image, mask, det, on_device: bool = False):
        g, s = self._where(stream)
        if on_device:
            raise ValueError("device-resident inputs live on one GPU; queue host frames")
        self.A[g].set_frame(s, None, mask, det)    # Stage I reads no image: mask + detections only
        self.B[g].set_frame(s, image, mask, det)

    def step(self):
        lib = self.A[0].ctx.lib
        for g in range(self.groups):
            L.check(lib.lc_tracker_step_stage(self.A[g].handle, 1))
            L.check(lib.lc_tracker_pipe(self.B[g].handle, self.A[g].handle, 1))
            L.check(lib.lc_tracker_step_stage(self.B[g].handle, 2))
            L.check(lib.lc_tracker_pipe(self.A[g].handle, self.B[g].handle, 2))

    def result(self, stream: int, with_report: bool = True):
        g, s = self._where(stream)
        return self.B[g].result(s, with_report)

    def synchronize(self):
        for c in self.ctx_a + self.ctx_b:
            c.synchronize()

    def close(self):
        for t in self.A + self.B:
            t.close()


class BatchTracker:
    """`n_streams` streams split into `groups` trackers, each on its own
    library context (CUDA solve / preprocessing / copy streams), stepped
    together.  Each group's kernel chain runs independently, so one group's
    raster / contour phases overlap another's solver phases and a slow stream
    only holds back its own group.  Same API as `Tracker` (global stream
    indices); results are identical to a single tracker's.
    """

    def __init__(self, actor, camera, config: SequenceConfig | None = None, n_streams: int = 1,
                 groups: int = 1, device: int = 0, priority_streams: bool = True,
                 host_threads: bool = True):
        groups = max(1, min(groups, n_streams))
        base, extra = divmod(n_streams, groups)
        self.sizes = [base + (1 if g < extra else 0) for g in range(groups)]
        self.starts = np.cumsum([0] + self.sizes[:-1]).tolist()
        self.torch_streams = []
        self.ctxs = []
        for _ in range(groups):
            st = 0
            if priority_streams:
                try:
                    import torch
                    ts = torch.cuda.Stream(device=device, priority=-1)
                    self.torch_streams.append(ts)
                    st = ts.cuda_stream
                except Exception:   # noqa: BLE001 - torch only provides the high-priority stream
                    st = 0
            self.ctxs.append(L.Context(device, st))
        self.trackers = [Tracker(actor, camera, config, n, ctx=c) for n, c in zip(self.sizes, self.ctxs)]
        self.S = n_streams
        # one host thread per group enqueues that group's step: the library
        # calls release the GIL (ctypes) and contexts share no mutable state,
        # so the groups' host-side launch work (~0.3 ms per group step) runs
        # in parallel instead of serialising in front of the device
        self._pool = None
        if host_threads and groups > 1:
            from concurrent.futures import ThreadPoolExecutor
            self._pool = ThreadPoolExecutor(max_workers=groups, thread_name_prefix="lc-group")

    def _where(self, stream):
        for g, (a, n) in enumerate(zip(self.starts, self.sizes)):
            if a <= stream < a + n:
                return g, stream - a
        raise IndexError("stream index out of range")

    def set_frame(self, stream, image, mask, det, on_device=False):
        g, s = self._where(stream)
        self.trackers[g].set_frame(s, image, mask, det, on_device)

    def step(self):
        if self._pool is None:
            for t in self.trackers:
                t.step()
            return
        for f in [self._pool.submit(t.step) for t in self.trackers]:
            f.result()

    def set_graph(self, on: bool = True):
        for t in self.trackers:
            t.set_graph(on)

    def graph_stats(self):
        st = [t.graph_stats() for t in self.trackers]
        return sum(g for g, _ in st), sum(r for _, r in st)

    def result(self, stream, with_report=True):
        g, s = self._where(stream)
        return self.trackers[g].result(s, with_report)

    def result_async(self, stream, pose_out, verts_out):
        g, s = self._where(stream)
        self.trackers[g].result_async(s, pose_out, verts_out)

    def set_state(self, stream, state):
        g, s = self._where(stream)
        self.trackers[g].set_state(s, state)

    def get_state(self, stream):
        g, s = self._where(stream)
        return self.trackers[g].get_state(s)

    def counters(self, stream):
        g, s = self._where(stream)
        return self.trackers[g].counters(s)

    def phase_times(self, stream):
        g, s = self._where(stream)
        return self.trackers[g].phase_times(s)

    def synchronize(self):
        for c in self.ctxs:
            c.synchronize()

    def launches(self) -> int:
        return sum(c.launches() for c in self.ctxs)

    def profile_kernel(self, name):
        for c in self.ctxs:
            c.profile_kernel(name)

    def profile_busy_ms(self) -> float:
        """Length of the union of the profiled kernel's launch intervals over
        all groups (the time the device spent in that kernel, concurrency
        counted once)."""
        iv = np.concatenate([c.profile_intervals() for c in self.ctxs]) if self.ctxs else np.zeros((0, 2))
        if len(iv) == 0:
            return 0.0
        iv = iv[np.argsort(iv[:, 0])]
        busy, cur_s, cur_e = 0.0, iv[0, 0], iv[0, 1]
        for a, b in iv[1:]:
            if a > cur_e:
                busy += cur_e - cur_s
                cur_s, cur_e = a, b
            else:
                cur_e = max(cur_e, b)
        return float(busy + (cur_e - cur_s))

    def profile_read(self):
        ms, n = 0.0, 0
        for c in self.ctxs:
            a, b = c.profile_read()
            ms += a
            n += b
        return ms, n

    def close(self):
        if self._pool is not None:
            self._pool.shutdown()
            self._pool = None
        for t in self.trackers:
            t.close()
