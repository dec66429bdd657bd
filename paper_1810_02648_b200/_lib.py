"""ctypes binding of liblivecap.so (include/livecap.h).

The product path: every compute call goes through these entry points.  If the
library is missing or no CUDA device is usable, `lib()` raises -- there is no
CPU fallback.  ctypes releases the GIL during calls, so the reference's
pipelined worker threads keep overlapping.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LIVECAP_LIB: an alternative build of the same sources (e.g. the sanitizer
# variant from _build.build_variant); default the in-tree library
LIB_PATH = os.environ.get("LIVECAP_LIB") or os.path.join(HERE, "liblivecap.so")

LC_OK, LC_EINVAL, LC_ECUDA, LC_ENOMEM, LC_ECAP = 0, 1, 2, 3, 4
LC_MAX_LOG = 64
LC_MAX_JOINTS = 32

P = C.c_void_p
i32, i64, f64, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64


class Camera(C.Structure):
    _fields_ = [("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64), ("width", i32), ("height", i32)]


class ActorDesc(C.Structure):
    _fields_ = [("n_vertices", i32), ("n_triangles", i32), ("n_edges", i32), ("n_joints", i32),
                ("rest_vertices", P), ("triangles", P), ("vertex_colors", P), ("vertex_labels", P),
                ("edges", P), ("edge_tris", P), ("degrees", P), ("directed_weights", P),
                ("parents", P), ("local_offsets", P), ("dof_joint", P), ("dof_axes", P),
                ("theta_min", P), ("theta_max", P), ("marker_offsets", P), ("head_index", i32),
                ("temporal_group", P), ("joint_parts", P), ("skin_indices", P), ("skin_weights", P)]


class PoseHyper(C.Structure):
    _fields_ = [("lambda_2d", f64), ("lambda_3d", f64), ("lambda_sil", f64),
                ("lambda_temporal", f64), ("lambda_anatomic", f64), ("face_weight", f64),
                ("group_weights", f64 * 8), ("gn_iterations", i32), ("max_halvings", i32)]


class NonrigidHyper(C.Structure):
    _fields_ = [("w_photo", f64), ("w_sil", f64), ("w_smooth", f64), ("w_edge", f64),
                ("w_velocity", f64), ("w_acceleration", f64), ("tau_color", f64),
                ("gn_iterations", i32), ("pcg_iterations", i32), ("max_halvings", i32),
                ("n_levels", i32), ("pyramid_kernels", i32 * 4), ("pyramid_taps", (f64 * 32) * 4),
                ("part_dilation", i32),
                ("snap_step", f64), ("snap_max_steps", i32), ("snap_band", f64)]


class Config(C.Structure):
    _fields_ = [("mode", i32), ("directional", i32), ("enable_warping", i32),
                ("enable_part_mask", i32), ("enable_snapping", i32), ("frame0_rounds", i32),
                ("frame0_iteration_scale", i32), ("pose", PoseHyper), ("nonrigid", NonrigidHyper)]


class Detections(C.Structure):
    _fields_ = [("joints2d", P), ("joints3d", P), ("valid2d", P), ("valid3d", P)]


class PcgInfo(C.Structure):
    _fields_ = [("iterations", i32), ("breakdown", i32), ("residual_norms", f64 * LC_MAX_LOG)]


class DenseInfo(C.Structure):
    _fields_ = [("damped", i32), ("damping", f64)]


class PoseReport(C.Structure):
    _fields_ = [("n_iterations", i32), ("behind_camera", i32), ("gimbal", i32),
                ("energy_before", f64 * LC_MAX_LOG), ("energy_after", f64 * LC_MAX_LOG),
                ("step_norm", f64 * LC_MAX_LOG), ("terms", (f64 * 5) * LC_MAX_LOG),
                ("halvings", i32 * LC_MAX_LOG), ("rejected", i32 * LC_MAX_LOG),
                ("damped", i32 * LC_MAX_LOG), ("n_contour", i32), ("has_temporal", i32)]


class NonrigidReport(C.Structure):
    _fields_ = [("n_iterations", i32), ("pruned", i32), ("degenerate_edges", i32),
                ("behind_camera", i32), ("level", i32 * LC_MAX_LOG),
                ("energy_before", f64 * LC_MAX_LOG), ("energy_after", f64 * LC_MAX_LOG),
                ("terms", (f64 * 6) * LC_MAX_LOG), ("has_temporal", i32),
                ("halvings", i32 * LC_MAX_LOG), ("rejected", i32 * LC_MAX_LOG),
                ("pcg_breakdown", i32 * LC_MAX_LOG), ("snapped", i32), ("snap_walked", i32),
                ("snap_reached", i32), ("snap_stuck", i32), ("snap_moved", i32),
                ("n_visible", i32), ("n_boundary", i32), ("n_enabled", i32)]


class FrameReport(C.Structure):
    _fields_ = [("pose", PoseReport), ("nonrigid", NonrigidReport), ("rescale_fallbacks", i32)]


class PoseProblemC(C.Structure):
    _fields_ = [("mask", P), ("joints2d", P), ("joints3d", P), ("valid2d", P), ("valid3d", P),
                ("n_contour", i32), ("contour_indices", P), ("contour_normals2d", P),
                ("contour_rest", P), ("contour_enabled", P), ("prev_positions", P),
                ("directional", i32), ("hyper", PoseHyper)]


class NonrigidProblemC(C.Structure):
    _fields_ = [("mask", P), ("n_levels", i32), ("pyramid", P), ("skinned", P),
                ("n_visible", i32), ("visible", P), ("n_boundary", i32), ("boundary", P),
                ("normals2d", P), ("enabled", P), ("prev", P), ("prev2", P),
                ("directional", i32), ("enable_photo", i32), ("enable_sil", i32),
                ("hyper", NonrigidHyper)]


# name -> (restype, argtypes)
_SIGS = {
    "lc_last_error": (C.c_char_p, []),
    "lc_version": (C.c_int, []),
    "lc_ctx_create": (C.c_int, [i32, u64, P]),
    "lc_ctx_destroy": (C.c_int, [P]),
    "lc_ctx_synchronize": (C.c_int, [P]),
    "lc_ctx_set_team_sizes": (C.c_int, [P, i32, i32]),
    "lc_ctx_set_pyramid_margin": (C.c_int, [P, i32]),
    "lc_tracker_set_pose": (C.c_int, [P, i32, P]),
    "lc_field_dt": (C.c_int, [P, P]),
    "lc_edt_squared": (C.c_int, [P, i32, i32, P, P]),
    "lc_surface_sets": (C.c_int, [P, P, P, P, i32, i32, i32, P, P, P, P, P, P, P]),
    "lc_kernel_launches": (C.c_int, [P, P]),
    "lc_process_launches": (C.c_int, [P]),
    "lc_tracker_set_graph": (C.c_int, [P, i32]),
    "lc_tracker_graph_stats": (C.c_int, [P, P, P]),
    "lc_rng_normal": (C.c_int, [P, P, P, f64, f64, P, i64, i32, P, P, P, i32, P]),
    "lc_rng_uniform": (C.c_int, [P, P, P, P, i64]),
    "lc_rng_scatter": (C.c_int, [P, P, P, i32, P]),
    "lc_rng_gather": (C.c_int, [P, P, i32, P, P]),
    "lc_rng_tables": (C.c_int, [P, P, P]),
    "lc_actor_upload": (C.c_int, [P, P, P]),
    "lc_actor_destroy": (C.c_int, [P]),
    "lc_pcg_solve_bsr": (C.c_int, [P, i32, i64, P, P, P, P, P, i32, P, P]),
    "lc_dense_solve": (C.c_int, [P, i32, P, P, P, P]),
    "lc_smooth_trajectory": (C.c_int, [P, i32, C.c_int64, P, i32, P, P]),
    "lc_mask_overlap": (C.c_int, [P, i32, C.c_int64, P, P, P, P]),
    "lc_mean_vertex_error": (C.c_int, [P, i32, C.c_int64, P, P, P, C.c_int64, i32, i32, P]),
    "lc_aligned_error": (C.c_int, [P, i32, i32, P, P, i32, i32, P, P, P, P]),
    "lc_gaussian_pyramid": (C.c_int, [P, i32, i32, i32, P, i32, P, P, P]),
    "lc_render": (C.c_int, [P, P, i32, P, i32, P, i32, P, i32, P, f64, i64, P, P, P]),
    "lc_field_create": (C.c_int, [P, i32, i32, P, P]),
    "lc_field_destroy": (C.c_int, [P]),
    "lc_field_n_contour": (C.c_int, [P, P]),
    "lc_field_query": (C.c_int, [P, i64, P, i32, P]),
    "lc_forward_kinematics": (C.c_int, [P, P, P, P, P, P, P, P]),
    "lc_skin_points": (C.c_int, [P, P, P, i32, P, P, P, P, P]),
    "lc_contour_vertices": (C.c_int, [P, P, P, P, P, P, P]),
    "lc_pose_solve": (C.c_int, [P, P, P, P, P, P, P]),
    "lc_nonrigid_solve": (C.c_int, [P, P, P, P, P, i32, i32, P, P]),
    "lc_tracker_create": (C.c_int, [P, P, P, P, i32, P]),
    "lc_tracker_destroy": (C.c_int, [P]),
    "lc_tracker_set_frame": (C.c_int, [P, i32, P, P, P, i32]),
    "lc_tracker_get_result_async": (C.c_int, [P, i32, P, P]),
    "lc_tracker_set_frame_u8": (C.c_int, [P, i32, P, P, P, i32]),
    "lc_tracker_step_stage": (C.c_int, [P, i32]),
    "lc_tracker_pipe": (C.c_int, [P, P, i32]),
    "lc_trace_dump": (C.c_int, [P, C.c_char_p, C.c_int64]),
    "lc_profile_intervals": (C.c_int, [P, P, C.c_int64, P]),
    "lc_tracker_step": (C.c_int, [P]),
    "lc_tracker_get_result": (C.c_int, [P, i32, P, P, P, P]),
    "lc_tracker_set_state": (C.c_int, [P, i32, P, P, P, P, P, P]),
    "lc_tracker_get_state": (C.c_int, [P, i32, P, P, P, P, P, P, P]),
    "lc_tracker_device_vertices": (C.c_int, [P, i32, P]),
    "lc_debug_tables": (C.c_int, [i32, P, P]),
    "lc_tracker_counters": (C.c_int, [P, i32, P]),
    "lc_tracker_inspect": (C.c_int, [P, i32, i32, P, i64, P]),
    "lc_tracker_phase_times": (C.c_int, [P, i32, P, P]),
    "lc_profile_kernel": (C.c_int, [P, C.c_char_p]),
    "lc_profile_read": (C.c_int, [P, P, P]),
}
EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


class LivecapError(RuntimeError):
    pass


def load_library(path: str = LIB_PATH):
    """Load and bind the shared library (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise LivecapError(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(code: int):
    if code == LC_OK:
        return
    msg = _lib.lc_last_error().decode(errors="replace")
    if code == LC_EINVAL:
        raise ValueError(msg)
    if code == LC_ENOMEM:
        raise MemoryError(msg)
    raise LivecapError(msg)


def gaussian_taps(size: int) -> np.ndarray:
    """Normalized Gaussian taps exactly as the reference computes them with
    numpy (imageproc.py:264-273); passed to the device so the pyramid is
    bit-exact whatever libm's exp rounds to."""
    if size == 1:
        return np.ones(1)
    sigma = (size - 1) / 6.0
    x = np.arange(size) - (size - 1) / 2.0
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def f64c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64c(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def u8c(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


class Context:
    """A CUDA device + stream owned by the library (one per host thread)."""

    def __init__(self, device: int = 0, stream: int = 0):
        lib = load_library()
        h = P()
        check(lib.lc_ctx_create(device, stream, C.byref(h)))
        self.device = int(device)
        self.handle = h
        self.lib = lib
        self._dependents = []   # weakrefs to objects holding device memory of this context

    def register(self, obj):
        """`obj.close()` frees device objects of this context: close() calls
        it first, so nothing is freed after its context."""
        if len(self._dependents) > 64:
            self._dependents = [r for r in self._dependents if r() is not None]
        self._dependents.append(weakref.ref(obj))

    def launches(self) -> int:
        n = C.c_int64()
        check(self.lib.lc_kernel_launches(self.handle, C.byref(n)))
        return n.value

    def profile_kernel(self, name: str | None):
        check(self.lib.lc_profile_kernel(self.handle, None if name is None else name.encode()))

    def profile_read(self):
        ms, n = C.c_double(), C.c_int64()
        check(self.lib.lc_profile_read(self.handle, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def profile_intervals(self):
        out = np.zeros(2 * 65536)
        n = C.c_int64()
        check(self.lib.lc_profile_intervals(self.handle, out.ctypes.data, 65536, C.byref(n)))
        return out[:2 * n.value].reshape(-1, 2)

    def synchronize(self):
        check(self.lib.lc_ctx_synchronize(self.handle))

    def set_team_sizes(self, pose: int = 0, surface: int = 0):
        """CTAs per stream of the pose / surface solver teams (0 = default)."""
        check(self.lib.lc_ctx_set_team_sizes(self.handle, int(pose), int(surface)))

    def set_pyramid_margin(self, margin_px: int):
        """Blur pyramid region of interest in pixels around the observed
        silhouette (-1: every tile, -2: none -- every sample on the exact
        on-demand path)."""
        check(self.lib.lc_ctx_set_pyramid_margin(self.handle, int(margin_px)))

    def close(self):
        if self.handle:
            for r in reversed(self._dependents):   # (trackers before the actors they use)
                obj = r()
                if obj is not None:
                    obj.close()
            self._dependents = []
            self.lib.lc_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def process_launches() -> int:
    """Kernels launched by every library context of this process (the
    per-thread default contexts of worker threads included)."""
    n = C.c_int64()
    check(load_library().lc_process_launches(C.byref(n)))
    return n.value


_tls = threading.local()


def default_context() -> Context:
    """Per-thread default context (the reference's pipelined stages run on
    worker threads; one library context per host thread keeps them independent)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(int(os.environ.get("LIVECAP_DEVICE", "0")))
        _tls.ctx = ctx
    return ctx
