/*
 * livecap.h -- C-ABI of liblivecap.so, the sm_100a implementation of the
 * LiveCap pose + non-rigid Gauss-Newton hot path.
 *
 * Plain C types only (pointers + sizes).  All host pointers are owned by the
 * caller for the duration of the call and never retained; device state lives
 * inside the opaque handles.  Every entry point returns LC_OK or an error
 * code; lc_last_error() describes the last failure on the calling thread.
 * Numerical events (damping, PCG breakdown, halvings, rejected steps,
 * behind-camera points, gimbal, pruned colours, degenerate edges, snap
 * walked/reached/stuck) are report fields, never errors -- the reference's
 * convention (reference pkg/src/montrack/solvers.py:48-54,
 * pose_stage.py:407-426, nonrigid_stage.py:352-369).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/montrack/).
 */
#ifndef LIVECAP_H
#define LIVECAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LC_OK      0
#define LC_EINVAL  1   /* maps to ValueError (reference raises at construction) */
#define LC_ECUDA   2   /* maps to RuntimeError */
#define LC_ENOMEM  3   /* maps to MemoryError / RuntimeError */
#define LC_ECAP    4   /* a capacity-bounded buffer overflowed (RuntimeError) */

#define LC_MAX_JOINTS 32
#define LC_N_POSE 36
#define LC_MAX_LOG 64

typedef struct lc_ctx lc_ctx;
typedef struct lc_actor lc_actor;
typedef struct lc_tracker lc_tracker;
typedef struct lc_field lc_field;

typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
} lc_camera;   /* camera.py:20-33 */

/* Actor upload: TemplateMesh + derived connectivity, Skeleton, SkinningWeights
 * (template.py:68-256).  Derived arrays are passed exactly as the reference's
 * TemplateMesh.__post_init__ computes them (template.py:84-129). */
typedef struct {
    int32_t n_vertices, n_triangles, n_edges, n_joints;
    const double  *rest_vertices;     /* N*3 */
    const int64_t *triangles;         /* T*3 */
    const double  *vertex_colors;     /* N*3 */
    const int64_t *vertex_labels;     /* N, classes 1..7 */
    const int64_t *edges;             /* E*2, i<j, lexicographic */
    const int64_t *edge_tris;         /* E*2, -1 for open boundary */
    const int64_t *degrees;           /* N */
    const double  *directed_weights;  /* 2E material weights s_ij */
    /* skeleton */
    const int64_t *parents;           /* J */
    const double  *local_offsets;     /* J*3 */
    const int64_t *dof_joint;         /* 27 */
    const double  *dof_axes;          /* 27*3 unit */
    const double  *theta_min;         /* 27 */
    const double  *theta_max;         /* 27 */
    const double  *marker_offsets;    /* 4*3 */
    int32_t head_index;
    const int32_t *temporal_group;    /* J, index into lc_pose_hyper.group_weights */
    const int32_t *joint_parts;       /* J, body part ids (nonrigid_stage.py:55-84) */
    /* skinning */
    const int64_t *skin_indices;      /* N*4, -1 padding */
    const double  *skin_weights;      /* N*4 */
} lc_actor_desc;

typedef struct {   /* pose_stage.py:37-48 */
    double lambda_2d, lambda_3d, lambda_sil, lambda_temporal, lambda_anatomic, face_weight;
    double group_weights[8];   /* temporal weight per group id */
    int32_t gn_iterations, max_halvings;
} lc_pose_hyper;

typedef struct {   /* nonrigid_stage.py:33-49 */
    double w_photo, w_sil, w_smooth, w_edge, w_velocity, w_acceleration, tau_color;
    int32_t gn_iterations, pcg_iterations, max_halvings;
    int32_t n_levels;
    int32_t pyramid_kernels[4];
    /* optional normalized taps per level (gaussian_kernel, imageproc.py:264-273);
     * all-zero rows are computed by the library */
    double pyramid_taps[4][32];
    int32_t part_dilation;
    double snap_step;
    int32_t snap_max_steps;
    double snap_band;
} lc_nonrigid_hyper;

typedef struct {   /* pipeline.py:48-61 */
    int32_t mode;              /* 0 full, 1 pose_only, 2 detections_only */
    int32_t directional, enable_warping, enable_part_mask, enable_snapping;
    int32_t frame0_rounds, frame0_iteration_scale;
    lc_pose_hyper pose;
    lc_nonrigid_hyper nonrigid;
} lc_config;

typedef struct {   /* FrameDetections, pose_stage.py:51-64 (joints3d raw, not rescaled) */
    const double  *joints2d;   /* (J+4)*2 */
    const double  *joints3d;   /* J*3 root-relative */
    const uint8_t *valid2d;    /* J+4 */
    const uint8_t *valid3d;    /* J */
} lc_detections;

typedef struct {   /* solvers.py:97-101 */
    int32_t iterations, breakdown;
    double residual_norms[LC_MAX_LOG];
} lc_pcg_info;

typedef struct {   /* solvers.py:35-38 */
    int32_t damped;
    double damping;
} lc_dense_info;

typedef struct {   /* pose_stage.py:407-426 (one PoseIterationLog per entry) */
    int32_t n_iterations, behind_camera, gimbal;
    double energy_before[LC_MAX_LOG], energy_after[LC_MAX_LOG], step_norm[LC_MAX_LOG];
    double terms[LC_MAX_LOG][5];      /* detection2d, detection3d, silhouette, temporal, anatomic */
    int32_t halvings[LC_MAX_LOG], rejected[LC_MAX_LOG], damped[LC_MAX_LOG];
    int32_t n_contour, has_temporal;
} lc_pose_report;

typedef struct {   /* nonrigid_stage.py:352-369,409-414 */
    int32_t n_iterations, pruned, degenerate_edges, behind_camera;
    int32_t level[LC_MAX_LOG];
    double energy_before[LC_MAX_LOG], energy_after[LC_MAX_LOG];
    double terms[LC_MAX_LOG][6];      /* photo, silhouette, smooth, edge, velocity, acceleration */
    int32_t has_temporal;
    int32_t halvings[LC_MAX_LOG], rejected[LC_MAX_LOG], pcg_breakdown[LC_MAX_LOG];
    int32_t snapped, snap_walked, snap_reached, snap_stuck, snap_moved;
    int32_t n_visible, n_boundary, n_enabled;
} lc_nonrigid_report;

typedef struct {
    lc_pose_report pose;
    lc_nonrigid_report nonrigid;
    int32_t rescale_fallbacks;
} lc_frame_report;

/* Per-call problem descriptors (the reference's PoseProblem / NonrigidProblem
 * fields, pose_stage.py:284-297, nonrigid_stage.py:160-176). */
typedef struct {
    const uint8_t *mask;              /* H*W observed silhouette (DistanceField.mask) or NULL */
    const double  *joints2d;          /* (J+4)*2 */
    const double  *joints3d;          /* J*3, already bone-length rescaled */
    const uint8_t *valid2d, *valid3d;
    int32_t n_contour;
    const int64_t *contour_indices;   /* B */
    const double  *contour_normals2d; /* B*2 */
    const double  *contour_rest;      /* B*3 */
    const uint8_t *contour_enabled;   /* B or NULL */
    const double  *prev_positions;    /* J*3 or NULL */
    int32_t directional;
    lc_pose_hyper hyper;
} lc_pose_problem;

typedef struct {
    const uint8_t *mask;              /* H*W or NULL (no silhouette field) */
    int32_t n_levels;
    const double  *pyramid;           /* n_levels*H*W*3, coarse first */
    const double  *skinned;           /* N*3 V^S */
    int32_t n_visible;
    const int64_t *visible;           /* P */
    int32_t n_boundary;
    const int64_t *boundary;          /* B */
    const double  *normals2d;         /* B*2 */
    const uint8_t *enabled;           /* B */
    const double  *prev, *prev2;      /* N*3 or NULL */
    int32_t directional, enable_photo, enable_sil;
    lc_nonrigid_hyper hyper;
} lc_nonrigid_problem;

/* ---- context / errors ---- */
const char *lc_last_error(void);
int lc_version(void);
int lc_ctx_create(int32_t device, uint64_t cuda_stream, lc_ctx **out);
int lc_ctx_destroy(lc_ctx *ctx);
int lc_ctx_synchronize(lc_ctx *ctx);
/* team (thread-block cluster) sizes of the pose / surface solvers launched
 * from this context: 1, 2, 4, 8 or 16 CTAs per stream, 0 = default policy
 * (overrides LIVECAP_POSE_CLUSTER / LIVECAP_SURFACE_CLUSTER) */
int lc_ctx_set_team_sizes(lc_ctx *ctx, int32_t pose_ctas, int32_t surface_ctas);
/* blur pyramid region of interest (gaussian_pyramid, imageproc.py:276-285):
 * trackers blur only the tiles within margin_px of the observed silhouette's
 * bounding box and sample the others with the same arithmetic on demand
 * (bit-identical).  -1: every tile; -2: no tile (test hook); default 64 or
 * LIVECAP_PYR_MARGIN */
int lc_ctx_set_pyramid_margin(lc_ctx *ctx, int32_t margin_px);
int lc_kernel_launches(lc_ctx *ctx, int64_t *count);   /* kernels launched on ctx so far */
int lc_process_launches(int64_t *count);               /* kernels launched by every context of the process */

/* ---- actor (template.py:68-256; uploaded once, immutable) ---- */
int lc_actor_upload(lc_ctx *ctx, const lc_actor_desc *desc, lc_actor **out);
int lc_actor_destroy(lc_actor *actor);

/* ---- kernel-level seams ---- */
/* solvers.py:104-145 pcg_solve(BlockSparseSystem) -- explicit layout */
int lc_pcg_solve_bsr(lc_ctx *ctx, int32_t n, int64_t m, const double *diag, const double *off,
                     const int64_t *rows, const int64_t *cols, const double *rhs,
                     int32_t iterations, double *x_out, lc_pcg_info *info);
/* smooth_trajectory (pipeline.py:308-325): centred weighted average of an
 * (F, D) stack along F, truncated and renormalised at the ends; bit-identical */
int lc_smooth_trajectory(lc_ctx *ctx, int32_t F, int64_t D, const double *values, int32_t K,
                         const double *stencil, double *out);
/* metrics.iou support: per-frame |a & b| and |a | b| of two (F, HW) mask stacks */
int lc_mask_overlap(lc_ctx *ctx, int32_t F, int64_t HW, const uint8_t *a, const uint8_t *b,
                    uint64_t *inter_out, uint64_t *union_out);
/* metrics.py:26-46 mean_vertex_error, batched over F frames of (N,3) vertex
 * arrays (pred, gt: F*N*3).  indices (n_idx, ascending or any order; negative
 * = from the end) selects vertices after centring on the full clouds, NULL =
 * all.  center 0/1.  on_device: pred, gt, indices are device pointers.
 * Bit-identical to numpy (sequential axis-0 means, pairwise mean). */
int lc_mean_vertex_error(lc_ctx *ctx, int32_t F, int64_t N, const double *pred, const double *gt,
                         const int64_t *indices, int64_t n_idx, int32_t center, int32_t on_device, double *out);
/* metrics.py:49-84 umeyama_alignment + aligned_joint_error, batched over F
 * frames of M 3-D points: per frame scale, rot (3x3 row-major), t (3) and the
 * mean distance after alignment (scale/rot/t outputs may be NULL). */
int lc_aligned_error(lc_ctx *ctx, int32_t F, int32_t M, const double *pred, const double *gt,
                     int32_t with_scaling, int32_t on_device, double *scale_out, double *rot_out,
                     double *t_out, double *err_out);
/* solvers.py:41-56 dense_solve(DenseNormalSystem) */
int lc_dense_solve(lc_ctx *ctx, int32_t n, const double *a, const double *b, double *x_out,
                   lc_dense_info *info);
/* imageproc.py:264-285 gaussian_pyramid; image H*W*C, out n_levels*H*W*C */
int lc_gaussian_pyramid(lc_ctx *ctx, int32_t h, int32_t w, int32_t c, const double *image,
                        int32_t n_levels, const int32_t *kernel_sizes, const double *taps /*n_levels*32 or NULL*/,
                        double *out);
/* debug: the library's own tap / rim-probe tables (for host-side checks) */
int lc_debug_tables(int32_t size, double *taps_out, double *probe_out);
/* rasterizer.py:77-120 render_depth / render_attributes / render_vertex_ids.
 * mode 0 depth, 1 attributes (n_attr), 2 vertex ids. */
int lc_render(lc_ctx *ctx, const lc_camera *cam, int32_t n, const double *verts, int32_t t,
              const int64_t *tris, int32_t mode, const double *attrs, int32_t n_attr,
              const int64_t *ids, double bg_attr, int64_t bg_id,
              double *zbuf_out, double *attr_out, int64_t *id_out);
/* imageproc.py:177-261 DistanceField: exact nearest contour-pixel centre */
int lc_field_create(lc_ctx *ctx, int32_t h, int32_t w, const uint8_t *mask, lc_field **out);
int lc_field_destroy(lc_field *f);
int lc_field_n_contour(lc_field *f, int32_t *k);
/* imageproc.py:117-124 euclidean_dt of the field's mask (DistanceField.dt,
 * :182): H*W doubles, bit-identical to the reference */
int lc_field_dt(lc_field *f, double *out);
/* imageproc.py:52-115 _edt_squared of a feature image (nonzero = feature):
 * H*W doubles, 1e18 in rows without any feature (bit-identical) */
int lc_edt_squared(lc_ctx *ctx, int32_t h, int32_t w, const uint8_t *feature, double *out);
/* kind 0: value(dist, clamped) 1: interface 2: residual(res, grad2) 3: gradient(vec2)
 * 4: inside.  out layout: n * 4 doubles [a, b, c, flag]. */
int lc_field_query(lc_field *f, int64_t n, const double *pos, int32_t kind, double *out);
/* skinning.py:206-246 forward_kinematics */
int lc_forward_kinematics(lc_ctx *ctx, const lc_actor *actor, const double *x36,
                          double *rot_out /*J*9*/, double *pos_out /*J*3*/,
                          double *markers_out /*12*/, double *dqs_out /*J*8*/, int32_t *gimbal);
/* skinning.py:378-398 skin_points (subset may be NULL) + optional jac (M*3*36) */
int lc_skin_points(lc_ctx *ctx, const lc_actor *actor, const double *x36, int32_t m,
                   const double *rest, const int64_t *subset, double *pos_out, double *rot_out,
                   double *jac_out);
/* pose_stage.py:151-191 extract_contour_vertices (+ visibility via own raster);
 * returns indices/normals, n_out = B; capacity = N. */
int lc_contour_vertices(lc_ctx *ctx, const lc_actor *actor, const lc_camera *cam,
                        const double *verts, int32_t *n_out, int64_t *idx_out, double *n2d_out);

/* The tracker's Stage I / II index and set work on caller vertices (N*3):
 * contour indices + normals2d (capacity N), the rim keep flags (stage 1:
 * outer_rim_mask with thickness probes AND rigidity >= 2, pipeline.py:211;
 * stage 2: outer_rim_mask(min_thickness=0), AND the part gating of
 * pipeline.py:241-249 when part_gate), visible ids (stage 2; capacity N),
 * optional full part label image (H*W int32, nonrigid_stage.py:102-128). */
int lc_surface_sets(lc_ctx *ctx, const lc_actor *actor, const lc_camera *cam, const double *verts,
                    int32_t stage, int32_t part_gate, int32_t dilation, int32_t *n_contour,
                    int64_t *idx_out, double *n2d_out, uint8_t *keep_out, int32_t *n_visible,
                    int64_t *vis_out, int32_t *labels_out);

/* ---- stage solvers ---- */
/* pose_stage.py:429-459 solve_pose */
int lc_pose_solve(lc_ctx *ctx, const lc_actor *actor, const lc_camera *cam,
                  const lc_pose_problem *pb, const double *x0, double *x_out,
                  lc_pose_report *report);
/* nonrigid_stage.py:372-403 solve_nonrigid (+ optional snap_vertices :417-500) */
int lc_nonrigid_solve(lc_ctx *ctx, const lc_actor *actor, const lc_camera *cam,
                      const lc_nonrigid_problem *pb, const double *v0, int32_t do_solve,
                      int32_t do_snap, double *v_out, lc_nonrigid_report *report);

/* ---- batched multi-stream tracker (pipeline.py:263-302 solve_frame, per stream) ---- */
int lc_tracker_create(lc_ctx *ctx, const lc_actor *actor, const lc_camera *cam,
                      const lc_config *cfg, int32_t n_streams, lc_tracker **out);
int lc_tracker_destroy(lc_tracker *tr);
/* queue the next frame of one stream: image H*W*3 f64, mask H*W u8.
 * on_device != 0: pointers are device pointers (already resident in HBM).
 * Up to 3 frames may be queued per stream; host inputs are uploaded
 * asynchronously (pinned memory must stay valid until the frame is solved),
 * and a queued frame is preprocessed while the one before it is solved
 * (the reference's pipelined driver, pipeline.py:432-499). */
int lc_tracker_set_frame(lc_tracker *tr, int32_t stream, const double *image,
                         const uint8_t *mask, const lc_detections *det, int32_t on_device);
/* the same with a uint8 RGB image (real-data ingest, imageproc.py:297-299):
 * 1 byte per channel is uploaded and converted on the device as / 255.0 */
int lc_tracker_set_frame_u8(lc_tracker *tr, int32_t stream, const uint8_t *image_rgb,
                            const uint8_t *mask, const lc_detections *det, int32_t on_device);
/* condition + solve_frame for the oldest queued frame of every stream
 * (asynchronous); launches the preprocessing of the next queued frames */
int lc_tracker_step(lc_tracker *tr);
/* CUDA-graph mode: once every stream's track state is warm and frames are
 * queued one ahead, each lc_tracker_step replays one captured graph per
 * frame-queue phase (the preprocessing of the next frame, both stages, the
 * state update) instead of enqueueing its ~60 kernels; results are
 * bit-identical.  Off by default; not while tracing or kernel profiling. */
int lc_tracker_set_graph(lc_tracker *tr, int32_t on);
int lc_tracker_graph_stats(lc_tracker *tr, int64_t *graphs, int64_t *replays);
int lc_tracker_get_result(lc_tracker *tr, int32_t stream, double *pose_out, double *verts_out,
                          double *skinned_out, lc_frame_report *report);
/* developer timeline (LIVECAP_TRACE=1 at context creation): text lines
 * "lane name t_ms" for the marks recorded since the last dump */
int lc_trace_dump(lc_ctx *ctx, char *buf, int64_t cap);
/* one solve stage of the oldest queued frame of every stream, which it then
 * consumes: 1 = conditioning + Stage I, 2 = Stage II + state update, 3 = both
 * (= lc_tracker_step); a stage-1 tracker and a stage-2 tracker joined by
 * lc_tracker_pipe split solve_frame across two GPUs */
int lc_tracker_step_stage(lc_tracker *tr, int32_t stages);
/* stage handoff between two matching trackers, possibly on two GPUs (the
 * paper's pose -> non-rigid GPU-pair pipeline): what = 1 copies the solved
 * poses src -> dst, what = 2 the Stage-I track state (x_prev, x_prev2,
 * joints_prev, disp_rest, flags); peer copies ordered by events */
int lc_tracker_pipe(lc_tracker *dst, lc_tracker *src, int32_t what);
/* streaming readout (the pipelined driver's emit, pipeline.py:449-499):
 * enqueue D2H copies of the last stepped frame's pose (36) and surface
 * (N*3) on the context's stream and return immediately; the host buffers
 * (pinned for full asynchrony) hold the data once the stream passes this
 * point, so frame f can be read while frame f+1 is solved. */
int lc_tracker_get_result_async(lc_tracker *tr, int32_t stream, double *pose_out, double *verts_out);
/* TrackState injection / readout (pipeline.py:135-142); NULL pointers = None */
int lc_tracker_set_state(lc_tracker *tr, int32_t stream, const double *x_prev,
                         const double *x_prev2, const double *joints_prev,
                         const double *disp_rest, const double *v_prev, const double *v_prev2);
/* set the Stage I pose (36 doubles) the next lc_tracker_step_stage(tr, 2)
 * solves Stage II from (per-stage teacher forcing) */
int lc_tracker_set_pose(lc_tracker *tr, int32_t stream, const double *x36);
int lc_tracker_get_state(lc_tracker *tr, int32_t stream, int32_t *flags, double *x_prev,
                         double *x_prev2, double *joints_prev, double *disp_rest,
                         double *v_prev, double *v_prev2);
/* cumulative per-stream work counters of the Stage II solver (for algorithmic
 * byte accounting): [frames, gn_steps, pcg_iterations, energy_evaluations
 * (line-search trials), sum visible P, sum boundary B, sum contour pixels K, 0] */
#define LC_NCOUNTERS 8
int lc_tracker_counters(lc_tracker *tr, int32_t stream, int64_t *out);
/* per-kernel timing: CUDA events around every launch of `kernel_name` on the
 * context's stream (NULL disables); read returns total ms and launch count */
int lc_profile_kernel(lc_ctx *ctx, const char *kernel_name);
int lc_profile_read(lc_ctx *ctx, double *total_ms, int64_t *count);
/* (start, end) ms of every profiled launch after the profiling origin */
int lc_profile_intervals(lc_ctx *ctx, double *out, int64_t cap, int64_t *count);
/* introspection of a stream's last Stage II setup (tests / debugging):
 * what 0: boundary vertex ids (int64), 1: boundary enabled (as int64 0/1),
 * 2: visible vertex ids (int64), 3: normals2d (B*2 f64), 4: v_init (N*3 f64),
 * 5: V^S (N*3 f64).  n_out = element count written (rows for 0-3). */
int lc_tracker_inspect(lc_tracker *tr, int32_t stream, int32_t what, void *out, int64_t capacity,
                       int64_t *n_out);
/* %globaltimer stamps (ns) at the phase boundaries of the last pose / surface
 * solve of a stream (64 slots each; profiling aid) */
int lc_tracker_phase_times(lc_tracker *tr, int32_t stream, int64_t *pose_ns, int64_t *surf_ns);
/* device pointer of a stream's resident vertices (N*3) for zero-copy readers */
int lc_tracker_device_vertices(lc_tracker *tr, int32_t stream, uint64_t *dptr);

/* ---- synthetic-generator random stream on the device (lc_rng.cu) ----------
 * numpy Generator(PCG64) as the reference's generator draws it
 * (synthetic.py:170-203: default_rng(seed).normal / .random).  state / inc:
 * the PCG64 128-bit state and increment as {hi, lo} 64-bit words. */
/* n normals loc + scale*z into device `out` (add_clip != 0: out = clip(out +
 * noise, 0, 1), the image noise).  *consumed = draws taken (advance the
 * stream by it).  Tail samples (layer 0, libm log1p) are left for the host:
 * tails[2t] = element, tails[2t+1] = draws of the sample, tail_draws[31 t ..]
 * = its first 31 draws; the host writes them with lc_rng_scatter. */
int lc_rng_normal(lc_ctx *ctx, const uint64_t *state, const uint64_t *inc, double loc, double scale,
                  double *out, int64_t n, int32_t add_clip, int64_t *consumed, int64_t *tails,
                  uint64_t *tail_draws, int32_t max_tails, int32_t *n_tails);
/* n doubles of Generator.random() into device `out` (consumes n draws) */
int lc_rng_uniform(lc_ctx *ctx, const uint64_t *state, const uint64_t *inc, double *out, int64_t n);
/* device out[idx[k]] = v[k] / host out[k] = device src[idx[k]] (host idx, v) */
int lc_rng_scatter(lc_ctx *ctx, const int64_t *idx, const double *v, int32_t n, double *out);
int lc_rng_gather(lc_ctx *ctx, const int64_t *idx, int32_t n, const double *src, double *out);
/* the device's ziggurat tables (numpy's ki_double / wi_double / fi_double) */
int lc_rng_tables(uint64_t *ki, double *wi, double *fi);

#ifdef __cplusplus
}
#endif
#endif
