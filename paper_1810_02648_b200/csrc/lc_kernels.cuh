// Kernel declarations and the per-stream job descriptors they consume.
#pragma once
#include "lc_kinematics.cuh"

// ----- blur pyramid (imageproc.py:264-285) ---------------------------------
struct PyrJob {
    const double *src;   // H*W*C
    double *tmp;         // H*W*C
    double *dst;         // H*W*C
};
__global__ void k_blur_axis(JobArg<PyrJob> jobs, int H, int W, int C, const double *taps, int half,
                            int axis);
// all levels of an (H,W,3) image from one haloed tile per CTA (levels*H*W*3 out)
#define LC_PYR_TILE 32
#define LC_PYR_HALO 7
struct PyrAllJob {
    const double *src;   // H*W*3
    double *dst;         // levels*H*W*3
    const int *roi;      // non-null: tile_flag was decided by k_pyr_roi; null: every tile
    uint8_t *tile_flag;  // per LC_PYR_TILE^2 tile: 1 = computed (null: no flags)
};
// the pyramid's region of interest: the LC_PYR_TILE tiles within `margin`
// pixels (rounded up to whole tiles) of a foreground tile of the observed
// mask, inside the margin-dilated bounding box of its contour cells
struct PyrRoiJob {
    const int *cell_count;   // ncx*ncy contour pixels per grid cell
    int *roi;                // out: [tx0, ty0, tx1, ty1] (tx0 > tx1: empty)
    const uint8_t *fg_rows;  // H x tiles_x foreground flags (GridJob::fg_rows)
    uint8_t *tile_flag;      // out: 1 = the pyramid computes the tile
};
__global__ void k_pyr_roi(JobArg<PyrRoiJob> jobs, int ncx, int ncy, int tiles_x, int tiles_y, int margin, int H);
__global__ void k_pyramid_fused(JobArg<PyrAllJob> jobs, int H, int W, int levels, const double *taps,
                                int h0, int h1, int h2, int h3);
size_t pyramid_fused_smem();

// ----- mask contour + NN grid (imageproc.py:34-49,186-193) -----------------
struct GridJob {
    const uint8_t *mask;   // H*W
    int *row_count;        // H
    int *row_start;        // H+1
    int2 *pts;             // capacity H*W
    int *cell_count;       // ncx*ncy
    int *cell_start;       // ncx*ncy+1
    int *cell_fill;        // ncx*ncy
    int *cell_pts;         // capacity H*W
    int *K;                // out: contour pixel count
    int *cand_pts;         // ncells * LC_CAND_MAX: fixed-capacity per-cell lists of site keys y << 16 | x
    int *cand_blk;         // ncells * 32: {start, count, LC_CAND_HEAD keys}
    int *quad;             // site-count quadtree (see NnGridDev)
    int qP, qL;
    double max_u2;         // cells whose bound U^2 exceeds this keep the quadtree search
    int *cell_seed;        // ncells: a nearby site per cell (jump flooding), -1 = none
    uint8_t *fg_rows;      // H x ceil(W / LC_PYR_TILE): foreground in the row's tile segment (or null)
};
__global__ void k_contour_rows(JobArg<GridJob> jobs, int H, int W);
__global__ void k_contour_scan_rows(JobArg<GridJob> jobs, int H, int ncells);
__global__ void k_contour_emit(JobArg<GridJob> jobs, int H, int W, int ncx);
__global__ void k_contour_scan_cells(JobArg<GridJob> jobs, int ncells);
__global__ void k_contour_fill(JobArg<GridJob> jobs, int ncx);
__global__ void k_cand_build(JobArg<GridJob> jobs, int H, int W);
__global__ void k_cell_jfa(JobArg<GridJob> jobs, int ncx, int ncy);
__global__ void k_quad_build(JobArg<GridJob> jobs, int ncx, int ncy);

// ----- rasterizer (rasterizer.py:18-120) -----------------------------------
// Tile-binned rasterizer scratch.  Triangles are set up once (projection,
// inverse area, clipped bbox) into TriRec, binned into 16x16-pixel tiles,
// and every tile resolves its pixels in one pass.
#define LC_RT_TILE 16
#define LC_RT_SHIFT 4
struct TriRec {
    double P[6];   // projected vertices (x0 y0 x1 y1 x2 y2)
    double D[3];   // depths
    double inv;    // 1 / signed area
    int bb[4];     // clipped pixel bbox x0 x1 y0 y1; bb[0] > bb[1] marks a culled triangle
};
struct RasterJob {
    const double *verts;        // N*3
    unsigned long long *zbuf;   // H*W, fp64 bit patterns (+inf = empty)
    int *tri_id;                // H*W, INT_MAX = empty
    uint8_t *mask;              // H*W out (isfinite(zbuf)), may be null
    TriRec *rec;                // T
    int *tcount;                // ntiles triangles per tile
    int *toff;                  // ntiles+1 list offsets
    int *tfill;                 // ntiles append counters
    int *tlist;                 // tcap triangle ids, grouped by tile
    int tcap;
    int *ioff;                  // ntiles+1 work-item offsets (chunks of LC_RT_CHUNK triangles)
    unsigned long long *pz;     // items x 256 per-chunk partial depths (multi-chunk tiles);
    int *pid;                   // items <= 2 ntiles + tcap / LC_RT_CHUNK
};
#define LC_RT_CHUNK 256
__global__ void k_rt_clear(JobArg<RasterJob> jobs, int n);
__global__ void k_rt_setup(JobArg<RasterJob> jobs, CamDev cam, const int *tris, int T);
template <int FILL>
__global__ void k_rt_bin(JobArg<RasterJob> jobs, int T, int ntx);
__global__ void k_rt_scan(JobArg<RasterJob> jobs, int n, int T);
__global__ void k_rt_tiles(JobArg<RasterJob> jobs, CamDev cam, int T, int ntx, int nt);
__global__ void k_rt_merge(JobArg<RasterJob> jobs, CamDev cam, int ntx, int nt);
__global__ void k_raster_resolve(JobArg<RasterJob> jobs, CamDev cam, const int *tris, int mode,
                                 const double *attrs, int n_attr, const int *ids,
                                 double bg_attr, long long bg_id, double *zout, double *aout,
                                 long long *iout);

// ----- kinematics / skinning (skinning.py:206-398) -------------------------
struct FkJob {
    const double *x;     // 36
    FkState *fk;         // out
    int active;
};
__global__ void k_fk(JobArg<FkJob> jobs, const SkelDev *sk);
struct SkinJob {
    const FkState *fk;
    const double *rest;      // M*3 rest points (already gathered for subsets)
    const double *disp;      // optional N*3 displacement added to rest (may be null)
    const int *subset;       // optional M vertex ids (skinning rows); null = identity
    double *pos;             // M*3 out
    double *rot;             // M*4 out or null
    double *jac;             // M*3*36 out or null
    int M;
    int active;
};
__global__ void k_skin(JobArg<SkinJob> jobs, ActorDev A);

// ----- occluding contour + rim filter + part gating -------------------------
struct ContourJob {
    const double *verts;            // N*3
    const unsigned long long *zbuf; // H*W
    uint8_t *tri_front;             // T
    double *tri_n;                  // T*3
    uint8_t *vflag;                 // N
    int *idx;                       // N capacity
    double *n2d;                    // N*2
    int *B;                         // out count
    int *vis;                       // N capacity (visible_vertices), may be null
    int *P;                         // out count
    int active;
};
__global__ void k_tri_front(JobArg<ContourJob> jobs, ActorDev A);
__global__ void k_sil_edges(JobArg<ContourJob> jobs, ActorDev A);
__global__ void k_vis_flags(JobArg<ContourJob> jobs, ActorDev A, CamDev cam);
__global__ void k_contour_compact(JobArg<ContourJob> jobs, ActorDev A, CamDev cam);

// own-silhouette contour pixels bucketed by 16x16 cell (fixed 256 slots per
// cell, row-major within a cell): all the rim's bounded queries need
struct OwnCellsJob {
    const uint8_t *mask;       // H*W own mask
    int *cnt;                  // ncells
    int *keys;                 // ncells*256 site keys y << 16 | x
};
__global__ void k_own_cells(JobArg<OwnCellsJob> jobs, int H, int W, int ncx);

struct RimJob {
    const double *verts;       // N*3
    const int *idx;            // B
    const int *B;
    NnGridDev own;             // own-mask field (mask, grid dims)
    const int *own_cnt;        // per-cell contour counts (k_own_cells)
    const int *own_keys;       // per-cell contour keys
    uint8_t *keep;             // B out
    int stage1;                // 1: thickness probes + rigidity gate
    int active;
    // stage-2 part gating
    const int *tri_id;         // H*W winning triangle (Stage-II raster)
    int part_gate;
    int dilation;
};
__global__ void __launch_bounds__(256) k_rim(JobArg<RimJob> jobs, ActorDev A, CamDev cam, const double *probe_offs);
__global__ void k_part_labels(ActorDev A, CamDev cam, const double *verts, const int *tri_id, int dilation,
                              int *labels);

// ----- surface solve (nonrigid_stage.py:189-500) ---------------------------
struct SurfJob;
struct PoseJob;
