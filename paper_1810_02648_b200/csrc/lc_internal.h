// Internal host/device layout of liblivecap (not part of the C-ABI).
//
// HBM layout (all fp64 AoS (.,3) like the reference's numpy arrays, int32
// indices):
//   actor tables   : uploaded once per actor, shared by every stream
//   stream slots   : per capture stream, resident for the tracker's life
//                    (pyramid, observed-contour grid, state, scratch)
#pragma once
#include <cstdint>

#define LC_MAXJ 32
#define LC_NDOF 27
#define LC_NROT 30       // 3 root Euler + 27 joint angles
#define LC_NP 36
#define LC_ELL 8  // ELL adjacency slots per vertex
#define LC_GRID_CELL 16  // NN grid cell edge in pixels
#define LC_GRID_SHIFT 4
#define LC_NCOUNTERS 8

struct SkelDev {
    int J, head, n_tree_levels;
    int parents[LC_MAXJ];
    double off[LC_MAXJ][3];
    double rest[LC_MAXJ][3];
    int dof_joint[LC_NDOF];
    double dof_axes[LC_NDOF][3];
    double tmin[LC_NDOF], tmax[LC_NDOF];
    double marker[4][3];
    unsigned moves_pos[LC_NDOF];    // bit j: dof k moves joint position j
    unsigned moves_frame[LC_NDOF];  // bit j: dof k moves joint frame j
    int dof_start[LC_MAXJ + 1];     // dofs of joint i: dof_list[dof_start[i]..dof_start[i+1])
    int dof_list[LC_NDOF];
    int level_start[LC_MAXJ + 1];   // FK schedule: joints grouped by tree depth
    int level_joint[LC_MAXJ];
    int group[LC_MAXJ];
    int joint_part[LC_MAXJ];
};

struct ActorDev {
    int N, T, E, J;
    const double *rest;        // N*3
    const int *tris;           // T*3
    const double *colors;      // N*3
    const int *edges;          // E*2
    const int *edge_tris;      // E*2
    const double *rest_len;    // E
    const double *rest_dir;    // E*3 unit rest direction (degenerate-edge fallback)
    const int *adj_ptr;        // N+1 : incident undirected edges per vertex, in the
    const int *adj_edge;       //       reference's directed order (as src: forward
    const int *adj_nbr;        //       edges asc., then reversed edges asc.)
    const int *degrees;        // N
    // ELL copy of the first LC_ELL incident edges of each vertex (slot k of
    // vertex i at k*N + i, the CSR order above): coalesced and independent
    // loads in the assembly / matvec; degrees beyond LC_ELL use the CSR tail
    const int *ell_nbr;        // LC_ELL*N neighbour vertex
    const int *ell_cnt;        // N incident edge count (= CSR degree)
    const int *epos;           // 2E ELL position of edge e at its src (2e) / dst (2e+1), -1 = CSR tail
    int n_heavy;               // vertices with more than LC_ELL incident edges (poles)
    const int *heavy;          // n_heavy ascending vertex ids
    const int *heavy_id;       // N: index into `heavy`, -1 for ELL-only vertices
    const double *w_dir;       // 2E directed material weights
    const int *skin_idx;       // N*4 (-1 padding)
    const double *skin_w;      // N*4
    const int *dominant;       // N
    const int *vt_ptr;         // N+1 : incident triangles in (slot, triangle) order
    const int *vt_tri;
    const double *rigidity;    // N (Table-1 class weight)
    const int *vpart;          // N body part of the dominant joint
    const SkelDev *skel;
};

struct CamDev {
    double fx, fy, cx, cy;
    int W, H;
};

// exact nearest-contour index over one mask
struct NnGridDev {
    int K;                 // contour pixels
    int W, H, ncx, ncy;
    const int2 *pts;       // K (x, y), np.argwhere row-major order
    const int *cell_start; // ncx*ncy+1
    const int *cell_pts;   // point ids grouped by cell
    const uint8_t *mask;   // H*W, for inside()
    // exact per-cell candidate lists (fixed capacity LC_CAND_MAX per cell)
    const int *cand_pts;    // per-cell lists of site keys y << 16 | x (16 B aligned)
    // per-cell 128 B blocks: {list start, list count, first LC_CAND_HEAD keys}
    // so a query gets its cell's range and the head of its list in one line
    const int *cand_blk;
    // site-count quadtree over the cells padded to qP x qP (qP = 2^qL):
    // level l (leaves l = 0) stores (qP>>l)^2 counts at offset quad_off(l)
    const int *quad;
    int qP, qL;
};
__host__ __device__ __forceinline__ int quad_off(int P, int l) {
    int o = 0;
    for (int k = 0; k < l; ++k) o += (P >> k) * (P >> k);
    return o;
}
#define LC_CAND_MAX 1024       // per-cell cap before falling back to the ring search
#define LC_CAND_HEAD 30        // keys stored inline in each cell's 128 B block

// per-config constants of the surface energy
struct EdgeConstDev {
    const double *cs_f, *cs_r;  // E : sqrt(w_smooth s / deg(src)) forward / reversed half
    const double *ce_f, *ce_r;  // E : sqrt(w_edge s / deg(src))
    const double *alpha;        // E : cs_f^2 + cs_r^2
    const double *beta;         // E : ce_f^2 + ce_r^2
    const double *ell_a, *ell_b; // LC_ELL*N alpha / beta gathered into the ELL slots
};

struct PoseHyperDev {
    double l2d, l3d, lsil, ltemp, lanat, face;
    double tw[LC_MAXJ];   // lambda-free temporal group weight per joint
    int gn, max_halvings;
    int first_trials;     // line-search trials evaluated in the first batch (then 4 at a time)
};

struct SurfHyperDev {
    double w_photo, w_sil, w_smooth, w_edge, w_vel, w_acc, tau;
    int gn, pcg, max_halvings, n_levels, dilation;
    double snap_step, snap_band;
    int snap_max_steps;
    int first_trials;     // line-search trials evaluated in the first batch
    int next_trials;      // ... and in each later batch
    const double *taps;   // levels*32 pyramid taps (for the on-demand blur outside the pyramid's region)
    int half[4];
};

// Job descriptors of a batched launch, passed by value as a kernel parameter
// (up to LC_JOB_INLINE streams; larger batches use a device array staged by
// k_stage).  Parameters live in the constant bank, so no copy engine and no
// extra launch is needed to get them to the device.
#define LC_JOB_INLINE 8
template <typename T>
struct JobArg {
    const T *ptr;              // device array (n > LC_JOB_INLINE), else null
    int n;
    T inl[LC_JOB_INLINE];
    __host__ __device__ __forceinline__ const T &operator[](int i) const { return ptr ? ptr[i] : inl[i]; }
};

// Programmatic dependent launch: kernels are launched with
// programmaticStreamSerialization, so a kernel's CTAs may be scheduled
// before the previous kernel on the stream has finished; every kernel waits
// here for that grid's completion (and memory flush) before touching its
// inputs.  This hides the launch latency between the many short kernels of
// a frame.
__device__ __forceinline__ void lc_pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef LC_PDL_EARLY_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
#endif
}
