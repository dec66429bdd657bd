// Job descriptors of the two persistent stage solvers.
#pragma once
#include "livecap.h"
#include "lc_kernels.cuh"

struct PoseJob {
    int active;
    const double *x0;
    double *x_out;
    NnGridDev obs;            // observed-silhouette field (K read from obs_K)
    const int *obs_K;
    int has_field;
    const int *B;             // contour count (device)
    const int *cidx;          // B contour vertex ids
    const double *n2d;        // B*2
    const double *crest;      // B*3 gathered rest points, or null -> drest[cidx]
    const double *drest;      // N*3 displaced rest
    const uint8_t *enabled;   // B or null
    const double *j2d, *j3d;  // detections (j3d rescaled)
    const uint8_t *v2d, *v3d;
    const double *prev_pos;   // J*3 or null
    PoseHyperDev hp;
    int directional;
    lc_pose_report *report;
    int log_offset;
    long long *phase;         // LC_NPHASE timestamps (or null)
    int *nn_hint;             // B: last nearest contour pixel per silhouette row (or null)
    FkState *fk_out;          // FK of x_out at exit (rank 0; null: not written)
};

struct SurfJob {
    int active;
    int do_solve, do_snap;
    const double *v0;         // N*3 start
    double *v;                // N*3 result
    const double *vs;         // N*3 skinned V^S
    const double *pyr;        // levels*H*W*3
    const uint8_t *pyr_tile;  // per pyramid tile: 1 = computed; null: every tile is
    const double *image;      // H*W*3 raw frame (the on-demand blur of uncomputed tiles)
    NnGridDev obs;
    const int *obs_K;
    int has_field;
    const int *vis;           // P visible ids
    const int *P;
    const int *bidx;          // B boundary ids
    const int *B;
    const double *n2d;        // B*2
    const uint8_t *enabled;   // B
    const double *prev, *prev2;
    int directional, enable_photo, enable_sil;
    // scratch
    double *diag;             // N*6 (sym: xx xy xz yy yz zz)
    double *minv;             // N*9 np.linalg.inv of each diagonal block
    double *rhs, *x, *r, *z, *p, *ap, *best;   // N*3
    double *edir, *eg;        // E*3
    double *ell_d, *ell_g;    // 3*LC_ELL*N edge direction / signed gradient per ELL slot (SoA)
    double *off0, *off1;      // N*3 snap offsets
    uint8_t *hold;            // N
    lc_nonrigid_report *report;
    int *nn_hint;             // B: last nearest contour pixel per boundary row (or null)
    long long *counters;      // cumulative: frames, gn, pcg iters, trials, P, B, K (or null)
    long long *phase;         // LC_NPHASE timestamps (or null)
};

template <int CS>
__global__ void k_pose_solve_t(JobArg<PoseJob> jobs, const SkelDev *skg, ActorDev A, CamDev cam);
size_t pose_smem_bytes(int n_joints);
int pose_block_threads();

template <int CS>
__global__ void k_surface_solve_t(JobArg<SurfJob> jobs, ActorDev A, CamDev cam, EdgeConstDev ec,
                                  SurfHyperDev hp, int H, int W, int pcg_mode);
int surface_block_threads();
int surface_pcg_mode(int N, int cs, size_t *smem_bytes);
