// Host-side runtime objects behind the C-ABI handles.
#pragma once
#include <cuda_runtime.h>
#include <string>
#include <map>
#include <vector>
#include "livecap.h"
#include "lc_pose.cuh"
#include "lc_bsr.cuh"

struct DevArena {
    std::vector<void *> ptrs;
    template <typename T>
    T *alloc(size_t count) {
        void *p = nullptr;
        if (count == 0) count = 1;
        if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) throw std::bad_alloc();
        ptrs.push_back(p);
        return static_cast<T *>(p);
    }
    template <typename T>
    T *upload(const T *host, size_t count, cudaStream_t st) {
        T *d = alloc<T>(count);
        if (count) cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, st);
        return d;
    }
    void release() {
        for (void *p : ptrs) cudaFree(p);
        ptrs.clear();
    }
    ~DevArena() { release(); }
};

struct lc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // auxiliary stream for work independent of Stage I (pyramid, observed grid)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_obs = nullptr, ev_pyr = nullptr;
    // host->device uploads of queued frames (copy engine, overlaps both)
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_pipe = nullptr;   // cross-device handoff point (lc_tracker_pipe)
    struct JobRing *ring = nullptr;  // descriptor staging ring (owned)
    // optional timeline (LIVECAP_TRACE=1): timing events at phase boundaries
    bool tracing = false;
    struct Mark { const char *name; int lane; cudaEvent_t ev; };
    std::vector<Mark> marks;
    long long launches = 0;
    // optional per-kernel timing: CUDA events around every launch of `prof_name`
    std::string prof_name;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    cudaEvent_t prof_ref = nullptr;   // recorded when profiling starts (interval origin)
    struct Slot *call_slot = nullptr;          // scratch slot for single-call entry points
    const lc_actor *call_actor = nullptr;
    int call_w = 0, call_h = 0;
    // team (thread-block cluster) sizes of the two solvers; 0 = default policy
    int pose_cs = 0, surf_cs = 0;
    // blur pyramid region of interest: tiles within this many pixels of the
    // observed silhouette's bounding box (INT_MIN: LIVECAP_PYR_MARGIN or 64;
    // -1: every tile; -2: none, every sample on the exact on-demand path)
    int pyr_margin = INT_MIN;
    // a tracker step is being captured into a CUDA graph: events that order
    // work across steps become external event record / wait nodes
    bool capturing = false;
    cudaEvent_t ev_join = nullptr;   // the auxiliary stream rejoins the captured stream
    // lc_rng_normal's scratch, kept across calls (grow-only)
    struct RngScratch {
        DevArena mem;
        long long M = 0;
        int mt = 0;
        size_t tb1 = 0, tb2 = 0;
        uint64_t *u = nullptr, *ddraws = nullptr;
        double *val = nullptr;
        int *len = nullptr, *n_slow = nullptr, *sst = nullptr, *err = nullptr, *nt = nullptr;
        unsigned char *kind = nullptr, *start = nullptr, *flag = nullptr;
        long long *num = nullptr, *slow = nullptr, *cons = nullptr, *dtails = nullptr;
        void *tmp1 = nullptr, *tmp2 = nullptr;
    } *rng = nullptr;
};

// device allocation list owned by an object

struct lc_actor {
    lc_ctx *ctx = nullptr;
    DevArena mem;
    ActorDev dev{};
    SkelDev skel{};
    SkelDev *skel_dev = nullptr;
    std::vector<int> host_edges;      // E*2
    std::vector<int> host_degrees;    // N
    std::vector<double> host_wdir;    // 2E
    std::vector<int> host_ell_edge;   // LC_ELL*N edge id per ELL slot (-1 = empty)
};

// NN grid buffers for one mask
struct GridBufs {
    int *row_count, *row_start, *cell_count, *cell_start, *cell_fill, *cell_pts, *K;
    int2 *pts;
    int *cand_pts;
    int *cand_blk;
    int *cell_seed;
    int *quad;
    int qP, qL;
    uint8_t *fg_rows;   // H x ceil(W / LC_PYR_TILE): any foreground in the row's 32-px segment
};

#define LC_QUEUE 3   // queued frames per tracker stream (solve, preprocess, upload)

// One queued frame of a tracker stream: inputs plus their preprocessing
// products (pipeline.py:156-162).  A stream has two, so the next frame can be
// uploaded and preprocessed while the current one is solved (the
// reference's pipelined driver, pipeline.py:432-499); a third lets the
// upload of frame f+2 overlap frame f+1's preprocessing and frame f's solve.
struct FrameIn {
    double *image = nullptr;           // own copy (host inputs)
    uint8_t *image_u8 = nullptr;       // raw RGB bytes of the uint8 upload path
    uint8_t *mask = nullptr;
    const double *image_src = nullptr;  // own copy or the caller's device pointer
    const uint8_t *mask_src = nullptr;
    double *pyr = nullptr;
    uint8_t *pyr_tile = nullptr;       // per pyramid tile: computed (1) or left to the on-demand path (0)
    int *pyr_roi = nullptr;            // [tx0, ty0, tx1, ty1] the pyramid's region of interest
    double *tmp = nullptr;             // blur scratch (the slot's, shared by its queue)
    GridBufs obs{};
    double *j2d = nullptr, *j3d_raw = nullptr;
    uint8_t *v2d = nullptr, *v3d = nullptr;
    cudaEvent_t ready_obs = nullptr;   // observed-silhouette grid built (aux stream)
    cudaEvent_t ready = nullptr;       // all preprocessing done (aux stream)
    cudaEvent_t freed = nullptr;       // last solve that read this buffer done (main stream)
    cudaEvent_t uploaded = nullptr;    // host inputs copied (copy stream)
    bool pending_upload = false;
    bool has_image = true;             // false: mask + detections only (a Stage-I-only tracker)
    bool used = false;                 // `freed` has been recorded at least once
    int state = 0;                     // 0 empty, 1 staged, 2 preprocessing launched
};

// per-stream device state + scratch
struct Slot {
    DevArena mem;
    int N = 0, T = 0, E = 0, H = 0, W = 0, levels = 0;
    // frame inputs
    double *image = nullptr;          // H*W*3 (own copy)
    const double *image_src = nullptr; // resident source (own copy or caller's device pointer)
    uint8_t *mask = nullptr;          // H*W
    const uint8_t *mask_src = nullptr;
    double *pyr = nullptr, *blur_tmp = nullptr;
    uint8_t *pyr_tile = nullptr;
    int *pyr_roi = nullptr;
    GridBufs obs{}, own{};
    uint8_t *own_mask = nullptr;
    int *own_cnt = nullptr, *own_keys = nullptr;   // own-silhouette contour buckets (rim)
    // detections
    double *j2d, *j3d_raw, *j3d;
    uint8_t *v2d, *v3d;
    int *fallbacks;
    // state (TrackState)
    double *x_prev, *x_prev2, *joints_prev, *disp, *v_prev, *v_prev2;
    bool has_prev = false, has_prev2 = false, has_vprev = false, has_vprev2 = false, has_disp = false;
    // per-frame
    double *x, *x0, *drest, *model, *vs, *rot, *vinit, *v;
    FkState *fk;
    unsigned long long *zbuf;
    int *tri_id;
    // tile-binned raster scratch (RasterJob)
    TriRec *rt_rec;
    int *rt_diff, *rt_off, *rt_fill, *rt_list, *rt_ioff, *rt_pid;
    unsigned long long *rt_pz;
    int rt_cap = 0;
    uint8_t *tri_front, *vflag, *enabled;
    double *tri_n, *n2d, *crest;
    int *cidx, *B, *vis, *P;
    int *nn_hint;
    // surface scratch
    double *diag, *minv, *rhs, *sx, *sr, *sz, *sp, *sap, *sbest, *edir, *eg, *off0, *off1;
    double *ell_d, *ell_g;   // 3*LC_ELL*N current edge directions / signed gradients in ELL slots (SoA)
    uint8_t *hold;
    // reports (device)
    lc_pose_report *pose_rep;
    lc_nonrigid_report *nr_rep;
    long long *counters;   // LC_NCOUNTERS cumulative work counters (device)
    long long *phase_pose, *phase_surf;   // LC_NPHASE timestamps of the last solves
    // tracker input queue, a ring of LC_QUEUE frames (in[0] aliases the buffers above)
    FrameIn in[LC_QUEUE];
    int in_head = 0, in_tail = 0;
    void allocate(int N_, int T_, int E_, int H_, int W_, int levels_, int J);
    void allocate_queue();
    void view(const FrameIn &f);
    ~Slot();
};

struct lc_field {
    lc_ctx *ctx = nullptr;
    DevArena mem;
    int H = 0, W = 0;
    uint8_t *mask = nullptr;
    GridBufs g{};
    int K = 0;
};

struct ConfigDev {
    DevArena mem;
    EdgeConstDev ec{};
    SurfHyperDev shp{};
    PoseHyperDev php{};
    double *taps = nullptr;   // levels * 32
    int half[4] = {0, 0, 0, 0};
    double *probe = nullptr;  // 128*2
};

struct lc_tracker {
    lc_ctx *ctx = nullptr;
    const lc_actor *actor = nullptr;
    lc_camera cam{};
    lc_config cfg{};
    int S = 0;
    std::vector<Slot *> slots;
    ConfigDev conf;
    DevArena mem;
    // device job arrays (rebuilt when needed)
    void *jobs_dev = nullptr;
    size_t jobs_bytes = 0;
    int frame_counter = 0;
    // CUDA-graph mode (lc_tracker_set_graph): steady-state steps replay one
    // captured graph per frame-queue phase
    bool graph_mode = false;
    struct Graph { cudaGraphExec_t exec = nullptr, exec_aux = nullptr; long long kernels = 0; };
    std::map<std::vector<long long>, Graph> graphs;
    long long graph_replays = 0;
};
