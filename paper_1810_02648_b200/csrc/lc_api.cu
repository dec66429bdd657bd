// C-ABI entry points (include/livecap.h) and the host runtime that schedules
// the kernels: actor upload, per-stream slots, the per-frame stage schedule
// of solve_frame (reference pipeline.py:156-302) batched over streams, and
// the single-call seams used by the Python mirror of the reference API.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>
#include "lc_runtime.h"
#include "lc_rng.cuh"

// ---------------------------------------------------------------------------
// errors

struct ApiError : std::exception {
    std::string m;
    explicit ApiError(std::string s) : m(std::move(s)) {}
    const char *what() const noexcept override { return m.c_str(); }
};
static void require(bool ok, const char *msg) {
    if (!ok) throw ApiError(msg);
}

static thread_local std::string g_err;
// kernels launched by every context of the process (contexts are per host
// thread; the reference's pipelined driver solves on worker threads)
static std::atomic<long long> g_launches{0};

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(expr)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess) return fail(LC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define API_BEGIN try {
#define API_END                                                                            \
    }                                                                                      \
    catch (const std::bad_alloc &) { return fail(LC_ENOMEM, "device allocation failed"); } \
    catch (const std::exception &ex) { return fail(LC_EINVAL, ex.what()); }


// programmatic dependent launch for every kernel (LIVECAP_NO_PDL=1 disables)
static bool lc_pdl_enabled() {
    static const bool on = getenv("LIVECAP_NO_PDL") == nullptr;
    return on;
}

template <typename K, typename... Args>
static void launch_named(const char *name, lc_ctx *c, K kernel, dim3 g, dim3 b, size_t smem, Args... args) {
    if (g.x == 0 || g.y == 0 || g.z == 0) return;   // empty batch / empty mesh
    const bool prof = !c->prof_name.empty() && c->prof_name == name;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, c->stream);
    }
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = g;
        cfg.blockDim = b;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = lc_pdl_enabled() ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kernel, args...);
    }
    if (prof) {
        cudaEventRecord(e1, c->stream);
        c->prof_events.push_back({e0, e1});
    }
    c->launches++;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw ApiError(std::string("launch of ") + name + " failed: " + cudaGetErrorString(e));
    }
}
#define launch(c, kernel, ...) launch_named(#kernel, c, kernel, __VA_ARGS__)

// timeline marks (LIVECAP_TRACE=1): an event with timing on the context's
// current stream; lane 0 = solve stream, 1 = auxiliary, 2 = copy
static void mark(lc_ctx *c, const char *name) {
    if (!c->tracing) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->stream);
    const int lane = c->stream == c->aux ? 1 : (c->stream == c->copy ? 2 : 0);
    c->marks.push_back({name, lane, e});
}

// temporarily route a context's launches to another stream
struct OnStream {
    lc_ctx *c;
    cudaStream_t saved;
    OnStream(lc_ctx *c_, cudaStream_t s) : c(c_), saved(c_->stream) { c->stream = s; }
    ~OnStream() { c->stream = saved; }
};

// cluster launch: `streams` teams of `cs` CTAs (one thread-block cluster per stream)
template <typename... KArgs, typename... Args>
static void launch_cluster(const char *name, lc_ctx *c, void (*kernel)(KArgs...), int streams, int cs,
                           dim3 block, size_t smem, Args... args) {
    if (streams <= 0) return;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(streams * cs);
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = lc_pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const bool prof = !c->prof_name.empty() && c->prof_name == name;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, c->stream);
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
    if (prof) {
        cudaEventRecord(e1, c->stream);
        c->prof_events.push_back({e0, e1});
    }
    c->launches++;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e == cudaSuccess) e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw ApiError(std::string("cluster launch of ") + name + " failed: " + cudaGetErrorString(e));
    }
}

// per-solver override (LIVECAP_POSE_CLUSTER / LIVECAP_SURFACE_CLUSTER), else LIVECAP_CLUSTER
static int cluster_size_for(const char *var) {
    const char *v = getenv(var);
    if (!v) return -1;
    const int x = atoi(v);
    return (x == 1 || x == 2 || x == 4 || x == 8 || x == 16) ? x : -1;
}

static int cluster_size() {
    static int cs = [] {
        const char *v = getenv("LIVECAP_CLUSTER");
        int x = v ? atoi(v) : 4;
        return (x == 1 || x == 2 || x == 4 || x == 8 || x == 16) ? x : 4;
    }();
    return cs;
}

static int last_launch_status() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(LC_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    return LC_OK;
}

extern "C" const char *lc_last_error(void) { return g_err.c_str(); }
extern "C" int lc_version(void) { return 1; }

// ---------------------------------------------------------------------------
// job staging: small per-launch descriptor arrays copied H2D in stream order

// Job descriptors reach the device as kernel parameters: a one-CTA
// k_stage launch carries the bytes by value and writes them into a device
// ring slot (or a given buffer) in stream order.  No copy engine is
// involved, so descriptor staging never queues behind a large host upload
// of a queued frame (which would stall the solve for the whole transfer),
// and the host never blocks.  Before the ring wraps, the streams are
// drained so no pending kernel still reads a slot.
template <int CAP>
struct StageBlob { uint4 w[CAP / 16]; };

template <int CAP>
__global__ void k_stage(unsigned char *dst, int bytes, StageBlob<CAP> blob) {
    lc_pdl_wait();
    const unsigned char *src = reinterpret_cast<const unsigned char *>(blob.w);
    const bool vec = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    const int nv = vec ? bytes / 16 : 0;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) reinterpret_cast<uint4 *>(dst)[i] = blob.w[i];
    for (int i = 16 * nv + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

template <int CAP>
static void stage_launch(cudaStream_t st, void *dst, const void *src, size_t bytes) {
    StageBlob<CAP> b;
    std::memcpy(b.w, src, bytes);
    k_stage<CAP><<<1, 128, 0, st>>>(static_cast<unsigned char *>(dst), (int)bytes, b);
}

static void stage_bytes(cudaStream_t st, void *dst, const void *src, size_t bytes) {
    if (bytes <= 512) stage_launch<512>(st, dst, src, bytes);
    else if (bytes <= 4096) stage_launch<4096>(st, dst, src, bytes);
    else if (bytes <= 16384) stage_launch<16384>(st, dst, src, bytes);
    else {
        for (size_t o = 0; o < bytes; o += 16384)
            stage_launch<16384>(st, static_cast<char *>(dst) + o, static_cast<const char *>(src) + o,
                                std::min<size_t>(16384, bytes - o));
    }
}

struct JobRing {
    char *dev = nullptr;
    size_t cap = 0, off = 0;
    cudaStream_t main = nullptr, aux = nullptr;
    void *put(cudaStream_t st, const void *src, size_t bytes, void *dst = nullptr) {
        void *d = dst;
        if (!d) {
            const size_t padded = (bytes + 255) & ~size_t(255);
            if (padded > cap) throw ApiError("job descriptor larger than the staging ring");
            if (off + padded > cap) {
                cudaStreamSynchronize(st);
                cudaStreamSynchronize(main);
                if (aux) cudaStreamSynchronize(aux);
                off = 0;
            }
            d = dev + off;
            off += padded;
        }
        stage_bytes(st, d, src, bytes);
        return d;
    }
};
static JobRing &ring_of(lc_ctx *c) {
    if (!c->ring) {
        JobRing *jr = new JobRing();
        jr->cap = 16 << 20;
        jr->main = c->stream;
        jr->aux = c->aux;
        if (cudaMalloc(&jr->dev, jr->cap) != cudaSuccess) {
            delete jr;
            throw std::bad_alloc();
        }
        c->ring = jr;
    }
    return *c->ring;
}
template <typename T>
static JobArg<T> stage(lc_ctx *c, const std::vector<T> &v) {
    JobArg<T> a{};
    a.n = (int)v.size();
    if (v.size() <= LC_JOB_INLINE) {
        a.ptr = nullptr;
        for (size_t i = 0; i < v.size(); ++i) a.inl[i] = v[i];
    } else {
        a.ptr = static_cast<const T *>(ring_of(c).put(c->stream, v.data(), v.size() * sizeof(T)));
    }
    return a;
}
// small host array -> existing device buffer, in stream order
static void stage_to(lc_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes) ring_of(c).put(c->stream, src, bytes, dst);
}

// ---------------------------------------------------------------------------
// context

extern "C" int lc_ctx_create(int32_t device, uint64_t cuda_stream, lc_ctx **out) {
    API_BEGIN
    require(out != nullptr, "out is null");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, "device ordinal out of range");
    CK(cudaSetDevice(device));
    lc_ctx *c = new lc_ctx();
    c->device = device;
    // the solve stream gets the highest priority and the preprocessing
    // (auxiliary) stream the lowest, so queued-frame preprocessing fills the
    // SMs the solve leaves idle instead of delaying its cluster launches
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    if (cuda_stream) {
        c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    } else {
        CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi));
        c->own_stream = true;
    }
    CK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, prio_lo));
    CK(cudaStreamCreateWithPriority(&c->copy, cudaStreamNonBlocking, prio_lo));
    c->tracing = getenv("LIVECAP_TRACE") != nullptr;
    CK(cudaEventCreateWithFlags(&c->ev_pipe, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_obs, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_pyr, cudaEventDisableTiming));
    {
        const int sm = (int)pose_smem_bytes(LC_MAXJ);
        CK(cudaFuncSetAttribute(k_pose_solve_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_pose_solve_t<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_pose_solve_t<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_pose_solve_t<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_pose_solve_t<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_pose_solve_t<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(k_surface_solve_t<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        for (auto k : {k_surface_solve_t<1>, k_surface_solve_t<2>, k_surface_solve_t<4>, k_surface_solve_t<8>,
                       k_surface_solve_t<16>})
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024));
        CK(cudaFuncSetAttribute(k_pyramid_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pyramid_fused_smem()));
    }
    *out = c;
    return LC_OK;
    API_END
}

extern "C" int lc_ctx_destroy(lc_ctx *c) {
    if (!c) return LC_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    delete c->call_slot;
    cudaStreamSynchronize(c->aux);
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->aux);
    cudaStreamDestroy(c->copy);
    cudaEventDestroy(c->ev_fork);
    if (c->ev_pipe) cudaEventDestroy(c->ev_pipe);
    if (c->ring) {
        cudaFree(c->ring->dev);
        delete c->ring;
        c->ring = nullptr;
    }
    cudaEventDestroy(c->ev_obs);
    cudaEventDestroy(c->ev_pyr);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    delete c->rng;
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return LC_OK;
}

// timeline dump: one line per mark "lane name t_ms" (t relative to the first mark), marks cleared
extern "C" int lc_trace_dump(lc_ctx *c, char *buf, int64_t cap) {
    require(c && buf && cap > 0, "null argument");
    cudaDeviceSynchronize();
    std::string out;
    if (!c->marks.empty()) {
        for (auto &m : c->marks) {
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, c->marks[0].ev, m.ev);
            char line[160];
            snprintf(line, sizeof line, "%d %s %.4f\n", m.lane, m.name, ms);
            out += line;
        }
        for (auto &m : c->marks) cudaEventDestroy(m.ev);
        c->marks.clear();
    }
    const size_t n = std::min<size_t>(out.size(), (size_t)cap - 1);
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
    return LC_OK;
}

extern "C" int lc_ctx_synchronize(lc_ctx *c) {
    require(c != nullptr, "null ctx");
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamSynchronize(c->aux));
    CK(cudaStreamSynchronize(c->copy));
    return last_launch_status();
}

extern "C" int lc_profile_kernel(lc_ctx *c, const char *name) {
    if (!c) return fail(LC_EINVAL, "null ctx");
    cudaStreamSynchronize(c->stream);
    for (auto &p : c->prof_events) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    c->prof_events.clear();
    c->prof_name = name ? name : "";
    if (!c->prof_ref) cudaEventCreate(&c->prof_ref);
    cudaEventRecord(c->prof_ref, c->stream);
    return LC_OK;
}

// (start, end) of every profiled launch in ms after the profiling origin
// (the event recorded by lc_profile_kernel on this context's stream): with
// several contexts profiled right after a device-wide synchronisation the
// origins coincide, so the intervals of concurrent launches can be unioned
extern "C" int lc_profile_intervals(lc_ctx *c, double *out, int64_t cap, int64_t *count) {
    if (!c || !out || !count) return fail(LC_EINVAL, "null argument");
    CK(cudaStreamSynchronize(c->stream));
    int64_t n = 0;
    for (auto &p : c->prof_events) {
        if (n >= cap) break;
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, c->prof_ref, p.first));
        CK(cudaEventElapsedTime(&b, c->prof_ref, p.second));
        out[2 * n] = a;
        out[2 * n + 1] = b;
        ++n;
    }
    *count = n;
    return LC_OK;
}

extern "C" int lc_profile_read(lc_ctx *c, double *total_ms, int64_t *count) {
    if (!c || !total_ms || !count) return fail(LC_EINVAL, "null argument");
    CK(cudaStreamSynchronize(c->stream));
    double tot = 0.0;
    for (auto &p : c->prof_events) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p.first, p.second));
        tot += ms;
    }
    *total_ms = tot;
    *count = (int64_t)c->prof_events.size();
    return LC_OK;
}

extern "C" int lc_process_launches(int64_t *count) {
    if (!count) return fail(LC_EINVAL, "null argument");
    *count = (int64_t)g_launches.load(std::memory_order_relaxed);
    return LC_OK;
}

extern "C" int lc_kernel_launches(lc_ctx *c, int64_t *count) {
    if (!c || !count) return fail(LC_EINVAL, "null argument");
    *count = c->launches;
    return LC_OK;
}

// ---------------------------------------------------------------------------
// actor upload (template.py:68-256 layout -> device tables)

static const double kClassWeight[8] = {0.0, 1.0, 2.0, 2.5, 3.0, 50.0, 100.0, 200.0};

extern "C" int lc_actor_upload(lc_ctx *c, const lc_actor_desc *d, lc_actor **out) {
    API_BEGIN
    require(c && d && out, "null argument");
    const int N = d->n_vertices, T = d->n_triangles, E = d->n_edges, J = d->n_joints;
    require(N > 0 && T >= 0 && E >= 0, "mesh needs vertices");
    require(J > 0 && J <= LC_MAXJ, "skeleton must have 1..32 joints");
    require(d->head_index >= 0 && d->head_index < J, "head index out of range");
    CK(cudaSetDevice(c->device));
    lc_actor *a = new lc_actor();
    a->ctx = c;
    cudaStream_t st = c->stream;

    // ---- skeleton
    SkelDev &s = a->skel;
    std::memset(&s, 0, sizeof(s));
    s.J = J;
    s.head = d->head_index;
    for (int i = 0; i < J; ++i) {
        s.parents[i] = (int)d->parents[i];
        require(i == 0 ? s.parents[i] == -1 : (s.parents[i] >= 0 && s.parents[i] < i),
                "parents must precede children with a single root");
        for (int k = 0; k < 3; ++k) s.off[i][k] = d->local_offsets[3 * i + k];
        for (int k = 0; k < 3; ++k)
            s.rest[i][k] = s.off[i][k] + (i > 0 ? s.rest[s.parents[i]][k] : 0.0);
        s.group[i] = d->temporal_group ? d->temporal_group[i] : 0;
        s.joint_part[i] = d->joint_parts ? d->joint_parts[i] : 1;
    }
    for (int k = 0; k < LC_NDOF; ++k) {
        s.dof_joint[k] = (int)d->dof_joint[k];
        require(s.dof_joint[k] >= 0 && s.dof_joint[k] < J, "dof joint out of range");
        for (int q = 0; q < 3; ++q) s.dof_axes[k][q] = d->dof_axes[3 * k + q];
        s.tmin[k] = d->theta_min[k];
        s.tmax[k] = d->theta_max[k];
    }
    for (int m = 0; m < 4; ++m)
        for (int q = 0; q < 3; ++q) s.marker[m][q] = d->marker_offsets[3 * m + q];
    // ancestor masks: dof k moves positions strictly below its joint, frames at/below
    for (int k = 0; k < LC_NDOF; ++k) {
        unsigned pos = 0, frame = 0;
        for (int i = 0; i < J; ++i) {
            int q = i;
            bool below = false;
            while (q != -1) {
                if (q == s.dof_joint[k]) { below = true; break; }
                q = s.parents[q];
            }
            if (below) {
                frame |= 1u << i;
                if (i != s.dof_joint[k]) pos |= 1u << i;
            }
        }
        s.moves_pos[k] = pos;
        s.moves_frame[k] = frame;
    }
    int cur = 0;
    for (int i = 0; i < J; ++i) {
        s.dof_start[i] = cur;
        for (int k = 0; k < LC_NDOF; ++k)
            if (s.dof_joint[k] == i) s.dof_list[cur++] = k;
    }
    s.dof_start[J] = cur;
    std::vector<int> depth(J, 0);
    int maxd = 0;
    for (int i = 1; i < J; ++i) {
        depth[i] = depth[s.parents[i]] + 1;
        maxd = std::max(maxd, depth[i]);
    }
    cur = 0;
    for (int L = 0; L <= maxd; ++L) {
        s.level_start[L] = cur;
        for (int i = 0; i < J; ++i)
            if (depth[i] == L) s.level_joint[cur++] = i;
    }
    s.level_start[maxd + 1] = cur;
    s.n_tree_levels = maxd + 1;
    for (int L = 0; L <= maxd; ++L)
        require(s.level_start[L + 1] - s.level_start[L] <= 32, "too many joints at one depth");
    a->skel_dev = a->mem.upload(&s, 1, st);

    // ---- mesh tables
    std::vector<int> tris(3 * (size_t)T), edges(2 * (size_t)E), etris(2 * (size_t)E), deg(N);
    for (size_t i = 0; i < tris.size(); ++i) {
        tris[i] = (int)d->triangles[i];
        require(tris[i] >= 0 && tris[i] < N, "triangle index out of range");
    }
    for (size_t i = 0; i < edges.size(); ++i) {
        edges[i] = (int)d->edges[i];
        etris[i] = (int)d->edge_tris[i];
    }
    for (int i = 0; i < N; ++i) deg[i] = (int)d->degrees[i];
    std::vector<double> rest_len(E), rest_dir(3 * (size_t)E);
    for (int e = 0; e < E; ++e) {
        const double *pa = d->rest_vertices + 3 * (size_t)edges[2 * e];
        const double *pb = d->rest_vertices + 3 * (size_t)edges[2 * e + 1];
        const double dx = pa[0] - pb[0], dy = pa[1] - pb[1], dz = pa[2] - pb[2];
        const double l = std::sqrt(dx * dx + dy * dy + dz * dz);
        rest_len[e] = l;
        rest_dir[3 * e] = dx / l;
        rest_dir[3 * e + 1] = dy / l;
        rest_dir[3 * e + 2] = dz / l;
    }
    // incident edges per vertex in the directed "as source" order of the
    // reference (forward edges ascending, then reversed edges ascending)
    std::vector<int> adj_ptr(N + 1, 0), adj_edge(2 * (size_t)E), adj_nbr(2 * (size_t)E);
    for (int e = 0; e < E; ++e) {
        adj_ptr[edges[2 * e] + 1]++;
        adj_ptr[edges[2 * e + 1] + 1]++;
    }
    for (int i = 0; i < N; ++i) adj_ptr[i + 1] += adj_ptr[i];
    {
        std::vector<int> fill(adj_ptr.begin(), adj_ptr.end() - 1);
        for (int e = 0; e < E; ++e) {
            const int i = edges[2 * e];
            adj_edge[fill[i]] = e;
            adj_nbr[fill[i]++] = edges[2 * e + 1];
        }
        for (int e = 0; e < E; ++e) {
            const int i = edges[2 * e + 1];
            adj_edge[fill[i]] = e;
            adj_nbr[fill[i]++] = edges[2 * e];
        }
    }
    // incident triangles per vertex in np.add.at slot order
    std::vector<int> vt_ptr(N + 1, 0), vt_tri(3 * (size_t)T);
    for (int t = 0; t < T; ++t)
        for (int k = 0; k < 3; ++k) vt_ptr[tris[3 * t + k] + 1]++;
    for (int i = 0; i < N; ++i) vt_ptr[i + 1] += vt_ptr[i];
    {
        std::vector<int> fill(vt_ptr.begin(), vt_ptr.end() - 1);
        for (int k = 0; k < 3; ++k)
            for (int t = 0; t < T; ++t) vt_tri[fill[tris[3 * t + k]]++] = t;
    }
    std::vector<int> sidx(4 * (size_t)N), dom(N), vpart(N);
    std::vector<double> rig(N);
    for (int i = 0; i < N; ++i) {
        int best = 0;
        for (int k = 0; k < 4; ++k) {
            sidx[4 * i + k] = (int)d->skin_indices[4 * i + k];
            require(sidx[4 * i + k] < J, "skinning references a joint outside the skeleton");
            if (d->skin_weights[4 * i + k] > d->skin_weights[4 * i + best]) best = k;
        }
        dom[i] = sidx[4 * i + best];
        require(dom[i] >= 0, "dominant skinning slot is padding");
        vpart[i] = s.joint_part[dom[i]];
        const int lab = (int)d->vertex_labels[i];
        require(lab >= 1 && lab <= 7, "invalid material class");
        rig[i] = kClassWeight[lab];
    }
    ActorDev &A = a->dev;
    A.N = N; A.T = T; A.E = E; A.J = J;
    A.rest = a->mem.upload(d->rest_vertices, 3 * (size_t)N, st);
    A.tris = a->mem.upload(tris.data(), tris.size(), st);
    A.colors = a->mem.upload(d->vertex_colors, 3 * (size_t)N, st);
    A.edges = a->mem.upload(edges.data(), edges.size(), st);
    A.edge_tris = a->mem.upload(etris.data(), etris.size(), st);
    A.rest_len = a->mem.upload(rest_len.data(), rest_len.size(), st);
    A.rest_dir = a->mem.upload(rest_dir.data(), rest_dir.size(), st);
    A.adj_ptr = a->mem.upload(adj_ptr.data(), adj_ptr.size(), st);
    A.adj_edge = a->mem.upload(adj_edge.data(), adj_edge.size(), st);
    A.adj_nbr = a->mem.upload(adj_nbr.data(), adj_nbr.size(), st);
    A.degrees = a->mem.upload(deg.data(), deg.size(), st);
    {
        std::vector<int> ell_nbr((size_t)LC_ELL * N, 0), ell_edge((size_t)LC_ELL * N, -1), ell_cnt(N),
            epos(2 * (size_t)E, -1);
        for (int i = 0; i < N; ++i) {
            const int cnt = adj_ptr[i + 1] - adj_ptr[i];
            ell_cnt[i] = cnt;
            for (int k = 0; k < std::min(cnt, LC_ELL); ++k) {
                const int idx = adj_ptr[i] + k, e = adj_edge[idx], pos = k * N + i;
                ell_nbr[pos] = adj_nbr[idx];
                ell_edge[pos] = e;
                epos[2 * (size_t)e + (edges[2 * e] == i ? 0 : 1)] = pos;
            }
        }
        std::vector<int> heavy, heavy_id(N, -1);
        for (int i = 0; i < N; ++i)
            if (ell_cnt[i] > LC_ELL) {
                heavy_id[i] = (int)heavy.size();
                heavy.push_back(i);
            }
        A.n_heavy = (int)heavy.size();
        A.heavy = heavy.empty() ? nullptr : a->mem.upload(heavy.data(), heavy.size(), st);
        A.heavy_id = a->mem.upload(heavy_id.data(), heavy_id.size(), st);
        A.ell_nbr = a->mem.upload(ell_nbr.data(), ell_nbr.size(), st);
        A.ell_cnt = a->mem.upload(ell_cnt.data(), ell_cnt.size(), st);
        A.epos = a->mem.upload(epos.data(), epos.size(), st);
        a->host_ell_edge = ell_edge;
    }
    A.w_dir = a->mem.upload(d->directed_weights, 2 * (size_t)E, st);
    A.skin_idx = a->mem.upload(sidx.data(), sidx.size(), st);
    A.skin_w = a->mem.upload(d->skin_weights, 4 * (size_t)N, st);
    A.dominant = a->mem.upload(dom.data(), dom.size(), st);
    A.vt_ptr = a->mem.upload(vt_ptr.data(), vt_ptr.size(), st);
    A.vt_tri = a->mem.upload(vt_tri.data(), vt_tri.size(), st);
    A.rigidity = a->mem.upload(rig.data(), rig.size(), st);
    A.vpart = a->mem.upload(vpart.data(), vpart.size(), st);
    A.skel = a->skel_dev;
    a->host_edges = edges;
    a->host_degrees = deg;
    a->host_wdir.assign(d->directed_weights, d->directed_weights + 2 * (size_t)E);
    CK(cudaStreamSynchronize(st));
    *out = a;
    return LC_OK;
    API_END
}

// per-context team sizes of the pose / surface solvers (1, 2, 4, 8 or 16
// CTAs per stream; 0 restores the default policy).  Results do not depend on
// the team size beyond fp64 reduction order.
extern "C" int lc_ctx_set_team_sizes(lc_ctx *c, int32_t pose_ctas, int32_t surface_ctas) {
    API_BEGIN
    require(c != nullptr, "null context");
    auto ok = [](int x) { return x == 0 || x == 1 || x == 2 || x == 4 || x == 8 || x == 16; };
    require(ok(pose_ctas) && ok(surface_ctas), "team sizes must be 0 (default), 1, 2, 4, 8 or 16");
    c->pose_cs = pose_ctas;
    c->surf_cs = surface_ctas;
    return LC_OK;
    API_END
}

extern "C" int lc_ctx_set_pyramid_margin(lc_ctx *c, int32_t margin_px) {
    API_BEGIN
    require(c != nullptr, "null context");
    require(margin_px >= -2, "margin must be >= 0, -1 (every tile) or -2 (no tile)");
    c->pyr_margin = margin_px;
    return LC_OK;
    API_END
}

extern "C" int lc_actor_destroy(lc_actor *a) {
    if (!a) return LC_OK;
    cudaSetDevice(a->ctx->device);
    cudaStreamSynchronize(a->ctx->stream);
    if (a->ctx->call_actor == a) a->ctx->call_actor = nullptr;
    delete a;
    return LC_OK;
}

// ---------------------------------------------------------------------------
// slots

static void alloc_grid(DevArena &m, GridBufs &g, int H, int W) {
    const int ncx = (W + LC_GRID_CELL - 1) / LC_GRID_CELL, ncy = (H + LC_GRID_CELL - 1) / LC_GRID_CELL;
    g.row_count = m.alloc<int>(H);
    g.row_start = m.alloc<int>(H + 1);
    g.cell_count = m.alloc<int>(ncx * ncy);
    g.cell_start = m.alloc<int>(ncx * ncy + 1);
    g.cell_fill = m.alloc<int>(ncx * ncy);
    g.pts = m.alloc<int2>((size_t)H * W);
    g.cell_pts = m.alloc<int>((size_t)H * W);
    g.K = m.alloc<int>(1);
    g.cand_pts = m.alloc<int>((size_t)ncx * ncy * LC_CAND_MAX);   // fixed-capacity per-cell lists
    g.cand_blk = m.alloc<int>((size_t)ncx * ncy * 32);
    g.cell_seed = m.alloc<int>(ncx * ncy);
    g.fg_rows = m.alloc<uint8_t>((size_t)H * ((W + LC_PYR_TILE - 1) / LC_PYR_TILE));
    g.qP = 1;
    g.qL = 0;
    while (g.qP < std::max(ncx, ncy)) { g.qP *= 2; g.qL++; }
    g.quad = m.alloc<int>(quad_off(g.qP, g.qL + 1));
}

static size_t pyr_tiles(int H, int W) {
    return (size_t)((W + LC_PYR_TILE - 1) / LC_PYR_TILE) * ((H + LC_PYR_TILE - 1) / LC_PYR_TILE);
}

void Slot::allocate(int N_, int T_, int E_, int H_, int W_, int levels_, int J) {
    N = N_; T = T_; E = E_; H = H_; W = W_; levels = levels_;
    const size_t HW = (size_t)H * W;
    image = mem.alloc<double>(HW * 3);
    mask = mem.alloc<uint8_t>(HW);
    image_src = image;
    mask_src = mask;
    pyr = mem.alloc<double>(HW * 3 * std::max(levels, 1));
    pyr_tile = mem.alloc<uint8_t>(pyr_tiles(H, W));
    pyr_roi = mem.alloc<int>(4);
    blur_tmp = mem.alloc<double>(HW * 3);
    alloc_grid(mem, obs, H, W);   // (the own silhouette uses cell buckets, own_cnt / own_keys)
    own_mask = mem.alloc<uint8_t>(HW);
    {
        const size_t nc = (size_t)((W + LC_GRID_CELL - 1) / LC_GRID_CELL) * ((H + LC_GRID_CELL - 1) / LC_GRID_CELL);
        own_cnt = mem.alloc<int>(nc);
        own_keys = mem.alloc<int>(nc * 256);
    }
    j2d = mem.alloc<double>(2 * (LC_MAXJ + 4));
    j3d_raw = mem.alloc<double>(3 * LC_MAXJ);
    j3d = mem.alloc<double>(3 * LC_MAXJ);
    v2d = mem.alloc<uint8_t>(LC_MAXJ + 4);
    v3d = mem.alloc<uint8_t>(LC_MAXJ);
    fallbacks = mem.alloc<int>(1);
    x_prev = mem.alloc<double>(LC_NP);
    x_prev2 = mem.alloc<double>(LC_NP);
    joints_prev = mem.alloc<double>(3 * LC_MAXJ);
    disp = mem.alloc<double>(3 * (size_t)N);
    v_prev = mem.alloc<double>(3 * (size_t)N);
    v_prev2 = mem.alloc<double>(3 * (size_t)N);
    x = mem.alloc<double>(LC_NP);
    x0 = mem.alloc<double>(LC_NP);
    drest = mem.alloc<double>(3 * (size_t)N);
    model = mem.alloc<double>(3 * (size_t)N);
    vs = mem.alloc<double>(3 * (size_t)N);
    rot = mem.alloc<double>(4 * (size_t)N);
    vinit = mem.alloc<double>(3 * (size_t)N);
    v = mem.alloc<double>(3 * (size_t)N);
    fk = mem.alloc<FkState>(1);
    zbuf = mem.alloc<unsigned long long>(HW);
    tri_id = mem.alloc<int>(HW);
    {
        const int ntx = (W + LC_RT_TILE - 1) / LC_RT_TILE, nty = (H + LC_RT_TILE - 1) / LC_RT_TILE;
        rt_rec = mem.alloc<TriRec>(std::max(T, 1));
        rt_diff = mem.alloc<int>((size_t)ntx * nty);
        rt_off = mem.alloc<int>((size_t)ntx * nty + 1);
        rt_fill = mem.alloc<int>((size_t)ntx * nty);
        rt_cap = std::max(1 << 20, 64 * T);
        rt_list = mem.alloc<int>(rt_cap);
        rt_ioff = mem.alloc<int>((size_t)ntx * nty + 1);
        const size_t items = 2 * (size_t)ntx * nty + rt_cap / LC_RT_CHUNK + 1;
        rt_pz = mem.alloc<unsigned long long>(items * 256);
        rt_pid = mem.alloc<int>(items * 256);
    }
    tri_front = mem.alloc<uint8_t>(T);
    vflag = mem.alloc<uint8_t>(N);
    enabled = mem.alloc<uint8_t>(N);
    tri_n = mem.alloc<double>(3 * (size_t)T);
    n2d = mem.alloc<double>(2 * (size_t)N);
    crest = mem.alloc<double>(3 * (size_t)N);
    cidx = mem.alloc<int>(N);
    nn_hint = mem.alloc<int>(N);
    B = mem.alloc<int>(1);
    vis = mem.alloc<int>(N);
    P = mem.alloc<int>(1);
    diag = mem.alloc<double>(6 * (size_t)N);
    minv = mem.alloc<double>(9 * (size_t)N);
    rhs = mem.alloc<double>(3 * (size_t)N);
    sx = mem.alloc<double>(3 * (size_t)N);
    sr = mem.alloc<double>(3 * (size_t)N);
    sz = mem.alloc<double>(3 * (size_t)N);
    sp = mem.alloc<double>(3 * (size_t)N);
    sap = mem.alloc<double>(3 * (size_t)N);
    sbest = mem.alloc<double>(3 * (size_t)N);
    edir = mem.alloc<double>(3 * (size_t)E);
    eg = mem.alloc<double>(3 * (size_t)E);
    ell_d = mem.alloc<double>(3 * (size_t)LC_ELL * N);
    ell_g = mem.alloc<double>(3 * (size_t)LC_ELL * N);
    off0 = mem.alloc<double>(3 * (size_t)N);
    off1 = mem.alloc<double>(3 * (size_t)N);
    hold = mem.alloc<uint8_t>(N);
    pose_rep = mem.alloc<lc_pose_report>(1);
    nr_rep = mem.alloc<lc_nonrigid_report>(1);
    counters = mem.alloc<long long>(LC_NCOUNTERS);
    phase_pose = mem.alloc<long long>(LC_NPHASE);
    phase_surf = mem.alloc<long long>(LC_NPHASE);
    cudaMemset(phase_pose, 0, sizeof(long long) * LC_NPHASE);
    cudaMemset(phase_surf, 0, sizeof(long long) * LC_NPHASE);
    cudaMemset(counters, 0, sizeof(long long) * LC_NCOUNTERS);
}

// the other input buffers + events of a tracker stream; in[0] is the slot's own
void Slot::allocate_queue() {
    const size_t HW = (size_t)H * W;
    FrameIn &a = in[0];
    a.image = image; a.mask = mask; a.image_src = image; a.mask_src = mask;
    a.pyr = pyr; a.obs = obs; a.j2d = j2d; a.j3d_raw = j3d_raw; a.v2d = v2d; a.v3d = v3d;
    a.pyr_tile = pyr_tile; a.pyr_roi = pyr_roi;
    a.tmp = blur_tmp;
    for (int q = 1; q < LC_QUEUE; ++q) {
        FrameIn &b = in[q];
        b.image = mem.alloc<double>(HW * 3);
        b.mask = mem.alloc<uint8_t>(HW);
        b.image_src = b.image; b.mask_src = b.mask;
        b.pyr = mem.alloc<double>(HW * 3 * std::max(levels, 1));
        b.pyr_tile = mem.alloc<uint8_t>(pyr_tiles(H, W));
        b.pyr_roi = mem.alloc<int>(4);
        alloc_grid(mem, b.obs, H, W);
        b.j2d = mem.alloc<double>(2 * (LC_MAXJ + 4));
        b.j3d_raw = mem.alloc<double>(3 * LC_MAXJ);
        b.v2d = mem.alloc<uint8_t>(LC_MAXJ + 4);
        b.v3d = mem.alloc<uint8_t>(LC_MAXJ);
        b.tmp = blur_tmp;
    }
    for (FrameIn &f : in) f.image_u8 = mem.alloc<uint8_t>(HW * 3);
    for (FrameIn &f : in) {
        cudaEventCreateWithFlags(&f.ready_obs, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&f.ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&f.freed, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&f.uploaded, cudaEventDisableTiming);
    }
}

// point the slot's per-frame input fields at queued frame `f`
void Slot::view(const FrameIn &f) {
    image_src = f.image_src; mask_src = f.mask_src; pyr = f.pyr; obs = f.obs;
    pyr_tile = f.pyr_tile; pyr_roi = f.pyr_roi;
    j2d = f.j2d; j3d_raw = f.j3d_raw; v2d = f.v2d; v3d = f.v3d;
}

Slot::~Slot() {
    for (FrameIn &f : in) {
        if (f.ready_obs) cudaEventDestroy(f.ready_obs);
        if (f.ready) cudaEventDestroy(f.ready);
        if (f.freed) cudaEventDestroy(f.freed);
        if (f.uploaded) cudaEventDestroy(f.uploaded);
    }
}

static CamDev cam_dev(const lc_camera &c) {
    CamDev d;
    d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy; d.W = c.width; d.H = c.height;
    return d;
}

static NnGridDev grid_dev(const GridBufs &g, const uint8_t *mask, int H, int W) {
    NnGridDev d;
    d.K = 0;
    d.W = W; d.H = H;
    d.ncx = (W + LC_GRID_CELL - 1) / LC_GRID_CELL;
    d.ncy = (H + LC_GRID_CELL - 1) / LC_GRID_CELL;
    d.pts = g.pts;
    d.cell_start = g.cell_start;
    d.cell_pts = g.cell_pts;
    d.mask = mask;
    d.cand_pts = g.cand_pts;
    d.cand_blk = g.cand_blk;
    d.quad = g.quad;
    d.qP = g.qP;
    d.qL = g.qL;
    return d;
}

// Candidate lists are built for cells whose bound U (the farthest point of
// the cell to a nearby site) is at most this many pixels; queries in farther
// cells take the exact quadtree search (slower per query than a list).  On
// the in-track bench workload, with rim-disabled rows skipping their
// queries, 192 px measured best (frames/s: all cells 4036, 192: 4244, 128:
// 4167, 64: 3876, 48: 3579): the far cells' long lists cost more to build
// than their few queries save.  LIVECAP_LIST_RADIUS overrides.
static double obs_list_radius() {
    static double r = [] {
        const char *v = getenv("LIVECAP_LIST_RADIUS");
        return v ? atof(v) : 192.0;
    }();
    return r;
}

// contour pixels + NN grid (+ candidate lists) for a batch of masks
static void build_grids(lc_ctx *c, const std::vector<std::pair<const GridBufs *, const uint8_t *>> &gs,
                        int H, int W, double max_u = 1e30, bool lists = true) {
    if (gs.empty()) return;
    std::vector<GridJob> jobs;
    for (auto &p : gs) {
        GridJob j;
        j.mask = p.second;
        j.row_count = p.first->row_count; j.row_start = p.first->row_start;
        j.pts = p.first->pts; j.cell_count = p.first->cell_count; j.cell_start = p.first->cell_start;
        j.cell_fill = p.first->cell_fill; j.cell_pts = p.first->cell_pts; j.K = p.first->K;
        j.cand_pts = p.first->cand_pts;
        j.cand_blk = p.first->cand_blk;
        j.max_u2 = max_u * max_u;
        j.quad = p.first->quad; j.qP = p.first->qP; j.qL = p.first->qL;
        j.fg_rows = p.first->fg_rows;
        j.cell_seed = p.first->cell_seed;
        jobs.push_back(j);
    }
    const auto dj = stage(c, jobs);
    const int S = (int)jobs.size();
    const int ncx = (W + LC_GRID_CELL - 1) / LC_GRID_CELL, ncy = (H + LC_GRID_CELL - 1) / LC_GRID_CELL;
    const int rows_grid = std::min(H, 1024);
    launch(c, k_contour_rows, dim3(rows_grid, S), dim3(256), 0, dj, H, W);
    launch(c, k_contour_scan_rows, dim3(S), dim3(1024), 0, dj, H, ncx * ncy);
    launch(c, k_contour_emit, dim3(rows_grid, S), dim3(256), 0, dj, H, W, ncx);
    launch(c, k_contour_scan_cells, dim3(S), dim3(1024), 0, dj, ncx * ncy);
    launch(c, k_quad_build, dim3(S), dim3(1024), 0, dj, ncx, ncy);
    launch(c, k_contour_fill, dim3(64, S), dim3(256), 0, dj, ncx);
    if (!lists) return;
    launch(c, k_cell_jfa, dim3(S), dim3(1024), sizeof(int) * 2 * ncx * ncy, dj, ncx, ncy);
    // (measurement knob: LIVECAP_CAND_GRID caps the CTAs per stream of this
    // grid-stride kernel, bounding the SMs the auxiliary stream can hold)
    static const int cand_cap = [] {
        const char *v = getenv("LIVECAP_CAND_GRID");
        return v ? atoi(v) : 0;
    }();
    int cand_grid = (ncx * ncy + 3) / 4;
    if (cand_cap > 0) cand_grid = std::min(cand_grid, cand_cap);
    launch(c, k_cand_build, dim3(cand_grid, S), dim3(128), 0, dj, H, W);
}

// depth buffer + winning triangle ids (+ mask) of a batch of meshes with
// the same triangles (rasterizer.py:18-68): tile-binned single pass
static void raster_tris(lc_ctx *c, const CamDev &cd, const int *tris, int T, const std::vector<RasterJob> &jobs) {
    if (jobs.empty()) return;
    const auto dj = stage(c, jobs);
    const unsigned S = (unsigned)jobs.size();
    const int ntx = (cd.W + LC_RT_TILE - 1) / LC_RT_TILE, nty = (cd.H + LC_RT_TILE - 1) / LC_RT_TILE;
    const int nt = ntx * nty;
    launch(c, k_rt_clear, dim3((nt + 255) / 256, S), dim3(256), 0, dj, nt);
    launch(c, k_rt_setup, dim3((T + 127) / 128, S), dim3(128), 0, dj, cd, tris, T);
    launch(c, k_rt_bin<0>, dim3((T + 3) / 4, S), dim3(128), 0, dj, T, ntx);
    launch(c, k_rt_scan, dim3(S), dim3(1024), 0, dj, nt, T);
    launch(c, k_rt_bin<1>, dim3((T + 3) / 4, S), dim3(128), 0, dj, T, ntx);
    mark(c, "raster:bin");
    launch(c, k_rt_tiles, dim3(std::max(1, 1184 / (int)S), S), dim3(256), 0, dj, cd, T, ntx, nt);
    launch(c, k_rt_merge, dim3(std::max(1, 1184 / (int)S), S), dim3(256), 0, dj, cd, ntx, nt);
    mark(c, "raster:tiles");
}

static RasterJob raster_job(Slot *s, const double *verts, uint8_t *mask) {
    RasterJob j{};
    j.verts = verts; j.zbuf = s->zbuf; j.tri_id = s->tri_id; j.mask = mask;
    j.rec = s->rt_rec; j.tcount = s->rt_diff; j.toff = s->rt_off; j.tfill = s->rt_fill; j.tlist = s->rt_list;
    j.tcap = s->rt_cap;
    j.ioff = s->rt_ioff; j.pz = s->rt_pz; j.pid = s->rt_pid;
    return j;
}

static void raster(lc_ctx *c, const lc_actor *a, const lc_camera &cam, const std::vector<RasterJob> &jobs) {
    raster_tris(c, cam_dev(cam), a->dev.tris, a->dev.T, jobs);
}

// ---------------------------------------------------------------------------
// config -> device constants

// Line-search batching (the halvings are exact, so any batching gives the
// sequential search's decisions; only the work differs).  On the in-track
// bench stream (oracle logs, frames 1-5) the pose accepts the full step in 29
// of 30 GN steps: its first batch is the full step alone (pose 638 -> 552 us
// per frame).  The surface takes 1-3 halvings or rejects in 14 of 15; trying
// every trial at once shortens an isolated solve (715 -> 669 us) but measured
// 3% fewer frames/s under the bench's concurrency (4170 vs 4310), so it also
// starts with the full step alone; later batches take the remaining halvings
// together (batches of 1 / 2 / 4 after the full step: 4317 / 4394 / 4368
// frames/s, within noise).  LIVECAP_{POSE,SURF}_FIRST_TRIALS and
// LIVECAP_SURF_NEXT_TRIALS override (1..4).
static int trials_env(const char *var, int dflt) {
    const char *v = getenv(var);
    const int n = v ? atoi(v) : dflt;
    return n < 1 ? 1 : (n > 4 ? 4 : n);
}

static void fill_pose_hyper(PoseHyperDev &h, const lc_pose_hyper &p, const SkelDev &s) {
    h.l2d = p.lambda_2d; h.l3d = p.lambda_3d; h.lsil = p.lambda_sil; h.ltemp = p.lambda_temporal;
    h.lanat = p.lambda_anatomic; h.face = p.face_weight;
    for (int i = 0; i < LC_MAXJ; ++i) h.tw[i] = i < s.J ? p.group_weights[s.group[i] & 7] : 0.0;
    h.gn = p.gn_iterations;
    h.max_halvings = p.max_halvings;
    h.first_trials = trials_env("LIVECAP_POSE_FIRST_TRIALS", 1);
}

static void fill_surf_hyper(SurfHyperDev &h, const lc_nonrigid_hyper &p) {
    h.w_photo = p.w_photo; h.w_sil = p.w_sil; h.w_smooth = p.w_smooth; h.w_edge = p.w_edge;
    h.w_vel = p.w_velocity; h.w_acc = p.w_acceleration; h.tau = p.tau_color;
    h.gn = p.gn_iterations; h.pcg = p.pcg_iterations; h.max_halvings = p.max_halvings;
    h.n_levels = p.n_levels; h.dilation = p.part_dilation;
    h.snap_step = p.snap_step; h.snap_band = p.snap_band; h.snap_max_steps = p.snap_max_steps;
    h.first_trials = trials_env("LIVECAP_SURF_FIRST_TRIALS", 1);
    h.next_trials = trials_env("LIVECAP_SURF_NEXT_TRIALS", 4);
}

// numpy-compatible pairwise sum (n <= 128 blocks of 8)
static double np_sum(const std::vector<double> &a) {
    const size_t n = a.size();
    if (n < 8) {
        double s = 0.0;
        for (double v : a) s += v;
        return s;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    size_t i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) s += a[i];
    return s;
}

// gaussian_kernel (imageproc.py:264-273)
static std::vector<double> gaussian_taps(int size) {
    if (size == 1) return {1.0};
    const double sigma = (size - 1) / 6.0;
    std::vector<double> k(size);
    for (int i = 0; i < size; ++i) {
        const double x = (double)i - (size - 1) / 2.0;
        const double q = x / sigma;
        k[i] = std::exp(-0.5 * (q * q));
    }
    const double s = np_sum(k);
    for (double &v : k) v = v / s;
    return k;
}

// outer_rim_mask probe offsets (pose_stage.py:255-259): 16 directions x radii 1..8
static std::vector<double> probe_offsets() {
    std::vector<double> o(128 * 2);
    const double step = (2.0 * M_PI - 0.0) / 16.0;
    for (int a = 0; a < 16; ++a) {
        const double ang = 0.0 + a * step;
        const double cs = std::cos(ang), sn = std::sin(ang);
        for (int r = 0; r < 8; ++r) {
            o[2 * (a * 8 + r)] = cs * (double)(r + 1);
            o[2 * (a * 8 + r) + 1] = sn * (double)(r + 1);
        }
    }
    return o;
}

extern "C" int lc_debug_tables(int32_t size, double *taps_out, double *probe_out) {
    if (taps_out) {
        auto k = gaussian_taps(size);
        std::memcpy(taps_out, k.data(), k.size() * sizeof(double));
    }
    if (probe_out) {
        auto p = probe_offsets();
        std::memcpy(probe_out, p.data(), p.size() * sizeof(double));
    }
    return LC_OK;
}

static void build_config(lc_ctx *c, const lc_actor *a, const lc_nonrigid_hyper *nh,
                         const lc_pose_hyper *ph, ConfigDev &cf) {
    cudaStream_t st = c->stream;
    const int E = a->dev.E;
    if (nh) {
        std::vector<double> csf(E), csr(E), cef(E), cer(E), al(E), be(E);
        const auto &ed = a->host_edges;
        const auto &dg = a->host_degrees;
        const auto &w = a->host_wdir;
        for (int e = 0; e < E; ++e) {
            const double da = (double)dg[ed[2 * e]], db = (double)dg[ed[2 * e + 1]];
            csf[e] = std::sqrt(nh->w_smooth * w[e] / da);
            csr[e] = std::sqrt(nh->w_smooth * w[e + E] / db);
            cef[e] = std::sqrt(nh->w_edge * w[e] / da);
            cer[e] = std::sqrt(nh->w_edge * w[e + E] / db);
            al[e] = csf[e] * csf[e] + csr[e] * csr[e];
            be[e] = cef[e] * cef[e] + cer[e] * cer[e];
        }
        cf.ec.cs_f = cf.mem.upload(csf.data(), E, st);
        cf.ec.cs_r = cf.mem.upload(csr.data(), E, st);
        cf.ec.ce_f = cf.mem.upload(cef.data(), E, st);
        cf.ec.ce_r = cf.mem.upload(cer.data(), E, st);
        cf.ec.alpha = cf.mem.upload(al.data(), E, st);
        cf.ec.beta = cf.mem.upload(be.data(), E, st);
        const int N = a->dev.N;
        std::vector<double> ea((size_t)LC_ELL * N, 0.0), eb((size_t)LC_ELL * N, 0.0);
        for (size_t q = 0; q < ea.size(); ++q) {
            const int e = a->host_ell_edge[q];
            if (e >= 0) { ea[q] = al[e]; eb[q] = be[e]; }
        }
        cf.ec.ell_a = cf.mem.upload(ea.data(), ea.size(), st);
        cf.ec.ell_b = cf.mem.upload(eb.data(), eb.size(), st);
        fill_surf_hyper(cf.shp, *nh);
        std::vector<double> taps(4 * 32, 0.0);
        for (int l = 0; l < nh->n_levels && l < 4; ++l) {
            const int k = nh->pyramid_kernels[l];
            require(k >= 1 && k % 2 == 1 && k <= 31, "pyramid kernel sizes must be odd and <= 31");
            bool given = false;
            for (int q = 0; q < 32; ++q) given = given || nh->pyramid_taps[l][q] != 0.0;
            if (given) std::copy(nh->pyramid_taps[l], nh->pyramid_taps[l] + 32, taps.begin() + 32 * l);
            else {
                auto t = gaussian_taps(k);
                std::copy(t.begin(), t.end(), taps.begin() + 32 * l);
            }
            cf.half[l] = k / 2;
        }
        cf.taps = cf.mem.upload(taps.data(), taps.size(), st);
        cf.shp.taps = cf.taps;
        for (int l = 0; l < 4; ++l) cf.shp.half[l] = cf.half[l];
    }
    if (ph) fill_pose_hyper(cf.php, *ph, a->skel);
    auto pr = probe_offsets();
    cf.probe = cf.mem.upload(pr.data(), pr.size(), st);
}

// gaussian_pyramid (imageproc.py:276-285) of a batch of images
struct PyrTarget {
    const double *src; double *dst; double *tmp;
    const int *roi = nullptr; uint8_t *tile_flag = nullptr;   // region of interest (tracker frames)
};

static void pyramid(lc_ctx *c, const ConfigDev &cf, const std::vector<PyrTarget> &ts, int H, int W, int levels) {
    if (ts.empty()) return;
    bool fused = levels <= 4;
    for (int l = 0; l < levels; ++l) fused = fused && cf.half[l] <= LC_PYR_HALO;
    if (fused) {
        std::vector<PyrAllJob> jobs;
        for (const PyrTarget &t : ts) jobs.push_back(PyrAllJob{t.src, t.dst, t.roi, t.tile_flag});
        int tiles = ((W + LC_PYR_TILE - 1) / LC_PYR_TILE) * ((H + LC_PYR_TILE - 1) / LC_PYR_TILE);
        // at most 296 CTAs per frame (two per SM), each striding over tiles:
        // the low-priority preprocessing holds fewer SM slots at a time
        // (frames/s 4528-4545 with one CTA per tile, 4564-4574 capped at
        // 148-592; LIVECAP_PYR_GRID overrides, 0 = one CTA per tile)
        static const int pyr_cap = [] {
            const char *v = getenv("LIVECAP_PYR_GRID");
            return v ? atoi(v) : 296;
        }();
        if (pyr_cap > 0) tiles = std::min(tiles, pyr_cap);
        launch(c, k_pyramid_fused, dim3(tiles, (unsigned)ts.size()), dim3(256), pyramid_fused_smem(),
               stage(c, jobs), H, W, levels, (const double *)cf.taps, cf.half[0], cf.half[1], cf.half[2],
               cf.half[3]);
        return;
    }
    const long long n = (long long)H * W * 3;
    const int grid = (int)std::min<long long>((n + 255) / 256, 2368);
    for (const PyrTarget &t : ts)   // (the two-pass path computes every tile)
        if (t.tile_flag) cudaMemsetAsync(t.tile_flag, 1, pyr_tiles(H, W), c->stream);
    for (int l = 0; l < levels; ++l) {
        std::vector<PyrJob> jobs;
        for (const PyrTarget &t : ts) jobs.push_back(PyrJob{t.src, t.tmp, t.dst + (size_t)l * n});
        const auto dj = stage(c, jobs);
        launch(c, k_blur_axis, dim3(grid, (unsigned)ts.size()), dim3(256), 0, dj, H, W, 3,
               (const double *)(cf.taps + 32 * l), cf.half[l], 0);
        launch(c, k_blur_axis, dim3(grid, (unsigned)ts.size()), dim3(256), 0, dj, H, W, 3,
               (const double *)(cf.taps + 32 * l), cf.half[l], 1);
    }
}


// ---------------------------------------------------------------------------
// small per-stream kernels of the frame schedule

struct PrepJob {
    const double *rest, *disp;   // disp may be null
    double *drest;
    // detection conditioning (pose_stage.py:92-116) + extrapolation (:119-127)
    const double *j3d_raw;
    double *j3d;
    const uint8_t *v3d;
    int *fallbacks;
    const double *x_prev, *x_prev2;  // null when absent
    double *x;                       // out: initial pose
    lc_pose_report *pose_rep;        // zeroed here (or null)
    lc_nonrigid_report *nr_rep;      // zeroed here (or null)
    int N;
};

__global__ void k_prep(JobArg<PrepJob> jobs, const SkelDev *skg) {
    lc_pdl_wait();
    const PrepJob J = jobs[blockIdx.y];
    const SkelDev &sk = *skg;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 3 * J.N; i += gridDim.x * blockDim.x)
        J.drest[i] = J.disp ? J.rest[i] + J.disp[i] : J.rest[i];
    if (blockIdx.x == 1) {   // the frame's reports start from zero
        for (int i = threadIdx.x; J.pose_rep && i < (int)(sizeof(lc_pose_report) / 4); i += blockDim.x)
            reinterpret_cast<int *>(J.pose_rep)[i] = 0;
        for (int i = threadIdx.x; J.nr_rep && i < (int)(sizeof(lc_nonrigid_report) / 4); i += blockDim.x)
            reinterpret_cast<int *>(J.nr_rep)[i] = 0;
        return;
    }
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    // rescale_detections: root outward, bone lengths from local offsets.  One
    // warp, lane = joint; the tree levels in order (FK schedule), so every
    // joint reads its parent's final value: the sequential loop's arithmetic
    const int lane = threadIdx.x;
    int fb = 0;
    if (lane == 0)
        for (int k = 0; k < 3; ++k) J.j3d[k] = J.j3d_raw[k];
    __syncwarp();
    for (int L = 1; L < sk.n_tree_levels; ++L) {
        const int q = sk.level_start[L] + lane;
        if (q < sk.level_start[L + 1]) {
            const int i = sk.level_joint[q];
            const int p = sk.parents[i];
            double d[3] = {J.j3d_raw[3 * i] - J.j3d_raw[3 * p], J.j3d_raw[3 * i + 1] - J.j3d_raw[3 * p + 1],
                           J.j3d_raw[3 * i + 2] - J.j3d_raw[3 * p + 2]};
            double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            const bool usable = n > 1e-9 && J.v3d[i] && J.v3d[p];
            if (!usable) {
                for (int k = 0; k < 3; ++k) d[k] = sk.rest[i][k] - sk.rest[p][k];
                n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                ++fb;
            }
            const double bl =
                sqrt(sk.off[i][0] * sk.off[i][0] + sk.off[i][1] * sk.off[i][1] + sk.off[i][2] * sk.off[i][2]);
            for (int k = 0; k < 3; ++k) J.j3d[3 * i + k] = J.j3d[3 * p + k] + bl * d[k] / n;
        }
        __syncwarp();
    }
    for (int o = 16; o > 0; o >>= 1) fb += __shfl_xor_sync(0xffffffffu, fb, o);
    if (lane == 0) *J.fallbacks = fb;
    if (J.x) {
        for (int k = lane; k < LC_NP; k += 32) {
            double v = 0.0;
            if (J.x_prev) v = J.x_prev2 ? 2.0 * J.x_prev[k] - J.x_prev2[k] : J.x_prev[k];
            if (J.x_prev && k >= 6 && k < 6 + LC_NDOF) v = fmin(fmax(v, sk.tmin[k - 6]), sk.tmax[k - 6]);
            J.x[k] = v;
        }
    }
}

struct FinishJob {
    const double *x, *v, *vs, *rot;
    const FkState *fk;
    double *x_prev, *x_prev2, *joints_prev, *disp, *v_prev, *v_prev2;
    int shift_x2, shift_v2;   // copy prev -> prev2 first
    int warp;                 // 1 rotate, 0 plain delta, -1 zero (pose_only)
    int N, J;
};

__global__ void k_finish(JobArg<FinishJob> jobs) {
    lc_pdl_wait();
    const FinishJob F = jobs[blockIdx.y];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F.N; i += gridDim.x * blockDim.x) {
        const V3 v = ld3(F.v + 3 * (size_t)i);
        if (F.shift_v2) st3(F.v_prev2 + 3 * (size_t)i, ld3(F.v_prev + 3 * (size_t)i));
        st3(F.v_prev + 3 * (size_t)i, v);
        V3 d = v3(0, 0, 0);
        if (F.warp >= 0) {
            d = v - ld3(F.vs + 3 * (size_t)i);
            if (F.warp == 1) {
                const double *q = F.rot + 4 * (size_t)i;
                d = qrot(qconj(Q4{q[0], q[1], q[2], q[3]}), d);
            }
        }
        st3(F.disp + 3 * (size_t)i, d);
    }
    if (blockIdx.x == 0) {
        for (int k = threadIdx.x; k < LC_NP; k += blockDim.x) {
            if (F.shift_x2) F.x_prev2[k] = F.x_prev[k];
        }
        __syncthreads();
        for (int k = threadIdx.x; k < LC_NP; k += blockDim.x) F.x_prev[k] = F.x[k];
        for (int k = threadIdx.x; k < 3 * F.J; k += blockDim.x) F.joints_prev[k] = F.fk->pos[k / 3][k % 3];
    }
}

// ---------------------------------------------------------------------------
// frame schedule (solve_frame, pipeline.py:263-302) for a batch of slots

struct FrameBatch {
    lc_ctx *c;
    const lc_actor *a;
    lc_camera cam;
    const lc_config *cfg;
    ConfigDev *cf;
    std::vector<Slot *> slots;
    std::vector<FrameIn *> in;    // the frame each slot solves (its preprocessing is launched)
};

// Events that order work across tracker steps (frame buffers freed /
// uploaded / preprocessed): while a step is captured into a CUDA graph they
// become external event record / wait nodes, so the replayed graph still
// synchronises with the previous and next steps and the copy stream.
static void ev_record_x(lc_ctx *c, cudaEvent_t e, cudaStream_t st) {
    if (c->capturing) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
}
static void ev_wait_x(lc_ctx *c, cudaStream_t st, cudaEvent_t e) {
    cudaStreamWaitEvent(st, e, c->capturing ? cudaEventWaitExternal : 0);
}

static int pyr_margin(const lc_ctx *c) {
    if (c->pyr_margin != INT_MIN) return c->pyr_margin;
    static const int env = [] {
        const char *v = getenv("LIVECAP_PYR_MARGIN");
        return v ? atoi(v) : 64;
    }();
    return env;
}

// Preprocessing of queued frames (pipeline.py:156-162) on the auxiliary
// stream: observed-silhouette contour + NN grid, then the blur pyramid.  A
// buffer is rebuilt only after the solve that last read it has finished.
static void launch_preprocess(lc_ctx *c, const ConfigDev &cf, const lc_config &cfg,
                              const std::vector<FrameIn *> &fs, int H, int W) {
    if (fs.empty()) return;
    // (while the auxiliary stream is captured on its own, the fork point is
    // recorded on the solve stream right before the graph launch)
    if (!c->capturing) cudaEventRecord(c->ev_fork, c->stream);
    ev_wait_x(c, c->aux, c->ev_fork);
    for (FrameIn *f : fs) {
        if (f->used) ev_wait_x(c, c->aux, f->freed);
        if (f->pending_upload) ev_wait_x(c, c->aux, f->uploaded);
        f->pending_upload = false;
    }
    OnStream on(c, c->aux);
    mark(c, "pre:start");
    // performance probe only (never set in tests or the bench): reuse the
    // buffers' previous preprocessing instead of rebuilding it
    static const bool skip_prep = getenv("LIVECAP_PROBE_SKIP_PREP") != nullptr;
    bool all_used = true;
    for (FrameIn *f : fs) all_used = all_used && f->used;
    if (skip_prep && all_used) {
        for (FrameIn *f : fs) {
            ev_record_x(c, f->ready_obs, c->aux);
            ev_record_x(c, f->ready, c->aux);
            f->state = 2;
        }
        return;
    }
    // finer probes (performance measurement only): skip just the grid or
    // just the pyramid rebuild
    static const bool skip_grid = getenv("LIVECAP_PROBE_SKIP_GRID") != nullptr;
    static const bool skip_pyr = getenv("LIVECAP_PROBE_SKIP_PYR") != nullptr;
    std::vector<std::pair<const GridBufs *, const uint8_t *>> gs;
    for (FrameIn *f : fs) gs.push_back({&f->obs, f->mask_src});
    if (!(skip_grid && all_used)) build_grids(c, gs, H, W, obs_list_radius());
    mark(c, "pre:grid");
    for (FrameIn *f : fs) ev_record_x(c, f->ready_obs, c->aux);
    if (cfg.mode == 0 && !(skip_pyr && all_used)) {
        std::vector<PyrTarget> ts;
        // region of interest: only the tiles near the observed silhouette
        // are blurred; samples elsewhere take the exact on-demand path
        const int margin = pyr_margin(c);
        std::vector<PyrRoiJob> rj;
        for (FrameIn *f : fs)
            if (f->has_image) {
                ts.push_back(PyrTarget{f->image_src, f->pyr, f->tmp, margin == -1 ? nullptr : f->pyr_roi,
                                       f->pyr_tile});
                rj.push_back(PyrRoiJob{f->obs.cell_count, f->pyr_roi, f->obs.fg_rows, f->pyr_tile});
            }
        if (!rj.empty() && margin != -1) {
            const int ncx = (W + LC_GRID_CELL - 1) / LC_GRID_CELL, ncy = (H + LC_GRID_CELL - 1) / LC_GRID_CELL;
            launch(c, k_pyr_roi, dim3((unsigned)rj.size()), dim3(1024), 0, stage(c, rj), ncx, ncy,
                   (W + LC_PYR_TILE - 1) / LC_PYR_TILE, (H + LC_PYR_TILE - 1) / LC_PYR_TILE, margin, H);
        }
        if (!ts.empty()) pyramid(c, cf, ts, H, W, cfg.nonrigid.n_levels);
    }
    mark(c, "pre:pyramid");
    for (FrameIn *f : fs) {
        ev_record_x(c, f->ready, c->aux);
        f->state = 2;
    }
}

// FK of each slot's pose (optional) then DQ skinning of the actor rest shape
// (use_drest = false) or the slot's displaced rest shape (use_drest = true)
static void fk_skin(FrameBatch &fb, const std::vector<Slot *> &ss, bool from_x, bool use_drest,
                    double *Slot::*out, double *Slot::*rot_out) {
    lc_ctx *c = fb.c;
    std::vector<FkJob> fj;
    std::vector<SkinJob> sj;
    for (Slot *s : ss) {
        fj.push_back(FkJob{s->x, s->fk, 1});
        SkinJob k{};
        k.fk = s->fk;
        k.rest = use_drest ? s->drest : fb.a->dev.rest;
        k.pos = s->*out;
        k.rot = rot_out ? s->*rot_out : nullptr;
        k.M = s->N;
        k.active = 1;
        sj.push_back(k);
    }
    if (from_x) launch(c, k_fk, dim3((unsigned)ss.size()), dim3(32), 0, stage(c, fj), (const SkelDev *)fb.a->skel_dev);
    launch(c, k_skin, dim3((fb.a->dev.N + 127) / 128, (unsigned)ss.size()), dim3(128), 0, stage(c, sj), fb.a->dev);
}

static void contour_and_rim(FrameBatch &fb, const std::vector<Slot *> &ss, double *Slot::*verts,
                            bool stage1) {
    lc_ctx *c = fb.c;
    const lc_actor *a = fb.a;
    const int H = fb.cam.height, W = fb.cam.width;
    std::vector<RasterJob> rj;
    for (Slot *s : ss) rj.push_back(raster_job(s, s->*verts, s->own_mask));
    raster(c, a, fb.cam, rj);
    // own-silhouette contour buckets: the rim's bounded queries need nothing else
    {
        std::vector<OwnCellsJob> oj;
        for (Slot *s : ss) oj.push_back(OwnCellsJob{s->own_mask, s->own_cnt, s->own_keys});
        const int ncx = (W + LC_GRID_CELL - 1) / LC_GRID_CELL, ncy = (H + LC_GRID_CELL - 1) / LC_GRID_CELL;
        launch(c, k_own_cells, dim3((ncx * ncy + 7) / 8, (unsigned)ss.size()), dim3(256), 0, stage(c, oj), H, W, ncx);
    }
    std::vector<ContourJob> cj;
    for (Slot *s : ss) {
        ContourJob j{};
        j.verts = s->*verts; j.zbuf = s->zbuf; j.tri_front = s->tri_front; j.tri_n = s->tri_n;
        j.vflag = s->vflag; j.idx = s->cidx; j.n2d = s->n2d; j.B = s->B;
        j.vis = stage1 ? nullptr : s->vis;
        j.P = stage1 ? nullptr : s->P;
        j.active = 1;
        cj.push_back(j);
    }
    const auto dcj = stage(c, cj);
    const unsigned S = (unsigned)ss.size();
    launch(c, k_tri_front, dim3(64, S), dim3(256), 0, dcj, a->dev);
    launch(c, k_sil_edges, dim3(64, S), dim3(256), 0, dcj, a->dev);
    launch(c, k_vis_flags, dim3((a->dev.N + 255) / 256, S), dim3(256), 0, dcj, a->dev, cam_dev(fb.cam));
    launch(c, k_contour_compact, dim3(S), dim3(1024), 0, dcj, a->dev, cam_dev(fb.cam));
    std::vector<RimJob> rjs;
    for (Slot *s : ss) {
        RimJob r{};
        r.verts = s->*verts; r.idx = s->cidx; r.B = s->B;
        r.own = grid_dev(s->own, s->own_mask, H, W);
        r.own_cnt = s->own_cnt;
        r.own_keys = s->own_keys;
        r.keep = s->enabled;
        r.stage1 = stage1;
        r.active = 1;
        r.tri_id = s->tri_id;
        r.part_gate = !stage1 && fb.cfg->enable_part_mask;
        r.dilation = fb.cfg->nonrigid.part_dilation;
        rjs.push_back(r);
    }
    launch(c, k_rim, dim3(128, S), dim3(256), 0, stage(c, rjs), a->dev, cam_dev(fb.cam),
           (const double *)fb.cf->probe);
}

static void pose_launch(lc_ctx *c, const lc_actor *a, const lc_camera &cam, const std::vector<PoseJob> &jobs) {
    const size_t smem = pose_smem_bytes(a->skel.J);
    static const int cs_env = cluster_size_for("LIVECAP_POSE_CLUSTER");
    const int cs = c->pose_cs > 0 ? c->pose_cs : cs_env > 0 ? cs_env : cluster_size();
    auto k = cs == 1 ? k_pose_solve_t<1> : cs == 2 ? k_pose_solve_t<2> : cs == 4 ? k_pose_solve_t<4> : cs == 8 ? k_pose_solve_t<8>
                                                                           : k_pose_solve_t<16>;
    launch_cluster("k_pose_solve", c, k, (int)jobs.size(), cs, dim3(pose_block_threads()), smem,
                   stage(c, jobs), (const SkelDev *)a->skel_dev, a->dev, cam_dev(cam));
}

static void surface_launch(lc_ctx *c, const lc_actor *a, const lc_camera &cam, const ConfigDev &cf,
                           const std::vector<SurfJob> &jobs) {
    // A stream's solve is latency-bound; the team size trades SMs per stream
    // against latency.  The default surface team grows with the mesh: the
    // smallest of 4, 8, 16 CTAs that leaves at most 3 vertices per thread
    // (x5k: 8; x20k: 16).  Measured at the bench's 16 streams in 4 groups
    // with the owner-computes assembly: x5k 8-CTA teams 3669 frames/s and
    // 1.34 ms per launch vs 3498 and 2.04 ms on 4 (round 1, before the
    // preprocessing contention was visible: 4/4 3.93k, 4/8 3.76k); x20k
    // cfg4 16: 1998 frames/s vs 1790 on 8 and 1362 on 4.  A single
    // latency-critical stream solves fastest with LIVECAP_POSE_CLUSTER=8
    // LIVECAP_SURFACE_CLUSTER=16.
    static const int cs_env = cluster_size_for("LIVECAP_SURFACE_CLUSTER");
    static const bool cs_global = getenv("LIVECAP_CLUSTER") != nullptr;
    int cs = c->surf_cs > 0 ? c->surf_cs : cs_env > 0 ? cs_env : cluster_size();
    if (c->surf_cs <= 0 && cs_env <= 0 && !cs_global)
        while (cs < 16 && (long long)a->dev.N > 3LL * cs * surface_block_threads()) cs *= 2;
    auto k = cs == 1 ? k_surface_solve_t<1> : cs == 2 ? k_surface_solve_t<2> : cs == 4 ? k_surface_solve_t<4>
             : cs == 8 ? k_surface_solve_t<8> : k_surface_solve_t<16>;
    size_t smem = 0;
    const int mode = surface_pcg_mode(a->dev.N, cs, &smem);
    launch_cluster("k_surface_solve", c, k, (int)jobs.size(), cs, dim3(surface_block_threads()), smem,
                   stage(c, jobs), a->dev, cam_dev(cam), cf.ec, cf.shp, cam.height, cam.width, mode);
}

// stages: 1 = conditioning + Stage I, 2 = Stage II + state update, 3 = both
// (a Stage-II-only run derives the displaced rest itself and keeps the pose
// already in the slot, imported from the Stage I device by lc_tracker_pipe)
static void run_frame(FrameBatch &fb, int stages = 3) {
    lc_ctx *c = fb.c;
    const lc_actor *a = fb.a;
    const lc_config &cfg = *fb.cfg;
    const int H = fb.cam.height, W = fb.cam.width;
    auto &ss = fb.slots;
    const unsigned S = (unsigned)ss.size();
    // ---- preprocessing (pipeline.py:156-162) was launched on the auxiliary
    // stream by lc_tracker_step (possibly during the previous frame's solve);
    // the observed grid is joined before the pose solve, the pyramid before
    // the surface solve.
    // ---- condition (pipeline.py:165-170) + displaced rest + initial pose
    {
        std::vector<PrepJob> pj;
        for (Slot *s : ss) {
            PrepJob p{};
            p.rest = a->dev.rest; p.disp = s->has_disp ? s->disp : nullptr; p.drest = s->drest;
            p.j3d_raw = s->j3d_raw; p.j3d = s->j3d; p.v3d = s->v3d; p.fallbacks = s->fallbacks;
            p.x_prev = s->has_prev ? s->x_prev : nullptr;
            p.x_prev2 = s->has_prev2 ? s->x_prev2 : nullptr;
            p.x = (stages & 1) ? s->x : nullptr;
            p.pose_rep = (stages & 1) ? s->pose_rep : nullptr;
            p.nr_rep = (stages & 2) ? s->nr_rep : nullptr;
            p.N = a->dev.N;
            pj.push_back(p);
        }
        mark(c, "frame:start");
        launch(c, k_prep, dim3(16, S), dim3(256), 0, stage(c, pj), (const SkelDev *)a->skel_dev);
    }
    if (stages & 1) {
    // ---- Stage I (pipeline.py:173-224)
    int max_rounds = 0;
    std::vector<int> rounds(S);
    for (unsigned i = 0; i < S; ++i) {
        // frame 0: [{l2d=0, lsil=0}, {lsil=0}] + [{}] * max(1, rounds - 2)  (pipeline.py:191-193)
        rounds[i] = ss[i]->has_prev ? 1 : 2 + std::max(1, cfg.frame0_rounds - 2);
        max_rounds = std::max(max_rounds, rounds[i]);
    }
    std::vector<int> log_off(S, 0);
    for (int r = 0; r < max_rounds; ++r) {
        std::vector<Slot *> act;
        for (unsigned i = 0; i < S; ++i)
            if (r < rounds[i]) act.push_back(ss[i]);
        fk_skin(fb, act, true, true, &Slot::model, nullptr);
        mark(c, "s1:skin");
        contour_and_rim(fb, act, &Slot::model, true);
        mark(c, "s1:contour+rim");
        std::vector<PoseJob> pj;
        int k = 0;
        for (unsigned i = 0; i < S; ++i) {
            if (r >= rounds[i]) continue;
            Slot *s = ss[i];
            PoseJob p{};
            p.active = 1;
            p.x0 = s->x;
            p.x_out = s->x;
            p.obs = grid_dev(s->obs, s->mask_src, H, W);
            p.obs_K = s->obs.K;
            p.has_field = 1;
            p.B = s->B; p.cidx = s->cidx; p.n2d = s->n2d; p.crest = nullptr; p.drest = s->drest;
            p.enabled = s->enabled;
            p.j2d = s->j2d; p.j3d = s->j3d; p.v2d = s->v2d; p.v3d = s->v3d;
            p.prev_pos = s->has_prev ? s->joints_prev : nullptr;
            lc_pose_hyper h = cfg.pose;
            if (cfg.mode == 2) h.lambda_sil = 0.0;
            if (!s->has_prev) {
                h.gn_iterations *= cfg.frame0_iteration_scale;
                if (r == 0) { h.lambda_2d = 0.0; h.lambda_sil = 0.0; }
                if (r == 1) h.lambda_sil = 0.0;
            }
            fill_pose_hyper(p.hp, h, a->skel);
            p.directional = cfg.directional;
            p.report = s->pose_rep;
            p.log_offset = log_off[i];
            p.phase = s->phase_pose;
            p.nn_hint = s->nn_hint;
            p.fk_out = s->fk;
            log_off[i] += h.gn_iterations;
            pj.push_back(p);
            ++k;
        }
        if (r == 0)
            for (FrameIn *f : fb.in) ev_wait_x(c, c->stream, f->ready_obs);
        mark(c, "s1:waited-grid");
        pose_launch(c, a, fb.cam, pj);
        mark(c, "s1:pose");
    }
    }
    if (!(stages & 2)) return;
    // ---- Stage II (pipeline.py:227-260) or the pose-only surface
    // the pose kernel leaves FK(x) in s->fk when Stage I ran in this step
    const bool fk_from_x = !(stages & 1) || cfg.pose.gn_iterations <= 0;
    if (cfg.mode == 0) {
        fk_skin(fb, ss, fk_from_x, true, &Slot::vinit, nullptr);
        fk_skin(fb, ss, false, false, &Slot::vs, &Slot::rot);
    } else {
        fk_skin(fb, ss, fk_from_x, false, &Slot::vs, &Slot::rot);
    }
    if (cfg.mode == 0) {
        mark(c, "s2:skin");
        contour_and_rim(fb, ss, &Slot::vinit, false);
        mark(c, "s2:contour+rim");
        std::vector<SurfJob> sj;
        for (Slot *s : ss) {
            SurfJob j{};
            j.active = 1;
            j.do_solve = 1;
            j.do_snap = cfg.enable_snapping;
            j.v0 = s->vinit; j.v = s->v; j.vs = s->vs;
            j.pyr = s->pyr;
            j.pyr_tile = s->pyr_tile;
            j.image = s->image_src;
            j.obs = grid_dev(s->obs, s->mask_src, H, W);
            j.obs_K = s->obs.K;
            j.has_field = 1;
            j.vis = s->vis; j.P = s->P; j.bidx = s->cidx; j.B = s->B; j.n2d = s->n2d; j.enabled = s->enabled;
            j.prev = s->has_vprev ? s->v_prev : nullptr;
            j.prev2 = s->has_vprev2 ? s->v_prev2 : nullptr;
            j.directional = cfg.directional; j.enable_photo = 1; j.enable_sil = 1;
            j.diag = s->diag; j.minv = s->minv; j.rhs = s->rhs; j.x = s->sx; j.r = s->sr; j.z = s->sz;
            j.p = s->sp; j.ap = s->sap; j.best = s->sbest; j.edir = s->edir; j.eg = s->eg;
            j.ell_d = s->ell_d; j.ell_g = s->ell_g;
            j.off0 = s->off0; j.off1 = s->off1; j.hold = s->hold;
            j.report = s->nr_rep;
            j.nn_hint = s->nn_hint;
            j.counters = s->counters;
            j.phase = s->phase_surf;
            sj.push_back(j);
        }
        for (FrameIn *f : fb.in) ev_wait_x(c, c->stream, f->ready);
        mark(c, "s2:waited-pyr");
        surface_launch(c, a, fb.cam, *fb.cf, sj);
        mark(c, "s2:surface");
    }
    for (FrameIn *f : fb.in) ev_wait_x(c, c->stream, f->ready);   // join the aux stream in every mode
    // ---- state update (pipeline.py:281-299)
    std::vector<FinishJob> fj;
    for (Slot *s : ss) {
        FinishJob f{};
        f.x = s->x; f.v = cfg.mode == 0 ? s->v : s->vs; f.vs = s->vs; f.rot = s->rot; f.fk = s->fk;
        f.x_prev = s->x_prev; f.x_prev2 = s->x_prev2; f.joints_prev = s->joints_prev; f.disp = s->disp;
        f.v_prev = s->v_prev; f.v_prev2 = s->v_prev2;
        f.shift_x2 = s->has_prev; f.shift_v2 = s->has_vprev;
        f.warp = cfg.mode == 0 ? (cfg.enable_warping ? 1 : 0) : -1;
        f.N = a->dev.N; f.J = a->skel.J;
        fj.push_back(f);
    }
    launch(c, k_finish, dim3(16, S), dim3(256), 0, stage(c, fj));
    mark(c, "frame:end");
    for (Slot *s : ss) {
        s->has_prev2 = s->has_prev;
        s->has_prev = true;
        s->has_vprev2 = s->has_vprev;
        s->has_vprev = true;
        s->has_disp = true;
    }
}

// ---------------------------------------------------------------------------
// tracker

extern "C" int lc_tracker_create(lc_ctx *c, const lc_actor *a, const lc_camera *cam, const lc_config *cfg,
                                 int32_t S, lc_tracker **out) {
    API_BEGIN
    require(c && a && cam && cfg && out, "null argument");
    require(S >= 1, "n_streams must be >= 1");
    require(cam->width >= 2 && cam->height >= 2 && cam->fx > 0 && cam->fy > 0, "invalid camera");
    require(cfg->mode >= 0 && cfg->mode <= 2, "invalid mode");
    require(cfg->nonrigid.n_levels >= 1 && cfg->nonrigid.n_levels <= 4, "1..4 pyramid levels");
    CK(cudaSetDevice(c->device));
    lc_tracker *t = new lc_tracker();
    t->ctx = c;
    t->actor = a;
    t->cam = *cam;
    t->cfg = *cfg;
    t->S = S;
    build_config(c, a, &cfg->nonrigid, &cfg->pose, t->conf);
    for (int i = 0; i < S; ++i) {
        Slot *s = new Slot();
        s->allocate(a->dev.N, a->dev.T, a->dev.E, cam->height, cam->width, cfg->nonrigid.n_levels, a->skel.J);
        s->allocate_queue();
        t->slots.push_back(s);
    }
    CK(cudaStreamSynchronize(c->stream));
    *out = t;
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_destroy(lc_tracker *t) {
    if (!t) return LC_OK;
    cudaSetDevice(t->ctx->device);
    cudaStreamSynchronize(t->ctx->stream);
    cudaStreamSynchronize(t->ctx->aux);   // queued frames may still be preprocessing
    cudaStreamSynchronize(t->ctx->copy);
    for (auto &g : t->graphs) {
        cudaGraphExecDestroy(g.second.exec);
        cudaGraphExecDestroy(g.second.exec_aux);
    }
    for (Slot *s : t->slots) delete s;
    delete t;
    return LC_OK;
}


// Queues the next frame of one stream (at most LC_QUEUE queued frames per
// stream: the one the next step solves and the ones after it, whose upload
// and preprocessing then overlap that solve).
extern "C" int lc_tracker_set_frame(lc_tracker *t, int32_t stream, const double *image, const uint8_t *mask,
                                    const lc_detections *det, int32_t on_device) {
    API_BEGIN
    require(t && det, "null argument");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    // image == NULL queues the mask and detections only: Stage I reads no
    // image, so the Stage-I tracker of a GPU pair skips the 8-byte-per-
    // channel upload and the blur pyramid (Stage II refuses such a frame)
    require(mask, "null mask");
    Slot *s = t->slots[stream];
    lc_ctx *c = t->ctx;
    FrameIn &f = s->in[s->in_tail];
    require(f.state == 0, "the stream's frame queue is full: call lc_tracker_step first");
    const size_t HW = (size_t)s->H * s->W;
    f.has_image = image != nullptr;
    if (on_device && t->graph_mode) {
        // graph mode bakes buffer addresses into the captured graphs: a
        // device frame is copied into the queue's own buffers (copy engine)
        if (f.used) CK(cudaStreamWaitEvent(c->copy, f.freed, 0));
        if (image) CK(cudaMemcpyAsync(f.image, image, HW * 3 * sizeof(double), cudaMemcpyDeviceToDevice, c->copy));
        CK(cudaMemcpyAsync(f.mask, mask, HW, cudaMemcpyDeviceToDevice, c->copy));
        CK(cudaEventRecord(f.uploaded, c->copy));
        f.pending_upload = true;
        f.image_src = image ? f.image : nullptr;
        f.mask_src = f.mask;
    } else if (on_device) {
        f.image_src = image;
        f.mask_src = mask;
    } else {
        // the host copies go on the copy stream, after the solve that last
        // read the buffer; the buffer's preprocessing waits for them
        if (f.used) CK(cudaStreamWaitEvent(c->copy, f.freed, 0));
        if (image) CK(cudaMemcpyAsync(f.image, image, HW * 3 * sizeof(double), cudaMemcpyHostToDevice, c->copy));
        CK(cudaMemcpyAsync(f.mask, mask, HW, cudaMemcpyHostToDevice, c->copy));
        CK(cudaEventRecord(f.uploaded, c->copy));
        f.pending_upload = true;
        f.image_src = image ? f.image : nullptr;
        f.mask_src = f.mask;
    }
    const int J = t->actor->skel.J;
    stage_to(c, f.j2d, det->joints2d, sizeof(double) * 2 * (J + 4));
    stage_to(c, f.j3d_raw, det->joints3d, sizeof(double) * 3 * J);
    stage_to(c, f.v2d, det->valid2d, J + 4);
    stage_to(c, f.v3d, det->valid3d, J);
    f.state = 1;
    s->in_tail = (s->in_tail + 1) % LC_QUEUE;
    return LC_OK;
    API_END
}

// colour bytes -> [0, 1] doubles with the reference's exact `/ 255.0`
// (imageproc.py:297-299: np.asarray(img, float64) / 255.0)
__global__ void k_u8_to_unit(const uint8_t *src, double *dst, long long n) {
    lc_pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = (double)src[i] / 255.0;
}

// uint8 RGB variant of lc_tracker_set_frame (real-data ingest): 1 byte per
// channel crosses PCIe, converted on the device on the copy stream
extern "C" int lc_tracker_set_frame_u8(lc_tracker *t, int32_t stream, const uint8_t *image_rgb,
                                       const uint8_t *mask, const lc_detections *det, int32_t on_device) {
    API_BEGIN
    require(t && det && image_rgb && mask, "null argument");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    Slot *s = t->slots[stream];
    lc_ctx *c = t->ctx;
    FrameIn &f = s->in[s->in_tail];
    require(f.state == 0, "the stream's frame queue is full: call lc_tracker_step first");
    const size_t HW = (size_t)s->H * s->W;
    if (f.used) CK(cudaStreamWaitEvent(c->copy, f.freed, 0));
    const uint8_t *src = image_rgb;
    if (!on_device) {
        CK(cudaMemcpyAsync(f.image_u8, image_rgb, HW * 3, cudaMemcpyHostToDevice, c->copy));
        CK(cudaMemcpyAsync(f.mask, mask, HW, cudaMemcpyHostToDevice, c->copy));
        src = f.image_u8;
        f.mask_src = f.mask;
    } else {
        f.mask_src = mask;
    }
    {
        OnStream on(c, c->copy);
        launch(c, k_u8_to_unit, dim3((unsigned)std::min<size_t>((3 * HW + 255) / 256, 2368)), dim3(256), 0, src,
               f.image, (long long)(3 * HW));
    }
    CK(cudaEventRecord(f.uploaded, c->copy));
    f.pending_upload = true;
    f.image_src = f.image;
    f.has_image = true;
    const int J = t->actor->skel.J;
    stage_to(c, f.j2d, det->joints2d, sizeof(double) * 2 * (J + 4));
    stage_to(c, f.j3d_raw, det->joints3d, sizeof(double) * 3 * J);
    stage_to(c, f.v2d, det->valid2d, J + 4);
    stage_to(c, f.v3d, det->valid3d, J);
    f.state = 1;
    s->in_tail = (s->in_tail + 1) % LC_QUEUE;
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_step(lc_tracker *t) { return lc_tracker_step_stage(t, 3); }

// One solve stage of the oldest queued frame of every stream, which it then
// consumes: 1 = conditioning + Stage I, 2 = Stage II + state update, 3 =
// both.  A tracker that runs only stage 1 and one that runs only stage 2,
// joined by lc_tracker_pipe, split solve_frame across a GPU pair.
extern "C" int lc_tracker_step_stage(lc_tracker *t, int32_t stages) {
    API_BEGIN
    require(t != nullptr, "null tracker");
    require(stages >= 1 && stages <= 3, "stages must be 1, 2 or 3");
    lc_ctx *c = t->ctx;
    CK(cudaSetDevice(c->device));
    std::vector<FrameIn *> cur, todo, next;
    bool all_next = true;
    for (Slot *s : t->slots) {
        FrameIn &f = s->in[s->in_head];
        require(f.state >= 1, "no frame queued for a stream: call lc_tracker_set_frame first");
        require(f.has_image || !(stages & 2), "Stage II needs the frame's image (it was queued without one)");
        cur.push_back(&f);
        if (f.state == 1) todo.push_back(&f);
        FrameIn &n = s->in[(s->in_head + 1) % LC_QUEUE];
        if (n.state == 1) next.push_back(&n);
        else all_next = false;
    }
    // CUDA-graph mode: the steady state -- every stream's frame preprocessed
    // during the previous step, its next frame queued (and uploaded by an
    // earlier step's buffer), its track state warm -- is one captured graph
    // per frame-queue phase; the host only does the queue bookkeeping
    std::vector<long long> key;
    bool steady = t->graph_mode && stages == 3 && todo.empty() && all_next && !c->tracing &&
                  c->prof_name.empty() && t->slots.size() <= LC_JOB_INLINE;
    for (size_t i = 0; steady && i < t->slots.size(); ++i) {
        const Slot *s = t->slots[i];
        const FrameIn *n = next[i];
        steady = s->has_prev && s->has_prev2 && s->has_vprev && s->has_vprev2 && s->has_disp && n->used &&
                 cur[i]->has_image && n->has_image;
        key.push_back(s->in_head);
        key.push_back(n->pending_upload ? 1 : 0);
        key.push_back((long long)(uintptr_t)cur[i]->image_src);
        key.push_back((long long)(uintptr_t)cur[i]->mask_src);
        key.push_back((long long)(uintptr_t)n->image_src);
        key.push_back((long long)(uintptr_t)n->mask_src);
    }
    auto bookkeeping = [&]() {
        for (FrameIn *f : next) {
            f->pending_upload = false;
            f->state = 2;
        }
        for (size_t i = 0; i < t->slots.size(); ++i) {
            t->slots[i]->view(*cur[i]);
            FrameIn &f = *cur[i];
            f.used = true;
            f.state = 0;
            t->slots[i]->in_head = (t->slots[i]->in_head + 1) % LC_QUEUE;
        }
        t->frame_counter++;
    };
    if (steady) {
        auto it = t->graphs.find(key);
        if (it == t->graphs.end()) {
            // capture the two branches separately, so that the next frame's
            // preprocessing (auxiliary stream) keeps overlapping this and the
            // following solves exactly as in the eager schedule
            lc_tracker::Graph gr;
            const long long l0 = c->launches;
            cudaGraph_t g = nullptr;
            c->capturing = true;
            try {
                CK(cudaStreamBeginCapture(c->aux, cudaStreamCaptureModeThreadLocal));
                launch_preprocess(c, t->conf, t->cfg, next, t->cam.height, t->cam.width);
                CK(cudaStreamEndCapture(c->aux, &g));
                CK(cudaGraphInstantiate(&gr.exec_aux, g, 0));
                cudaGraphDestroy(g);
                g = nullptr;
                for (size_t i = 0; i < next.size(); ++i) {   // (launch_preprocess's bookkeeping, undone:
                    next[i]->state = 1;                          //  the launch below redoes it)
                    next[i]->pending_upload = key[6 * i + 1] != 0;
                }
                CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
                for (size_t i = 0; i < t->slots.size(); ++i) t->slots[i]->view(*cur[i]);
                FrameBatch fb{c, t->actor, t->cam, &t->cfg, &t->conf, t->slots, cur};
                run_frame(fb, stages);
                for (size_t i = 0; i < t->slots.size(); ++i) ev_record_x(c, cur[i]->freed, c->stream);
                CK(cudaStreamEndCapture(c->stream, &g));
                CK(cudaGraphInstantiate(&gr.exec, g, 0));
                cudaGraphDestroy(g);
            } catch (...) {
                c->capturing = false;
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(c->aux, &junk);
                if (junk) cudaGraphDestroy(junk);
                junk = nullptr;
                cudaStreamEndCapture(c->stream, &junk);
                if (junk) cudaGraphDestroy(junk);
                throw;
            }
            c->capturing = false;
            gr.kernels = c->launches - l0;
            c->launches = l0;   // counted when the graphs run
            g_launches.fetch_sub(gr.kernels, std::memory_order_relaxed);
            it = t->graphs.emplace(key, gr).first;
        } else {
            t->graph_replays++;
        }
        bookkeeping();
        CK(cudaEventRecord(c->ev_fork, c->stream));
        CK(cudaGraphLaunch(it->second.exec_aux, c->aux));
        CK(cudaGraphLaunch(it->second.exec, c->stream));
        c->launches += it->second.kernels;
        g_launches.fetch_add(it->second.kernels, std::memory_order_relaxed);
        return last_launch_status();
    }
    const int H = t->cam.height, W = t->cam.width;
    launch_preprocess(c, t->conf, t->cfg, todo, H, W);
    // every stream already has its next frame: preprocess it during this solve
    if (all_next) launch_preprocess(c, t->conf, t->cfg, next, H, W);
    for (size_t i = 0; i < t->slots.size(); ++i) t->slots[i]->view(*cur[i]);
    FrameBatch fb{c, t->actor, t->cam, &t->cfg, &t->conf, t->slots, cur};
    run_frame(fb, stages);
    for (size_t i = 0; i < t->slots.size(); ++i) {
        FrameIn &f = *cur[i];
        CK(cudaEventRecord(f.freed, c->stream));
        f.used = true;
        f.state = 0;
        t->slots[i]->in_head = (t->slots[i]->in_head + 1) % LC_QUEUE;
    }
    t->frame_counter++;
    return last_launch_status();
    API_END
}

// CUDA-graph mode for the steady state of lc_tracker_step (see there)
extern "C" int lc_tracker_set_graph(lc_tracker *t, int32_t on) {
    API_BEGIN
    require(t != nullptr, "null tracker");
    t->graph_mode = on != 0;
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_graph_stats(lc_tracker *t, int64_t *graphs, int64_t *replays) {
    API_BEGIN
    require(t && graphs && replays, "null argument");
    *graphs = (int64_t)t->graphs.size();
    *replays = t->graph_replays;
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_get_result(lc_tracker *t, int32_t stream, double *pose_out, double *verts_out,
                                     double *skinned_out, lc_frame_report *rep) {
    API_BEGIN
    require(t != nullptr, "null tracker");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    Slot *s = t->slots[stream];
    lc_ctx *c = t->ctx;
    const size_t N = s->N;
    if (pose_out) CK(cudaMemcpyAsync(pose_out, s->x_prev, sizeof(double) * LC_NP, cudaMemcpyDeviceToHost, c->stream));
    if (verts_out) CK(cudaMemcpyAsync(verts_out, s->v_prev, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, c->stream));
    if (skinned_out) CK(cudaMemcpyAsync(skinned_out, s->vs, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, c->stream));
    if (rep) {
        CK(cudaMemcpyAsync(&rep->pose, s->pose_rep, sizeof(lc_pose_report), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&rep->nonrigid, s->nr_rep, sizeof(lc_nonrigid_report), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&rep->rescale_fallbacks, s->fallbacks, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return last_launch_status();
    API_END
}

// Stage handoff between two trackers of the same actor / camera / stream
// count, possibly on different GPUs (the paper's pose -> non-rigid stage
// pipeline over a GPU pair):
//   what = 1: the solved pose of every stream, src -> dst (Stage I device ->
//             Stage II device, 36 doubles per stream);
//   what = 2: the track state Stage I needs, src -> dst (x_prev, x_prev2,
//             joints_prev, disp_rest + their flags; Stage II device -> Stage I
//             device, ~0.13 MB per stream at x5k).
// The copies are peer copies over NVLink on the destination's stream, after
// an event on the source's stream, so they are ordered after the source
// stage and before the destination's next stage.
extern "C" int lc_tracker_pipe(lc_tracker *dst, lc_tracker *src, int32_t what) {
    API_BEGIN
    require(dst && src && dst != src, "two distinct trackers required");
    require(dst->S == src->S && dst->actor->dev.N == src->actor->dev.N, "trackers do not match");
    require(what == 1 || what == 2, "what must be 1 (pose) or 2 (state)");
    lc_ctx *cd = dst->ctx, *cs = src->ctx;
    if (cd->device != cs->device) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, cd->device, cs->device);
        if (can) {
            CK(cudaSetDevice(cd->device));
            const cudaError_t e = cudaDeviceEnablePeerAccess(cs->device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else CK(e);
        }
    }
    CK(cudaSetDevice(cs->device));
    CK(cudaEventRecord(cs->ev_pipe, cs->stream));
    CK(cudaSetDevice(cd->device));
    CK(cudaStreamWaitEvent(cd->stream, cs->ev_pipe, 0));
    const size_t N = dst->actor->dev.N;
    for (int i = 0; i < dst->S; ++i) {
        Slot *d = dst->slots[i], *s = src->slots[i];
        auto cp = [&](void *to, const void *from, size_t bytes) {
            CK(cudaMemcpyPeerAsync(to, cd->device, from, cs->device, bytes, cd->stream));
        };
        if (what == 1) {
            cp(d->x, s->x, sizeof(double) * LC_NP);
        } else {
            cp(d->x_prev, s->x_prev, sizeof(double) * LC_NP);
            cp(d->x_prev2, s->x_prev2, sizeof(double) * LC_NP);
            cp(d->joints_prev, s->joints_prev, sizeof(double) * 3 * LC_MAXJ);
            cp(d->disp, s->disp, sizeof(double) * 3 * N);
            d->has_prev = s->has_prev;
            d->has_prev2 = s->has_prev2;
            d->has_disp = s->has_disp;
        }
    }
    return LC_OK;
    API_END
}

// Streaming readout: enqueue the D2H copies of the last stepped frame's pose
// and surface on the solve stream and return at once (pinned destinations
// make it fully asynchronous).  The data is on the host once the stream has
// passed this point (an event recorded after it, or lc_ctx_synchronize), so
// a caller can read frame f while frame f+1 is being solved.
extern "C" int lc_tracker_get_result_async(lc_tracker *t, int32_t stream, double *pose_out, double *verts_out) {
    API_BEGIN
    require(t != nullptr, "null tracker");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    Slot *s = t->slots[stream];
    lc_ctx *c = t->ctx;
    if (pose_out) CK(cudaMemcpyAsync(pose_out, s->x_prev, sizeof(double) * LC_NP, cudaMemcpyDeviceToHost, c->stream));
    if (verts_out)
        CK(cudaMemcpyAsync(verts_out, s->v_prev, sizeof(double) * 3 * s->N, cudaMemcpyDeviceToHost, c->stream));
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_set_state(lc_tracker *t, int32_t stream, const double *x_prev, const double *x_prev2,
                                    const double *joints_prev, const double *disp_rest, const double *v_prev,
                                    const double *v_prev2) {
    API_BEGIN
    require(t != nullptr, "null tracker");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    Slot *s = t->slots[stream];
    lc_ctx *c = t->ctx;
    const size_t N = s->N;
    const int J = t->actor->skel.J;
    auto put = [&](double *dst, const double *src, size_t n) {
        if (src) cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, c->stream);
    };
    require(!(x_prev && !joints_prev), "joints_prev is required with pose_prev");
    put(s->x_prev, x_prev, LC_NP);
    put(s->x_prev2, x_prev2, LC_NP);
    put(s->joints_prev, joints_prev, 3 * J);
    put(s->disp, disp_rest, 3 * N);
    put(s->v_prev, v_prev, 3 * N);
    put(s->v_prev2, v_prev2, 3 * N);
    s->has_prev = x_prev != nullptr;
    s->has_prev2 = x_prev2 != nullptr;
    s->has_disp = disp_rest != nullptr;
    s->has_vprev = v_prev != nullptr;
    s->has_vprev2 = v_prev2 != nullptr;
    CK(cudaStreamSynchronize(c->stream));
    return LC_OK;
    API_END
}

// Stage I output of one stream (36 doubles, host): the pose the next
// lc_tracker_step_stage(t, 2) solves Stage II from (per-stage teacher forcing
// in the parity tests; the GPU-pair pipeline moves it with lc_tracker_pipe)
extern "C" int lc_tracker_set_pose(lc_tracker *t, int32_t stream, const double *x36) {
    API_BEGIN
    require(t && x36, "null argument");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));
    for (int k = 0; k < LC_NP; ++k) require(std::isfinite(x36[k]), "non-finite pose");
    CK(cudaMemcpyAsync(t->slots[stream]->x, x36, sizeof(double) * LC_NP, cudaMemcpyHostToDevice, t->ctx->stream));
    CK(cudaStreamSynchronize(t->ctx->stream));
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_get_state(lc_tracker *t, int32_t stream, int32_t *flags, double *x_prev,
                                    double *x_prev2, double *joints_prev, double *disp_rest, double *v_prev,
                                    double *v_prev2) {
    API_BEGIN
    require(t != nullptr, "null tracker");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    Slot *s = t->slots[stream];
    lc_ctx *c = t->ctx;
    const size_t N = s->N;
    const int J = t->actor->skel.J;
    auto get = [&](double *dst, const double *src, size_t n) {
        if (dst) cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    };
    get(x_prev, s->x_prev, LC_NP);
    get(x_prev2, s->x_prev2, LC_NP);
    get(joints_prev, s->joints_prev, 3 * J);
    get(disp_rest, s->disp, 3 * N);
    get(v_prev, s->v_prev, 3 * N);
    get(v_prev2, s->v_prev2, 3 * N);
    if (flags) {
        flags[0] = s->has_prev; flags[1] = s->has_prev2; flags[2] = s->has_disp;
        flags[3] = s->has_vprev; flags[4] = s->has_vprev2;
    }
    CK(cudaStreamSynchronize(c->stream));
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_counters(lc_tracker *t, int32_t stream, int64_t *out) {
    API_BEGIN
    require(t && out, "null argument");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    CK(cudaMemcpyAsync(out, t->slots[stream]->counters, sizeof(long long) * LC_NCOUNTERS,
                       cudaMemcpyDeviceToHost, t->ctx->stream));
    CK(cudaStreamSynchronize(t->ctx->stream));
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_inspect(lc_tracker *t, int32_t stream, int32_t what, void *out, int64_t cap,
                                  int64_t *n_out) {
    API_BEGIN
    require(t && out && n_out, "null argument");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    Slot *s = t->slots[stream];
    cudaStream_t st = t->ctx->stream;
    int B = 0, P = 0;
    CK(cudaMemcpyAsync(&B, s->B, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&P, s->P, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const size_t N = s->N;
    if (what == 0 || what == 2) {
        const int n = what == 0 ? B : P;
        require(n <= cap, "capacity too small");
        std::vector<int> tmp(n);
        if (n) CK(cudaMemcpy(tmp.data(), what == 0 ? s->cidx : s->vis, sizeof(int) * n, cudaMemcpyDeviceToHost));
        for (int i = 0; i < n; ++i) static_cast<int64_t *>(out)[i] = tmp[i];
        *n_out = n;
    } else if (what == 1) {
        require(B <= cap, "capacity too small");
        std::vector<uint8_t> tmp(B);
        if (B) CK(cudaMemcpy(tmp.data(), s->enabled, B, cudaMemcpyDeviceToHost));
        for (int i = 0; i < B; ++i) static_cast<int64_t *>(out)[i] = tmp[i];
        *n_out = B;
    } else if (what == 3) {
        require(2 * (int64_t)B <= cap, "capacity too small");
        if (B) CK(cudaMemcpy(out, s->n2d, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost));
        *n_out = B;
    } else if (what == 4 || what == 5) {
        require((int64_t)(3 * N) <= cap, "capacity too small");
        CK(cudaMemcpy(out, what == 4 ? s->vinit : s->vs, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost));
        *n_out = (int64_t)N;
    } else if (what >= 6 && what <= 9) {
        // the last Stage II GN step's normal system: 6 diag (N*6 sym), 7 rhs,
        // 8 the PCG's best iterate (N*3), 9 the Jacobi inverse (N*9)
        const size_t w = what == 6 ? 6 : what == 9 ? 9 : 3;
        require((int64_t)(w * N) <= cap, "capacity too small");
        const double *src = what == 6 ? s->diag : what == 7 ? s->rhs : what == 8 ? s->sbest : s->minv;
        CK(cudaMemcpy(out, src, sizeof(double) * w * N, cudaMemcpyDeviceToHost));
        *n_out = (int64_t)N;
    } else {
        return fail(LC_EINVAL, "unknown inspect target");
    }
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_phase_times(lc_tracker *t, int32_t stream, int64_t *pose_ns, int64_t *surf_ns) {
    API_BEGIN
    require(t != nullptr, "null tracker");
    require(stream >= 0 && stream < t->S, "stream index out of range");
    CK(cudaSetDevice(t->ctx->device));   // the tracker's streams belong to its device
    Slot *s = t->slots[stream];
    if (pose_ns) CK(cudaMemcpy(pose_ns, s->phase_pose, sizeof(long long) * LC_NPHASE, cudaMemcpyDeviceToHost));
    if (surf_ns) CK(cudaMemcpy(surf_ns, s->phase_surf, sizeof(long long) * LC_NPHASE, cudaMemcpyDeviceToHost));
    return LC_OK;
    API_END
}

extern "C" int lc_tracker_device_vertices(lc_tracker *t, int32_t stream, uint64_t *dptr) {
    if (!t || !dptr || stream < 0 || stream >= t->S) return fail(LC_EINVAL, "bad argument");
    *dptr = reinterpret_cast<uint64_t>(t->slots[stream]->v_prev);
    return LC_OK;
}

// ---------------------------------------------------------------------------
// single-call seams (a scratch slot per context, sized to actor + camera)

static Slot *call_slot(lc_ctx *c, const lc_actor *a, int H, int W, int levels) {
    if (!c->call_slot || c->call_actor != a || c->call_w != W || c->call_h != H || c->call_slot->levels < levels) {
        cudaStreamSynchronize(c->stream);
        delete c->call_slot;
        c->call_slot = new Slot();
        c->call_slot->allocate(a->dev.N, a->dev.T, a->dev.E, H, W, std::max(levels, 3), a->skel.J);
        c->call_actor = a;
        c->call_w = W;
        c->call_h = H;
    }
    return c->call_slot;
}

extern "C" int lc_pose_solve(lc_ctx *c, const lc_actor *a, const lc_camera *cam, const lc_pose_problem *pb,
                             const double *x0, double *x_out, lc_pose_report *report) {
    API_BEGIN
    require(c && a && cam && pb && x0 && x_out, "null argument");
    require(pb->n_contour >= 0 && pb->n_contour <= a->dev.N, "contour size out of range");
    CK(cudaSetDevice(c->device));
    const int H = cam->height, W = cam->width, J = a->skel.J;
    Slot *s = call_slot(c, a, H, W, 1);
    cudaStream_t st = c->stream;
    const bool has_field = pb->mask != nullptr;
    if (has_field) {
        CK(cudaMemcpyAsync(s->mask, pb->mask, (size_t)H * W, cudaMemcpyHostToDevice, st));
        build_grids(c, {{&s->obs, s->mask}}, H, W);
    }
    CK(cudaMemcpyAsync(s->j2d, pb->joints2d, sizeof(double) * 2 * (J + 4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->j3d, pb->joints3d, sizeof(double) * 3 * J, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->v2d, pb->valid2d, J + 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->v3d, pb->valid3d, J, cudaMemcpyHostToDevice, st));
    const int B = pb->n_contour;
    std::vector<int> idx(B);
    for (int i = 0; i < B; ++i) {
        idx[i] = (int)pb->contour_indices[i];
        require(idx[i] >= 0 && idx[i] < a->dev.N, "contour index out of range");
    }
    if (B) {
        CK(cudaMemcpyAsync(s->cidx, idx.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(s->n2d, pb->contour_normals2d, sizeof(double) * 2 * B, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(s->crest, pb->contour_rest, sizeof(double) * 3 * B, cudaMemcpyHostToDevice, st));
        if (pb->contour_enabled)
            CK(cudaMemcpyAsync(s->enabled, pb->contour_enabled, B, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(s->B, &B, sizeof(int), cudaMemcpyHostToDevice, st));
    if (pb->prev_positions)
        CK(cudaMemcpyAsync(s->joints_prev, pb->prev_positions, sizeof(double) * 3 * J, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->x0, x0, sizeof(double) * LC_NP, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(s->pose_rep, 0, sizeof(lc_pose_report), st));
    PoseJob p{};
    p.active = 1;
    p.x0 = s->x0;
    p.x_out = s->x;
    p.obs = grid_dev(s->obs, s->mask, H, W);
    p.obs_K = s->obs.K;
    p.has_field = has_field;
    p.B = s->B; p.cidx = s->cidx; p.n2d = s->n2d; p.crest = s->crest; p.drest = nullptr;
    p.enabled = pb->contour_enabled ? s->enabled : nullptr;
    p.j2d = s->j2d; p.j3d = s->j3d; p.v2d = s->v2d; p.v3d = s->v3d;
    p.prev_pos = pb->prev_positions ? s->joints_prev : nullptr;
    fill_pose_hyper(p.hp, pb->hyper, a->skel);
    p.directional = pb->directional;
    p.report = s->pose_rep;
    p.log_offset = 0;
    p.nn_hint = s->nn_hint;
    require(pb->hyper.gn_iterations <= LC_MAX_LOG, "too many GN iterations for the report");
    pose_launch(c, a, *cam, {p});
    CK(cudaMemcpyAsync(x_out, s->x, sizeof(double) * LC_NP, cudaMemcpyDeviceToHost, st));
    if (report) CK(cudaMemcpyAsync(report, s->pose_rep, sizeof(lc_pose_report), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

extern "C" int lc_nonrigid_solve(lc_ctx *c, const lc_actor *a, const lc_camera *cam, const lc_nonrigid_problem *pb,
                                 const double *v0, int32_t do_solve, int32_t do_snap, double *v_out,
                                 lc_nonrigid_report *report) {
    API_BEGIN
    require(c && a && cam && pb && v0 && v_out, "null argument");
    require(pb->n_levels >= 1 && pb->n_levels <= 4, "1..4 pyramid levels");
    require(pb->hyper.gn_iterations <= LC_MAX_LOG, "too many GN iterations for the report");
    CK(cudaSetDevice(c->device));
    const int H = cam->height, W = cam->width, N = a->dev.N;
    Slot *s = call_slot(c, a, H, W, pb->n_levels);
    cudaStream_t st = c->stream;
    const bool has_field = pb->mask != nullptr;
    if (has_field) {
        CK(cudaMemcpyAsync(s->mask, pb->mask, (size_t)H * W, cudaMemcpyHostToDevice, st));
        build_grids(c, {{&s->obs, s->mask}}, H, W);
    }
    const size_t HW3 = (size_t)H * W * 3;
    if (pb->pyramid)
        CK(cudaMemcpyAsync(s->pyr, pb->pyramid, sizeof(double) * HW3 * pb->n_levels, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->vs, pb->skinned, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->vinit, v0, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    auto put_idx = [&](int *dst, const int64_t *src, int n) {
        std::vector<int> t(n);
        for (int i = 0; i < n; ++i) {
            t[i] = (int)src[i];
            require(t[i] >= 0 && t[i] < N, "vertex index out of range");
        }
        if (n) cudaMemcpyAsync(dst, t.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
    };
    put_idx(s->vis, pb->visible, pb->n_visible);
    put_idx(s->cidx, pb->boundary, pb->n_boundary);
    CK(cudaMemcpyAsync(s->P, &pb->n_visible, sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->B, &pb->n_boundary, sizeof(int), cudaMemcpyHostToDevice, st));
    if (pb->n_boundary) {
        CK(cudaMemcpyAsync(s->n2d, pb->normals2d, sizeof(double) * 2 * pb->n_boundary, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(s->enabled, pb->enabled, pb->n_boundary, cudaMemcpyHostToDevice, st));
    }
    if (pb->prev) CK(cudaMemcpyAsync(s->v_prev, pb->prev, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    if (pb->prev2) CK(cudaMemcpyAsync(s->v_prev2, pb->prev2, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(s->nr_rep, 0, sizeof(lc_nonrigid_report), st));
    ConfigDev cf;
    lc_nonrigid_hyper nh = pb->hyper;
    nh.n_levels = pb->n_levels;
    build_config(c, a, &nh, nullptr, cf);
    SurfJob j{};
    j.active = 1;
    j.do_solve = do_solve;
    j.do_snap = do_snap;
    j.v0 = s->vinit; j.v = s->v; j.vs = s->vs; j.pyr = s->pyr;
    j.obs = grid_dev(s->obs, s->mask, H, W);
    j.obs_K = s->obs.K;
    j.has_field = has_field;
    j.vis = s->vis; j.P = s->P; j.bidx = s->cidx; j.B = s->B; j.n2d = s->n2d; j.enabled = s->enabled;
    j.prev = pb->prev ? s->v_prev : nullptr;
    j.prev2 = pb->prev2 ? s->v_prev2 : nullptr;
    j.directional = pb->directional; j.enable_photo = pb->enable_photo; j.enable_sil = pb->enable_sil;
    j.diag = s->diag; j.minv = s->minv; j.rhs = s->rhs; j.x = s->sx; j.r = s->sr; j.z = s->sz;
    j.p = s->sp; j.ap = s->sap; j.best = s->sbest; j.edir = s->edir; j.eg = s->eg;
    j.ell_d = s->ell_d; j.ell_g = s->ell_g;
    j.off0 = s->off0; j.off1 = s->off1; j.hold = s->hold;
    j.report = s->nr_rep;
    j.nn_hint = s->nn_hint;
    surface_launch(c, a, *cam, cf, {j});
    CK(cudaMemcpyAsync(v_out, s->v, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, st));
    if (report) CK(cudaMemcpyAsync(report, s->nr_rep, sizeof(lc_nonrigid_report), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

extern "C" int lc_forward_kinematics(lc_ctx *c, const lc_actor *a, const double *x36, double *rot_out,
                                     double *pos_out, double *markers_out, double *dqs_out, int32_t *gimbal) {
    API_BEGIN
    require(c && a && x36, "null argument");
    CK(cudaSetDevice(c->device));
    DevArena m;
    double *dx = m.upload(x36, LC_NP, c->stream);
    FkState *f = m.alloc<FkState>(1);
    launch(c, k_fk, dim3(1), dim3(32), 0, stage(c, std::vector<FkJob>{FkJob{dx, f, 1}}),
           (const SkelDev *)a->skel_dev);
    FkState h;
    CK(cudaMemcpyAsync(&h, f, sizeof(FkState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const int J = a->skel.J;
    for (int j = 0; j < J; ++j) {
        if (rot_out) std::memcpy(rot_out + 9 * j, h.rot[j], 9 * sizeof(double));
        if (pos_out) std::memcpy(pos_out + 3 * j, h.pos[j], 3 * sizeof(double));
        if (dqs_out) std::memcpy(dqs_out + 8 * j, h.dq[j], 8 * sizeof(double));
    }
    if (markers_out) std::memcpy(markers_out, h.markers, 12 * sizeof(double));
    if (gimbal) *gimbal = h.gimbal;
    return last_launch_status();
    API_END
}

__global__ void k_skin_jac(const FkState *fk, const SkelDev *skg, ActorDev A, int M, const double *rest,
                           const int *subset, double *jac);

extern "C" int lc_skin_points(lc_ctx *c, const lc_actor *a, const double *x36, int32_t M, const double *rest,
                              const int64_t *subset, double *pos_out, double *rot_out, double *jac_out) {
    API_BEGIN
    require(c && a && x36 && rest && pos_out, "null argument");
    require(M >= 0, "negative point count");
    if (!subset) require(M == a->dev.N, "without a subset, rest points must cover every vertex");
    CK(cudaSetDevice(c->device));
    if (M == 0) return LC_OK;
    DevArena m;
    cudaStream_t st = c->stream;
    double *dx = m.upload(x36, LC_NP, st);
    FkState *f = m.alloc<FkState>(1);
    double *dr = m.upload(rest, 3 * (size_t)M, st);
    int *ds = nullptr;
    if (subset) {
        std::vector<int> t(M);
        for (int i = 0; i < M; ++i) {
            t[i] = (int)subset[i];
            require(t[i] >= 0 && t[i] < a->dev.N, "subset index out of range");
        }
        ds = m.upload(t.data(), M, st);
        CK(cudaStreamSynchronize(st));
    }
    double *dp = m.alloc<double>(3 * (size_t)M);
    double *dq = rot_out ? m.alloc<double>(4 * (size_t)M) : nullptr;
    launch(c, k_fk, dim3(1), dim3(32), 0, stage(c, std::vector<FkJob>{FkJob{dx, f, 1}}),
           (const SkelDev *)a->skel_dev);
    SkinJob j{};
    j.fk = f; j.rest = dr; j.subset = ds; j.pos = dp; j.rot = dq; j.M = M; j.active = 1;
    launch(c, k_skin, dim3((M + 127) / 128), dim3(128), 0, stage(c, std::vector<SkinJob>{j}), a->dev);
    double *dj = nullptr;
    if (jac_out) {
        dj = m.alloc<double>((size_t)M * 3 * LC_NP);
        launch(c, k_skin_jac, dim3((M + 127) / 128), dim3(128), 0, (const FkState *)f,
               (const SkelDev *)a->skel_dev, a->dev, M, (const double *)dr, (const int *)ds, dj);
    }
    CK(cudaMemcpyAsync(pos_out, dp, sizeof(double) * 3 * M, cudaMemcpyDeviceToHost, st));
    if (rot_out) CK(cudaMemcpyAsync(rot_out, dq, sizeof(double) * 4 * M, cudaMemcpyDeviceToHost, st));
    if (jac_out) CK(cudaMemcpyAsync(jac_out, dj, sizeof(double) * 3 * LC_NP * M, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

extern "C" int lc_contour_vertices(lc_ctx *c, const lc_actor *a, const lc_camera *cam, const double *verts,
                                   int32_t *n_out, int64_t *idx_out, double *n2d_out) {
    API_BEGIN
    require(c && a && cam && verts && n_out, "null argument");
    CK(cudaSetDevice(c->device));
    const int H = cam->height, W = cam->width, N = a->dev.N;
    Slot *s = call_slot(c, a, H, W, 1);
    cudaStream_t st = c->stream;
    CK(cudaMemcpyAsync(s->model, verts, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    raster(c, a, *cam, {raster_job(s, s->model, nullptr)});
    ContourJob j{};
    j.verts = s->model; j.zbuf = s->zbuf; j.tri_front = s->tri_front; j.tri_n = s->tri_n; j.vflag = s->vflag;
    j.idx = s->cidx; j.n2d = s->n2d; j.B = s->B; j.vis = nullptr; j.P = nullptr; j.active = 1;
    const auto dj = stage(c, std::vector<ContourJob>{j});
    launch(c, k_tri_front, dim3(64), dim3(256), 0, dj, a->dev);
    launch(c, k_sil_edges, dim3(64), dim3(256), 0, dj, a->dev);
    launch(c, k_vis_flags, dim3((a->dev.N + 255) / 256), dim3(256), 0, dj, a->dev, cam_dev(*cam));
    launch(c, k_contour_compact, dim3(1), dim3(1024), 0, dj, a->dev, cam_dev(*cam));
    int B = 0;
    CK(cudaMemcpyAsync(&B, s->B, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int> idx(B);
    if (B) {
        CK(cudaMemcpyAsync(idx.data(), s->cidx, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
        if (n2d_out) CK(cudaMemcpyAsync(n2d_out, s->n2d, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    *n_out = B;
    if (idx_out)
        for (int i = 0; i < B; ++i) idx_out[i] = idx[i];
    return last_launch_status();
    API_END
}

// The tracker's own index / set work on caller vertices (test seam for the
// bit-exact set parity): raster, contour vertices +
// normals (extract_contour_vertices, pose_stage.py:139-191), visible ids
// (visible_vertices, nonrigid_stage.py:87-99, stage 2), the rim filter
// (outer_rim_mask, pose_stage.py:218-264: stage 1 with the thickness probes
// and the rigidity >= 2 gate of pipeline.py:211, stage 2 without), the part
// gating of pipeline.py:241-249 (stage 2, part_gate) and optionally the full
// part label image (build_body_part_mask, nonrigid_stage.py:102-128).
extern "C" int lc_surface_sets(lc_ctx *c, const lc_actor *a, const lc_camera *cam, const double *verts,
                               int32_t stage, int32_t part_gate, int32_t dilation, int32_t *n_contour,
                               int64_t *idx_out, double *n2d_out, uint8_t *keep_out, int32_t *n_visible,
                               int64_t *vis_out, int32_t *labels_out) {
    API_BEGIN
    require(c && a && cam && verts && n_contour, "null argument");
    require(stage == 1 || stage == 2, "stage must be 1 or 2");
    require(dilation >= 0 && dilation <= 64, "dilation out of range");
    CK(cudaSetDevice(c->device));
    const int H = cam->height, W = cam->width, N = a->dev.N;
    Slot *s = call_slot(c, a, H, W, 1);
    cudaStream_t st = c->stream;
    CK(cudaMemcpyAsync(s->vinit, verts, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    lc_config cfg{};
    cfg.enable_part_mask = part_gate;
    cfg.nonrigid.part_dilation = dilation;
    ConfigDev cf;
    auto pr = probe_offsets();
    cf.probe = cf.mem.upload(pr.data(), pr.size(), st);
    FrameBatch fb{c, a, *cam, &cfg, &cf, {s}, {}};
    contour_and_rim(fb, {s}, &Slot::vinit, stage == 1);
    DevArena m;
    int *lab = nullptr;
    if (labels_out) {
        lab = m.alloc<int>((size_t)H * W);
        launch(c, k_part_labels, dim3(592), dim3(256), 0, a->dev, cam_dev(*cam), (const double *)s->vinit,
               (const int *)s->tri_id, (int)dilation, lab);
    }
    int B = 0, P = 0;
    CK(cudaMemcpyAsync(&B, s->B, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (stage == 2) CK(cudaMemcpyAsync(&P, s->P, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int> idx(B), vis(P);
    if (B) {
        CK(cudaMemcpyAsync(idx.data(), s->cidx, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
        if (n2d_out) CK(cudaMemcpyAsync(n2d_out, s->n2d, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost, st));
        if (keep_out) CK(cudaMemcpyAsync(keep_out, s->enabled, B, cudaMemcpyDeviceToHost, st));
    }
    if (P) CK(cudaMemcpyAsync(vis.data(), s->vis, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
    if (labels_out) CK(cudaMemcpyAsync(labels_out, lab, sizeof(int) * H * W, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *n_contour = B;
    if (n_visible) *n_visible = P;
    if (idx_out)
        for (int i = 0; i < B; ++i) idx_out[i] = idx[i];
    if (vis_out)
        for (int i = 0; i < P; ++i) vis_out[i] = vis[i];
    return last_launch_status();
    API_END
}

// ---------------------------------------------------------------------------
// stateless seams: render, pyramid, distance field, PCG, dense solve

extern "C" int lc_render(lc_ctx *c, const lc_camera *cam, int32_t n, const double *verts, int32_t t,
                         const int64_t *tris, int32_t mode, const double *attrs, int32_t n_attr,
                         const int64_t *ids, double bg_attr, int64_t bg_id, double *zbuf_out,
                         double *attr_out, int64_t *id_out) {
    API_BEGIN
    require(c && cam && verts && tris && zbuf_out, "null argument");
    require(mode >= 0 && mode <= 2, "mode must be 0, 1 or 2");
    require(mode != 1 || (attrs && attr_out && n_attr > 0), "attribute mode needs attrs");
    require(mode != 2 || (ids && id_out), "id mode needs ids");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t HW = (size_t)cam->width * cam->height;
    std::vector<int> tt(3 * (size_t)t), ii;
    for (size_t k = 0; k < tt.size(); ++k) {
        tt[k] = (int)tris[k];
        require(tt[k] >= 0 && tt[k] < n, "triangle index out of range");
    }
    double *dv = m.upload(verts, 3 * (size_t)n, st);
    int *dt = m.upload(tt.data(), tt.size(), st);
    unsigned long long *zb = m.alloc<unsigned long long>(HW);
    int *tid = m.alloc<int>(HW);
    double *za = m.alloc<double>(HW);
    double *da = nullptr, *ao = nullptr;
    int *di = nullptr;
    long long *io = nullptr;
    if (mode == 1) {
        da = m.upload(attrs, (size_t)n * n_attr, st);
        ao = m.alloc<double>(HW * n_attr);
    }
    if (mode == 2) {
        ii.resize(n);
        for (int k = 0; k < n; ++k) ii[k] = (int)ids[k];
        di = m.upload(ii.data(), ii.size(), st);
        io = m.alloc<long long>(HW);
    }
    const CamDev cd = cam_dev(*cam);
    RasterJob rj{};
    {
        const int ntx = (cam->width + LC_RT_TILE - 1) / LC_RT_TILE, nty = (cam->height + LC_RT_TILE - 1) / LC_RT_TILE;
        rj.verts = dv; rj.zbuf = zb; rj.tri_id = tid; rj.mask = nullptr;
        rj.rec = m.alloc<TriRec>(std::max(t, 1));
        rj.tcount = m.alloc<int>((size_t)ntx * nty);
        rj.toff = m.alloc<int>((size_t)ntx * nty + 1);
        rj.tfill = m.alloc<int>((size_t)ntx * nty);
        rj.tcap = std::max(1 << 20, 64 * t);
        rj.tlist = m.alloc<int>(rj.tcap);
        rj.ioff = m.alloc<int>((size_t)ntx * nty + 1);
        const size_t items = 2 * (size_t)ntx * nty + rj.tcap / LC_RT_CHUNK + 1;
        rj.pz = m.alloc<unsigned long long>(items * 256);
        rj.pid = m.alloc<int>(items * 256);
    }
    raster_tris(c, cd, dt, t, {rj});
    const auto dj = stage(c, std::vector<RasterJob>{rj});
    launch(c, k_raster_resolve, dim3(592), dim3(256), 0, dj, cd, (const int *)dt, mode, (const double *)da,
           n_attr, (const int *)di, bg_attr, (long long)bg_id, za, ao, io);
    CK(cudaMemcpyAsync(zbuf_out, za, HW * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (mode == 1) CK(cudaMemcpyAsync(attr_out, ao, HW * n_attr * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (mode == 2) CK(cudaMemcpyAsync(id_out, io, HW * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

extern "C" int lc_gaussian_pyramid(lc_ctx *c, int32_t h, int32_t w, int32_t ch, const double *image,
                                   int32_t n_levels, const int32_t *kernel_sizes, const double *given_taps,
                                   double *out) {
    API_BEGIN
    require(c && image && kernel_sizes && out, "null argument");
    require(h >= 1 && w >= 1 && ch >= 1, "bad image shape");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t n = (size_t)h * w * ch;
    double *src = m.upload(image, n, st);
    double *tmp = m.alloc<double>(n);
    double *dst = m.alloc<double>(n * n_levels);
    const int grid = (int)std::min<size_t>((n + 255) / 256, 2368);
    bool fused = ch == 3 && n_levels <= 4 && given_taps;
    for (int l = 0; l < n_levels && fused; ++l) fused = kernel_sizes[l] <= 2 * LC_PYR_HALO + 1;
    if (fused) {
        std::vector<double> taps(given_taps, given_taps + 32 * n_levels);
        taps.resize(4 * 32, 0.0);
        double *dt = m.upload(taps.data(), taps.size(), st);
        int hs[4] = {0, 0, 0, 0};
        for (int l = 0; l < n_levels; ++l) {
            require(kernel_sizes[l] >= 1 && kernel_sizes[l] % 2 == 1, "kernel size must be odd and positive");
            hs[l] = kernel_sizes[l] / 2;
        }
        const int tiles = ((w + LC_PYR_TILE - 1) / LC_PYR_TILE) * ((h + LC_PYR_TILE - 1) / LC_PYR_TILE);
        const auto dj = stage(c, std::vector<PyrAllJob>{PyrAllJob{src, dst}});
        launch(c, k_pyramid_fused, dim3(tiles), dim3(256), pyramid_fused_smem(), dj, h, w, n_levels,
               (const double *)dt, hs[0], hs[1], hs[2], hs[3]);
        CK(cudaMemcpyAsync(out, dst, n * n_levels * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return last_launch_status();
    }
    for (int l = 0; l < n_levels; ++l) {
        const int k = kernel_sizes[l];
        require(k >= 1 && k % 2 == 1, "kernel size must be odd and positive");
        require(k <= 31 || !given_taps, "kernel sizes above 31 need library taps");
        auto taps = given_taps ? std::vector<double>(given_taps + 32 * l, given_taps + 32 * l + k) : gaussian_taps(k);
        double *dt = m.upload(taps.data(), taps.size(), st);
        const auto dj = stage(c, std::vector<PyrJob>{PyrJob{src, tmp, dst + n * l}});
        launch(c, k_blur_axis, dim3(grid), dim3(256), 0, dj, h, w, ch, (const double *)dt, k / 2, 0);
        launch(c, k_blur_axis, dim3(grid), dim3(256), 0, dj, h, w, ch, (const double *)dt, k / 2, 1);
    }
    CK(cudaMemcpyAsync(out, dst, n * n_levels * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

__global__ void k_edt_cols(const uint8_t *mask, int H, int W, int contour, double *g);
__global__ void k_edt_rows(const double *g, int H, int W, int take_sqrt, long long *vs, double *zs, double *out);

static void edt_launch(lc_ctx *c, const uint8_t *dmask, int H, int W, int contour, int take_sqrt, double *dout,
                       DevArena &m) {
    double *g = m.alloc<double>((size_t)H * W);
    long long *vs = m.alloc<long long>((size_t)H * W);
    double *zs = m.alloc<double>((size_t)H * (W + 1));
    launch(c, k_edt_cols, dim3((unsigned)((W + 127) / 128)), dim3(128), 0, dmask, (int)H, (int)W, (int)contour, g);
    launch(c, k_edt_rows, dim3((unsigned)((H + 127) / 128)), dim3(128), 0, (const double *)g, (int)H, (int)W,
           (int)take_sqrt, vs, zs, dout);
}

// imageproc.py:52-115 _edt_squared of a feature image (H*W bytes, nonzero =
// feature) -> H*W doubles (1e18 where a row has no feature at all)
extern "C" int lc_edt_squared(lc_ctx *c, int32_t h, int32_t w, const uint8_t *feature, double *out) {
    API_BEGIN
    require(c && feature && out, "null argument");
    require(h >= 1 && w >= 1, "bad image shape");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t HW = (size_t)h * w;
    const uint8_t *df = m.upload(feature, HW, st);
    double *dout = m.alloc<double>(HW);
    edt_launch(c, df, h, w, 0, 0, dout, m);
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * HW, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

// imageproc.py:117-124 euclidean_dt / DistanceField.dt (:182): distance of
// every pixel centre to the nearest contour pixel centre of the field's mask
extern "C" int lc_field_dt(lc_field *f, double *out) {
    API_BEGIN
    require(f && out, "null argument");
    lc_ctx *c = f->ctx;
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t HW = (size_t)f->H * f->W;
    double *dout = m.alloc<double>(HW);
    edt_launch(c, f->mask, f->H, f->W, 1, 1, dout, m);
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * HW, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

extern "C" int lc_field_create(lc_ctx *c, int32_t h, int32_t w, const uint8_t *mask, lc_field **out) {
    API_BEGIN
    require(c && mask && out, "null argument");
    require(h >= 1 && w >= 1, "bad mask shape");
    CK(cudaSetDevice(c->device));
    lc_field *f = new lc_field();
    f->ctx = c;
    f->H = h;
    f->W = w;
    f->mask = f->mem.upload(mask, (size_t)h * w, c->stream);
    alloc_grid(f->mem, f->g, h, w);
    build_grids(c, {{&f->g, f->mask}}, h, w);
    CK(cudaMemcpyAsync(&f->K, f->g.K, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (f->K == 0) {
        delete f;
        return fail(LC_EINVAL, "mask has no foreground, distance transform undefined");
    }
    *out = f;
    return last_launch_status();
    API_END
}

extern "C" int lc_field_destroy(lc_field *f) {
    delete f;
    return LC_OK;
}

extern "C" int lc_field_n_contour(lc_field *f, int32_t *k) {
    if (!f || !k) return fail(LC_EINVAL, "null argument");
    *k = f->K;
    return LC_OK;
}

__global__ void k_field_query(NnGridDev g, long long n, const double *pos, int kind, double *out) {
    lc_pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double x = pos[2 * i], y = pos[2 * i + 1];
        double *o = out + 4 * i;
        if (kind == 4) {
            o[0] = field_inside(g, x, y) ? 1.0 : 0.0;
            o[1] = o[2] = o[3] = 0.0;
            continue;
        }
        const NnResult r = field_nearest(g, x, y);
        if (kind == 0) { o[0] = r.dist; o[1] = 0.0; o[2] = 0.0; }
        else if (kind == 1) { o[0] = field_interface(r); o[1] = 0.0; o[2] = 0.0; }
        else if (kind == 2) { double v, gx, gy; field_residual(r, v, gx, gy); o[0] = v; o[1] = gx; o[2] = gy; }
        else { o[0] = r.dist; o[1] = r.vx; o[2] = r.vy; }
        o[3] = r.clamped ? 1.0 : 0.0;
    }
}

extern "C" int lc_field_query(lc_field *f, int64_t n, const double *pos, int32_t kind, double *out) {
    API_BEGIN
    require(f && pos && out, "null argument");
    require(kind >= 0 && kind <= 4, "kind must be 0..4");
    lc_ctx *c = f->ctx;
    CK(cudaSetDevice(c->device));
    if (n == 0) return LC_OK;
    DevArena m;
    double *dp = m.upload(pos, 2 * (size_t)n, c->stream);
    double *dout = m.alloc<double>(4 * (size_t)n);
    NnGridDev g = grid_dev(f->g, f->mask, f->H, f->W);
    g.K = f->K;
    launch(c, k_field_query, dim3((unsigned)std::min<long long>((n + 255) / 256, 4096)), dim3(256), 0, g,
           (long long)n, (const double *)dp, kind, dout);
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return last_launch_status();
    API_END
}

extern "C" int lc_pcg_solve_bsr(lc_ctx *c, int32_t n, int64_t m_, const double *diag, const double *off,
                                const int64_t *rows, const int64_t *cols, const double *rhs, int32_t iterations,
                                double *x_out, lc_pcg_info *info) {
    API_BEGIN
    require(c && diag && rhs && x_out, "null argument");
    require(n >= 1, "empty system");
    require(m_ >= 0 && m_ < INT_MAX, "too many off-diagonal blocks");
    require(iterations >= 0 && iterations < LC_MAX_LOG, "iterations out of range");
    const int m = (int)m_;
    for (int i = 0; i < m; ++i)
        require(rows[i] >= 0 && rows[i] < n && cols[i] >= 0 && cols[i] < n, "block index out of range");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena mem;
    BsrJob J{};
    J.n = n; J.m = m; J.iters = iterations;
    J.diag = mem.upload(diag, 9 * (size_t)n, st);
    J.off = mem.upload(off, 9 * (size_t)std::max(m, 1), st);
    std::vector<int> cc(std::max(m, 1));
    for (int i = 0; i < m; ++i) cc[i] = (int)cols[i];
    J.cols = mem.upload(cc.data(), cc.size(), st);
    long long *drows = mem.upload(reinterpret_cast<const long long *>(rows), std::max(m, 1), st);
    int *keys = mem.alloc<int>(std::max(m, 1)), *vals = mem.alloc<int>(std::max(m, 1));
    int *skeys = mem.alloc<int>(std::max(m, 1)), *order = mem.alloc<int>(std::max(m, 1));
    int *count = mem.alloc<int>(n);
    int *rowptr = mem.alloc<int>(n + 1);
    CK(cudaMemsetAsync(count, 0, sizeof(int) * n, st));
    if (m) {
        launch(c, k_bsr_keys, dim3(std::min((m + 255) / 256, 1024)), dim3(256), 0, m, (const long long *)drows,
               keys, vals, count);
        const size_t tb = bsr_sort_temp_bytes(m);
        void *tmp = mem.alloc<char>(tb);
        int bits = 1;
        while ((1 << bits) < n && bits < 31) ++bits;
        CK(bsr_sort(tmp, tb, keys, skeys, vals, order, m, bits, st));
        c->launches++;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    launch(c, k_bsr_rowptr, dim3(1), dim3(1024), 0, n, (const int *)count, rowptr);
    J.rowptr = rowptr;
    J.order = order;
    J.rhs = mem.upload(rhs, 3 * (size_t)n, st);
    J.minv = mem.alloc<double>(9 * (size_t)n);
    J.x = mem.alloc<double>(3 * (size_t)n); J.r = mem.alloc<double>(3 * (size_t)n);
    J.z = mem.alloc<double>(3 * (size_t)n); J.p = mem.alloc<double>(3 * (size_t)n);
    J.ap = mem.alloc<double>(3 * (size_t)n); J.best = mem.alloc<double>(3 * (size_t)n);
    J.norms = mem.alloc<double>(LC_MAX_LOG);
    J.info = mem.alloc<int>(4);
    launch(c, k_pcg_bsr, dim3(1), dim3(1024), 0, J);
    CK(cudaMemcpyAsync(x_out, J.best, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
    int hinfo[4] = {0, 0, 0, 0};
    double norms[LC_MAX_LOG];
    CK(cudaMemcpyAsync(hinfo, J.info, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(norms, J.norms, sizeof(double) * LC_MAX_LOG, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (info) {
        info->iterations = hinfo[0];
        info->breakdown = hinfo[1];
        for (int k = 0; k <= hinfo[0] && k < LC_MAX_LOG; ++k) info->residual_norms[k] = norms[k];
    }
    return last_launch_status();
    API_END
}

__global__ void k_smooth_trajectory(const double *v, int F, long long D, const double *w, int K, double *out);
__global__ void k_mask_overlap(const uint8_t *a, const uint8_t *b, long long HW, unsigned long long *inter,
                               unsigned long long *uni);

// smooth_trajectory (pipeline.py:308-325) of an (F, D) stack, bit-identical
extern "C" int lc_smooth_trajectory(lc_ctx *c, int32_t F, int64_t D, const double *values, int32_t K,
                                    const double *stencil, double *out) {
    API_BEGIN
    require(c && values && stencil && out, "null argument");
    require(K >= 1 && K % 2 == 1, "stencil length must be odd");
    require(F >= 1 && D >= 1, "empty trajectory");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t n = (size_t)F * D;
    double *dv = m.upload(values, n, st), *dw = m.upload(stencil, K, st), *dout = m.alloc<double>(n);
    launch(c, k_smooth_trajectory, dim3((unsigned)std::min<size_t>((n + 255) / 256, 4096)), dim3(256), 0,
           (const double *)dv, (int)F, (long long)D, (const double *)dw, (int)K, dout);
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

// per-frame intersection / union pixel counts of two (F, H, W) mask stacks (metrics.iou)
extern "C" int lc_mask_overlap(lc_ctx *c, int32_t F, int64_t HW, const uint8_t *a, const uint8_t *b,
                               uint64_t *inter_out, uint64_t *union_out) {
    API_BEGIN
    require(c && a && b && inter_out && union_out, "null argument");
    require(F >= 1 && HW >= 1, "empty masks");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t n = (size_t)F * HW;
    uint8_t *da = m.upload(a, n, st), *db = m.upload(b, n, st);
    unsigned long long *di = m.alloc<unsigned long long>(F), *du = m.alloc<unsigned long long>(F);
    CK(cudaMemsetAsync(di, 0, sizeof(unsigned long long) * F, st));
    CK(cudaMemsetAsync(du, 0, sizeof(unsigned long long) * F, st));
    launch(c, k_mask_overlap, dim3(64, (unsigned)F), dim3(256), 0, (const uint8_t *)da, (const uint8_t *)db,
           (long long)HW, di, du);
    CK(cudaMemcpyAsync(inter_out, di, sizeof(uint64_t) * F, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(union_out, du, sizeof(uint64_t) * F, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

__global__ void k_vertex_error(int F, long long N, const double *pred, const double *gt, const long long *idx,
                               long long n_sel, int center, double *dist, double *out);
__global__ void k_umeyama(int F, int M, const double *src_all, const double *dst_all, int with_scaling,
                          double *scale_out, double *rot_out, double *t_out, double *err_out, double *scratch);

// metrics.mean_vertex_error over F frames (bit-identical to numpy)
extern "C" int lc_mean_vertex_error(lc_ctx *c, int32_t F, int64_t N, const double *pred, const double *gt,
                                    const int64_t *indices, int64_t n_idx, int32_t center, int32_t on_device,
                                    double *out) {
    API_BEGIN
    require(c && pred && gt && out, "null argument");
    require(F >= 1 && N >= 1, "empty vertex arrays");
    require(!indices || n_idx >= 1, "empty index selection");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t n = (size_t)F * N * 3;
    const long long n_sel = indices ? n_idx : N;
    if (indices && !on_device)
        for (int64_t k = 0; k < n_idx; ++k) require(indices[k] >= -N && indices[k] < N, "index out of range");
    const double *dp = on_device ? pred : m.upload(pred, n, st);
    const double *dg = on_device ? gt : m.upload(gt, n, st);
    const long long *di = nullptr;
    if (indices) {
        if (on_device) di = reinterpret_cast<const long long *>(indices);
        else {
            std::vector<long long> ix(n_idx);
            for (int64_t k = 0; k < n_idx; ++k) ix[k] = indices[k] < 0 ? indices[k] + N : indices[k];
            di = m.upload(ix.data(), ix.size(), st);
        }
    }
    double *dist = m.alloc<double>((size_t)F * n_sel), *dout = m.alloc<double>(F);
    launch(c, k_vertex_error, dim3((unsigned)F), dim3(256), 0, (int)F, (long long)N, dp, dg, di, n_sel,
           (int)center, dist, dout);
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * F, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

// metrics.umeyama_alignment + aligned_joint_error over F frames of M 3-D points
extern "C" int lc_aligned_error(lc_ctx *c, int32_t F, int32_t M, const double *pred, const double *gt,
                                int32_t with_scaling, int32_t on_device, double *scale_out, double *rot_out,
                                double *t_out, double *err_out) {
    API_BEGIN
    require(c && pred && gt && err_out, "null argument");
    require(F >= 1, "no frames");
    require(M >= 3, "need at least 3 points to align");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    const size_t n = (size_t)F * M * 3;
    const double *dp = on_device ? pred : m.upload(pred, n, st);
    const double *dg = on_device ? gt : m.upload(gt, n, st);
    double *sc = m.alloc<double>(F), *rot = m.alloc<double>(9 * (size_t)F), *tt = m.alloc<double>(3 * (size_t)F);
    double *err = m.alloc<double>(F), *scr = m.alloc<double>((size_t)F * M);
    launch(c, k_umeyama, dim3((unsigned)((F + 63) / 64)), dim3(64), 0, (int)F, (int)M, dp, dg, (int)with_scaling,
           sc, rot, tt, err, scr);
    CK(cudaMemcpyAsync(err_out, err, sizeof(double) * F, cudaMemcpyDeviceToHost, st));
    if (scale_out) CK(cudaMemcpyAsync(scale_out, sc, sizeof(double) * F, cudaMemcpyDeviceToHost, st));
    if (rot_out) CK(cudaMemcpyAsync(rot_out, rot, sizeof(double) * 9 * F, cudaMemcpyDeviceToHost, st));
    if (t_out) CK(cudaMemcpyAsync(t_out, tt, sizeof(double) * 3 * F, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return last_launch_status();
    API_END
}

extern "C" int lc_dense_solve(lc_ctx *c, int32_t n, const double *a, const double *b, double *x_out,
                              lc_dense_info *info) {
    API_BEGIN
    require(c && a && b && x_out, "null argument");
    require(n >= 1 && n <= 64, "dense solve supports 1 <= n <= 64");
    for (int i = 0; i < n * n; ++i) require(std::isfinite(a[i]), "non-finite entries in normal system");
    for (int i = 0; i < n; ++i) require(std::isfinite(b[i]), "non-finite entries in normal system");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DevArena m;
    double *da = m.upload(a, (size_t)n * n, st), *db = m.upload(b, n, st);
    double *dx = m.alloc<double>(n), *di = m.alloc<double>(2);
    launch(c, k_dense_solve, dim3(1), dim3(256), 0, n, (const double *)da, (const double *)db, dx, di);
    double hi[2];
    CK(cudaMemcpyAsync(x_out, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hi, di, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (info) {
        info->damped = hi[0] != 0.0;
        info->damping = hi[1];
    }
    return last_launch_status();
    API_END
}

// ---------------------------------------------------------------------------
// numpy Generator(PCG64).normal on the device (lc_rng.cu)

// n normals loc + scale * z of the PCG64 stream (state, inc: hi, lo words)
// into the device array `out` (add_clip: out = clip(out + noise, 0, 1), the
// generator's image noise).  Returns the draws consumed (advance the stream
// by it) and the tail samples the host completes: tails[2t] = element,
// tails[2t+1] = draws, tail_draws[t*31 ..] = the sample's first 31 draws.
extern "C" int lc_rng_normal(lc_ctx *c, const uint64_t *state, const uint64_t *inc, double loc, double scale,
                             double *out, int64_t n, int32_t add_clip, int64_t *consumed, int64_t *tails,
                             uint64_t *tail_draws, int32_t max_tails, int32_t *n_tails) {
    API_BEGIN
    require(c && state && inc && out && consumed && n_tails, "null argument");
    require(n >= 0, "negative count");
    CK(cudaSetDevice(c->device));
    *consumed = 0;
    *n_tails = 0;
    if (n == 0) return LC_OK;
    cudaStream_t st = c->stream;
    for (long long M = n + n / 32 + 4096;; M *= 2) {
        if (!c->rng) c->rng = new lc_ctx::RngScratch();
        lc_ctx::RngScratch &R = *c->rng;
        const int mt = std::max(max_tails, 1);
        if (M > R.M || mt > R.mt) {   // (grow-only: the generator calls this once per frame)
            cudaStreamSynchronize(st);
            R.mem.release();
            R.M = std::max(M, R.M);
            R.mt = std::max(mt, R.mt);
            const long long m = R.M;
            R.u = R.mem.alloc<uint64_t>(m);
            R.val = R.mem.alloc<double>(m);
            R.len = R.mem.alloc<int>(m);
            R.kind = R.mem.alloc<unsigned char>(m);
            R.start = R.mem.alloc<unsigned char>(m);
            R.flag = R.mem.alloc<unsigned char>(m);
            R.num = R.mem.alloc<long long>(m);
            R.slow = R.mem.alloc<long long>(m);
            R.n_slow = R.mem.alloc<int>(1);
            R.sst = R.mem.alloc<int>(m);
            R.err = R.mem.alloc<int>(1);
            R.nt = R.mem.alloc<int>(1);
            R.cons = R.mem.alloc<long long>(1);
            R.dtails = R.mem.alloc<long long>(2 * (size_t)R.mt);
            R.ddraws = R.mem.alloc<uint64_t>((size_t)R.mt * LC_TAIL_DRAWS);
            R.tb1 = R.tb2 = 0;
            CK(rng_select_slow(nullptr, R.tb1, R.flag, R.slow, R.n_slow, m, st));
            CK(rng_scan_starts(nullptr, R.tb2, R.start, R.num, m, st));
            R.tmp1 = R.mem.alloc<char>(R.tb1);
            R.tmp2 = R.mem.alloc<char>(R.tb2);
        }
        uint64_t *u = R.u, *ddraws = R.ddraws;
        double *val = R.val;
        int *len = R.len, *n_slow = R.n_slow, *sst = R.sst, *err = R.err, *nt = R.nt;
        unsigned char *kind = R.kind, *start = R.start, *flag = R.flag;
        long long *num = R.num, *slow = R.slow, *cons = R.cons, *dtails = R.dtails;
        CK(cudaMemsetAsync(err, 0, sizeof(int), st));
        CK(cudaMemsetAsync(nt, 0, sizeof(int), st));
        CK(cudaMemsetAsync(cons, 0xff, sizeof(long long), st));
        const int grid = 148 * 8;
        launch(c, k_rng_draws, dim3(grid), dim3(256), 0, state[0], state[1], inc[0], inc[1], u, M);
        launch(c, k_zig_walk, dim3(grid), dim3(256), 0, (const uint64_t *)u, M, val, len, kind,
                     start);
        launch(c, k_slow_flags, dim3(grid), dim3(256), 0, (const int *)len, M, flag);
        {
            size_t tb = 0;
            CK(rng_select_slow(nullptr, tb, flag, slow, n_slow, M, st));
            require(tb <= R.tb1, "rng scratch too small");
            CK(rng_select_slow(R.tmp1, tb, flag, slow, n_slow, M, st));
        }
        launch(c, k_zig_starts, dim3(1), dim3(1024), 0, (const long long *)slow,
                     (const int *)n_slow, (const int *)len, start, sst, M, err);
        {
            size_t tb = 0;
            CK(rng_scan_starts(nullptr, tb, start, num, M, st));
            require(tb <= R.tb2, "rng scratch too small");
            CK(rng_scan_starts(R.tmp2, tb, start, num, M, st));
        }
        launch(c, k_zig_emit, dim3(grid), dim3(256), 0, (const unsigned char *)start,
                     (const long long *)num, (const double *)val, (const int *)len, (const unsigned char *)kind,
                     (const uint64_t *)u, M, (long long)n, loc, scale, out, (int)add_clip, cons, dtails, ddraws, nt,
                     mt, err);
        int h_err = 0, h_nt = 0;
        long long h_cons = -1;
        CK(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&h_nt, nt, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&h_cons, cons, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        require(h_err != 1, "ziggurat sample spans more than 64 draws (unsupported)");
        if (h_cons < 0 || h_err == 2) continue;   // fewer than n samples in M draws: a longer buffer
        require(h_nt <= max_tails, "more tail samples than max_tails");
        *consumed = h_cons;
        *n_tails = h_nt;
        if (h_nt > 0) {
            if (tails) CK(cudaMemcpyAsync(tails, dtails, sizeof(long long) * 2 * h_nt, cudaMemcpyDeviceToHost, st));
            if (tail_draws)
                CK(cudaMemcpyAsync(tail_draws, ddraws, sizeof(uint64_t) * LC_TAIL_DRAWS * h_nt, cudaMemcpyDeviceToHost,
                                   st));
            CK(cudaStreamSynchronize(st));
        }
        return LC_OK;
    }
    API_END
}

// out[idx[k]] = v[k] (host-completed tail samples); idx / v host arrays
extern "C" int lc_rng_scatter(lc_ctx *c, const int64_t *idx, const double *v, int32_t n, double *out) {
    API_BEGIN
    require(c && out && (n == 0 || (idx && v)), "null argument");
    CK(cudaSetDevice(c->device));
    if (n == 0) return LC_OK;
    DevArena mem;
    long long *di = mem.alloc<long long>(n);
    double *dv = mem.alloc<double>(n);
    CK(cudaMemcpyAsync(di, idx, sizeof(long long) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dv, v, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    launch(c, k_rng_scatter, dim3((n + 255) / 256), dim3(256), 0, (const long long *)di,
                 (const double *)dv, (int)n, out);
    CK(cudaStreamSynchronize(c->stream));
    return LC_OK;
    API_END
}

// out[k] = src[idx[k]] (device src; host idx / out)
extern "C" int lc_rng_gather(lc_ctx *c, const int64_t *idx, int32_t n, const double *src, double *out) {
    API_BEGIN
    require(c && src && (n == 0 || (idx && out)), "null argument");
    CK(cudaSetDevice(c->device));
    if (n == 0) return LC_OK;
    DevArena mem;
    long long *di = mem.alloc<long long>(n);
    double *dv = mem.alloc<double>(n);
    CK(cudaMemcpyAsync(di, idx, sizeof(long long) * n, cudaMemcpyHostToDevice, c->stream));
    launch(c, k_rng_gather, dim3((n + 255) / 256), dim3(256), 0, (const long long *)di, (int)n,
                 src, dv);
    CK(cudaMemcpyAsync(out, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return LC_OK;
    API_END
}

// n doubles of Generator.random() (draws 0..n-1 of the stream) into device `out`
extern "C" int lc_rng_uniform(lc_ctx *c, const uint64_t *state, const uint64_t *inc, double *out, int64_t n) {
    API_BEGIN
    require(c && state && inc && (n == 0 || out), "null argument");
    CK(cudaSetDevice(c->device));
    if (n == 0) return LC_OK;
    launch(c, k_rng_uniform, dim3((unsigned)std::min<long long>((n + 255) / 256, 148 * 8)), dim3(256), 0, state[0],
           state[1], inc[0], inc[1], out, (long long)n);
    return last_launch_status();
    API_END
}

// the ziggurat tables the device draws with (256 entries each)
extern "C" int lc_rng_tables(uint64_t *ki, double *wi, double *fi) {
    API_BEGIN
    require(ki && wi && fi, "null argument");
    CK(rng_tables(ki, wi, fi));
    return LC_OK;
    API_END
}
