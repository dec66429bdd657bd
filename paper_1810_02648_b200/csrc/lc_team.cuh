// A "team" is the set of CTAs that cooperate on one capture stream: a thread
// block cluster of CS CTAs (CS = 1: a single CTA).  Phases are separated by
// cluster barriers (barrier.cluster arrive.release / wait.acquire, which also
// order the global-memory writes of one phase before the reads of the next),
// and reductions are deterministic: every CTA tree-reduces its threads, then
// every CTA sums the per-CTA partials in rank order through distributed
// shared memory, so all CTAs hold bit-identical totals whatever the timing.
#pragma once
#include <cooperative_groups.h>
#include "lc_device.cuh"

namespace cg = cooperative_groups;

template <int CS, int NT>
struct Team {
    static constexpr int size = CS * NT;
    static constexpr int ctas = CS;

    __device__ __forceinline__ static int rank() {
        if constexpr (CS == 1) return 0;
        else return (int)cg::this_cluster().block_rank();
    }
    // stream index of this CTA (clusters are laid out contiguously along x)
    __device__ __forceinline__ static int stream() { return blockIdx.x / CS; }
    __device__ __forceinline__ static int tid() { return rank() * NT + (int)threadIdx.x; }

    __device__ __forceinline__ static void sync() {
        if constexpr (CS == 1) __syncthreads();
        else cg::this_cluster().sync();
    }

    // Layout of the shared reduction buffer (the same offsets in every CTA):
    // per-warp partials [kMaxSums][32], two parity slots of per-CTA partials,
    // the totals, and the parity flag.
    static constexpr int kMaxSums = 32;
    static constexpr int kSlot = kMaxSums * 32;
    static constexpr int kRes = kSlot + 2 * kMaxSums;
    static constexpr int kPar = kRes + kMaxSums;
    static constexpr int kBar = kPar + 2;   // mbarrier of sums_light + its phase count
    static constexpr int red_doubles = kBar + 2;

    // (every CTA calls this before the kernel's first team barrier, which
    // makes the mbarrier initialisation visible to the peers' remote arrives)
    __device__ __forceinline__ static void init_red(double *red) {
        if (threadIdx.x == 0) {
            *reinterpret_cast<int *>(red + kPar) = 0;
            *reinterpret_cast<int *>(red + kBar + 1) = 0;
            if constexpr (CS > 1) {
                const unsigned bar = (unsigned)__cvta_generic_to_shared(red + kBar);
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(CS) : "memory");
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
        }
    }

    // M simultaneous sums over every thread of the team.  Per-warp shuffle
    // trees, then warp m' sums partial m over the CTA's warps (fixed order),
    // then every CTA adds the per-CTA partials in rank order through DSMEM,
    // so every CTA holds bit-identical totals.  Per-CTA partials alternate
    // between two slots (`parity`, identical in every CTA because every CTA
    // makes the same sequence of calls), so one cluster barrier suffices: a
    // slot is rewritten two calls later, after an intermediate barrier that
    // every reader must have reached.
    template <int M>
    __device__ static void sums(double (&v)[M], double *red) {
        static_assert(M <= kMaxSums, "too many simultaneous sums");
        constexpr int NW = NT / 32;
        for (int m = 0; m < M; ++m)
            for (int o = 16; o > 0; o >>= 1) v[m] += __shfl_down_sync(0xffffffffu, v[m], o);
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        __syncthreads();
        if (l == 0)
            for (int m = 0; m < M; ++m) red[m * 32 + w] = v[m];
        int *par = reinterpret_cast<int *>(red + kPar);
        __syncthreads();
        const int parity = *par;
        double *slot = red + kSlot + kMaxSums * parity;   // this CTA's partials
        double *res = red + kRes;                          // local copy of the totals
        for (int m = w; m < M; m += NW) {
            double s = (l < NW) ? red[m * 32 + l] : 0.0;
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if (l == 0) {
                if constexpr (CS == 1) res[m] = s;
                else slot[m] = s;
            }
        }
        if constexpr (CS == 1) {
            __syncthreads();
        } else {
            auto cl = cg::this_cluster();
            cl.sync();
            if (threadIdx.x < M) {
                double s = 0.0;
                for (int r = 0; r < CS; ++r) s += cl.map_shared_rank(slot, r)[threadIdx.x];
                res[threadIdx.x] = s;
            }
            if (threadIdx.x == 0) *par = parity ^ 1;
            __syncthreads();
        }
        for (int m = 0; m < M; ++m) v[m] = res[m];
    }

    // sums() for phases that exchange only shared memory across the team
    // (the per-CTA partials here, and e.g. PCG vectors a CTA keeps in its own
    // shared memory and its peers read over DSMEM): the same deterministic
    // rank-order totals, but the cluster barrier is an mbarrier handshake
    // with release / acquire restricted to shared memory -- a CTA fences its
    // own shared-memory writes and arrives remotely on every peer's mbarrier,
    // then waits on its own.  No GPU-scope MEMBAR and no L1 invalidation
    // (cluster.sync emits MEMBAR.ALL.GPU + CCTL.IVALL), so global-memory
    // writes of one CTA are NOT ordered before another CTA's reads by this
    // call: use sums() / sync() where the phase boundary needs that.
    template <int M>
    __device__ static void sums_light(double (&v)[M], double *red) {
#ifdef LC_TEAM_FULL_SYNC
        // sanitizer build: compute-sanitizer racecheck does not model the
        // remote-mbarrier handshake, so this variant takes the cluster barrier
        sums<M>(v, red);
        return;
#endif
        if constexpr (CS == 1) {
            sums<M>(v, red);
        } else {
            static_assert(M <= kMaxSums, "too many simultaneous sums");
            constexpr int NW = NT / 32;
            for (int m = 0; m < M; ++m)
                for (int o = 16; o > 0; o >>= 1) v[m] += __shfl_down_sync(0xffffffffu, v[m], o);
            const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
            __syncthreads();
            if (l == 0)
                for (int m = 0; m < M; ++m) red[m * 32 + w] = v[m];
            int *par = reinterpret_cast<int *>(red + kPar);
            int *phase = reinterpret_cast<int *>(red + kBar + 1);
            __syncthreads();
            const int parity = *par;
            const int ph = *phase;
            double *slot = red + kSlot + kMaxSums * parity;
            double *res = red + kRes;
            for (int m = w; m < M; m += NW) {
                double s = (l < NW) ? red[m * 32 + l] : 0.0;
                for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
                if (l == 0) slot[m] = s;
            }
            __syncthreads();   // this CTA's slot is complete
            const unsigned bar = (unsigned)__cvta_generic_to_shared(red + kBar);
            if (threadIdx.x < CS) {   // lane r signals peer r (itself included)
                unsigned remote;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"((int)threadIdx.x));
                asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
                asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
            }
            unsigned done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2; "
                    "selp.u32 %0, 1, 0, p; }"
                    : "=r"(done) : "r"(bar), "r"(ph & 1) : "memory");
            asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
            if (threadIdx.x < M) {
                auto cl = cg::this_cluster();
                double s = 0.0;
                for (int r = 0; r < CS; ++r) s += cl.map_shared_rank(slot, r)[threadIdx.x];
                res[threadIdx.x] = s;
            }
            if (threadIdx.x == 0) {
                *par = parity ^ 1;
                *phase = ph + 1;
            }
            __syncthreads();
            for (int m = 0; m < M; ++m) v[m] = res[m];
        }
    }

    // the team barrier of sums_light alone, for shared-memory-only exchanges
    // (the same mbarrier and phase sequence; no GPU-scope fence)
    __device__ static void sync_light(double *red) {
#ifdef LC_TEAM_FULL_SYNC
        sync();
        return;
#endif
        if constexpr (CS == 1) {
            __syncthreads();
        } else {
            int *phase = reinterpret_cast<int *>(red + kBar + 1);
            const int ph = *phase;
            __syncthreads();   // this CTA's shared-memory writes are done (and every thread read ph)
            const unsigned bar = (unsigned)__cvta_generic_to_shared(red + kBar);
            if (threadIdx.x < CS) {
                unsigned remote;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"((int)threadIdx.x));
                asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
                asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
            }
            unsigned done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2; "
                    "selp.u32 %0, 1, 0, p; }"
                    : "=r"(done) : "r"(bar), "r"(ph & 1) : "memory");
            asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) *phase = ph + 1;
            __syncthreads();
        }
    }

    // sum_arrays over the light barrier: the per-CTA arrays and the totals
    // are shared memory only
    __device__ static void sum_arrays_light(const double *part, double *out, int n, double *red) {
        if constexpr (CS == 1) {
            for (int e = threadIdx.x; e < n; e += NT) out[e] = part[e];
            __syncthreads();
        } else {
            sync_light(red);
            auto cl = cg::this_cluster();
            for (int e = threadIdx.x; e < n; e += NT) {
                double s = 0.0;
                for (int r = 0; r < CS; ++r) s += cl.map_shared_rank(part, r)[e];
                out[e] = s;
            }
            sync_light(red);   // every peer has read this CTA's partials
        }
    }

    // element-wise sum of a per-CTA shared array `part[n]` over the team, in
    // rank order, into `out[n]` (shared, every CTA).  Caller syncs after.
    __device__ static void sum_arrays(const double *part, double *out, int n) {
        if constexpr (CS == 1) {
            for (int e = threadIdx.x; e < n; e += NT) out[e] = part[e];
            __syncthreads();
        } else {
            auto cl = cg::this_cluster();
            cl.sync();
            for (int e = threadIdx.x; e < n; e += NT) {
                double s = 0.0;
                for (int r = 0; r < CS; ++r) s += cl.map_shared_rank(part, r)[e];
                out[e] = s;
            }
            cl.sync();
        }
    }
};
