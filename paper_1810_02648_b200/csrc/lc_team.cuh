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
    static constexpr int kMaxSums = 24;
    static constexpr int kSlot = kMaxSums * 32;
    static constexpr int kRes = kSlot + 2 * kMaxSums;
    static constexpr int kPar = kRes + kMaxSums;
    static constexpr int red_doubles = kPar + 2;

    __device__ __forceinline__ static void init_red(double *red) {
        if (threadIdx.x == 0) *reinterpret_cast<int *>(red + kPar) = 0;
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
