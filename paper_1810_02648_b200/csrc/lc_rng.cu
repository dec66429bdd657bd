// numpy Generator(PCG64).normal on the device, bit for bit.
//
// The reference's synthetic generator (synthetic.py:170-203) draws the image
// noise of every frame -- H*W*3 normals, 3.1 M at 1024^2 -- and then the
// detection noise from one numpy PCG64 stream.  Each normal consumes a
// variable number of uint64 draws (the ziggurat's fast path takes one, the
// wedge and tail paths more), so the samples are data-dependent positions
// of the draw sequence.  On the device:
//   1. every draw u[k] of the stream (jump-ahead: thread t starts at
//      position t, then steps by the affine map of T LCG steps);
//   2. for every position k, the sample a walk starting at k would produce
//      and the draws it consumes (len 1 on the 99.3% fast path);
//   3. which positions start a sample: position 0 does, and a start k covers
//      k+1 .. k+len-1.  Only slow positions (len > 1) cover anything, so the
//      starts are resolved on the short sorted list of slow positions (a
//      fixed point over a bounded look-back, one CTA), then the covered
//      positions are cleared;
//   4. an exclusive scan of the start flags numbers the samples; sample i
//      goes to element i (image: clip(image + loc + scale * z, 0, 1)).
// Exactness: the fast path and the wedge's arithmetic are numpy's fp64
// operations; the wedge compares against exp(), which matches glibc's except
// possibly in the last bit (a decision can flip only if the comparand falls
// in that ulp, ~2^-52 per wedge test).  The tail (layer 0) VALUES use
// log1p, where CUDA and libm may differ in the last bit: tail samples (about
// 1 in 4000) are listed with their draws, and the host recomputes them with
// libm's log1p (paper_1810_02648_b200/rng.py), checks the draw counts, and
// scatters the values (lc_rng_scatter).
#include <cub/cub.cuh>
#include "lc_rng.cuh"
#include "lc_internal.h"
#include "lc_ziggurat_tables.h"

typedef unsigned __int128 u128;

namespace {

constexpr double kZigR = 3.6541528853610088;
constexpr double kZigInvR = 0.27366123732975828;
constexpr int kTailDraws = LC_TAIL_DRAWS;

__device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ u128 pcg_mult() { return mk128(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL); }

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned r = (unsigned)(s >> 122);
    return (x >> r) | (x << ((64u - r) & 63u));
}

// affine map of `delta` LCG steps: s -> am * s + ap
__device__ __forceinline__ void pcg_jump(u128 inc, unsigned long long delta, u128 &am, u128 &ap) {
    u128 acc_m = 1, acc_p = 0, cur_m = pcg_mult(), cur_p = inc;
    while (delta) {
        if (delta & 1) {
            acc_m = acc_m * cur_m;
            acc_p = acc_p * cur_m + cur_p;
        }
        cur_p = (cur_m + 1) * cur_p;
        cur_m = cur_m * cur_m;
        delta >>= 1;
    }
    am = acc_m;
    ap = acc_p;
}

__device__ __forceinline__ double u_double(uint64_t u) { return (double)(u >> 11) * (1.0 / 9007199254740992.0); }

}  // namespace

// draw k = output of the state after k+1 steps
__global__ void k_rng_draws(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t *u, long long M) {
    lc_pdl_wait();
    const long long T = (long long)gridDim.x * blockDim.x;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= M) return;
    const u128 inc = mk128(i_hi, i_lo);
    u128 am, ap, tm, tp;
    pcg_jump(inc, (unsigned long long)t + 1, am, ap);
    pcg_jump(inc, (unsigned long long)T, tm, tp);
    u128 s = am * mk128(s_hi, s_lo) + ap;
    for (long long k = t; k < M; k += T) {
        u[k] = pcg_out(s);
        s = tm * s + tp;
    }
}

namespace {
// the sample a walk from position k produces (random_standard_normal,
// numpy/random/src/distributions/distributions.c) and the draws it takes;
// len = -1 when the walk runs past the buffer.  kind: 0 fast, 1 wedge, 2 tail
__device__ __forceinline__ double zig_walk(const uint64_t *u, long long M, long long k, int &len, int &kind) {
    long long p = k;
    kind = 0;
    for (;;) {
        if (p >= M) { len = -1; return 0.0; }
        uint64_t r = u[p++];
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const int sign = (int)(r & 1);
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * lc_zig_wi[idx];
        if (sign) x = -x;
        if (rabs < lc_zig_ki[idx]) { len = (int)(p - k); return x; }
        if (idx == 0) {
            kind = 2;
            for (;;) {
                if (p + 1 >= M) { len = -1; return 0.0; }
                const double xx = -kZigInvR * log1p(-u_double(u[p++]));
                const double yy = -log1p(-u_double(u[p++]));
                if (yy + yy > xx * xx) {
                    len = (int)(p - k);
                    return ((rabs >> 8) & 0x1) ? -(kZigR + xx) : kZigR + xx;
                }
            }
        }
        if (kind == 0) kind = 1;
        if (p >= M) { len = -1; return 0.0; }
        if ((lc_zig_fi[idx - 1] - lc_zig_fi[idx]) * u_double(u[p++]) + lc_zig_fi[idx] < exp(-0.5 * x * x)) {
            len = (int)(p - k);
            return x;
        }
    }
}

}  // namespace

__global__ void k_zig_walk(const uint64_t *u, long long M, double *val, int *len, unsigned char *kind,
                           unsigned char *start) {
    lc_pdl_wait();
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < M;
         k += (long long)gridDim.x * blockDim.x) {
        int l, kd;
        val[k] = zig_walk(u, M, k, l, kd);
        len[k] = l;
        kind[k] = (unsigned char)kd;
        start[k] = 1;
    }
}

// slow positions (len != 1), ascending: their start status by a fixed point
// over the bounded look-back (a slow position is a start iff no earlier
// start's span reaches it), then the spans of the slow starts are cleared
__global__ void __launch_bounds__(1024) k_zig_starts(const long long *slow, const int *n_slow_p, const int *len,
                                                     unsigned char *start, int *sst, long long M, int *err) {
    lc_pdl_wait();
    const int n = *n_slow_p;
    __shared__ int changed;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sst[i] = 1;
    __syncthreads();
    for (int round = 0; round < 64; ++round) {
        if (threadIdx.x == 0) changed = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const long long s = slow[i];
            int st = 1;
            for (int j = i - 1; j >= 0; --j) {
                const long long q = slow[j];
                if (s - q > 64) break;   // spans are < 64 draws (checked below)
                if (sst[j] && q + len[q] > s) { st = 0; break; }
            }
            if (st != sst[i]) { sst[i] = st; changed = 1; }
        }
        __syncthreads();
        if (!changed) break;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const long long s = slow[i];
        const int L = len[s];
        if (L > 64) { atomicExch(err, 1); continue; }   // (never observed; the look-back assumes it)
        if (L < 0) {   // ran past the buffer: only a start among the first n samples matters (k_zig_emit)
            if (!sst[i]) start[s] = 0;
            continue;
        }
        if (!sst[i]) start[s] = 0;
        else
            for (int j = 1; j < L && s + j < M; ++j) start[s + j] = 0;
    }
}

__global__ void k_slow_flags(const int *len, long long M, unsigned char *flag) {
    lc_pdl_wait();
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < M;
         k += (long long)gridDim.x * blockDim.x)
        flag[k] = len[k] != 1;
}

// sample i (numbered by the scan) -> element i; tail samples are listed for
// the host instead (their value needs libm's log1p)
__global__ void k_zig_emit(const unsigned char *start, const long long *num, const double *val, const int *len,
                           const unsigned char *kind, const uint64_t *u, long long M, long long n, double loc,
                           double scale, double *out, int add_clip, long long *consumed, long long *tails,
                           uint64_t *tail_draws, int *n_tails, int max_tails, int *err) {
    lc_pdl_wait();
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < M;
         k += (long long)gridDim.x * blockDim.x) {
        if (!start[k]) continue;
        const long long i = num[k];
        if (i >= n) continue;
        if (len[k] < 0) { atomicExch(err, 2); continue; }   // walk ran past the buffer: a longer one
        if (i == n - 1) *consumed = k + len[k];
        if (kind[k] == 2) {
            const int t = atomicAdd(n_tails, 1);
            if (t < max_tails) {
                tails[2 * t] = i;
                tails[2 * t + 1] = len[k];
                for (int j = 0; j < kTailDraws; ++j) tail_draws[(size_t)t * kTailDraws + j] = k + j < M ? u[k + j] : 0;
            }
            continue;
        }
        const double nz = loc + scale * val[k];
        if (add_clip) out[i] = fmin(fmax(out[i] + nz, 0.0), 1.0);
        else out[i] = nz;
    }
}

__global__ void k_rng_scatter(const long long *idx, const double *v, int n, double *out) {
    lc_pdl_wait();
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[idx[k]] = v[k];
}

__global__ void k_rng_gather(const long long *idx, int n, const double *src, double *out) {
    lc_pdl_wait();
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[k] = src[idx[k]];
}

// the slow positions (flag != 0) in ascending order
cudaError_t rng_select_slow(void *temp, size_t &temp_bytes, const unsigned char *flag, long long *slow, int *n_slow,
                            long long M, cudaStream_t st) {
    cub::CountingInputIterator<long long> it(0);
    return cub::DeviceSelect::Flagged(temp, temp_bytes, it, flag, slow, n_slow, M, st);
}

// num[k] = number of starts before k
cudaError_t rng_scan_starts(void *temp, size_t &temp_bytes, const unsigned char *start, long long *num, long long M,
                            cudaStream_t st) {
    cub::TransformInputIterator<long long, cub::CastOp<long long>, const unsigned char *> fl(start, {});
    return cub::DeviceScan::ExclusiveSum(temp, temp_bytes, fl, num, M, st);
}


// the tables as the device uses them (the host completes tail samples with them)
cudaError_t rng_tables(uint64_t *ki, double *wi, double *fi) {
    cudaError_t e = cudaMemcpyFromSymbol(ki, lc_zig_ki, sizeof(uint64_t) * 256);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(wi, lc_zig_wi, sizeof(double) * 256);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(fi, lc_zig_fi, sizeof(double) * 256);
    return e;
}

// next_double of draws 0..n-1 (Generator.random)
__global__ void k_rng_uniform(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, double *out, long long n) {
    lc_pdl_wait();
    const long long T = (long long)gridDim.x * blockDim.x;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const u128 inc = mk128(i_hi, i_lo);
    u128 am, ap, tm, tp;
    pcg_jump(inc, (unsigned long long)t + 1, am, ap);
    pcg_jump(inc, (unsigned long long)T, tm, tp);
    u128 s = am * mk128(s_hi, s_lo) + ap;
    for (long long k = t; k < n; k += T) {
        out[k] = u_double(pcg_out(s));
        s = tm * s + tp;
    }
}
