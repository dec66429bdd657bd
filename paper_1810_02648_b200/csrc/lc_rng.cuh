// numpy Generator(PCG64).normal on the device (lc_rng.cu): kernels and scan
// helpers, launched by the C-ABI in lc_api.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

constexpr int LC_TAIL_DRAWS = 31;   // draws recorded per tail sample for the host

__global__ void k_rng_draws(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t *u, long long M);
__global__ void k_zig_walk(const uint64_t *u, long long M, double *val, int *len, unsigned char *kind,
                           unsigned char *start);
__global__ void k_zig_starts(const long long *slow, const int *n_slow_p, const int *len, unsigned char *start,
                             int *sst, long long M, int *err);
__global__ void k_slow_flags(const int *len, long long M, unsigned char *flag);
__global__ void k_zig_emit(const unsigned char *start, const long long *num, const double *val, const int *len,
                           const unsigned char *kind, const uint64_t *u, long long M, long long n, double loc,
                           double scale, double *out, int add_clip, long long *consumed, long long *tails,
                           uint64_t *tail_draws, int *n_tails, int max_tails, int *err);
__global__ void k_rng_scatter(const long long *idx, const double *v, int n, double *out);
__global__ void k_rng_gather(const long long *idx, int n, const double *src, double *out);
cudaError_t rng_select_slow(void *temp, size_t &temp_bytes, const unsigned char *flag, long long *slow, int *n_slow,
                            long long M, cudaStream_t st);
cudaError_t rng_scan_starts(void *temp, size_t &temp_bytes, const unsigned char *start, long long *num, long long M,
                            cudaStream_t st);
cudaError_t rng_tables(uint64_t *ki, double *wi, double *fi);
__global__ void k_rng_uniform(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, double *out, long long n);
