#pragma once
#include <cuda_runtime.h>
#include <cstddef>

struct BsrJob {
    int n, m, iters;
    const double *diag;    // n*9
    const double *off;     // m*9
    const int *cols;       // m
    const int *rowptr;     // n+1
    const int *order;      // m, block ids sorted by row (stable)
    const double *rhs;     // n*3
    double *minv;          // n*9
    double *x, *r, *z, *p, *ap, *best;   // n*3
    double *norms;         // LC_MAX_LOG
    int *info;             // iterations, breakdown, singular
};

__global__ void k_bsr_keys(int m, const long long *rows, int *keys, int *vals, int *count);
__global__ void k_bsr_rowptr(int n, const int *count, int *rowptr);
__global__ void k_pcg_bsr(BsrJob J);
__global__ void k_dense_solve(int n, const double *A, const double *b, double *x, double *info);
size_t bsr_sort_temp_bytes(int m);
cudaError_t bsr_sort(void *temp, size_t temp_bytes, const int *keys_in, int *keys_out,
                     const int *vals_in, int *vals_out, int m, int key_bits, cudaStream_t st);
