// microbenchmark: warp QR of a 36x36 SPD system (clock64 timing)
#include <cstdio>
#include <cstdlib>
#include "lc_qr.cuh"
__global__ void kq(const double *A, const double *b, double *x, long long *t) {
    __shared__ QrSmemT<36> s;
    double damping;
    long long t0 = clock64();
    for (int rep = 0; rep < 10; ++rep) dense_solve_block<256>(s, A, b, 36, damping);
    long long t1 = clock64();
    if (threadIdx.x < 36) x[threadIdx.x] = s.x[threadIdx.x];
    if (threadIdx.x == 0) *t = (t1 - t0) / 10;
}
int main() {
    const int n = 36;
    double A[n * n], b[n];
    srand(1);
    double M[n * n];
    for (int i = 0; i < n * n; ++i) M[i] = rand() / (double)RAND_MAX - 0.5;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
        double s = 0; for (int k = 0; k < n; ++k) s += M[i * n + k] * M[j * n + k];
        A[i * n + j] = s + (i == j ? 1.0 : 0.0);
    }
    for (int i = 0; i < n; ++i) b[i] = i;
    double *dA, *db, *dx; long long *dt;
    cudaMalloc(&dA, sizeof A); cudaMalloc(&db, sizeof b); cudaMalloc(&dx, sizeof b); cudaMalloc(&dt, 8);
    cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice); cudaMemcpy(db, b, sizeof b, cudaMemcpyHostToDevice);
    kq<<<1, 256>>>(dA, db, dx, dt);
    long long t; double x[n];
    cudaMemcpy(&t, dt, 8, cudaMemcpyDeviceToHost); cudaMemcpy(x, dx, sizeof x, cudaMemcpyDeviceToHost);
    double r = 0; for (int i = 0; i < n; ++i) { double s = -b[i]; for (int j = 0; j < n; ++j) s += A[i*n+j]*x[j]; r = fmax(r, fabs(s)); }
    printf("qr cycles per solve: %lld  residual %.3e\n", t, r);
}
