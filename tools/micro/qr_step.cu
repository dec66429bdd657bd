#include <cstdio>
#include "lc_qr.cuh"
// time one factor step's pieces (k = 0, n = 36)
__global__ void ks(const double *A, const double *b, long long *out) {
    __shared__ QrSmemT<36> s;
    const int t = threadIdx.x;
    if (t < 64) qr_load_pair(s, A, b, 36, 0.0);
    const int n = 36, k = 0;
    long long c0 = clock64();
    const double akk = s.c[k][k];
    double v[36];
#pragma unroll
    for (int i = 0; i < 36; ++i) v[i] = (i > k && i < n) ? s.c[k][i] : 0.0;
    double q[4] = {akk * akk, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 36; ++i) q[(i + 1) & 3] = fma(v[i], v[i], q[(i + 1) & 3]);
    const double ss = (q[0] + q[1]) + (q[2] + q[3]);
    long long c1 = clock64();
    const double nrm = sqrt(ss);
    long long c2 = clock64();
    const double alpha = akk >= 0.0 ? -nrm : nrm;
    const double v0 = akk - alpha;
    const double vn2 = ss - akk * akk + v0 * v0;
    const double tau = 2.0 / vn2;
    long long c3 = clock64();
    double *cj = s.c[t + 1];
    double col[36];
#pragma unroll
    for (int i = 0; i < 36; ++i) col[i] = (i > k && i < n) ? cj[i] : 0.0;
    const double ck = cj[k];
    double d[4] = {v0 * ck, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 36; ++i) d[(i + 1) & 3] = fma(v[i], col[i], d[(i + 1) & 3]);
    const double w = tau * ((d[0] + d[1]) + (d[2] + d[3]));
    long long c4 = clock64();
#pragma unroll
    for (int i = 0; i < 36; ++i)
        if (i > k && i < n) cj[i] = fma(-w, v[i], col[i]);
    cj[k] = fma(-w, v0, ck);
    long long c5 = clock64();
    asm volatile("bar.sync 1, 64;" ::: "memory");
    long long c6 = clock64();
    if (t == 0) { out[0] = c1 - c0; out[1] = c2 - c1; out[2] = c3 - c2; out[3] = c4 - c3; out[4] = c5 - c4; out[5] = c6 - c5; }
}
int main() {
    double A[36 * 36], b[36];
    for (int i = 0; i < 36 * 36; ++i) A[i] = (i % 37 == 0) ? 4.0 : 0.01 * (i % 7);
    for (int i = 0; i < 36; ++i) b[i] = 1;
    double *dA, *db; long long *d;
    cudaMalloc(&dA, sizeof A); cudaMalloc(&db, sizeof b); cudaMalloc(&d, 64);
    cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice); cudaMemcpy(db, b, sizeof b, cudaMemcpyHostToDevice);
    ks<<<1, 64>>>(dA, db, d);
    ks<<<1, 64>>>(dA, db, d);
    long long o[6]; cudaMemcpy(o, d, 48, cudaMemcpyDeviceToHost);
    printf("loads+norm %lld sqrt %lld div %lld col+dot %lld update %lld bar %lld\n", o[0], o[1], o[2], o[3], o[4], o[5]);
}
