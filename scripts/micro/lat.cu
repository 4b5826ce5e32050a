// Latency microbenchmarks (dependent chains) on sm_100a: DFMA, FFMA, F2F, LDS.64, bar.sync.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, float fin) {
    __shared__ double sm[1024];
    __shared__ int idx[1024];
    const int t = threadIdx.x;
    sm[t] = 1.0 + t * 1e-9; idx[t] = (t * 7 + 1) % blockDim.x;
    __syncthreads();
    double d = out[0] + t;
    float f = fin;
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) d = fma(d, 0.999999, 1e-7);
    long long c1 = clock64();
    for (int i = 0; i < n; ++i) f = fmaf(f, 0.999999f, 1e-7f);
    long long c2 = clock64();
    double e = d;
    for (int i = 0; i < n; ++i) e = (double)(float)e + 1e-3;           // F2F round trip
    long long c3 = clock64();
    int j = t;
    for (int i = 0; i < n; ++i) j = idx[j];                           // dependent LDS
    long long c4 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long c5 = clock64();
    double q = d;
    for (int i = 0; i < n; ++i) q = sqrt(q + 1.0);
    long long c6 = clock64();
    double r = d;
    for (int i = 0; i < n; ++i) r = 1.0 / (r + 1.0);
    long long c7 = clock64();
    if (t == 0) {
        cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4;
        cyc[5] = c6 - c5; cyc[6] = c7 - c6;
    }
    out[1 + t] = d + f + e + j + q + r;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8 * 2048); cudaMalloc(&c, 8 * 16);
    cudaMemset(o, 0, 8 * 2048);
    const int n = 1000;
    for (int th : {32, 512, 1024}) {
        k<<<1, th>>>(o, c, n, 1.f);
        long long h[16];
        cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
        printf("threads %4d per-op cycles: DFMA %.1f FFMA %.1f F2F-roundtrip %.1f LDS-chain %.1f bar.sync %.1f dsqrt %.1f ddiv %.1f\n",
               th, h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n, h[6] / (double)n);
    }
    return 0;
}
