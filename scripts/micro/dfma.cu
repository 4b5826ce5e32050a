// DFMA throughput on sm_100a: 148 x 8 warps, 16 independent fp64 FMA chains per thread.
#include <cstdio>
__global__ void k(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}
int main() {
    double* d; cudaMalloc(&d, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps = 4; warps <= 16; warps *= 2) {
        k<<<148, 32 * warps>>>(d, 100, 0.999, 0.001);
        cudaEventRecord(e0);
        k<<<148, 32 * warps>>>(d, iters, 0.999, 0.001);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 16 * iters * 148.0 * 32 * warps;
        printf("warps/SM %d: %.2f TFLOP/s fp64 FMA\n", warps, fl / ms / 1e9);
    }
    return 0;
}
