// Throughput of scalar vs packed (f32x2) FP32 instructions on sm_100a, at full occupancy and
// at k_wave's 8 warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int MODE>
__global__ void k(float* out, float s) {
    float a[kChains]; float2 b[kChains];
    for (int c = 0; c < kChains; ++c) { a[c] = threadIdx.x * 1e-3f + c; b[c] = make_float2(a[c], a[c] + 1.f); }
    const float2 s2 = make_float2(s, s), t2 = make_float2(1e-7f, 2e-7f);
    const float t = 1e-7f;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (MODE == 0) a[c] = fmaf(a[c], s, a[(c + 1) % kChains]);           // FFMA 3-reg
            if (MODE == 1) b[c] = __ffma2_rn(b[c], s2, b[(c + 1) % kChains]);    // FFMA2
            if (MODE == 2) a[c] = a[c] + a[(c + 3) % kChains];                    // FADD
            if (MODE == 3) b[c] = __fadd2_rn(b[c], b[(c + 3) % kChains]);         // FADD2
            if (MODE == 4) { a[c] = fmaf(a[c], s, a[(c + 1) % kChains]); a[c] = fmaxf(a[c], t); }   // FFMA + FMNMX
            if (MODE == 5) { b[c] = __ffma2_rn(b[c], s2, b[(c + 1) % kChains]); b[c].x = fmaxf(b[c].x, t); b[c].y = fmaxf(b[c].y, t); }
            if (MODE == 6) a[c] = fmaf(a[c], s, t);                               // FFMA imm-ish
            if (MODE == 7) b[c] = __ffma2_rn(b[c], s2, t2);
        }
    }
    float acc = 0.f;
    for (int c = 0; c < kChains; ++c) acc += a[c] + b[c].x + b[c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, int threads, int blocks_per_sm, int nsm, float* out) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int grid = nsm * blocks_per_sm;
    k<MODE><<<grid, threads>>>(out, 0.999f);
    cudaEventRecord(e0);
    k<MODE><<<grid, threads>>>(out, 0.999f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int ops_per = (MODE == 4 || MODE == 5) ? 2 : 1;
    double lanes = (MODE & 1) ? 2.0 : 1.0;                 // fp32 results per thread-instruction (FP part)
    double inst = (double)grid * threads * kIters * kChains;   // FP instructions (one of the ops_per)
    double cyc = ms * 1e-3 * 1.9e9;                          // nominal
    printf("%-22s threads %4d x %d/SM: %.3f ms  %.3e fp-results/s  %.2f warp-inst/clk/SM (@1.9GHz, x%d ops)\n",
           name, threads, blocks_per_sm, ms, inst * lanes / (ms * 1e-3), inst * ops_per / 32.0 / nsm / cyc, ops_per);
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, sizeof(float) * nsm * 2048);
    for (int cfg = 0; cfg < 2; ++cfg) {
        int th = cfg == 0 ? 1024 : 256, bps = cfg == 0 ? 2 : 1;     // 64 warps/SM, or 8 warps/SM
        run<0>("FFMA", th, bps, nsm, out);
        run<1>("FFMA2", th, bps, nsm, out);
        run<2>("FADD", th, bps, nsm, out);
        run<3>("FADD2", th, bps, nsm, out);
        run<4>("FFMA+FMNMX", th, bps, nsm, out);
        run<5>("FFMA2+2FMNMX", th, bps, nsm, out);
        run<6>("FFMA const", th, bps, nsm, out);
        run<7>("FFMA2 const", th, bps, nsm, out);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
