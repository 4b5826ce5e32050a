// uot_temporal.cuh -- two Algorithm-1 iterations per HBM pass (temporal blocking) for the
// fixed-marginal hot path (arXiv 1909.00149, Alg. 1 lines 3, 5-7; rho = inf).
//
// The per-iteration update of a pixel reads a at (j, i+1), (j+1, i) (div^*)
// and M' at (j, i-1), (j-1, i) (div), so one iteration shrinks the region on
// which a' is exact by one pixel on every side.  A CTA therefore loads a tile of
// TW x TH interior pixels plus a 2-pixel halo of Mx, My, r, a, f into shared memory
// (cp.async, zero-filled outside the grid and on the pinned flux components, L3), runs
// iteration k+1 on the region shrunk by 1 and iteration k+2 on the interior, and writes
// only the interior's M, r, a of iteration k+2: 36 B of HBM traffic per pixel per TWO
// iterations (the halo re-reads are neighbouring tiles' interiors and hit L2).
// The arithmetic of each iteration is k_iter's (uot_kernels.cuh), in the same order.
// Because neighbouring tiles read this tile's iteration-k values as their halo, the
// outputs go to the other ping-pong slot for M, a AND to a second r buffer (r_alt).
#pragma once
#include "uot_kernels.cuh"

namespace uotk {

constexpr int kTW = 64, kTH = 32, kHalo = 2;
constexpr int kRW = kTW + 2 * kHalo, kRH = kTH + 2 * kHalo, kRA = kRW * kRH;
constexpr int kT2Threads = 256;
constexpr size_t kT2Smem = 9 * (size_t)kRA * sizeof(float);

struct Iter2Args {
    int nx, ny, tiles_x, tiles_y;
    long long N;
    const float* f;
    const float* mx_in; const float* my_in; const float* a_in; const float* r_in;
    float* mx_out; float* my_out; float* a_out; float* r_out;
    float tau1, tau2, atau1;
    int r_mode;
    float r_scale;
    double* partials;           // [G * tiles][kRec] when reducing
    const int* stop;
};

// 4-byte async global -> shared copy; zero-fill when !valid (src-size 0)
__device__ __forceinline__ void cp_async4(float* s, const float* g, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    const int sz = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(g), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <bool RED>
__global__ void __launch_bounds__(kT2Threads, 2) k_iter2(const Iter2Args A) {
    extern __shared__ float sm[];
    __shared__ double red_sh[40];
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    float* MX0 = sm;            // iteration k (masked: pinned / outside = 0), later M^{k+2}
    float* MY0 = MX0 + kRA;
    float* R0 = MY0 + kRA;
    float* A0 = R0 + kRA;
    float* F = A0 + kRA;
    float* MX1 = F + kRA;       // iteration k+1
    float* MY1 = MX1 + kRA;
    float* R1 = MY1 + kRA;
    float* A1 = R1 + kRA;
    const int tiles = A.tiles_x * A.tiles_y;
    const int pair = blockIdx.x / tiles, tile = blockIdx.x - pair * tiles;
    const int tx = tile % A.tiles_x, ty = tile / A.tiles_x;
    const int nx = A.nx, ny = A.ny;
    const int gi0 = tx * kTW - kHalo, gj0 = ty * kTH - kHalo;
    const size_t po = (size_t)pair * (size_t)A.N;
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1;
    const int tid = threadIdx.x;

    // ---- load the tile + halo (iteration k) -------------------------------------------
    for (int e = tid; e < kRA; e += kT2Threads) {
        const int jj = e / kRW, ii = e - jj * kRW;
        const int gi = gi0 + ii, gj = gj0 + jj;
        const bool in = gi >= 0 && gi < nx && gj >= 0 && gj < ny;
        const size_t g = in ? po + (size_t)gj * nx + gi : po;
        cp_async4(MX0 + e, A.mx_in + g, in && gi < nx - 1);   // Mx[:, nx-1] pinned (L3)
        cp_async4(MY0 + e, A.my_in + g, in && gj < ny - 1);   // My[ny-1, :] pinned
        cp_async4(R0 + e, A.r_in + g, in);
        cp_async4(A0 + e, A.a_in + g, in);
        cp_async4(F + e, A.f + g, in);
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- iteration k+1, line 3: M' on [0, RH-2] x [0, RW-2] (needs a at +i, +j) -------
    for (int e = tid; e < (kRH - 1) * (kRW - 1); e += kT2Threads) {
        const int jj = e / (kRW - 1), ii = e - jj * (kRW - 1);
        const int idx = jj * kRW + ii;
        const int gi = gi0 + ii, gj = gj0 + jj;
        const bool in = gi >= 0 && gi < nx && gj >= 0 && gj < ny;
        const bool colx = in && gi < nx - 1, rowy = in && gj < ny - 1;
        const float a = A0[idx];
        const float gx = colx ? a - A0[idx + 1] : 0.f;
        const float gy = rowy ? a - A0[idx + kRW] : 0.f;
        const float qx = MX0[idx] - t1 * gx;
        const float qy = MY0[idx] - t1 * gy;
        const float n2 = qx * qx + qy * qy;
        const float s = shrink_factor(n2, rsqrtf(n2), t1);
        MX1[idx] = s * qx;
        MY1[idx] = s * qy;
    }
    __syncthreads();
    // ---- iteration k+1, lines 5-7: r', a' on [1, RH-2] x [1, RW-2] --------------------
    for (int e = tid; e < (kRH - 2) * (kRW - 2); e += kT2Threads) {
        const int jj = 1 + e / (kRW - 2), ii = 1 + e % (kRW - 2);
        const int idx = jj * kRW + ii;
        const int gi = gi0 + ii, gj = gj0 + jj;
        const bool in = gi >= 0 && gi < nx && gj >= 0 && gj < ny;
        const float r0 = R0[idx], a0 = A0[idx], f = F[idx];
        const float rn = in ? r_update(fmaf(t1, a0, r0), A.r_mode, at1, A.r_scale) : 0.f;
        const float divn = (MX1[idx] - MX1[idx - 1]) + (MY1[idx] - MY1[idx - kRW]);
        const float divk = (MX0[idx] - MX0[idx - 1]) + (MY0[idx] - MY0[idx - kRW]);
        const float Kn = divn - rn - f;
        const float Kk = divk - r0 - f;
        R1[idx] = rn;
        A1[idx] = in ? fmaf(t2, 2.f * Kn - Kk, a0) : 0.f;
    }
    __syncthreads();
    // ---- iteration k+2, line 3: M'' on [1, RH-3] x [1, RW-3] (into MX0/MY0) ------------
    for (int e = tid; e < (kRH - 3) * (kRW - 3); e += kT2Threads) {
        const int jj = 1 + e / (kRW - 3), ii = 1 + e % (kRW - 3);
        const int idx = jj * kRW + ii;
        const int gi = gi0 + ii, gj = gj0 + jj;
        const bool in = gi >= 0 && gi < nx && gj >= 0 && gj < ny;
        const bool colx = in && gi < nx - 1, rowy = in && gj < ny - 1;
        const float a = A1[idx];
        const float gx = colx ? a - A1[idx + 1] : 0.f;
        const float gy = rowy ? a - A1[idx + kRW] : 0.f;
        const float qx = MX1[idx] - t1 * gx;                 // M' is 0 on pinned / outside
        const float qy = MY1[idx] - t1 * gy;
        const float n2 = qx * qx + qy * qy;
        const float s = shrink_factor(n2, rsqrtf(n2), t1);
        MX0[idx] = s * qx;
        MY0[idx] = s * qy;
    }
    __syncthreads();
    // ---- iteration k+2, lines 5-7 on the interior; write M'', r'', a'' ----------------
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f;
    for (int e = tid; e < kTH * kTW; e += kT2Threads) {
        const int jj = kHalo + e / kTW, ii = kHalo + e % kTW;
        const int gi = gi0 + ii, gj = gj0 + jj;
        if (gi >= nx || gj >= ny) continue;
        const int idx = jj * kRW + ii;
        const float r1 = R1[idx], a1 = A1[idx], f = F[idx];
        const float rn = r_update(fmaf(t1, a1, r1), A.r_mode, at1, A.r_scale);
        const float mxn = MX0[idx], myn = MY0[idx];
        const float divn = (mxn - MX0[idx - 1]) + (myn - MY0[idx - kRW]);
        const float divk = (MX1[idx] - MX1[idx - 1]) + (MY1[idx] - MY1[idx - kRW]);
        const float Kn = divn - rn - f;
        const float Kk = divk - r1 - f;
        const float an = fmaf(t2, 2.f * Kn - Kk, a1);
        const size_t g = po + (size_t)gj * nx + gi;
        A.mx_out[g] = mxn;
        A.my_out[g] = myn;
        A.r_out[g] = rn;
        A.a_out[g] = an;
        if constexpr (RED) {
            const float dmx = mxn - MX1[idx], dmy = myn - MY1[idx], dr = rn - r1;
            s_tr += sqrtf(mxn * mxn + myn * myn);
            s_gr += pw(rn, A.r_mode);
            s_k2 += Kn * Kn;
            s_dz += dmx * dmx + dmy * dmy + dr * dr;
            s_ub += pw(divn - f, A.r_mode);
        }
    }
    if constexpr (RED) {
        // fixed-order block sums (warp butterfly, then warp 0 over the 8 warp sums)
        double v[5] = {s_tr, s_gr, s_k2, s_dz, s_ub};
        const int w = tid >> 5, l = tid & 31;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(kFull, v[q], o);
        }
        if (l == 0)
#pragma unroll
            for (int q = 0; q < 5; ++q) red_sh[q * 8 + w] = v[q];
        __syncthreads();
        if (tid == 0) {
            double* P = A.partials + ((size_t)pair * tiles + tile) * kRec;
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                double t = 0.0;
                for (int k = 0; k < kT2Threads / 32; ++k) t += red_sh[q * 8 + k];
                P[q] = t;
            }
            P[5] = 0.0; P[6] = 0.0; P[7] = 0.0;
        }
    }
}

}  // namespace uotk
