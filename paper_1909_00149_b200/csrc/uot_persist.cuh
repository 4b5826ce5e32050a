// uot_persist.cuh -- SMEM-resident persistent kernel for small grids
// (BASELINE configs[0..1]: 64^2 and 512^2 pairs), arXiv 1909.00149 Alg. 1.
//
// The streaming kernel (uot_kernels.cuh) is bound by launch latency and by
// its per-warp dependent-load chain when a whole iteration moves only a few
// MB.  Here the complete state of a pair (Mx, My, r, a, f [, x, p]) lives in
// shared memory, split into tiles of TW x TH pixels, one tile per CTA, and
// ALL iterations of a call run inside one cooperative launch:
//   phase A  M^{k+1} = shrink(M^k - tau1 div^*(a^k)) on the tile plus its left
//            column and top row (halo recompute, needs the a / M ring);
//   phase B  r^{k+1}, (x^{k+1}), K^k, K^{k+1}, a^{k+1} on the tile;
//   publish  the tile's edge rows/columns of a^{k+1} and M^{k+1} to a
//            double-buffered global exchange slot, then release a per-tile
//            iteration flag;
//   halo     wait (acquire) for the 6 neighbour tiles that feed the ring
//            (top, bottom, left, right, top-right, bottom-left) and load it.
// Only neighbour tiles synchronise; the residual reductions of a check
// iteration use one grid-wide barrier (last CTA reduces in fixed order and
// evaluates the stopping test, L13).  Arithmetic per pixel is the same as the
// streaming kernel's (same order of operations), so both paths agree to fp32
// rounding.  Prox mode is supported for chains of T = 2 (pairs), where the
// x-update needs only the tile's own dual.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "uot_kernels.cuh"

namespace uotk {

struct PersistArgs {
    int nx, ny, G, T, P;
    long long N;
    int TW, TH, tiles_x, tiles_y;     // tile geometry (per pair)
    int n_iters;                      // iterations in this launch
    int red_every;                    // reductions every red_every-th iteration (0: none) ...
    int red_last;                     // ... and on the last one
    long long iter0;                  // iteration count before the launch
    int slot0;                        // ping-pong slot holding iterate iter0
    int prox;                         // T == 2 prox mode
    const float* f;
    float* mxb[2]; float* myb[2]; float* ab[2];   // ping-pong slots; input = slot slot0
    float* r;
    float* xb[2]; const float* p;
    float tau1, tau2, atau1, c1, c2, c3;
    int r_mode; float r_scale; int fix_first;
    float* xchg;                      // [ctas][2][4*TW + 4*TH]
    int* flags;                       // [ctas], zeroed before the launch
    int* bar;                         // [2] grid barrier (count, generation), zeroed before the launch
    double* partials;                 // [ctas][kRec]
    double* pair_out;                 // [G][kRec]
    double* glob;
    int* stop;                        // nullable: device stopping test armed
    double tol, tau1d;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// dynamic SMEM layout (floats)
struct PLayout {
    int wa, wm;         // row pitch of the a ring (TW+2) and of M (TW+1)
    int na, nm, no;     // sizes
    __device__ __host__ PLayout(int TW, int TH) {
        wa = TW + 2; wm = TW + 1;
        na = (TH + 2) * wa; nm = (TH + 1) * wm; no = TH * TW;
    }
    __device__ __host__ size_t floats(bool prox) const {
        return (size_t)na + 4 * (size_t)nm + (prox ? 5 : 2) * (size_t)no;
    }
};

template <bool PROX>
__global__ void __launch_bounds__(512)
k_persist(const PersistArgs A) {
    extern __shared__ float sm[];
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    const int TW = A.TW, TH = A.TH, nx = A.nx, ny = A.ny;
    const PLayout L(TW, TH);
    float* sA = sm;                         // a ring: (jj+1)*wa + (ii+1), jj in [-1,TH], ii in [-1,TW]
    float* sMX[2] = {sA + L.na, sA + L.na + L.nm};        // M: (jj+1)*wm + (ii+1), jj in [-1,TH), ii in [-1,TW)
    float* sMY[2] = {sA + L.na + 2 * L.nm, sA + L.na + 3 * L.nm};
    float* sR = sA + L.na + 4 * L.nm;       // own: jj*TW + ii
    float* sF = sR + L.no;                  // fixed: f; prox: x0
    float* sX1 = sF + L.no;                 // prox only
    float* sP0 = sX1 + L.no;
    float* sP1 = sP0 + L.no;

    const int tiles = A.tiles_x * A.tiles_y;
    const int cta = blockIdx.x;
    const int pair = cta / tiles;
    const int tile = cta % tiles;
    const int ty = tile / A.tiles_x, tx = tile % A.tiles_x;
    const int i0 = tx * TW, j0 = ty * TH;
    const size_t po = (size_t)pair * A.N;
    const int tid = threadIdx.x, nth = blockDim.x;
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1;
    const int XS = 4 * TW + 4 * TH;         // exchange slot size
    // exchange slot sub-offsets
    const int oTop = 0, oBot = TW, oLeft = 2 * TW, oRight = 2 * TW + TH, oMxB = 2 * TW + 2 * TH,
              oMyB = 3 * TW + 2 * TH, oMxR = 4 * TW + 2 * TH, oMyR = 4 * TW + 3 * TH;
    auto nb_cta = [&](int dy, int dx) -> int {
        const int yy = ty + dy, xx = tx + dx;
        if (yy < 0 || yy >= A.tiles_y || xx < 0 || xx >= A.tiles_x) return -1;
        return pair * tiles + yy * A.tiles_x + xx;
    };
    const int nT = nb_cta(-1, 0), nB = nb_cta(1, 0), nL = nb_cta(0, -1), nR = nb_cta(0, 1);
    const int nTR = nb_cta(-1, 1), nBL = nb_cta(1, -1);

    // prox (T = 2): frames of this pair's chain
    const size_t f0 = PROX ? ((size_t)(pair / A.P) * A.T + (pair % A.P)) * (size_t)A.N : 0;

    // ---- initial load from global (iteration iter0); halos straight from neighbours' regions
    const int in = A.slot0;
    const float* gmx = A.mxb[in] + po; const float* gmy = A.myb[in] + po; const float* ga = A.ab[in] + po;
    auto gidx_ok = [&](int gj, int gi) { return gj >= 0 && gj < ny && gi >= 0 && gi < nx; };
    // the (-1,-1) and (TH,TW) corners are never used: not loaded (their owners are not
    // synchronised with this tile, and may already be writing the output slot)
    for (int e = tid; e < (TH + 2) * (TW + 2); e += nth) {
        const int jj = e / (TW + 2) - 1, ii = e % (TW + 2) - 1;
        const int gj = j0 + jj, gi = i0 + ii;
        const bool corner = (jj < 0 && ii < 0) || (jj == TH && ii == TW);
        sA[e] = (!corner && gidx_ok(gj, gi)) ? ga[(size_t)gj * nx + gi] : 0.f;
    }
    for (int e = tid; e < (TH + 1) * (TW + 1); e += nth) {
        const int jj = e / (TW + 1) - 1, ii = e % (TW + 1) - 1;
        const int gj = j0 + jj, gi = i0 + ii;
        const bool ok = gidx_ok(gj, gi) && !(jj < 0 && ii < 0);
        sMX[0][e] = (ok && gi < nx - 1) ? gmx[(size_t)gj * nx + gi] : 0.f;   // pinned read as 0 (L3)
        sMY[0][e] = (ok && gj < ny - 1) ? gmy[(size_t)gj * nx + gi] : 0.f;
    }
    for (int e = tid; e < TH * TW; e += nth) {
        const int jj = e / TW, ii = e % TW;
        const int gj = j0 + jj, gi = i0 + ii;
        const bool ok = gidx_ok(gj, gi);
        const size_t g = (size_t)gj * nx + gi;
        sR[e] = ok ? A.r[po + g] : 0.f;
        if constexpr (PROX) {
            sF[e] = ok ? A.xb[in][f0 + g] : 0.f;
            sX1[e] = ok ? A.xb[in][f0 + A.N + g] : 0.f;
            sP0[e] = ok ? A.p[f0 + g] : 0.f;
            sP1[e] = ok ? A.p[f0 + A.N + g] : 0.f;
        } else {
            sF[e] = ok ? A.f[po + g] : 0.f;
        }
    }
    __syncthreads();

    __shared__ double red_sh[32];
    __shared__ int s_flag;
    const int dA_i = nth % (TW + 1), dA_j = nth / (TW + 1);      // index increments per stride
    const int dB_i = nth % TW, dB_j = nth / TW;
    const bool lonely = nT < 0 && nB < 0 && nL < 0 && nR < 0 && nTR < 0 && nBL < 0;   // single tile: no exchange
    int cur = 0;                            // which sMX/sMY buffer holds M^k
    int done = 0;
    for (int k = 0; k < A.n_iters; ++k) {
        float* MXk = sMX[cur]; float* MYk = sMY[cur];
        float* MXn = sMX[cur ^ 1]; float* MYn = sMY[cur ^ 1];
        // ---------------- phase A: M^{k+1} on the tile + left column + top row (Alg.1 line 3)
        const int ext = (TH + 1) * (TW + 1);
        int jjA = tid / (TW + 1) - 1, iiA = tid % (TW + 1) - 1;   // running 2-D index of e
        for (int e = tid; e < ext; e += nth, iiA += dA_i, jjA += dA_j) {
            if (iiA >= TW) { iiA -= TW + 1; ++jjA; }
            const int jj = jjA, ii = iiA;
            if (jj < 0 && ii < 0) continue;                      // (-1,-1) is never used
            const int gj = j0 + jj, gi = i0 + ii;
            float mxn = 0.f, myn = 0.f;
            if (gidx_ok(gj, gi)) {
                const int ka = (jj + 1) * L.wa + (ii + 1);
                const float ac = sA[ka];
                const float gx = (gi < nx - 1) ? ac - sA[ka + 1] : 0.f;
                const float gy = (gj < ny - 1) ? ac - sA[ka + L.wa] : 0.f;
                const float qx = __fmaf_rn(-t1, gx, MXk[e]);
                const float qy = __fmaf_rn(-t1, gy, MYk[e]);
                const float n2 = norm2(qx, qy);
                const float s = shrink_factor(n2, rsqrtf(n2), t1);
                mxn = s * qx;
                myn = s * qy;
            }
            MXn[e] = mxn;
            MYn[e] = myn;
        }
        __syncthreads();
        // ---------------- phase B: r, x, K^k, K^{k+1}, a (Alg.1 lines 4-7)
        const bool red = (A.red_every > 0 && ((k + 1) % A.red_every == 0)) || (A.red_last && k == A.n_iters - 1);
        float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f, s_px = 0.f;
        int jjB = tid / TW, iiB = tid % TW;
        for (int e = tid; e < TH * TW; e += nth, iiB += dB_i, jjB += dB_j) {
            if (iiB >= TW) { iiB -= TW; ++jjB; }
            const int jj = jjB, ii = iiB;
            const int gj = j0 + jj, gi = i0 + ii;
            if (!gidx_ok(gj, gi)) continue;
            const int ka = (jj + 1) * L.wa + (ii + 1);
            const int km = (jj + 1) * L.wm + (ii + 1);
            const float ac = sA[ka];
            const float rk = sR[e];
            const float rn = r_update(fmaf(t1, ac, rk), A.r_mode, at1, A.r_scale);
            float fk, fn, x0n = 0.f, x1n = 0.f;
            if constexpr (PROX) {
                x0n = A.fix_first ? sF[e] : fmaxf(fmaf(A.c1, sP0[e], fmaf(A.c2, sF[e], -A.c3 * (ac - 0.f))), 0.f);
                x1n = fmaxf(fmaf(A.c1, sP1[e], fmaf(A.c2, sX1[e], -A.c3 * (0.f - ac))), 0.f);
                fk = sX1[e] - sF[e];
                fn = x1n - x0n;
            } else {
                fk = sF[e];
                fn = sF[e];
            }
            const float divn = (MXn[km] - MXn[km - 1]) + (MYn[km] - MYn[km - L.wm]);
            const float divk = (MXk[km] - MXk[km - 1]) + (MYk[km] - MYk[km - L.wm]);
            const float Kn = divn - rn - fn;
            const float Kk = divk - rk - fk;
            const float an = fmaf(t2, 2.f * Kn - Kk, ac);
            if (red) {
                const float mx2 = MXn[km] * MXn[km] + MYn[km] * MYn[km];
                const float dmx = MXn[km] - MXk[km], dmy = MYn[km] - MYk[km], dr = rn - rk;
                s_tr += sqrtf(mx2);
                s_gr += pw(rn, A.r_mode);
                s_k2 += Kn * Kn;
                s_dz += dmx * dmx + dmy * dmy + dr * dr;
                s_ub += pw(divn - fn, A.r_mode);
                if constexpr (PROX) {
                    const float d0 = x0n - sF[e], d1 = x1n - sX1[e], e0 = x0n - sP0[e], e1 = x1n - sP1[e];
                    s_dz += d0 * d0 + d1 * d1;
                    s_px += e0 * e0 + e1 * e1;
                }
            }
            sR[e] = rn;
            if constexpr (PROX) { sF[e] = x0n; sX1[e] = x1n; }
            sA[ka] = an;                      // own pixel only: in place is safe after phase A
        }
        cur ^= 1;
        done = k + 1;
        __syncthreads();
        // ---------------- reductions (check iterations): fixed-order, grid barrier
        if (red) {
            double d[6] = {s_tr, s_gr, s_k2, s_dz, s_ub, s_px};
            double out[6];
            for (int q = 0; q < 6; ++q) {
                double v = d[q];
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
                if ((tid & 31) == 0) red_sh[tid >> 5] = v;
                __syncthreads();
                double t = 0.0;
                if (tid == 0) for (int w = 0; w < (nth >> 5); ++w) t += red_sh[w];
                out[q] = t;
                __syncthreads();
            }
            int gen = 0;
            if (tid == 0) {
                double* P = A.partials + (size_t)cta * kRec;
                for (int q = 0; q < 6; ++q) P[q] = out[q];
                P[6] = 0.0; P[7] = 0.0;
                __threadfence();
                gen = *reinterpret_cast<volatile int*>(&A.bar[1]);
                s_flag = (atomicAdd(&A.bar[0], 1) == (int)gridDim.x - 1) ? 1 : 0;
            }
            __syncthreads();
            if (s_flag) {
                // last CTA: per (pair, field) one warp sums the tiles' records in fixed order
                __threadfence();
                const int nw = nth >> 5, w = tid >> 5, lane = tid & 31;
                for (int cq = w; cq < A.G * 6; cq += nw) {
                    const int g = cq / 6, q = cq % 6;
                    double v = 0.0;
                    for (int tt = lane; tt < tiles; tt += 32) v += __ldcg(A.partials + (size_t)(g * tiles + tt) * kRec + q);
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
                    if (lane == 0) A.pair_out[(size_t)g * kRec + q] = v;
                }
                __syncthreads();
                if (tid == 0) {
                    double tot[6] = {0, 0, 0, 0, 0, 0};
                    for (int g = 0; g < A.G; ++g)
                        for (int q = 0; q < 6; ++q) tot[q] += __ldcg(A.pair_out + (size_t)g * kRec + q);
                    bool nonf = false;
                    for (int q = 0; q < 6; ++q) { A.glob[q] = tot[q]; nonf |= !isfinite(tot[q]); }
                    const long long it = A.iter0 + k + 1;
                    A.glob[12] = (double)it;                        // GL_LASTRED
                    if (nonf) {
                        A.glob[11] = 1.0;                           // GL_NONF
                        if (A.stop) *A.stop = 1;
                    } else if (A.tol > 0.0 && A.stop) {
                        const double scale = A.tol * fmax(sqrt(A.glob[8]), 1e-30);   // GL_FSQ
                        if (sqrt(tot[2]) <= scale && sqrt(tot[3]) / A.tau1d <= scale) {
                            A.glob[10] = (double)it;                // GL_CONV
                            *A.stop = 1;
                        }
                    }
                    A.bar[0] = 0;
                    __threadfence();
                    atomicExch(&A.bar[1], gen + 1);
                }
            } else if (tid == 0) {
                while (*reinterpret_cast<volatile int*>(&A.bar[1]) == gen) __nanosleep(64);
                __threadfence();
            }
            __syncthreads();
            if (A.stop != nullptr && *reinterpret_cast<volatile int*>(A.stop)) break;
        }
        if (k == A.n_iters - 1) break;
        if (lonely) continue;                                   // ring = grid boundary (zeros)
        // ---------------- publish edges of a^{k+1}, M^{k+1}; release flag
        float* X = A.xchg + ((size_t)cta * 2 + ((k + 1) & 1)) * XS;
        const float* MXc = sMX[cur]; const float* MYc = sMY[cur];
        for (int e = tid; e < 2 * TW + 2 * TH; e += nth) {
            if (e < TW) {
                X[oTop + e] = sA[1 * L.wa + e + 1];
                X[oMxB + e] = MXc[TH * L.wm + e + 1];
                X[oMyB + e] = MYc[TH * L.wm + e + 1];
            } else if (e < 2 * TW) {
                const int ii = e - TW;
                X[oBot + ii] = sA[TH * L.wa + ii + 1];
            } else if (e < 2 * TW + TH) {
                const int jj = e - 2 * TW;
                X[oLeft + jj] = sA[(jj + 1) * L.wa + 1];
                X[oMxR + jj] = MXc[(jj + 1) * L.wm + TW];
                X[oMyR + jj] = MYc[(jj + 1) * L.wm + TW];
            } else {
                const int jj = e - 2 * TW - TH;
                X[oRight + jj] = sA[(jj + 1) * L.wa + TW];
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release(&A.flags[cta], k + 1);
            const int nbs[6] = {nT, nB, nL, nR, nTR, nBL};
            for (int q = 0; q < 6; ++q)
                if (nbs[q] >= 0)
                    while (ld_acquire(&A.flags[nbs[q]]) < k + 1) __nanosleep(20);
        }
        __syncthreads();
        // ---------------- halo ring from the neighbours' slots (L2, bypass L1)
        const size_t par = (size_t)((k + 1) & 1);
        auto slot = [&](int nbc) { return A.xchg + ((size_t)nbc * 2 + par) * XS; };
        for (int e = tid; e < 2 * TW + 2 * TH + 2; e += nth) {
            if (e < TW) {                                   // top ring row (jj = -1), from top nb bottom
                const float* S = nT >= 0 ? slot(nT) : nullptr;
                sA[0 * L.wa + e + 1] = S ? __ldcg(S + oBot + e) : 0.f;
                sMX[cur][0 * L.wm + e + 1] = S ? __ldcg(S + oMxB + e) : 0.f;
                sMY[cur][0 * L.wm + e + 1] = S ? __ldcg(S + oMyB + e) : 0.f;
            } else if (e < 2 * TW) {                        // bottom ring row (jj = TH), from bottom nb top
                const int ii = e - TW;
                const float* S = nB >= 0 ? slot(nB) : nullptr;
                sA[(TH + 1) * L.wa + ii + 1] = S ? __ldcg(S + oTop + ii) : 0.f;
            } else if (e < 2 * TW + TH) {                   // left ring col (ii = -1), from left nb right
                const int jj = e - 2 * TW;
                const float* S = nL >= 0 ? slot(nL) : nullptr;
                sA[(jj + 1) * L.wa + 0] = S ? __ldcg(S + oRight + jj) : 0.f;
                sMX[cur][(jj + 1) * L.wm + 0] = S ? __ldcg(S + oMxR + jj) : 0.f;
                sMY[cur][(jj + 1) * L.wm + 0] = S ? __ldcg(S + oMyR + jj) : 0.f;
            } else if (e < 2 * TW + 2 * TH) {               // right ring col (ii = TW), from right nb left
                const int jj = e - 2 * TW - TH;
                const float* S = nR >= 0 ? slot(nR) : nullptr;
                sA[(jj + 1) * L.wa + TW + 1] = S ? __ldcg(S + oLeft + jj) : 0.f;
            } else if (e == 2 * TW + 2 * TH) {              // top-right corner (-1, TW): top-right nb (TH-1, 0)
                const float* S = nTR >= 0 ? slot(nTR) : nullptr;
                sA[0 * L.wa + TW + 1] = S ? __ldcg(S + oBot + 0) : 0.f;
            } else {                                        // bottom-left corner (TH, -1): bottom-left nb (0, TW-1)
                const float* S = nBL >= 0 ? slot(nBL) : nullptr;
                sA[(TH + 1) * L.wa + 0] = S ? __ldcg(S + oTop + TW - 1) : 0.f;
            }
        }
        __syncthreads();
    }

    // ---- write the final iterate (iteration iter0 + done) to its ping-pong slot
    const int o = A.slot0 ^ (int)(done & 1);
    const float* MXc = sMX[cur]; const float* MYc = sMY[cur];
    for (int e = tid; e < TH * TW; e += nth) {
        const int jj = e / TW, ii = e % TW;
        const int gj = j0 + jj, gi = i0 + ii;
        if (!gidx_ok(gj, gi)) continue;
        const size_t g = (size_t)gj * nx + gi;
        const int km = (jj + 1) * L.wm + (ii + 1);
        A.mxb[o][po + g] = MXc[km];
        A.myb[o][po + g] = MYc[km];
        A.ab[o][po + g] = sA[(jj + 1) * L.wa + (ii + 1)];
        A.r[po + g] = sR[e];
        if constexpr (PROX) {
            A.xb[o][f0 + g] = sF[e];
            A.xb[o][f0 + A.N + g] = sX1[e];
        }
    }
}

}  // namespace uotk
