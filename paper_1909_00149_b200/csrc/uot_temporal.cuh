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
#include <cuda.h>                   // CUtensorMap (TMA descriptors; encoded on the host)
#include "uot_kernels.cuh"

namespace uotk {

constexpr int kTW = 64, kHalo = 2;
constexpr int kLW = 4;                              // loaded columns left of the interior (16-B aligned)
constexpr int kRW = kTW + 2 * kLW;                  // 72 loaded columns (18 float4), 2 extra unused
constexpr int kT2Threads = 320;             // 10 warps: 2 quads per thread in every phase at TH = 32
constexpr int kT2Wide = 640;                // 20 warps: grids with fewer tiles than SMs (latency-bound)
constexpr int kTH = 32;                             // default interior rows (tile 64 x kTH)
template <int TH, int S> struct TB {                // TH interior rows, S iterations (= halo rows)
    static_assert(S >= 1 && S <= kLW, "the 4 loaded columns per side bound S");
    static constexpr int RH = TH + 2 * S, RA = kRW * RH;
    static constexpr size_t smem = 6 * (size_t)RA * sizeof(float);   // Mx, My, r, a, f, K
    // CTAs per SM: SMEM-bound, at most 3 (320 threads x 3 keeps 64 registers per thread)
    static constexpr int fit = (int)((227u * 1024u) / (smem + 1024u));
    static constexpr int minb = fit < 1 ? 1 : (fit > 3 ? 3 : fit);
};

struct Iter2Args {
    int nx, ny, tiles_x, tiles_y;
    long long N;
    const float* f;
    const float* mx_in; const float* my_in; const float* a_in; const float* r_in;
    float* mx_out; float* my_out; float* a_out; float* r_out;
    float tau1, tau2, atau1;
    int r_mode;
    float r_scale;
    int vec;                    // 16-byte loads (nx % 4 == 0, aligned planes)
    int tma;                    // tile loads by TMA (Iter2Maps valid)
    double* partials;           // [G * tiles][kRec] when reducing
    const int* stop;
};
struct Iter2Maps {
    CUtensorMap tmap[5];        // [G][ny][nx] fp32 views of Mx, My, r, a, f (inputs of this pass);
                                // box 72 x RH x 1, out-of-bounds elements read as 0
};

// TMA: one thread arms an mbarrier with the tile's byte count and issues one 3-D bulk
// tensor copy per plane (coordinates may be negative: out-of-grid elements are zero-filled).
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_3d(float* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(reinterpret_cast<unsigned long long>(map)),
          "r"(x), "r"(y), "r"(z), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

// async global -> shared copies; zero-fill when !valid (src-size 0)
__device__ __forceinline__ void cp_async4(float* s, const float* g, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    const int sz = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(g), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async16(float* s, const float* g, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Region coordinates: row r in [0, RH) <-> gj = ty*TH - S + r; column c in [0, kRW)
// <-> gi = tx*kTW - kLW + c.  Interior: r in [S, TH + S), c in [4, 68).
// Iteration j (1..S) of the pass computes M^j on rows [j-1, RH-1-j] (it reads a^{j-1} at
// +i, +j) and r^j, a^j on rows [j, RH-1-j] (they read M^j at -i, -j): the exact region
// shrinks by one pixel per side and iteration, columns likewise (4 loaded columns per side
// bound S <= 4).  The extrapolated dual step (line 7) needs K^{j-1} = div M^{j-1} - r^{j-1} - f,
// which iteration j-1 computed: it is kept in its own plane (K^0 from the loaded state in a
// first phase), so M, r, a are all updated in place (6 planes) and the divergence of M is
// evaluated once per iteration.
// EDGE: the tile touches the grid border (bounds / pinned masks needed); else all in-grid.
template <int TH, int S, bool RED, bool EDGE, int NT, int RM>
__device__ __forceinline__ void iter_tile(const Iter2Args& A, float* sm, double* red_sh, int pair, int tile,
                                          int gi0, int gj0) {
    constexpr int kRH = TB<TH, S>::RH, kRA = TB<TH, S>::RA, kTH = TH;
    constexpr int Q = kRW / 4;                       // float4 quads per region row
    float* __restrict__ MX = sm;                     // M (masked: pinned / outside = 0)
    float* __restrict__ MY = sm + kRA;
    float* __restrict__ RR = sm + 2 * kRA;
    float* __restrict__ AA = sm + 3 * kRA;
    float* __restrict__ F = sm + 4 * kRA;
    float* __restrict__ KK = sm + 5 * kRA;           // K^{j-1}
    const int nx = A.nx, ny = A.ny;
    const size_t po = (size_t)pair * (size_t)A.N;
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    auto inside = [&](int r, int c) {
        if (!EDGE) return true;
        const int gi = gi0 + c, gj = gj0 + r;
        return gi >= 0 && gi < nx && gj >= 0 && gj < ny;
    };
    auto colx = [&](int r, int c) {                  // Mx exists (L3)
        if (!EDGE) return true;
        const int gi = gi0 + c, gj = gj0 + r;
        return gi >= 0 && gi < nx - 1 && gj >= 0 && gj < ny;
    };
    auto rowy = [&](int r, int c) {                  // My exists (L3)
        if (!EDGE) return true;
        const int gi = gi0 + c, gj = gj0 + r;
        return gi >= 0 && gi < nx && gj >= 0 && gj < ny - 1;
    };

    // ---- load the tile + halo (iteration k) -------------------------------------------
    if (A.tma) {
        // loaded by the kernel (TMA): complete and visible
    } else if (A.vec) {
        for (int e = threadIdx.x; e < kRH * Q; e += NT) {
            const int r = e / Q, c = 4 * (e - r * Q);
            const int gi = gi0 + c, gj = gj0 + r;
            const bool ok = gj >= 0 && gj < ny && gi >= 0 && gi < nx;   // whole float4 (nx % 4 == 0)
            const size_t g = ok ? po + (size_t)gj * nx + gi : po;
            const int s = r * kRW + c;
            cp_async16(MX + s, A.mx_in + g, ok);
            cp_async16(MY + s, A.my_in + g, ok);
            cp_async16(RR + s, A.r_in + g, ok);
            cp_async16(AA + s, A.a_in + g, ok);
            cp_async16(F + s, A.f + g, ok);
        }
    } else {
        for (int e = threadIdx.x; e < kRA; e += NT) {
            const int r = e / kRW, c = e - r * kRW;
            const int gi = gi0 + c, gj = gj0 + r;
            const bool ok = gi >= 0 && gi < nx && gj >= 0 && gj < ny;
            const size_t g = ok ? po + (size_t)gj * nx + gi : po;
            cp_async4(MX + e, A.mx_in + g, ok);
            cp_async4(MY + e, A.my_in + g, ok);
            cp_async4(RR + e, A.r_in + g, ok);
            cp_async4(AA + e, A.a_in + g, ok);
            cp_async4(F + e, A.f + g, ok);
        }
    }
    if (!A.tma) cp_async_wait_all();
    if (EDGE) {                                      // pinned flux components read as 0 (L3)
        __syncthreads();
        for (int e = threadIdx.x; e < kRA; e += NT) {
            const int r = e / kRW, c = e - r * kRW;
            if (!colx(r, c)) MX[e] = 0.f;
            if (!rowy(r, c)) MY[e] = 0.f;
        }
    }
    __syncthreads();

    // The phases before the last work on float4 quads of whole 72-column rows (18 quads
    // per row): 4 pixels per thread with 128-bit SMEM accesses; columns outside a phase's
    // exact range are computed from don't-care neighbours and never used.  The quad's
    // right / left neighbours come from the next / previous 4 floats.
    auto ld4 = [](const float* p) { return *reinterpret_cast<const float4*>(p); };
    auto st4 = [](float* p, float a, float b, float c, float d) { *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d); };
    // ---- K^0 = div M^k - r^k - f on rows [1, RH-2] (line 7's previous K) ----
#pragma unroll 2
    for (int e = threadIdx.x; e < (kRH - 2) * Q; e += NT) {
        const int rr = e / Q, r = 1 + rr, c = 4 * (e - rr * Q);
        const int idx = r * kRW + c;
        const float4 mx = ld4(MX + idx), my = ld4(MY + idx), myu = ld4(MY + idx - kRW);
        const float4 r4 = ld4(RR + idx), f4 = ld4(F + idx);
        const float mxl = MX[idx - 1];               // row start: don't-care column
        st4(KK + idx, ((mx.x - mxl) + (my.x - myu.x)) - r4.x - f4.x, ((mx.y - mx.x) + (my.y - myu.y)) - r4.y - f4.y,
            ((mx.z - mx.y) + (my.z - myu.z)) - r4.z - f4.z, ((mx.w - mx.z) + (my.w - myu.w)) - r4.w - f4.w);
    }
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f;
    // line 3 (in place): M^j = prox(M^{j-1} - tau1 div^* a^{j-1}) on rows [r0, r0 + nr);
    // LAST (reductions): accumulate |M^S - M^{S-1}|^2 over the tile's interior pixels
    auto m_phase = [&](int r0, int nr, bool last) {
#pragma unroll 2
        for (int e = threadIdx.x; e < nr * Q; e += NT) {
            const int rr = e / Q, r = r0 + rr, c = 4 * (e - rr * Q);
            const int idx = r * kRW + c;
            const float4 a4 = ld4(AA + idx), ad4 = ld4(AA + idx + kRW), mx4 = ld4(MX + idx), my4 = ld4(MY + idx);
            const float a5 = AA[idx + 4];           // right neighbour of the 4th pixel (row end: unused)
            const float av[5] = {a4.x, a4.y, a4.z, a4.w, a5}, adv[4] = {ad4.x, ad4.y, ad4.z, ad4.w};
            const float mxv[4] = {mx4.x, mx4.y, mx4.z, mx4.w}, myv[4] = {my4.x, my4.y, my4.z, my4.w};
            float ox[4], oy[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float gx = colx(r, c + v) ? av[v] - av[v + 1] : 0.f;
                const float gy = rowy(r, c + v) ? av[v] - adv[v] : 0.f;
                const float qx = __fmaf_rn(-t1, gx, mxv[v]);   // M is 0 on pinned / outside
                const float qy = __fmaf_rn(-t1, gy, myv[v]);
                const float n2 = norm2(qx, qy);
                const float sf = shrink_factor(n2, rsqrtf(n2), t1);
                ox[v] = sf * qx;
                oy[v] = sf * qy;
            }
            if (RED && last) {
                const int gi = gi0 + c, gj = gj0 + r;
                if (r >= S && r < S + kTH && c >= kLW && c < kLW + kTW && (!EDGE || gj < ny)) {
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        if (!EDGE || gi + v < nx) {
                            const float dmx = ox[v] - mxv[v], dmy = oy[v] - myv[v];
                            s_dz += dmx * dmx + dmy * dmy;
                        }
                }
            }
            st4(MX + idx, ox[0], ox[1], ox[2], ox[3]);
            st4(MY + idx, oy[0], oy[1], oy[2], oy[3]);
        }
    };
    // lines 5-7 (in place): r^j, a^j and K^j from M^j, K^{j-1} on rows [r0, r0 + nr)
    auto ra_phase = [&](int r0, int nr) {
#pragma unroll 2
        for (int e = threadIdx.x; e < nr * Q; e += NT) {
            const int rr = e / Q, r = r0 + rr, c = 4 * (e - rr * Q);
            const int idx = r * kRW + c;
            const float4 r04 = ld4(RR + idx), a04 = ld4(AA + idx), f4 = ld4(F + idx), k04 = ld4(KK + idx);
            const float4 mx1 = ld4(MX + idx), my1 = ld4(MY + idx), my1u = ld4(MY + idx - kRW);
            const float mx1l = MX[idx - 1];         // row start: don't-care column
            const float r0v[4] = {r04.x, r04.y, r04.z, r04.w}, a0v[4] = {a04.x, a04.y, a04.z, a04.w};
            const float fv[4] = {f4.x, f4.y, f4.z, f4.w}, kv[4] = {k04.x, k04.y, k04.z, k04.w};
            const float mxn[5] = {mx1l, mx1.x, mx1.y, mx1.z, mx1.w}, myn[4] = {my1.x, my1.y, my1.z, my1.w};
            const float mynu[4] = {my1u.x, my1u.y, my1u.z, my1u.w};
            float ro[4], ao[4], ko[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const bool in = inside(r, c + v);
                const float rn = in ? r_update(fmaf(t1, a0v[v], r0v[v]), RM, at1, A.r_scale) : 0.f;
                const float divn = (mxn[v + 1] - mxn[v]) + (myn[v] - mynu[v]);
                const float Kn = divn - rn - fv[v];
                ro[v] = rn;
                ko[v] = Kn;
                ao[v] = in ? fmaf(t2, 2.f * Kn - kv[v], a0v[v]) : 0.f;
            }
            st4(RR + idx, ro[0], ro[1], ro[2], ro[3]);
            st4(AA + idx, ao[0], ao[1], ao[2], ao[3]);
            st4(KK + idx, ko[0], ko[1], ko[2], ko[3]);
        }
    };
    __syncthreads();
#pragma unroll(S <= 2 ? S : 1)                     // S = 4: one copy of each phase (instruction cache)
    for (int j = 1; j <= S; ++j) {
        m_phase(j - 1, kRH - 2 * j + 1, j == S);
        __syncthreads();
        if (j < S) {
            ra_phase(j, kRH - 2 * j);
            __syncthreads();
        }
    }
    // ---- iteration S, lines 5-7 on the interior rows [S, S + TH), cols [4, 67]: one
    //      float4 (4 pixels) per thread, 128-bit SMEM reads and global stores -------------
    for (int e = threadIdx.x; e < kTH * (kTW / 4); e += NT) {
        const int rr = e >> 4, r = S + rr, c = kLW + 4 * (e & 15);
        const int gi = gi0 + c, gj = gj0 + r;
        if (EDGE && gj >= ny) continue;
        const int idx = r * kRW + c;
        const float4 R14 = ld4(RR + idx);
        const float4 A14 = ld4(AA + idx);
        const float4 F4 = ld4(F + idx);
        const float4 K4 = ld4(KK + idx);
        const float4 MXn = ld4(MX + idx);
        const float4 MYn = ld4(MY + idx);
        const float4 MYnu = ld4(MY + idx - kRW);
        const float mxnl = MX[idx - 1];
        const float r1v[4] = {R14.x, R14.y, R14.z, R14.w}, a1v[4] = {A14.x, A14.y, A14.z, A14.w};
        const float fv[4] = {F4.x, F4.y, F4.z, F4.w}, kv[4] = {K4.x, K4.y, K4.z, K4.w};
        const float mxn[4] = {MXn.x, MXn.y, MXn.z, MXn.w}, myn[4] = {MYn.x, MYn.y, MYn.z, MYn.w};
        const float mynu[4] = {MYnu.x, MYnu.y, MYnu.z, MYnu.w};
        float rn[4], an[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            rn[v] = r_update(fmaf(t1, a1v[v], r1v[v]), RM, at1, A.r_scale);
            const float divn = (mxn[v] - (v ? mxn[v - 1] : mxnl)) + (myn[v] - mynu[v]);
            const float Kn = divn - rn[v] - fv[v];
            an[v] = fmaf(t2, 2.f * Kn - kv[v], a1v[v]);
            if constexpr (RED) {
                if (!EDGE || gi + v < nx) {
                    const float dr = rn[v] - r1v[v];
                    s_tr += sqrtf(mxn[v] * mxn[v] + myn[v] * myn[v]);
                    s_gr += pw(rn[v], RM);
                    s_k2 += Kn * Kn;
                    s_dz += dr * dr;
                    s_ub += pw(divn - fv[v], RM);
                }
            }
        }
        const size_t g = po + (size_t)gj * nx + gi;
        if (A.vec && (!EDGE || gi + 3 < nx)) {
            *reinterpret_cast<float4*>(A.mx_out + g) = MXn;
            *reinterpret_cast<float4*>(A.my_out + g) = MYn;
            *reinterpret_cast<float4*>(A.r_out + g) = make_float4(rn[0], rn[1], rn[2], rn[3]);
            *reinterpret_cast<float4*>(A.a_out + g) = make_float4(an[0], an[1], an[2], an[3]);
        } else {
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (gi + v < nx) {
                    A.mx_out[g + v] = mxn[v];
                    A.my_out[g + v] = myn[v];
                    A.r_out[g + v] = rn[v];
                    A.a_out[g + v] = an[v];
                }
        }
    }
    if constexpr (RED) {
        // fixed-order block sums (warp butterfly, then the warp sums in order)
        double v[5] = {s_tr, s_gr, s_k2, s_dz, s_ub};
#pragma unroll
        for (int q = 0; q < 5; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(kFull, v[q], o);
        }
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 5; ++q) red_sh[q * NW + warp] = v[q];
        __syncthreads();
        if (threadIdx.x == 0) {
            const int tiles = A.tiles_x * A.tiles_y;
            double* P = A.partials + ((size_t)pair * tiles + tile) * kRec;
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                double t = 0.0;
                for (int k = 0; k < NW; ++k) t += red_sh[q * NW + k];
                P[q] = t;
            }
            P[5] = 0.0; P[6] = 0.0; P[7] = 0.0;
        }
    }
}

// S fused fixed-marginal iterations of one TW x TH tile (+ S-pixel halo) per CTA.
// RM: residual mode (0: l1 soft threshold, 1: l2 averaging, 2: balanced r = 0; Iter2Args.r_mode).
template <int TH, int S, bool RED, int NT, int RM>
__global__ void __launch_bounds__(NT, NT > kT2Threads ? 1 : TB<TH, S>::minb) k_iter2(const Iter2Args A,
                                                                       const __grid_constant__ Iter2Maps M) {
    constexpr int kTH = TH, kRH = TB<TH, S>::RH;
    extern __shared__ __align__(128) float4 sm4[];
    __shared__ double red_sh[5 * (NT / 32)];
    pdl_wait();
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    const int tiles = A.tiles_x * A.tiles_y;
    const int pair = blockIdx.x / tiles, tile = blockIdx.x - pair * tiles;
    const int tx = tile % A.tiles_x, ty = tile / A.tiles_x;
    const int gi0 = tx * kTW - kLW, gj0 = ty * kTH - S;
    // interior tile: every region pixel in the grid and off the pinned last row/column
    const bool edge = gi0 < 0 || gj0 < 0 || gi0 + kRW > A.nx - 1 || gj0 + kRH > A.ny - 1;
    float* sm = reinterpret_cast<float*>(sm4);
    if (A.tma) {                                     // one thread: 5 TMA tile copies on one mbarrier
        __shared__ alignas(8) unsigned long long tbar;
        constexpr int kRA = TB<TH, S>::RA;
        if (threadIdx.x == 0) {
            mbar_init(&tbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            mbar_expect_tx(&tbar, 5u * kRA * (unsigned)sizeof(float));
#pragma unroll
            for (int q = 0; q < 5; ++q) tma_load_3d(sm + q * kRA, &M.tmap[q], gi0, gj0, pair, &tbar);
        }
        __syncthreads();                             // barrier initialised before anyone waits
        mbar_wait(&tbar, 0);
    }
    if (edge) iter_tile<TH, S, RED, true, NT, RM>(A, sm, red_sh, pair, tile, gi0, gj0);
    else iter_tile<TH, S, RED, false, NT, RM>(A, sm, red_sh, pair, tile, gi0, gj0);
    pdl_trigger();
}

}  // namespace uotk
