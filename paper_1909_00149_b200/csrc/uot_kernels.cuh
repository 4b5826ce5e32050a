// uot_kernels.cuh -- sm_100a kernels of the fused Algorithm-1 iteration
// (arXiv 1909.00149).  Readings "Lnn" are DESIGN.md's.
//
// Design:
//  * One WARP marches down a vertical strip of 32*V pixels (V = 4: one float4
//    per lane) over a segment of H rows of one pair.  Per row it streams the
//    row's Mx, My, r, f and the NEXT row of a (a of the current row is kept
//    from the previous step), so every plane is read once from HBM:
//    20 B read + 16 B written per pixel-iteration (fixed marginals).
//  * div^*(a) (sync point #1 of P:326) needs a at (j, i+1) and (j+1, i):
//    the +i neighbour comes from the next lane by shuffle (lane 31: one halo
//    load), the +j neighbour is the prefetched next row.
//  * div(M^{k+1}) (sync point #2) needs M'x at (j, i-1) and M'y at (j-1, i):
//    M'x(j, i-1) comes from the previous lane by shuffle (lane 0 RECOMPUTES
//    the shrink of its left halo pixel), M'y(j-1, i) is carried from the
//    previous row (the segment's first row recomputes row j0-1: prologue).
//    Halo recomputation replaces both grid-wide synchronisations; a, M are
//    ping-ponged so the halo reads see iteration-k values.
//  * K^k = div(M^k) - r^k - f is recomputed from the incoming state, never
//    stored (L8).  r is updated in place (its update is pointwise).
//  * Optional fused reductions (transport, growth, ||K||^2, ||dz||^2,
//    ||div M - f||_1) -> fp32 per lane, fp64 warp butterfly -> one record per
//    warp; k_pair_reduce sums records in fixed order (deterministic).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace uotk {

constexpr int kWarps = 4;          // warps (work items) per CTA in k_iter
#ifndef UOT_PROX_MIN_BLOCKS
#define UOT_PROX_MIN_BLOCKS 4
#endif
constexpr int kMinBlocksProx = UOT_PROX_MIN_BLOCKS;   // prox/DF: cap registers for 4 CTAs (16 warps) per SM
constexpr int kRec = 8;            // doubles per partial record
constexpr unsigned kFull = 0xffffffffu;

struct IterArgs {
    int nx, ny;
    int strips, segs, H, items;
    int G, T, P;                      // pairs in context, frames / pairs per chain
    int sel, Gsel;                    // pair selection (UOT_PART_*) and number of selected pairs
    long long N;                      // nx*ny
    const float* f;                   // [G][N]            (fixed mode)
    const float* mx_in;               // [G][N] iteration k
    const float* my_in;
    const float* a_in;
    float* mx_out;                    // [G][N] iteration k+1
    float* my_out;
    float* a_out;
    float* r;                         // [G][N] in place
    float tau1, tau2, atau1;          // atau1 = alpha * tau1 (+inf when balanced)
    int r_mode;                       // 0: l1 soft threshold, 1: l2 averaging (p = 2), 2: balanced (r = 0)
    float r_scale;                    // 1/(1 + 2 alpha tau1) for r_mode 1
    int fix_first;                    // prox: frame 0 of each chain is constant
    // prox mode
    const float* x_in;                // [B][T][N] iteration k
    float* x_out;                     // [B][T][N] iteration k+1
    const float* p;                   // [B][T][N] prox centres (= frames)
    const float* a_prev_halo;         // [B][N] or nullptr
    const float* a_next_halo;         // [B][N] or nullptr
    float c1, c2, c3;                 // rho tau1/(1+rho tau1), 1/(1+rho tau1), tau1/(1+rho tau1)
    double* partials;                 // [items][kRec] when reducing
    const int* stop;                  // device stop flag or nullptr
    // UOT-DF ADMM (MODE 2): ADMM state in place, inner prox frames = (s0, z) in x_in/x_out
    const float* y;                   // [B][N] measurements (Phi = I)
    float* xa;                        // [B][N] ADMM x
    float* aa;                        // [B][N] ADMM scaled dual a
    float* ba;                        // [B][N] ADMM scaled dual b
    float* s_out;                     // [B][N] s^{k+1} (written on reducing iterations)
    float rho_admm, inv1prho;         // rho, 1/(1+rho)
};

template <int V>
__device__ __forceinline__ void ld_ro(float (&d)[V], const float* p) {
    if constexpr (V == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        d[0] = t.x; d[1] = t.y; d[2] = t.z; d[3] = t.w;
    } else if constexpr (V == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        d[0] = t.x; d[1] = t.y;
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) d[v] = __ldg(p + v);
    }
}

template <int V>
__device__ __forceinline__ void ld_rw(float (&d)[V], const float* p) {
    if constexpr (V == 4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        d[0] = t.x; d[1] = t.y; d[2] = t.z; d[3] = t.w;
    } else if constexpr (V == 2) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        d[0] = t.x; d[1] = t.y;
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) d[v] = p[v];
    }
}

template <int V>
__device__ __forceinline__ void st(float* p, const float (&d)[V]) {
    if constexpr (V == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(d[0], d[1], d[2], d[3]);
    } else if constexpr (V == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(d[0], d[1]);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) p[v] = d[v];
    }
}

template <int V>
__device__ __forceinline__ void zero(float (&d)[V]) {
#pragma unroll
    for (int v = 0; v < V; ++v) d[v] = 0.f;
}

// shrink^{l2}_{tau1} factor: max(||q|| - tau1, 0)/||q||, 0 at q = 0 (L7).
// rsqrt(0) = +inf -> 1 - tau1*inf = -inf -> 0.
// |q|^2 of the flux-prox argument in ONE association, fma(qy, qy, qx * qx), in every kernel (the
// packed-fp32x2 wavefronts compute it the same way): paths that must agree bitwise do
__device__ __forceinline__ float norm2(float qx, float qy) { return __fmaf_rn(qy, qy, __fmul_rn(qx, qx)); }

__device__ __forceinline__ float shrink_factor(float n2, float inv, float t1) {
    return fmaxf(fmaf(-t1, inv, 1.f), 0.f);
}

// shrink^{l1}_{s}(q) = sign(q) max(|q| - s, 0)
__device__ __forceinline__ float soft(float q, float s) {
    return copysignf(fmaxf(fabsf(q) - s, 0.f), q);
}

// r-update on q = r + tau1 a: l1 soft threshold, l2 averaging, or 0 (balanced)
__device__ __forceinline__ float r_update(float q, int mode, float at1, float rscale) {
    return mode == 0 ? soft(q, at1) : (mode == 1 ? q * rscale : 0.f);
}

// |v|^p for the growth / repaired-bound reductions
__device__ __forceinline__ float pw(float v, int mode) { return mode == 1 ? v * v : fabsf(v); }

// Programmatic dependent launch: a kernel launched with the PDL attribute may start while
// its predecessor on the stream drains; pdl_wait() blocks until the predecessor has
// completed and its writes are visible (no-op without the attribute).  It precedes every
// global read and write of the kernels that use it.  pdl_trigger() lets the successor
// launch once every CTA has triggered or exited.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Fused iteration.  PROX = false: fixed marginals (rho = inf), K = div M - r - f.
// PROX = true: Alg.1 line 4 as well: frames x are iterates with
// centres p; the warp of pair t also updates x_t (and x_{T-1} for the last
// pair of the chain) from a_{t-1}, a_t, a_{t+1} at the same pixel:
//   x_s' = max(0, c1 p_s + c2 x_s - c3 (A^T a)_s),  (A^T a)_s = a_s - a_{s-1},
//   c1 = rho tau1/(1+rho tau1), c2 = 1/(1+rho tau1), c3 = tau1/(1+rho tau1),
// with a_{-1} / a_{T-1} taken from the shard halos (or 0 at a chain end).
template <int V, bool RED, bool PROX, bool DF = false>
__global__ void __launch_bounds__(kWarps * 32, (PROX || DF) ? kMinBlocksProx : 1)
k_iter(const IterArgs A) {
    pdl_wait();
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    const int lane = threadIdx.x & 31;
    const int item = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (item >= A.items) return;                        // warp-uniform
    int strip, seg, pair;
    if constexpr (PROX) {
        // pair-fastest order: the 4 warps of a CTA are consecutive pairs at the same
        // (segment, strip), so the neighbour-pair planes they share hit in L1/L2
        const int q = item % A.Gsel;
        const int rest = item / A.Gsel;
        if (A.sel == 0) {
            pair = q;
        } else {
            const int nb = A.P >= 2 ? 2 : 1;              // boundary pairs per chain
            if (A.sel == 2) {
                const int b = q / nb, k = q % nb;
                pair = b * A.P + (k == 0 ? 0 : A.P - 1);
            } else {
                const int Pi = A.P - nb, b = q / Pi;
                pair = b * A.P + 1 + q % Pi;
            }
        }
        strip = rest % A.strips;
        seg = rest / A.strips;
    } else {
        strip = item % A.strips;
        const int rest = item / A.strips;
        seg = rest % A.segs;
        pair = rest / A.segs;
    }
    const int rec = (pair * A.segs + seg) * A.strips + strip;   // partial record (pair-contiguous)

    const int nx = A.nx, ny = A.ny;
    const int i0 = strip * 32 * V;
    const int ib = i0 + lane * V;
    const bool act = ib < nx;                           // whole vector inside (nx % V == 0)
    const int iL = i0 - 1, iR = i0 + 32 * V;
    const bool hasL = iL >= 0, hasR = iR < nx;
    const int j0 = seg * A.H;
    const int j1 = min(j0 + A.H, ny);
    const size_t po = (size_t)pair * (size_t)A.N;

    const float* __restrict__ mxi = A.mx_in + po;
    const float* __restrict__ myi = A.my_in + po;
    const float* __restrict__ ai = A.a_in + po;
    float* __restrict__ mxo = A.mx_out + po;
    float* __restrict__ myo = A.my_out + po;
    float* __restrict__ ao = A.a_out + po;
    float* __restrict__ rp = A.r + po;
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1;

    // fixed: f plane; prox: x_t, x_{t+1}, p_t, p_{t+1}, a_{t-1}, a_{t+1} planes, x' outputs
    const float* __restrict__ fp = nullptr;
    const float* __restrict__ x0i = nullptr; const float* __restrict__ x1i = nullptr;
    const float* __restrict__ p0i = nullptr; const float* __restrict__ p1i = nullptr;
    const float* __restrict__ ami = nullptr; const float* __restrict__ api = nullptr;
    float* __restrict__ x0o = nullptr; float* __restrict__ x1o = nullptr;
    bool last_pair = false, own_last = false;
    const float* __restrict__ ypi = nullptr;
    float* __restrict__ xap = nullptr; float* __restrict__ aap = nullptr; float* __restrict__ bap = nullptr;
    float* __restrict__ sop = nullptr;
    if constexpr (DF) {
        // pair g = problem b (T = 2): frame 0 = s0 (constant), frame 1 = z; x_out gets z^{k+1}
        const size_t f0 = (size_t)pair * 2 * (size_t)A.N;
        x0i = A.x_in + f0; x1i = x0i + A.N;
        x1o = A.x_out + f0 + A.N;
        ypi = A.y + po; xap = A.xa + po; aap = A.aa + po; bap = A.ba + po; sop = A.s_out + po;
    } else if constexpr (PROX) {
        const int b = pair / A.P, t = pair % A.P;
        const size_t f0 = ((size_t)b * A.T + t) * (size_t)A.N;
        x0i = A.x_in + f0; x1i = x0i + A.N;
        p0i = A.p + f0; p1i = p0i + A.N;
        x0o = A.x_out + f0;
        last_pair = (t == A.P - 1);
        // the shard's last frame is the next rank's first frame when a next halo exists: both
        // ranks update it (bit-identically), only the owner (the next rank) reduces its terms
        own_last = last_pair && A.a_next_halo == nullptr;
        if (last_pair) x1o = x0o + A.N;
        ami = (t > 0) ? A.a_in + po - A.N : (A.a_prev_halo ? A.a_prev_halo + (size_t)b * A.N : nullptr);
        api = (t < A.P - 1) ? A.a_in + po + A.N : (A.a_next_halo ? A.a_next_halo + (size_t)b * A.N : nullptr);
    } else {
        fp = A.f + po;
    }
    const float c1 = A.c1, c2 = A.c2, c3 = A.c3;

    bool colx[V];                                       // Mx exists / gx != 0: i < nx-1 (L3, L4)
#pragma unroll
    for (int v = 0; v < V; ++v) colx[v] = (ib + v) < nx - 1;

    // ---- prologue: a at row j0, and M'y / My at row j0-1 ------------------------------
    float a_c[V], myp_n[V], myp_o[V];
    float aL_c = 0.f, aR_c = 0.f;
    const size_t r0 = (size_t)j0 * nx;
    if (act) ld_ro<V>(a_c, ai + r0 + ib); else zero<V>(a_c);
    if (lane == 0 && hasL) aL_c = __ldg(ai + r0 + iL);
    if (lane == 31 && hasR) aR_c = __ldg(ai + r0 + iR);
    if (j0 > 0) {
        const size_t rp0 = (size_t)(j0 - 1) * nx;
        float a_p[V], mxp[V], myp[V];
        float aR_p = 0.f;
        if (act) { ld_ro<V>(a_p, ai + rp0 + ib); ld_ro<V>(mxp, mxi + rp0 + ib); ld_ro<V>(myp, myi + rp0 + ib); }
        else { zero<V>(a_p); zero<V>(mxp); zero<V>(myp); }
        if (lane == 31 && hasR) aR_p = __ldg(ai + rp0 + iR);
        const float nb = __shfl_down_sync(kFull, a_p[0], 1);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const float ar = (v < V - 1) ? a_p[(v + 1) % V] : (lane == 31 ? aR_p : nb);
            const float gx = colx[v] ? a_p[v] - ar : 0.f;
            const float gy = a_p[v] - a_c[v];            // row j0-1 < ny-1
            const float qx = __fmaf_rn(-t1, gx, (colx[v] ? mxp[v] : 0.f));
            const float qy = __fmaf_rn(-t1, gy, myp[v]);
            const float n2 = norm2(qx, qy);
            const float s = shrink_factor(n2, rsqrtf(n2), t1);
            myp_n[v] = s * qy;
            myp_o[v] = myp[v];
        }
    } else {
        zero<V>(myp_n); zero<V>(myp_o);
    }

    // ---- software-pipelined row loop ---------------------------------------------------
    float n_a[V], n_mx[V], n_my[V], n_r[V], n_f[V];
    float n_x0[V], n_x1[V], n_p0[V], n_p1[V], n_am[V], n_ap[V];
    float n_aL = 0.f, n_aR = 0.f, n_mxL = 0.f, n_myL = 0.f;
    auto fetch = [&](int j) {
        const size_t rj = (size_t)j * nx;
        const bool has_next = (j + 1) < ny;
        if (act) {
            ld_ro<V>(n_mx, mxi + rj + ib);
            ld_ro<V>(n_my, myi + rj + ib);
            ld_rw<V>(n_r, rp + rj + ib);
            if constexpr (DF) {
                ld_ro<V>(n_x0, x0i + rj + ib);            // s0
                ld_ro<V>(n_x1, x1i + rj + ib);            // z
                ld_ro<V>(n_p1, ypi + rj + ib);            // y
                ld_rw<V>(n_p0, xap + rj + ib);            // ADMM x
                ld_rw<V>(n_am, aap + rj + ib);            // ADMM a
                ld_rw<V>(n_ap, bap + rj + ib);            // ADMM b
            } else if constexpr (PROX) {
                ld_ro<V>(n_x0, x0i + rj + ib);
                ld_ro<V>(n_x1, x1i + rj + ib);
                ld_ro<V>(n_p0, p0i + rj + ib);
                ld_ro<V>(n_p1, p1i + rj + ib);
                if (ami) ld_ro<V>(n_am, ami + rj + ib); else zero<V>(n_am);
                if (api) ld_ro<V>(n_ap, api + rj + ib); else zero<V>(n_ap);
            } else {
                ld_ro<V>(n_f, fp + rj + ib);
            }
            if (has_next) ld_ro<V>(n_a, ai + rj + nx + ib); else zero<V>(n_a);
        } else {
            zero<V>(n_mx); zero<V>(n_my); zero<V>(n_r); zero<V>(n_a);
            if constexpr (PROX || DF) { zero<V>(n_x0); zero<V>(n_x1); zero<V>(n_p0); zero<V>(n_p1); zero<V>(n_am); zero<V>(n_ap); }
            else zero<V>(n_f);
        }
        if (lane == 0 && hasL) {
            n_mxL = __ldg(mxi + rj + iL);
            n_myL = __ldg(myi + rj + iL);
            n_aL = has_next ? __ldg(ai + rj + nx + iL) : 0.f;
        }
        if (lane == 31 && hasR) n_aR = has_next ? __ldg(ai + rj + nx + iR) : 0.f;
    };
    fetch(j0);

    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f, s_px = 0.f;

    for (int j = j0; j < j1; ++j) {
        float c_a[V], c_mx[V], c_my[V], c_r[V], c_f[V];
        float c_x0[V], c_x1[V], c_p0[V], c_p1[V], c_am[V], c_ap[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            c_a[v] = n_a[v]; c_mx[v] = n_mx[v]; c_my[v] = n_my[v]; c_r[v] = n_r[v];
            if constexpr (PROX || DF) {
                c_x0[v] = n_x0[v]; c_x1[v] = n_x1[v]; c_p0[v] = n_p0[v]; c_p1[v] = n_p1[v];
                c_am[v] = n_am[v]; c_ap[v] = n_ap[v];
            } else {
                c_f[v] = n_f[v];
            }
        }
        const float c_aL = n_aL, c_aR = n_aR, c_mxL = n_mxL, c_myL = n_myL;
        if (j + 1 < j1) fetch(j + 1);
        const bool lastrow = (j == ny - 1);

        // Alg.1 line 3: m <- shrink_{tau1}(m - tau1 div^*(a))
        const float nb = __shfl_down_sync(kFull, a_c[0], 1);
        float mxn[V], myn[V], mxk[V], myk[V], rn[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const float ar = (v < V - 1) ? a_c[(v + 1) % V] : (lane == 31 ? aR_c : nb);
            const float gx = colx[v] ? a_c[v] - ar : 0.f;
            const float gy = lastrow ? 0.f : a_c[v] - c_a[v];
            mxk[v] = colx[v] ? c_mx[v] : 0.f;           // pinned components read as 0 (L3)
            myk[v] = lastrow ? 0.f : c_my[v];
            const float qx = __fmaf_rn(-t1, gx, mxk[v]);
            const float qy = __fmaf_rn(-t1, gy, myk[v]);
            const float n2 = norm2(qx, qy);
            const float inv = rsqrtf(n2);
            const float s = shrink_factor(n2, inv, t1);
            mxn[v] = s * qx;
            myn[v] = s * qy;
            // Alg.1 line 5: r <- shrink^{l1}_{alpha tau1}(r + tau1 a); p = 2 averaging
            // update; balanced: r dropped
            rn[v] = r_update(fmaf(t1, a_c[v], c_r[v]), A.r_mode, at1, A.r_scale);
            if constexpr (RED) s_tr += (n2 > 0.f) ? fmaxf(n2 * inv - t1, 0.f) : 0.f;
        }
        // Alg.1 line 4 (prox): x_t and x_{t+1} from the iteration-k duals
        float x0n[V], x1n[V], fk[V], fn[V];
        float sn[V], xan[V], aan[V], ban[V];
        const bool fix0 = PROX && A.fix_first && (pair % A.P == 0);     // constant first argument
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if constexpr (DF) {
                // Alg.2 lines 4-5 (L23: s-update from the printed augmented Lagrangian; Phi = I)
                sn[v] = fmaxf(0.5f * (c_p0[v] + c_am[v] + c_x1[v] + c_ap[v]), 0.f);
                xan[v] = (c_p1[v] + A.rho_admm * (sn[v] - c_am[v])) * A.inv1prho;
                // Alg.2 line 6: one warm-started Alg.1 iteration of prox_{kappa/rho V_{s0}}(s - b):
                // z' = Pi_+(c1 v + c2 z + c3 a_in) (A := I with K = div M - r - z + s0)
                x1n[v] = fmaxf(fmaf(c1, sn[v] - c_ap[v], fmaf(c2, c_x1[v], c3 * a_c[v])), 0.f);
                x0n[v] = c_x0[v];
                fk[v] = c_x1[v] - c_x0[v];
                fn[v] = x1n[v] - c_x0[v];
                // lines 7-8
                aan[v] = c_am[v] + xan[v] - sn[v];
                ban[v] = c_ap[v] + x1n[v] - sn[v];
            } else if constexpr (PROX) {
                x0n[v] = fix0 ? c_x0[v] : fmaxf(fmaf(c1, c_p0[v], fmaf(c2, c_x0[v], -c3 * (a_c[v] - c_am[v]))), 0.f);
                x1n[v] = fmaxf(fmaf(c1, c_p1[v], fmaf(c2, c_x1[v], -c3 * (c_ap[v] - a_c[v]))), 0.f);
                fk[v] = c_x1[v] - c_x0[v];
                fn[v] = x1n[v] - x0n[v];
            } else {
                fk[v] = c_f[v];
                fn[v] = c_f[v];
            }
        }
        // M'x and Mx at (j, i-1): previous lane, or recomputed halo for lane 0
        const float upn = __shfl_up_sync(kFull, mxn[V - 1], 1);
        const float upk = __shfl_up_sync(kFull, mxk[V - 1], 1);
        float lmn0 = upn, lmk0 = upk;
        if (lane == 0) {
            if (hasL) {
                const float gxL = aL_c - a_c[0];
                const float gyL = lastrow ? 0.f : aL_c - c_aL;
                const float kyL = lastrow ? 0.f : c_myL;
                const float qx = __fmaf_rn(-t1, gxL, c_mxL);
                const float qy = __fmaf_rn(-t1, gyL, kyL);
                const float n2 = norm2(qx, qy);
                lmn0 = shrink_factor(n2, rsqrtf(n2), t1) * qx;
                lmk0 = c_mxL;
            } else {
                lmn0 = 0.f; lmk0 = 0.f;
            }
        }
        // Alg.1 lines 6-7: b = 2K^{k+1} - K^k, a <- a + tau2 b
        float an[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const float lmn = v ? mxn[(v + V - 1) % V] : lmn0;
            const float lmk = v ? mxk[(v + V - 1) % V] : lmk0;
            const float divn = (mxn[v] - lmn) + (myn[v] - myp_n[v]);
            const float divk = (mxk[v] - lmk) + (myk[v] - myp_o[v]);
            const float Kn = divn - rn[v] - fn[v];
            const float Kk = divk - c_r[v] - fk[v];
            an[v] = fmaf(t2, 2.f * Kn - Kk, a_c[v]);
            if constexpr (RED && DF) {
                // ADMM residuals and the data term
                const float p0 = xan[v] - sn[v], p1 = x1n[v] - sn[v];
                const float d0 = xan[v] - c_p0[v], d1 = x1n[v] - c_x1[v];
                const float e = c_p1[v] - sn[v];
                s_gr += pw(rn[v], A.r_mode);
                s_k2 += Kn * Kn;
                s_dz += p0 * p0 + p1 * p1;
                s_ub += d0 * d0 + d1 * d1;
                s_px += 0.5f * e * e;
            } else if constexpr (RED) {
                const float dmx = mxn[v] - mxk[v], dmy = myn[v] - myk[v], dr = rn[v] - c_r[v];
                s_gr += pw(rn[v], A.r_mode);
                s_k2 += Kn * Kn;
                s_dz += dmx * dmx + dmy * dmy + dr * dr;
                s_ub += pw(divn - fn[v], A.r_mode);
                if constexpr (PROX) {
                    const float d0 = x0n[v] - c_x0[v], e0 = x0n[v] - c_p0[v];
                    s_dz += d0 * d0;
                    s_px += e0 * e0;
                    if (own_last) {
                        const float d1 = x1n[v] - c_x1[v], e1 = x1n[v] - c_p1[v];
                        s_dz += d1 * d1;
                        s_px += e1 * e1;
                    }
                }
            }
        }
        if (act) {
            const size_t rj = (size_t)j * nx + ib;
            st<V>(mxo + rj, mxn);
            st<V>(myo + rj, myn);
            st<V>(rp + rj, rn);
            st<V>(ao + rj, an);
            if constexpr (DF) {
                st<V>(x1o + rj, x1n);
                st<V>(xap + rj, xan);
                st<V>(aap + rj, aan);
                st<V>(bap + rj, ban);
                if constexpr (RED) st<V>(sop + rj, sn);
            } else if constexpr (PROX) {
                st<V>(x0o + rj, x0n);
                if (last_pair) st<V>(x1o + rj, x1n);
            }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) { myp_n[v] = myn[v]; myp_o[v] = myk[v]; a_c[v] = c_a[v]; }
        aL_c = c_aL;
        aR_c = c_aR;
    }

    if constexpr (RED) {
        double d0 = s_tr, d1 = s_gr, d2 = s_k2, d3 = s_dz, d4 = s_ub, d5 = s_px;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            d0 += __shfl_xor_sync(kFull, d0, o);
            d1 += __shfl_xor_sync(kFull, d1, o);
            d2 += __shfl_xor_sync(kFull, d2, o);
            d3 += __shfl_xor_sync(kFull, d3, o);
            d4 += __shfl_xor_sync(kFull, d4, o);
            if constexpr (PROX || DF) d5 += __shfl_xor_sync(kFull, d5, o);
        }
        if (lane == 0) {
            double* P = A.partials + (size_t)rec * kRec;
            P[0] = d0; P[1] = d1; P[2] = d2; P[3] = d3; P[4] = d4; P[5] = (PROX || DF) ? d5 : 0.0; P[6] = 0.0; P[7] = 0.0;
        }
    }
    pdl_trigger();
}

// ------------------------------------------------------------------------------------------
// Setup (row a0): f = x_{t+1} - x_t per pair, and per-block partial sums of f^2, |f|.
struct SetupArgs {
    int T, P;                 // frames / pairs per chain
    long long N;
    int bpp;                  // blocks per pair
    const float* frames;      // [B][T][N]
    float* f;                 // [G][N]
    double* partials;         // [G*bpp][kRec]
};

__global__ void __launch_bounds__(256) k_setup_f(const SetupArgs S);

// Objective / certificate of the current state: per block records
// {sum||M||, sum|r|, sum|div M - f|, sum a f, max||div^* a||, max|a|, sum (x-p)^2, 0}.
struct ObjArgs {
    int nx, ny, T, P;
    long long N;
    int bpp;
    const float* x;           // [B][T][N] frames (fixed) or x (prox)
    const float* p;           // [B][T][N] prox centres (prox) or nullptr
    const float* mx; const float* my; const float* r; const float* a;
    double* partials;
    int p2;                   // p = 2 sums (r^2, (div M - f)^2)
    int next_owns_last;       // shard with a next halo: its last frame is reduced by the next rank
};
__global__ void __launch_bounds__(256) k_objective(const ObjArgs O);

// Deterministic per-pair reduction of records (sum; bit k of max_mask -> max),
// then the last block reduces the pairs in order into glob[0..7] and, for
// iteration records, evaluates the stopping test (L13).
struct ReduceArgs {
    const double* partials;
    int recs_per_pair;
    int G;
    double* pair_out;         // [G][kRec]
    double* glob;             // global accumulators (see uot_api.cu)
    int* counter;
    int* stop;                // nullable
    unsigned max_mask;
    int is_iteration;         // 1: glob[0..7] iteration sums + stop test
    int is_setup;             // 1: write glob f-norm slots
    long long iteration;      // iteration index just completed
    double tol;               // <= 0: no stop test
    double tau1;
    int stop_kind;            // 0: L13 relative (K, dz); 1: ADMM absolute: sqrt(f3) < tol, rho sqrt(f4) < tol
    double rho_admm;
};
__global__ void __launch_bounds__(256) k_pair_reduce(const ReduceArgs R);

}  // namespace uotk
