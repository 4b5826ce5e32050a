// uot_single.cuh -- k_single: every iteration of a call on ONE small fixed-marginal pair in
// ONE CTA (arXiv 1909.00149, Alg. 1 lines 3, 5-7; rho = inf).  SURVEY 8(d)'s "K2"
// for grids the size of C1 (64 x 64): the whole state lives in registers, one thread per
// quad of four consecutive pixels of a row (nx % 4 == 0, nx/4 * ny <= 1024 threads), and the
// two couplings of an iteration -- div^*(a^k) needs a at (j, i+1), (j+1, i) (P:326 sync
// point #1) and div(M^{k+1}) needs M'_x at (j, i-1), M'_y at (j-1, i) (sync point #2) -- are
// exchanged through shared memory with one __syncthreads each.  The residual reductions of a
// checked iteration (L13) and the device-side stopping test run in the same CTA, so a call of
// n iterations is one launch with no grid-wide synchronisation at all.  Per pixel the
// arithmetic is k_iter's (same order; K^k carried instead of recomputed).
// Included by uot_api.cu after the report-slot enum (GL_*).
#pragma once
#include <type_traits>
#include "uot_wave_pk.cuh"

namespace uotk {

constexpr int kSingleThreads = 1024;
// block size: V = 8 pixels per thread when nx % 8 == 0 (fewer, busier threads), else 4

struct SingleArgs {
    int nx, ny;                          // nx % V == 0, (nx / V) * ny <= kSingleThreads
    const float* f;                      // [N] x_{t+1} - x_t
    const float* mx_in; const float* my_in; const float* a_in;   // iterate slot0
    float* mxb[2]; float* myb[2]; float* ab[2];                   // both ping-pong slots
    float* r;                            // in place
    int slot0;
    float tau1, tau2, atau1, r_scale;
    int n_iters, red_every, red_last;
    long long iter0;
    double* pair_out;                    // [kRec] this pair's row of the last reduction
    double* glob;                        // report / stop slots (GL_*)
    int* stop;                           // non-null: armed stop (exit once set)
    double tol, tau1d;
};

// V consecutive pixels of a row per thread (4 or 8: nx % V == 0, nx/V * ny <= 1024 threads);
// RD: the iteration also reduces (only checked iterations take that code).
template <int V>
__device__ __forceinline__ void ld4v(float (&d)[V], const float* p) {
#pragma unroll
    for (int u = 0; u < V; u += 4) {
        const float4 q = *reinterpret_cast<const float4*>(p + u);
        d[u] = q.x; d[u + 1] = q.y; d[u + 2] = q.z; d[u + 3] = q.w;
    }
}
template <int V>
__device__ __forceinline__ void st4v(float* p, const float (&d)[V]) {
#pragma unroll
    for (int u = 0; u < V; u += 4) *reinterpret_cast<float4*>(p + u) = make_float4(d[u], d[u + 1], d[u + 2], d[u + 3]);
}

// PK: the pointwise arithmetic as packed fp32x2 (FFMA2 / FADD2 / FMUL2, uot_wave_pk.cuh: same
// values as the scalar form; the two horizontal differences stay scalar).
template <int RM, int V, bool PK = true>
__global__ void __launch_bounds__(kSingleThreads * 4 / V, 1) k_single(const SingleArgs A) {
    __shared__ __align__(16) float As[kSingleThreads * 4];      // a^k, [ny][nx]
    __shared__ __align__(16) float Mys[kSingleThreads * 4];     // M'_y, [ny][nx]
    __shared__ float Mxw[kSingleThreads];                        // M'_x of each thread's last column
    __shared__ double red[kSingleThreads / 32][6];
    __shared__ int s_stop;
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    const int nx = A.nx, ny = A.ny, Q = nx / V;
    const int q = threadIdx.x, j = q / Q, iq = q - j * Q, i0 = V * iq;
    const bool act = j < ny;
    const bool lastc = iq == Q - 1;              // holds the pinned column nx - 1 (L3)
    const bool lastr = j == ny - 1;              // the pinned row ny - 1 (L3)
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1, rsc = A.r_scale;
    const int g = j * nx + i0;                   // N <= 8192
    float mx[V], my[V], a[V], r[V], f[V], K[V];
    if (act) {
        ld4v<V>(mx, A.mx_in + g); ld4v<V>(my, A.my_in + g); ld4v<V>(a, A.a_in + g);
        ld4v<V>(r, A.r + g); ld4v<V>(f, A.f + g);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) mx[v] = my[v] = a[v] = r[v] = f[v] = 0.f;
    }
    if (lastc) mx[V - 1] = 0.f;                  // pinned flux components read as 0
    if (lastr)
#pragma unroll
        for (int v = 0; v < V; ++v) my[v] = 0.f;
    // K^k = div M^k - r^k - f from the incoming state (L8)
    Mxw[q] = mx[V - 1];
    if (act) st4v<V>(Mys + g, my);
    if (q == 0) s_stop = 0;
    __syncthreads();
    {
        float mu[V];
        const float ml = (act && iq > 0) ? Mxw[q - 1] : 0.f;
        if (act && j > 0) ld4v<V>(mu, Mys + g - nx);
        else
#pragma unroll
            for (int v = 0; v < V; ++v) mu[v] = 0.f;
#pragma unroll
        for (int v = 0; v < V; ++v) K[v] = ((mx[v] - (v ? mx[v - 1] : ml)) + (my[v] - mu[v])) - r[v] - f[v];
    }
    const float t1xl = lastc ? 0.f : t1;         // gx = 0 on the pinned column (L4)
    const float t1y = lastr ? 0.f : t1;          // gy = 0 on the pinned row
    // One iteration (Alg. 1 lines 3, 5-7); with RD the reductions of a6 too (fixed order).
    // Two barriers: after the a^k exchange and after the M' exchange (the previous iteration's
    // readers of As / Mxw / Mys have passed one of them before the next write).
    auto iteration = [&](auto rd_tag, float* sums) {
        constexpr bool RD = decltype(rd_tag)::value;
        if (act) st4v<V>(As + g, a);
        __syncthreads();
        // line 3: M^{k+1} = shrink(M^k - tau1 div^*(a^k)), a at (j, i+1) and (j+1, i)
        float ad[V];
        const float aR = (act && !lastc) ? As[g + V] : 0.f;
        if (act && !lastr) ld4v<V>(ad, As + g + nx);
        else
#pragma unroll
            for (int v = 0; v < V; ++v) ad[v] = 0.f;
        float nmx[V], nmy[V], nrm[V], rn[V];
        if constexpr (PK && !RD) {
            const float2 nt1 = pk_dup(-t1), nt1y2 = pk_dup(-t1y), one = pk_dup(1.f), tt1 = pk_dup(t1);
#pragma unroll
            for (int v = 0; v < V; v += 2) {
                const float2 gx = make_float2(a[v] - a[v + 1], a[v + 1] - (v + 2 < V ? a[v + 2] : aR));
                const float2 av = make_float2(a[v], a[v + 1]);
                const float2 gy = pk_sub(av, make_float2(ad[v], ad[v + 1]));
                const float2 qx = pk_fma(v + 2 < V ? nt1 : make_float2(-t1, -t1xl), gx, make_float2(mx[v], mx[v + 1]));
                const float2 qy = pk_fma(nt1y2, gy, make_float2(my[v], my[v + 1]));
                const float2 n2 = pk_fma(qy, qy, pk_mul(qx, qx));
                float2 sf = pk_fma(nt1, make_float2(rsqrt_ftz(n2.x), rsqrt_ftz(n2.y)), one);
                sf = make_float2(fmaxf(sf.x, 0.f), fmaxf(sf.y, 0.f));
                const float2 m1 = pk_mul(sf, qx), m2 = pk_mul(sf, qy);
                nmx[v] = m1.x; nmx[v + 1] = m1.y; nmy[v] = m2.x; nmy[v + 1] = m2.y;
                const float2 q5 = pk_fma(tt1, av, make_float2(r[v], r[v + 1]));
                float2 r5;
                if constexpr (RM == 0) r5 = pk_sub(q5, make_float2(fminf(fmaxf(q5.x, -at1), at1), fminf(fmaxf(q5.y, -at1), at1)));
                else if constexpr (RM == 1) r5 = pk_mul(q5, pk_dup(rsc));
                else r5 = make_float2(0.f, 0.f);
                rn[v] = r5.x; rn[v + 1] = r5.y;
            }
        } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const float gx = a[v] - (v < V - 1 ? a[v + 1] : aR);
            const float gy = a[v] - ad[v];
            const float qx = __fmaf_rn(-(v == V - 1 ? t1xl : t1), gx, mx[v]);
            const float qy = __fmaf_rn(-t1y, gy, my[v]);
            const float n2 = norm2(qx, qy);
            const float inv = rsqrt_ftz(n2);
            const float sf = shrink_factor(n2, inv, t1);
            nmx[v] = sf * qx;
            nmy[v] = sf * qy;
            if constexpr (RD) nrm[v] = fmaxf(fmaf(n2, fminf(inv, 1e30f), -t1), 0.f);    // |M^{k+1}|
            // line 5: r^{k+1} = shrink_{alpha tau1}(r^k + tau1 a^k) (p = 2: averaging, L24)
            rn[v] = r_update(fmaf(t1, a[v], r[v]), RM, at1, rsc);
        }
        }
        Mxw[q] = nmx[V - 1];
        if (act) st4v<V>(Mys + g, nmy);
        __syncthreads();
        // lines 6-7: K^{k+1} = div M^{k+1} - r^{k+1} - f, a^{k+1} = a^k + tau2 (2K^{k+1} - K^k)
        float mu[V];
        const float ml = (act && iq > 0) ? Mxw[q - 1] : 0.f;
        if (act && j > 0) ld4v<V>(mu, Mys + g - nx);
        else
#pragma unroll
            for (int v = 0; v < V; ++v) mu[v] = 0.f;
        if constexpr (PK && !RD) {
            const float2 tt2 = pk_dup(t2), m2 = pk_dup(-2.f);
#pragma unroll
            for (int v = 0; v < V; v += 2) {
                const float2 dmx = make_float2(nmx[v] - (v ? nmx[v - 1] : ml), nmx[v + 1] - nmx[v]);
                const float2 divn = pk_add(dmx, pk_sub(make_float2(nmy[v], nmy[v + 1]), make_float2(mu[v], mu[v + 1])));
                // -K^{k+1} = (r - div M) + f (exact negation); a += tau2 (2K^{k+1} - K^k)
                const float2 nk = pk_add(pk_sub(make_float2(rn[v], rn[v + 1]), divn), make_float2(f[v], f[v + 1]));
                const float2 an = pk_fma(tt2, pk_fma(m2, nk, make_float2(-K[v], -K[v + 1])), make_float2(a[v], a[v + 1]));
                mx[v] = nmx[v]; mx[v + 1] = nmx[v + 1]; my[v] = nmy[v]; my[v + 1] = nmy[v + 1];
                r[v] = rn[v]; r[v + 1] = rn[v + 1]; a[v] = an.x; a[v + 1] = an.y;
                K[v] = -nk.x; K[v + 1] = -nk.y;
            }
        } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const float divn = (nmx[v] - (v ? nmx[v - 1] : ml)) + (nmy[v] - mu[v]);
            const float kn = divn - rn[v] - f[v];
            const float an = fmaf(t2, fmaf(2.f, kn, -K[v]), a[v]);
            if constexpr (RD) {
                const float w = act ? 1.f : 0.f;
                const float dmx = nmx[v] - mx[v], dmy = nmy[v] - my[v], dr = rn[v] - r[v];
                sums[0] = fmaf(w, nrm[v], sums[0]);
                sums[1] = fmaf(w, pw(rn[v], RM), sums[1]);
                sums[2] = fmaf(w * kn, kn, sums[2]);
                sums[3] = fmaf(w, dmx * dmx + dmy * dmy + dr * dr, sums[3]);
                sums[4] = fmaf(w, pw(divn - f[v], RM), sums[4]);
            }
            mx[v] = nmx[v]; my[v] = nmy[v]; r[v] = rn[v]; a[v] = an; K[v] = kn;
        }
        }
    };
    int done = 0;
    int to_red = A.red_every > 0 ? A.red_every : 0x7fffffff;      // iterations to the next checked one
    for (int k = 0; k < A.n_iters; ++k) {
        const bool rd = (A.red_last && k == A.n_iters - 1) || --to_red == 0;
        if (to_red == 0) to_red = A.red_every;
        done = k + 1;
        if (!rd) {
            iteration(std::false_type{}, nullptr);
            continue;
        }
        float sums[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
        iteration(std::true_type{}, sums);
        // fixed-order block sums (fp64), report + stop test (L13)
        double v[5];
        const int lane = q & 31, w = q >> 5;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            v[c] = sums[c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(kFull, v[c], o);
        }
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < 5; ++c) red[w][c] = v[c];
        __syncthreads();
        if (q < 5) {                              // field q summed over the warps in fixed order
            double t = 0.0;
            for (int w2 = 0; w2 < (int)(blockDim.x / 32); ++w2) t += red[w2][q];
            red[0][q] = t;
        }
        __syncwarp();
        if (q == 0) {
            double tot[5];
#pragma unroll
            for (int c = 0; c < 5; ++c) tot[c] = red[0][c];
            bool nonf = false;
            double* G = A.glob;
            for (int c = 0; c < 5; ++c) {
                A.pair_out[c] = tot[c];
                G[c] = tot[c];
                nonf |= !isfinite(tot[c]);
            }
            A.pair_out[5] = 0.0; A.pair_out[6] = 0.0; A.pair_out[7] = 0.0;
            G[GL_PX] = 0.0;                                        // fixed marginals
            const double it = (double)(A.iter0 + done);
            G[GL_LASTRED] = it;
            int st = 0;
            if (nonf) {
                G[GL_NONF] = 1.0;
                st = 1;
            } else if (A.tol > 0.0 && A.stop != nullptr) {
                const double scale = A.tol * fmax(sqrt(G[GL_FSQ]), 1e-30);
                if (sqrt(tot[2]) <= scale && sqrt(tot[3]) / A.tau1d <= scale) {
                    G[GL_CONV] = it;
                    st = 1;
                }
            }
            if (st && A.stop != nullptr) *A.stop = 1;
            s_stop = st && A.stop != nullptr;
        }
        __syncthreads();
        if (s_stop) break;
    }
    // iterate iter0 + done -> slot slot0 ^ (done & 1) (the host's persistent-launch bookkeeping)
    if (act) {
        const int o = A.slot0 ^ (done & 1);
        st4v<V>(A.mxb[o] + g, mx);
        st4v<V>(A.myb[o] + g, my);
        st4v<V>(A.ab[o] + g, a);
        st4v<V>(A.r + g, r);
    }
}

}  // namespace uotk
