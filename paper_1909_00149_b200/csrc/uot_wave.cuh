// uot_wave.cuh -- S fixed-marginal Algorithm-1 iterations per HBM pass as a register
// wavefront (arXiv 1909.00149, Alg. 1 lines 3, 5-7; rho = inf).
//
// One warp owns a strip of 128 columns (32 lanes x one float4 quad) and marches down H + 2S
// rows of one pair.  At step t it receives row t of the iterate (M, r, a, f; cp.async into a
// per-warp SMEM ring of 8 rows, 7 - S rows ahead) and advances every level j = 1..S by one
// row: level j updates row t - j from level j-1's rows t - j (carried in registers) and
// t - j + 1 (just produced), so the S iterations run as a wavefront with no block barrier
// and no SMEM traffic beyond the ring.  Horizontal neighbours (a at i+1 for div^*, M_x at
// i-1 for div) come from the adjacent lane by shuffle; vertical ones are the carried rows.
// Each iteration invalidates one more column at each strip side, so ceil(S/4) lanes per side
// are halo: the warp writes the 120 columns of lanes 1..30 (S <= 4) or the 112 of lanes
// 2..29 (S = 5); the S rows above / below the H output rows are halo likewise (re-read
// from L2 by the neighbours).  K^{j-1} (line 7's previous K) is carried with the level, so
// div M is evaluated once per pixel and iteration.  The arithmetic per pixel is k_iter's,
// in the same order.  HBM traffic: 36 B per pair-pixel per S iterations (+ column and 2S/H
// row halo, mostly from L2: ncu 1.004x algorithmic at S = 5, H = 512).
#pragma once
#include "uot_temporal.cuh"

namespace uotk {

constexpr int kWaveOut = 120;                   // columns written per warp strip (lanes 1..30), S <= 4
// S iterations invalidate S columns at each strip side: ceil(S/4) halo lanes per side
__host__ __device__ constexpr int wave_halo_lanes(int S) { return (S + 3) / 4; }
__host__ __device__ constexpr int wave_out(int S) { return 128 - 8 * wave_halo_lanes(S); }
// Strips of 128 loaded columns start at s * wave_out(S): neighbouring strips overlap by the two
// halos, the first strip starts at column 0 (nothing is unknown left of the grid) and the last
// one reaches the right edge (nothing unknown right of it), so those two need no halo lanes on
// the grid side.  Strips needed for nx columns:
__host__ __device__ constexpr int wave_strips(int nx, int S) {
    return nx <= 128 ? 1 : (nx - 128 + wave_out(S) - 1) / wave_out(S) + 1;
}
constexpr int kWaveRing = 8;                    // rows per warp in the SMEM ring
constexpr int kWaveWarps = 1;                   // warps (independent strips) per CTA
template <int S, bool RED> struct WaveCfg {     // warps per SM: registers <= 255 (S >= 4; a 168 cap for
    static constexpr int minb = (S >= 4 ? 8 : 10) / kWaveWarps;   // 10 warps / SM spills and is slower) / 204
};
constexpr size_t kWaveSmem = (size_t)kWaveWarps * kWaveRing * 5 * 32 * sizeof(float4);   // 20 KB per warp

struct WaveArgs {
    int nx, ny;                 // nx % 4 == 0, 16-byte aligned planes
    int strips, segs, H;        // units per pair: strips x segs (segment = H output rows)
    int G;
    long long N;
    const float* f;
    const float* mx_in; const float* my_in; const float* a_in; const float* r_in;
    float* mx_out; float* my_out; float* a_out; float* r_out;
    float tau1, tau2, atau1, r_scale;
    double* partials;           // [G][strips * segs][kRec] when reducing
    const int* stop;
};

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// rsqrt without the denormal-input rescaling (n2 < 2^-126 flushes to 0 -> +inf -> shrink
// factor 0, the value the unflushed rsqrt gives through max(1 - tau1 * huge, 0) anyway)
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float f4c(const float4& q, int v) { return v == 0 ? q.x : (v == 1 ? q.y : (v == 2 ? q.z : q.w)); }

template <int S, int RM, bool RED>
__global__ void __launch_bounds__(kWaveWarps * 32, WaveCfg<S, RED>::minb) k_wave(const WaveArgs A) {
    static_assert(S >= 1 && S <= 5, "ring of 8 rows: S + prefetch + 1 <= 8");
    constexpr int HL = wave_halo_lanes(S), OUT = wave_out(S);
    constexpr int P = kWaveRing - S - 1;        // rows in flight ahead of the current one
    extern __shared__ __align__(16) float4 wring[];
    pdl_wait();
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int upp = A.strips * A.segs;
    const long long unit = (long long)blockIdx.x * kWaveWarps + w;
    if (unit >= (long long)A.G * upp) return;   // whole warp: no block-level synchronisation below
    const int pair = (int)(unit / upp), u = (int)(unit - (long long)pair * upp);
    const int sy = u / A.strips, sx = u - sy * A.strips;
    const int nx = A.nx, ny = A.ny;
    const int gs = sx * OUT;                                     // first loaded column of the strip
    const int gi = gs + 4 * lane;                                // first column of this lane's quad
    const bool lane_in = gi < nx;                                // whole quad in the grid (nx % 4 == 0)
    const bool last_q = gi + 3 == nx - 1;                        // holds the pinned column nx-1 (L3)
    const bool left_edge = lane == 0 && sx == 0;                 // column -1 is outside: M_x there = 0
    const bool writer = lane_in && (lane >= HL || sx == 0) && (lane <= 31 - HL || gs + 128 >= nx);
    const int y0 = sy * A.H, y1 = min(y0 + A.H, ny);             // output rows [y0, y1)
    const size_t po = (size_t)pair * (size_t)A.N;
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1, rsc = A.r_scale;
    float* const mx_out = A.mx_out; float* const my_out = A.my_out;
    float* const r_out = A.r_out; float* const a_out = A.a_out;
    // Boundary handling without per-pixel masks: r, a, f, M are 0 outside the grid (zero-filled
    // loads) and stay 0 there as long as div^* a is cut at the two places where one side of the
    // difference is in the grid: column -1 / row -1 (outside, next to the grid) and the pinned
    // column nx-1 / row ny-1 (L3).  Scaling tau1 by 0 there keeps those M components 0 exactly
    // (then div M, K, r, a outside are exact zeros).  Column cut: the 4th pixel of the lane
    // holding column -1 or nx-1; row cut: a row-uniform scale.
    const float t1x3 = last_q ? 0.f : t1;
    float4* ring = wring + (size_t)w * (kWaveRing * 5 * 32) + lane;   // [slot][plane][lane]

    auto issue = [&](int t) {                                    // row t -> slot t & 7 (zero outside)
        const bool ok = lane_in && t >= 0 && t < ny;
        const size_t g = ok ? po + (size_t)t * nx + gi : po;
        float4* s = ring + (t & (kWaveRing - 1)) * (5 * 32);
        cp_async16(reinterpret_cast<float*>(s), A.mx_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 32), A.my_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 64), A.r_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 96), A.a_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 128), A.f + g, ok);
        cp_commit();
    };

    const int t0 = y0 - S, t1r = y1 - 1 + S;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    // The first steps' deeper levels read f of rows above t0 that are never loaded: clear the
    // ring so those discarded rows are finite (a NaN there would poison the weight-0 terms of
    // the reductions).  Each lane clears and later reads only its own slots.
#pragma unroll
    for (int q = 0; q < kWaveRing * 5; ++q) ring[q * 32] = z4;
#pragma unroll
    for (int p = 0; p < P; ++p) issue(t0 + p);
    // Level j-1's outputs (M, r, a, K) at one row, in two register sets: a step reads the
    // previous row from one set and writes the current row into the other, and the next
    // step swaps them (two steps per loop trip: no register copies).
    struct Lv { float4 mx, my, r, a, k; };
    Lv SA[S], SB[S];
    float4 upY[S + 1];                            // level j's M_y at its previous row
#pragma unroll
    for (int j = 0; j < S; ++j) { SA[j] = {z4, z4, z4, z4, z4}; SB[j] = SA[j]; }
#pragma unroll
    for (int j = 0; j <= S; ++j) upY[j] = z4;
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f;

    auto step = [&](const int t, Lv (&Pv)[S], Lv (&Cv)[S]) {
        if (t + P <= t1r) issue(t + P);
        else cp_commit();                                        // empty group: uniform wait count
        cp_wait<P>();                                            // row t has landed (own lane's copies)
        const float4* s = ring + (t & (kWaveRing - 1)) * (5 * 32);
        float4 Mx = s[0], My = s[32];
        const float4 R = s[64], F = s[128];
        if (last_q) Mx.w = 0.f;                                  // pinned flux components (L3)
        if (t == ny - 1) My = z4;
        // ---- level 0: K^0 = div M - r - f at row t ----
        const float sh0 = __shfl_up_sync(kFull, Mx.w, 1);   // all lanes shuffle, then select
        const float mxl0 = left_edge ? 0.f : sh0;
        Cv[0].mx = Mx; Cv[0].my = My; Cv[0].r = R; Cv[0].a = s[96];
        Cv[0].k.x = ((Mx.x - mxl0) + (My.x - upY[0].x)) - R.x - F.x;
        Cv[0].k.y = ((Mx.y - Mx.x) + (My.y - upY[0].y)) - R.y - F.y;
        Cv[0].k.z = ((Mx.z - Mx.y) + (My.z - upY[0].z)) - R.z - F.z;
        Cv[0].k.w = ((Mx.w - Mx.z) + (My.w - upY[0].w)) - R.w - F.w;
        upY[0] = My;
#pragma unroll
        for (int j = 1; j <= S; ++j) {
            const int rho = t - j;
            const float4 qmx = Pv[j - 1].mx, qmy = Pv[j - 1].my, qr = Pv[j - 1].r, qa = Pv[j - 1].a, qk = Pv[j - 1].k;
            const float4 cA = Cv[j - 1].a;                       // a^{j-1} at rho + 1
            const float t1y = (rho == -1 || rho == ny - 1) ? 0.f : t1;
            // line 3: M^j(rho) = prox(M^{j-1} - tau1 div^* a^{j-1}); a at (rho, i+1) and (rho+1, i)
            const float a5 = __shfl_down_sync(kFull, qa.x, 1);
            const float av[5] = {qa.x, qa.y, qa.z, qa.w, a5};
            float nmx[4], nmy[4], nrm[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float gx = av[v] - av[v + 1];
                const float gy = av[v] - f4c(cA, v);
                const float qx = __fmaf_rn(-(v == 3 ? t1x3 : t1), gx, f4c(qmx, v));
                const float qy = __fmaf_rn(-t1y, gy, f4c(qmy, v));
                const float n2 = norm2(qx, qy);
                const float inv = rsqrt_ftz(n2);
                const float sf = shrink_factor(n2, inv, t1);
                nmx[v] = sf * qx;
                nmy[v] = sf * qy;
                // |M^j| = max(|q| - tau1, 0) (the l2 shrink); the clamp keeps n2 * inv
                // finite where n2 is 0 or flushed (inv = +inf) -- those give 0
                if (RED && j == S) nrm[v] = fmaxf(fmaf(n2, fminf(inv, 1e30f), -t1), 0.f);
            }
            // lines 5-7: r^j, a^j, K^j at rho from M^j (left neighbour by shuffle, up carried)
            const float shl = __shfl_up_sync(kFull, nmx[3], 1);   // all lanes shuffle, then select
            const float mxl = left_edge ? 0.f : shl;
            const float wr = (writer && rho >= y0 && rho < y1) ? 1.f : 0.f;   // output pixel (reductions)
            const float4 Fr = ring[(rho & (kWaveRing - 1)) * (5 * 32) + 128];
            const float mxv[5] = {mxl, nmx[0], nmx[1], nmx[2], nmx[3]};
            float rn[4], an[4], kn[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                rn[v] = r_update(fmaf(t1, f4c(qa, v), f4c(qr, v)), RM, at1, rsc);
                const float divn = (mxv[v + 1] - mxv[v]) + (nmy[v] - f4c(upY[j], v));
                kn[v] = divn - rn[v] - f4c(Fr, v);
                an[v] = fmaf(t2, fmaf(2.f, kn[v], -f4c(qk, v)), f4c(qa, v));
                if (RED && j == S) {                             // branch-free: weight 0 off the output
                    const float dmx = nmx[v] - f4c(qmx, v), dmy = nmy[v] - f4c(qmy, v), dr = rn[v] - f4c(qr, v);
                    s_tr = fmaf(wr, nrm[v], s_tr);
                    s_gr = fmaf(wr, pw(rn[v], RM), s_gr);
                    s_k2 = fmaf(wr * kn[v], kn[v], s_k2);
                    s_dz = fmaf(wr, dmx * dmx + dmy * dmy + dr * dr, s_dz);
                    s_ub = fmaf(wr, pw(divn - f4c(Fr, v), RM), s_ub);
                }
            }
            upY[j] = make_float4(nmy[0], nmy[1], nmy[2], nmy[3]);
            if (j < S) {
                Cv[j].mx = make_float4(nmx[0], nmx[1], nmx[2], nmx[3]);
                Cv[j].my = upY[j];
                Cv[j].r = make_float4(rn[0], rn[1], rn[2], rn[3]);
                Cv[j].a = make_float4(an[0], an[1], an[2], an[3]);
                Cv[j].k = make_float4(kn[0], kn[1], kn[2], kn[3]);
            } else if (writer && rho >= y0 && rho < y1) {
                const size_t g = po + (size_t)rho * nx + gi;
                *reinterpret_cast<float4*>(mx_out + g) = make_float4(nmx[0], nmx[1], nmx[2], nmx[3]);
                *reinterpret_cast<float4*>(my_out + g) = upY[j];
                *reinterpret_cast<float4*>(r_out + g) = make_float4(rn[0], rn[1], rn[2], rn[3]);
                *reinterpret_cast<float4*>(a_out + g) = make_float4(an[0], an[1], an[2], an[3]);
            }
        }
    };
    int t = t0;
#pragma unroll 1
    for (; t + 1 <= t1r; t += 2) {
        step(t, SA, SB);
        step(t + 1, SB, SA);
    }
    if (t <= t1r) step(t, SA, SB);
    cp_wait<0>();
    pdl_trigger();
    if constexpr (RED) {                                         // fixed-order warp sums -> one record
        double v[5] = {s_tr, s_gr, s_k2, s_dz, s_ub};
#pragma unroll
        for (int q = 0; q < 5; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(kFull, v[q], o);
        }
        if (lane == 0) {
            double* Pp = A.partials + ((size_t)pair * upp + u) * kRec;
#pragma unroll
            for (int q = 0; q < 5; ++q) Pp[q] = v[q];
            Pp[5] = 0.0; Pp[6] = 0.0; Pp[7] = 0.0;
        }
    }
}

// ============================================================================================
// k_wave_df: S UOT-DF ADMM iterations (Algorithm 2 with Phi = I and one warm-started Alg.1
// iteration per ADMM iteration) per HBM pass, as the same register
// wavefront.  Per pixel and iteration (the fused k_iter<DF>'s arithmetic, same order):
//   M' = shrink(M - tau1 div^* a)                               (inner line 3)
//   r' = shrink_{mu tau1}(r + tau1 a)                            (inner line 5)
//   s  = max((x + a_x + z + b) / 2, 0)                           (line 4, L23)
//   x' = (y + rho (s - a_x)) / (1 + rho)                         (line 5)
//   z' = max(c1 (s - b) + c2 z + c3 a, 0)                        (line 6: inner line 4, fixed s0)
//   K' = div M' - r' - (z' - s0),  a' = a + tau2 (2K' - K)       (inner lines 6-7)
//   a_x' = a_x + x' - s,  b' = b + z' - s                        (lines 7-8)
// Everything but M' and div M' is pointwise, so a level carries (M, r, a, K, z, x, a_x, b) of
// its previous row; y and s0 come from a constant-plane ring at the level's row.  All
// pointwise planes are ping-ponged by the host (the strip/segment halos of neighbouring warps
// read this warp's iteration-k values).
struct WaveDfArgs {
    int nx, ny, strips, segs, H, G;
    long long N;
    const float* y; const float* s0;
    const float* mx_in; const float* my_in; const float* a_in; const float* z_in;    // z: [G][2][N] frame 1
    const float* r_in; const float* x_in; const float* ax_in; const float* b_in;
    float* mx_out; float* my_out; float* a_out; float* z_out;
    float* r_out; float* x_out; float* ax_out; float* b_out;
    float* s_out;                   // s of the last level (RED only)
    float tau1, tau2, atau1, r_scale, c1, c2, c3, rho, inv1prho;
    double* partials;               // [G][strips * segs][kRec]
    const int* stop;
};

constexpr int kWaveDfState = 4;     // rows of the state ring (current + 3 in flight)
#ifndef UOT_WAVE_DF_WARPS
#define UOT_WAVE_DF_WARPS 1
#endif
constexpr int kWaveDfWarps = UOT_WAVE_DF_WARPS;    // warps (independent strips) per CTA
constexpr size_t kWaveDfSmem = (size_t)kWaveDfWarps * (kWaveDfState * 8 + kWaveRing * 2) * 32 * sizeof(float4);

template <int S, int RM, bool RED>
__global__ void __launch_bounds__(kWaveDfWarps * 32, 8 / kWaveDfWarps) k_wave_df(const WaveDfArgs A) {
    static_assert(S >= 1 && S <= 4, "lanes 0 and 31 hold a 4-column halo");
    constexpr int P = kWaveDfState - 1;          // rows in flight ahead of the current one
    static_assert(S + P + 1 <= kWaveRing, "constant ring holds rows t-S .. t+P");
    extern __shared__ __align__(16) float4 wdring[];
    pdl_wait();
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int upp = A.strips * A.segs;
    const long long unit = (long long)blockIdx.x * kWaveDfWarps + w;
    if (unit >= (long long)A.G * upp) return;
    const int pair = (int)(unit / upp), u = (int)(unit - (long long)pair * upp);
    const int sy = u / A.strips, sx = u - sy * A.strips;
    const int nx = A.nx, ny = A.ny;
    const int gs = sx * kWaveOut;                                // strip layout as k_wave (wave_strips)
    const int gi = gs + 4 * lane;
    const bool lane_in = gi < nx;
    const bool last_q = gi + 3 == nx - 1;
    const bool left_edge = lane == 0 && sx == 0;
    const bool writer = lane_in && (lane >= 1 || sx == 0) && (lane <= 30 || gs + 128 >= nx);
    const int y0 = sy * A.H, y1 = min(y0 + A.H, ny);
    const size_t po = (size_t)pair * (size_t)A.N, pz = ((size_t)pair * 2 + 1) * (size_t)A.N;
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1, rsc = A.r_scale;
    const float c1 = A.c1, c2 = A.c2, c3 = A.c3, rho = A.rho, i1r = A.inv1prho;
    const float t1x3 = last_q ? 0.f : t1;
    float4* sring = wdring + (size_t)w * ((kWaveDfState * 8 + kWaveRing * 2) * 32) + lane;   // [slot][8][lane]
    float4* cring = sring + kWaveDfState * 8 * 32;                                            // [slot][2][lane]

    auto issue = [&](int t) {
        const bool ok = lane_in && t >= 0 && t < ny;
        const size_t off = ok ? (size_t)t * nx + gi : 0;
        float4* s = sring + (t & (kWaveDfState - 1)) * (8 * 32);
        float4* c = cring + (t & (kWaveRing - 1)) * (2 * 32);
        cp_async16(reinterpret_cast<float*>(s), A.mx_in + po + off, ok);
        cp_async16(reinterpret_cast<float*>(s + 32), A.my_in + po + off, ok);
        cp_async16(reinterpret_cast<float*>(s + 64), A.r_in + po + off, ok);
        cp_async16(reinterpret_cast<float*>(s + 96), A.a_in + po + off, ok);
        cp_async16(reinterpret_cast<float*>(s + 128), A.z_in + pz + off, ok);
        cp_async16(reinterpret_cast<float*>(s + 160), A.x_in + po + off, ok);
        cp_async16(reinterpret_cast<float*>(s + 192), A.ax_in + po + off, ok);
        cp_async16(reinterpret_cast<float*>(s + 224), A.b_in + po + off, ok);
        cp_async16(reinterpret_cast<float*>(c), A.y + po + off, ok);
        cp_async16(reinterpret_cast<float*>(c + 32), A.s0 + po + off, ok);
        cp_commit();
    };

    const int t0 = y0 - S, t1r = y1 - 1 + S;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < kWaveDfState * 8; ++q) sring[q * 32] = z4;       // (see k_wave: rows never loaded)
#pragma unroll
    for (int q = 0; q < kWaveRing * 2; ++q) cring[q * 32] = z4;
#pragma unroll
    for (int p = 0; p < P; ++p) issue(t0 + p);
    struct Lv { float4 mx, my, r, a, k, z, x, ax, b; };
    Lv SA[S], SB[S];
    float4 upY[S + 1];
#pragma unroll
    for (int j = 0; j < S; ++j) { SA[j] = {z4, z4, z4, z4, z4, z4, z4, z4, z4}; SB[j] = SA[j]; }
#pragma unroll
    for (int j = 0; j <= S; ++j) upY[j] = z4;
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f, s_px = 0.f;

    auto step = [&](const int t, Lv (&Pv)[S], Lv (&Cv)[S]) {
        if (t + P <= t1r) issue(t + P);
        else cp_commit();
        cp_wait<P>();
        const float4* s = sring + (t & (kWaveDfState - 1)) * (8 * 32);
        const float4* cc = cring + (t & (kWaveRing - 1)) * (2 * 32);
        float4 Mx = s[0], My = s[32];
        const float4 R = s[64], Z = s[128], S0 = cc[32];
        if (last_q) Mx.w = 0.f;                                  // pinned flux components (L3)
        if (t == ny - 1) My = z4;
        // level 0: K^0 = div M - r - (z - s0)
        const float sh0 = __shfl_up_sync(kFull, Mx.w, 1);   // all lanes shuffle, then select
        const float mxl0 = left_edge ? 0.f : sh0;
        Cv[0].mx = Mx; Cv[0].my = My; Cv[0].r = R; Cv[0].a = s[96]; Cv[0].z = Z;
        Cv[0].x = s[160]; Cv[0].ax = s[192]; Cv[0].b = s[224];
        Cv[0].k.x = ((Mx.x - mxl0) + (My.x - upY[0].x)) - R.x - (Z.x - S0.x);
        Cv[0].k.y = ((Mx.y - Mx.x) + (My.y - upY[0].y)) - R.y - (Z.y - S0.y);
        Cv[0].k.z = ((Mx.z - Mx.y) + (My.z - upY[0].z)) - R.z - (Z.z - S0.z);
        Cv[0].k.w = ((Mx.w - Mx.z) + (My.w - upY[0].w)) - R.w - (Z.w - S0.w);
        upY[0] = My;
#pragma unroll
        for (int j = 1; j <= S; ++j) {
            const int rho_ = t - j;
            const Lv q = Pv[j - 1];
            const float4 cA = Cv[j - 1].a;                       // a^{j-1} at rho + 1
            const float t1y = (rho_ == -1 || rho_ == ny - 1) ? 0.f : t1;
            const float a5 = __shfl_down_sync(kFull, q.a.x, 1);
            const float av[5] = {q.a.x, q.a.y, q.a.z, q.a.w, a5};
            float nmx[4], nmy[4], nrm[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float gx = av[v] - av[v + 1];
                const float gy = av[v] - f4c(cA, v);
                const float qx = __fmaf_rn(-(v == 3 ? t1x3 : t1), gx, f4c(q.mx, v));
                const float qy = __fmaf_rn(-t1y, gy, f4c(q.my, v));
                const float n2 = norm2(qx, qy);
                const float inv = rsqrt_ftz(n2);
                const float sf = shrink_factor(n2, inv, t1);
                nmx[v] = sf * qx;
                nmy[v] = sf * qy;
                if (RED && j == S) nrm[v] = fmaxf(fmaf(n2, fminf(inv, 1e30f), -t1), 0.f);
            }
            const float shl = __shfl_up_sync(kFull, nmx[3], 1);   // all lanes shuffle, then select
            const float mxl = left_edge ? 0.f : shl;
            const float wr = (writer && rho_ >= y0 && rho_ < y1) ? 1.f : 0.f;
            const float4* cr = cring + (rho_ & (kWaveRing - 1)) * (2 * 32);
            const float4 Yr = cr[0], S0r = cr[32];
            const float mxv[5] = {mxl, nmx[0], nmx[1], nmx[2], nmx[3]};
            float rn[4], an[4], kn[4], zn[4], xn[4], axn[4], bn[4], sn[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float av0 = f4c(q.a, v), zv = f4c(q.z, v), xv = f4c(q.x, v), axv = f4c(q.ax, v), bv = f4c(q.b, v);
                rn[v] = r_update(fmaf(t1, av0, f4c(q.r, v)), RM, at1, rsc);
                sn[v] = fmaxf(0.5f * (xv + axv + zv + bv), 0.f);
                xn[v] = (f4c(Yr, v) + rho * (sn[v] - axv)) * i1r;
                zn[v] = fmaxf(fmaf(c1, sn[v] - bv, fmaf(c2, zv, c3 * av0)), 0.f);
                const float fnv = zn[v] - f4c(S0r, v);
                const float divn = (mxv[v + 1] - mxv[v]) + (nmy[v] - f4c(upY[j], v));
                kn[v] = divn - rn[v] - fnv;
                an[v] = fmaf(t2, 2.f * kn[v] - f4c(q.k, v), av0);
                axn[v] = axv + xn[v] - sn[v];
                bn[v] = bv + zn[v] - sn[v];
                if (RED && j == S) {
                    const float p0 = xn[v] - sn[v], p1 = zn[v] - sn[v];
                    const float d0 = xn[v] - xv, d1 = zn[v] - zv;
                    const float e = f4c(Yr, v) - sn[v];
                    s_tr = fmaf(wr, nrm[v], s_tr);
                    s_gr = fmaf(wr, pw(rn[v], RM), s_gr);
                    s_k2 = fmaf(wr * kn[v], kn[v], s_k2);
                    s_dz = fmaf(wr, p0 * p0 + p1 * p1, s_dz);
                    s_ub = fmaf(wr, d0 * d0 + d1 * d1, s_ub);
                    s_px = fmaf(wr, 0.5f * e * e, s_px);
                }
            }
            upY[j] = make_float4(nmy[0], nmy[1], nmy[2], nmy[3]);
            if (j < S) {
                Cv[j].mx = make_float4(nmx[0], nmx[1], nmx[2], nmx[3]);
                Cv[j].my = upY[j];
                Cv[j].r = make_float4(rn[0], rn[1], rn[2], rn[3]);
                Cv[j].a = make_float4(an[0], an[1], an[2], an[3]);
                Cv[j].k = make_float4(kn[0], kn[1], kn[2], kn[3]);
                Cv[j].z = make_float4(zn[0], zn[1], zn[2], zn[3]);
                Cv[j].x = make_float4(xn[0], xn[1], xn[2], xn[3]);
                Cv[j].ax = make_float4(axn[0], axn[1], axn[2], axn[3]);
                Cv[j].b = make_float4(bn[0], bn[1], bn[2], bn[3]);
            } else if (writer && rho_ >= y0 && rho_ < y1) {
                const size_t g = po + (size_t)rho_ * nx + gi, gz = pz + (size_t)rho_ * nx + gi;
                *reinterpret_cast<float4*>(A.mx_out + g) = make_float4(nmx[0], nmx[1], nmx[2], nmx[3]);
                *reinterpret_cast<float4*>(A.my_out + g) = upY[j];
                *reinterpret_cast<float4*>(A.r_out + g) = make_float4(rn[0], rn[1], rn[2], rn[3]);
                *reinterpret_cast<float4*>(A.a_out + g) = make_float4(an[0], an[1], an[2], an[3]);
                *reinterpret_cast<float4*>(A.z_out + gz) = make_float4(zn[0], zn[1], zn[2], zn[3]);
                *reinterpret_cast<float4*>(A.x_out + g) = make_float4(xn[0], xn[1], xn[2], xn[3]);
                *reinterpret_cast<float4*>(A.ax_out + g) = make_float4(axn[0], axn[1], axn[2], axn[3]);
                *reinterpret_cast<float4*>(A.b_out + g) = make_float4(bn[0], bn[1], bn[2], bn[3]);
                if (RED) *reinterpret_cast<float4*>(A.s_out + g) = make_float4(sn[0], sn[1], sn[2], sn[3]);
            }
        }
    };
    int t = t0;
#pragma unroll 1
    for (; t + 1 <= t1r; t += 2) {
        step(t, SA, SB);
        step(t + 1, SB, SA);
    }
    if (t <= t1r) step(t, SA, SB);
    cp_wait<0>();
    pdl_trigger();
    if constexpr (RED) {
        double v[6] = {s_tr, s_gr, s_k2, s_dz, s_ub, s_px};
#pragma unroll
        for (int q = 0; q < 6; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(kFull, v[q], o);
        }
        if (lane == 0) {
            double* Pp = A.partials + ((size_t)pair * upp + u) * kRec;
#pragma unroll
            for (int q = 0; q < 6; ++q) Pp[q] = v[q];
            Pp[6] = 0.0; Pp[7] = 0.0;
        }
    }
}

}  // namespace uotk
