// uot_wave_n.cuh -- k_wave_n: the packed register wavefront on NARROW strips (64 columns: one
// fp32x2 column pair per lane).
//
// Same method and schedule as k_wave_pk (uot_wave_pk.cuh: S fixed-marginal Algorithm-1
// iterations per HBM pass, level j on row t - j at step t, horizontal neighbours by
// shuffle, vertical ones carried), with half the columns per lane.  Two things change:
//  * registers: a level carries M, r, a, -K as one pair each (10 registers instead of 20), so
//    a warp needs ~half of k_wave_pk's 222 registers and twice as many warps fit an SM
//    (16 instead of 8) -- the same pixels in flight per SM, twice the independent warps;
//  * strip width: halo lanes are ceil(S/2) per side (2 columns each), so a strip writes
//    64 - 4 ceil(S/2) columns.  A 256-column row (config C3) takes 5 strips of 64 (320 columns
//    computed, 1.25x) instead of 3 of 128 (384, 1.5x); a 1024-column row takes 20 (1.25x)
//    instead of 9 (1.125x), so the host picks the strip width per grid (uot_api.cu,
//    wave_model).
// The arithmetic per pixel is k_wave_pk's, op for op (same packed ops on the same operands,
// same rounding), so the iterates equal k_wave_pk's value for value; only the reductions'
// per-lane association differs.
#pragma once
#include "uot_wave_pk.cuh"

namespace uotk {

// S iterations invalidate S columns per strip side: ceil(S/2) halo lanes of 2 columns
__host__ __device__ constexpr int waven_halo_lanes(int S) { return (S + 1) / 2; }
__host__ __device__ constexpr int waven_out(int S) { return 64 - 4 * waven_halo_lanes(S); }
__host__ __device__ constexpr int waven_strips(int nx, int S) {
    return nx <= 64 ? 1 : (nx - 64 + waven_out(S) - 1) / waven_out(S) + 1;
}
constexpr int kWaveNMinB = 16;                  // warps (= CTAs of one warp) per SM: <= 128 registers
constexpr size_t kWaveNSmem = (size_t)kWaveRing * 5 * 32 * sizeof(float2);   // 10 KB per warp

__device__ __forceinline__ void cp_async8(float* s, const float* g, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(sz) : "memory");
}
__device__ __forceinline__ void st2_if(float* g, float2 v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.f32 [%0], {%1, %2};\n\t}"
                 :: "l"(g), "f"(v.x), "f"(v.y), "r"((int)p));
}

template <int S, int RM, bool RED>
__global__ void __launch_bounds__(32, kWaveNMinB) k_wave_n(const WaveArgs A) {
    static_assert(S >= 1 && S <= 5, "ring of 8 rows: S + prefetch + 1 <= 8");
    constexpr int HL = waven_halo_lanes(S), OUT = waven_out(S);
    constexpr int P = kWaveRing - S - 1;        // rows in flight ahead of the current one
    extern __shared__ __align__(16) float2 wring2[];
    pdl_wait();
    if (A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop)) return;
    const int lane = threadIdx.x & 31;
    const int upp = A.strips * A.segs;
    const long long unit = (long long)blockIdx.x;
    if (unit >= (long long)A.G * upp) return;
    const int pair = (int)(unit / upp), u = (int)(unit - (long long)pair * upp);
    const int sy = u / A.strips, sx = u - sy * A.strips;
    const int nx = A.nx, ny = A.ny;
    const int gs = sx * OUT;                                     // first loaded column of the strip
    const int gi = gs + 2 * lane;                                // first column of this lane's pair
    const bool lane_in = gi < nx;                                // whole pair in the grid (nx % 2 == 0)
    const bool last_q = gi + 1 == nx - 1;                        // holds the pinned column nx-1 (L3)
    const bool left_edge = lane == 0 && sx == 0;                 // column -1 is outside: M_x there = 0
    const bool writer = lane_in && (lane >= HL || sx == 0) && (lane <= 31 - HL || gs + 64 >= nx);
    const int y0 = sy * A.H, y1 = min(y0 + A.H, ny);             // output rows [y0, y1)
    const size_t po = (size_t)pair * (size_t)A.N;
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1, rsc = A.r_scale;
    float* const mx_out = A.mx_out; float* const my_out = A.my_out;
    float* const r_out = A.r_out; float* const a_out = A.a_out;
    // -tau1 per column; the pinned column nx-1 (2nd pixel of the last pair) takes 0 (k_wave)
    const float2 nt1 = pk_dup(-t1), nt1h = make_float2(-t1, last_q ? 0.f : -t1);
    float2* ring = wring2 + lane;                                // [slot][plane][lane]
    const int t0 = y0 - S, t1r = y1 - 1 + S;

    auto issue = [&](int t) {                                    // row t -> slot t & 7 (zero outside)
        const bool ok = lane_in && t >= 0 && t < ny && t <= t1r;     // past the segment: zero-fill only
        const size_t g = ok ? po + (size_t)t * nx + gi : po;
        float2* s = ring + (t & (kWaveRing - 1)) * (5 * 32);
        cp_async8(reinterpret_cast<float*>(s), A.mx_in + g, ok);
        cp_async8(reinterpret_cast<float*>(s + 32), A.my_in + g, ok);
        cp_async8(reinterpret_cast<float*>(s + 64), A.r_in + g, ok);
        cp_async8(reinterpret_cast<float*>(s + 96), A.a_in + g, ok);
        cp_async8(reinterpret_cast<float*>(s + 128), A.f + g, ok);
        cp_commit();
    };

    const float2 z2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < kWaveRing * 5; ++q) ring[q * 32] = z2;   // rows never loaded stay finite (k_wave)
#pragma unroll
    for (int p = 0; p < P; ++p) issue(t0 + p);
    struct Lv { float2 mx, my, r, a, nk; };   // level j-1's outputs at one row (nk = -K)
    Lv SA[S], SB[S];
    float2 upY[S + 1];                        // level j's M_y at its previous row
#pragma unroll
    for (int j = 0; j < S; ++j) { SA[j] = {z2, z2, z2, z2, z2}; SB[j] = SA[j]; }
#pragma unroll
    for (int j = 0; j <= S; ++j) upY[j] = z2;
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f;

    auto step = [&](const int t, Lv (&Pv)[S], Lv (&Cv)[S]) {
        issue(t + P);
        cp_wait<P>();                                            // row t has landed (own lane's copies)
        const float2* s = ring + (t & (kWaveRing - 1)) * (5 * 32);
        float2 Mx = s[0], My = s[32];
        if (last_q) Mx.y = 0.f;                                  // pinned flux components (L3)
        if (t == ny - 1) My = z2;
        // ---- level 0: -K^0 = (r - div M) + f at row t ----
        const float sh0 = __shfl_up_sync(kFull, Mx.y, 1);        // all lanes shuffle, then select
        const float2 qr = s[64];
        const float2 dl0 = make_float2(Mx.x - (left_edge ? 0.f : sh0), Mx.y - Mx.x);
        const float2 div0 = pk_add(dl0, pk_sub(My, upY[0]));
        Cv[0].mx = Mx; Cv[0].my = My; Cv[0].r = qr; Cv[0].a = s[96];
        Cv[0].nk = pk_add(pk_sub(qr, div0), s[128]);
        upY[0] = My;
#pragma unroll
        for (int j = 1; j <= S; ++j) {
            const int rho = t - j;
            const Lv& p = Pv[j - 1];
            const float2 cA = Cv[j - 1].a;                       // a^{j-1} at rho + 1
            const float2 nt1y = pk_dup((rho == -1 || rho == ny - 1) ? 0.f : -t1);
            // line 3: M^j(rho) = prox(M^{j-1} - tau1 div^* a^{j-1}); a at (rho, i+1) and (rho+1, i)
            const float a5 = __shfl_down_sync(kFull, p.a.x, 1);
            const float2 gx = make_float2(p.a.x - p.a.y, p.a.y - a5);
            const float2 gy = pk_sub(p.a, cA);
            const float2 qx = pk_fma(nt1h, gx, p.mx);
            const float2 qy = pk_fma(nt1y, gy, p.my);
            const float2 n2 = pk_fma(qy, qy, pk_mul(qx, qx));
            const float2 inv = make_float2(rsqrt_ftz(n2.x), rsqrt_ftz(n2.y));
            float2 sf = pk_fma(nt1, inv, make_float2(1.f, 1.f));
            sf = make_float2(fmaxf(sf.x, 0.f), fmaxf(sf.y, 0.f));
            const float2 nmx = pk_mul(sf, qx), nmy = pk_mul(sf, qy);
            // line 5: r^j = shrink_{alpha tau1}(r^{j-1} + tau1 a^{j-1})
            const float2 q5 = pk_fma(pk_dup(t1), p.a, p.r);
            float2 rn;
            if constexpr (RM == 0) {
                rn = pk_sub(q5, make_float2(fminf(fmaxf(q5.x, -at1), at1), fminf(fmaxf(q5.y, -at1), at1)));
            } else if constexpr (RM == 1) {
                rn = pk_mul(q5, pk_dup(rsc));
            } else {
                rn = z2;
            }
            // lines 6-7: -K^j = (r^j - div M^j) + f;  a^j = a^{j-1} + tau2 (2 K^j - K^{j-1})
            const float shl = __shfl_up_sync(kFull, nmx.y, 1);   // all lanes shuffle, then select
            const float2 Fr = ring[(rho & (kWaveRing - 1)) * (5 * 32) + 128];
            const float2 dl = make_float2(nmx.x - (left_edge ? 0.f : shl), nmx.y - nmx.x);
            const float2 divn = pk_add(dl, pk_sub(nmy, upY[j]));
            const float2 nkn = pk_add(pk_sub(rn, divn), Fr);
            const float2 an = pk_fma(pk_dup(t2), pk_fma(pk_dup(-2.f), nkn, p.nk), p.a);
            if (RED && j == S) {                                 // branch-free: weight 0 off the output
                const float wr = (writer && rho >= y0 && rho < y1) ? 1.f : 0.f;
                const float2 ic = make_float2(fminf(inv.x, 1e30f), fminf(inv.y, 1e30f));
                float2 nrm = pk_fma(n2, ic, pk_dup(-t1));        // |M^j| (k_wave)
                nrm = make_float2(fmaxf(nrm.x, 0.f), fmaxf(nrm.y, 0.f));
                const float2 k2 = pk_mul(nkn, nkn);
                const float2 dmx = pk_sub(nmx, p.mx), dmy = pk_sub(nmy, p.my), dr = pk_sub(rn, p.r);
                float2 dz = pk_fma(dmy, dmy, pk_mul(dmx, dmx));
                dz = pk_fma(dr, dr, dz);
                const float2 ub = pk_sub(divn, Fr);
                float gr, ubs;
                if constexpr (RM == 1) {
                    gr = rn.x * rn.x + rn.y * rn.y; ubs = ub.x * ub.x + ub.y * ub.y;
                } else {
                    gr = fabsf(rn.x) + fabsf(rn.y); ubs = fabsf(ub.x) + fabsf(ub.y);
                }
                s_tr = fmaf(wr, nrm.x + nrm.y, s_tr);
                s_gr = fmaf(wr, gr, s_gr);
                s_k2 = fmaf(wr, k2.x + k2.y, s_k2);
                s_dz = fmaf(wr, dz.x + dz.y, s_dz);
                s_ub = fmaf(wr, ubs, s_ub);
            }
            upY[j] = nmy;
            if (j < S) {
                Cv[j].mx = nmx; Cv[j].my = nmy; Cv[j].r = rn; Cv[j].a = an; Cv[j].nk = nkn;
            } else {
                const bool wp = writer && rho >= y0 && rho < y1;
                const size_t g = po + (size_t)rho * nx + gi;
                st2_if(mx_out + g, nmx, wp);
                st2_if(my_out + g, nmy, wp);
                st2_if(r_out + g, rn, wp);
                st2_if(a_out + g, an, wp);
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

}  // namespace uotk
