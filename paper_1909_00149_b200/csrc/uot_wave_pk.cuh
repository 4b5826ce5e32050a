// uot_wave_pk.cuh -- k_wave with packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2 / FMUL2).
//
// Same register wavefront as k_wave (uot_wave.cuh: S fixed-marginal Algorithm-1 iterations per
// HBM pass; strips, segments, ring, halos and edge handling unchanged), same
// arithmetic per pixel and iteration in the same order.  What changes is the instruction
// stream: k_wave<5> is issue-bound (29.6 SASS instructions per pixel-level, 19 of them scalar
// FADD/FFMA/FMUL; ncu issue-active 75% with 2 warps per scheduler), and sm_100a issues an
// fp32x2 instruction for two pixels in one slot at the same FP32-pipe throughput (measured:
// scripts/micro/ffma2.cu, 128 fp32 results / clk / SM either way).  A lane's quad of columns
// is held as two pairs l = (c, c+1), h = (c+2, c+3) -- the register pairs an LDS.128 /
// STG.128 fills -- so every vertical and pointwise step is one packed instruction per pair;
// only the two horizontal differences (div^* along i, div along i) stay scalar (their shifted
// operand pairs are not register-aligned; the scalar results land in pairs for free).
//
// Exactness: each packed op is the scalar op of k_wave with the same rounding (rn, no
// contraction across intrinsics); the previous K is carried negated (nK = -K, computed as
// (r - div M) + f, an exact negation) so line 7's 2K' - K is one fma(-2, nK', nK); the
// l1 soft threshold is evaluated as q - clamp(q, -s, s), equal to sign(q) max(|q| - s, 0)
// in round-to-nearest; |q|^2 is fma(qy, qy, qx * qx) as in every kernel (norm2).  So the
// iterates equal k_wave's value for value (zeros may differ in sign).
#pragma once
#include "uot_wave.cuh"

namespace uotk {

__device__ __forceinline__ float2 pk_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 pk_mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 pk_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 pk_sub(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 ra, rb, rr;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0, %1}, rr;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 pk_dup(float v) { return make_float2(v, v); }
// predicated 16-byte store: keeps the step loop one basic block (no branch around the level-S
// stores), so ptxas can interleave step t+1's upper levels with step t's lower ones
__device__ __forceinline__ void st4_if(float* g, float4 v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.v4.f32 [%0], {%1, %2, %3, %4};\n\t}"
                 :: "l"(g), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"((int)p));
}

struct Quad { float2 l, h; };     // columns (c, c+1) and (c+2, c+3) of one lane
__device__ __forceinline__ Quad qd(const float4& v) { return {make_float2(v.x, v.y), make_float2(v.z, v.w)}; }
__device__ __forceinline__ float4 f4(const Quad& q) { return make_float4(q.l.x, q.l.y, q.h.x, q.h.y); }
__device__ __forceinline__ Quad qadd(const Quad& a, const Quad& b) { return {pk_add(a.l, b.l), pk_add(a.h, b.h)}; }
__device__ __forceinline__ Quad qsub(const Quad& a, const Quad& b) { return {pk_sub(a.l, b.l), pk_sub(a.h, b.h)}; }
__device__ __forceinline__ Quad qmul(const Quad& a, const Quad& b) { return {pk_mul(a.l, b.l), pk_mul(a.h, b.h)}; }
__device__ __forceinline__ Quad qfma(float2 s, const Quad& b, const Quad& c) { return {pk_fma(s, b.l, c.l), pk_fma(s, b.h, c.h)}; }
__device__ __forceinline__ Quad qfma(const Quad& a, const Quad& b, const Quad& c) {
    return {pk_fma(a.l, b.l, c.l), pk_fma(a.h, b.h, c.h)};
}
__device__ __forceinline__ float qc(const Quad& q, int v) { return v == 0 ? q.l.x : (v == 1 ? q.l.y : (v == 2 ? q.h.x : q.h.y)); }
// columns c-1 .. c+2 minus c .. c+3 shifted: (q0 - q1, q1 - q2, q2 - q3, q3 - right) and
// (q0 - left, q1 - q0, q2 - q1, q3 - q2): scalar, results in pairs
__device__ __forceinline__ Quad qdiff_right(const Quad& q, float right) {
    return {make_float2(q.l.x - q.l.y, q.l.y - q.h.x), make_float2(q.h.x - q.h.y, q.h.y - right)};
}
__device__ __forceinline__ Quad qdiff_left(const Quad& q, float left) {
    return {make_float2(q.l.x - left, q.l.y - q.l.x), make_float2(q.h.x - q.l.y, q.h.y - q.h.x)};
}

template <int S, int RM, bool RED>
__global__ void __launch_bounds__(kWaveWarps * 32, WaveCfg<S, RED>::minb) k_wave_pk(const WaveArgs A) {
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
    // -tau1 per column pair; the pinned column nx-1 (4th pixel of the last quad) takes 0 (k_wave)
    const float2 nt1 = pk_dup(-t1), nt1h = make_float2(-t1, last_q ? 0.f : -t1);
    float4* ring = wring + (size_t)w * (kWaveRing * 5 * 32) + lane;   // [slot][plane][lane]
    const int t0 = y0 - S, t1r = y1 - 1 + S;

    auto issue = [&](int t) {                                    // row t -> slot t & 7 (zero outside)
        const bool ok = lane_in && t >= 0 && t < ny && t <= t1r;     // past the segment: zero-fill only
        const size_t g = ok ? po + (size_t)t * nx + gi : po;
        float4* s = ring + (t & (kWaveRing - 1)) * (5 * 32);
        cp_async16(reinterpret_cast<float*>(s), A.mx_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 32), A.my_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 64), A.r_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 96), A.a_in + g, ok);
        cp_async16(reinterpret_cast<float*>(s + 128), A.f + g, ok);
        cp_commit();
    };

    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const Quad zq = qd(z4);
#pragma unroll
    for (int q = 0; q < kWaveRing * 5; ++q) ring[q * 32] = z4;   // rows never loaded stay finite (k_wave)
#pragma unroll
    for (int p = 0; p < P; ++p) issue(t0 + p);
    // level j-1's outputs at one row (nk = -K), ping-ponged between two register sets (k_wave)
    struct Lv { Quad mx, my, r, a, nk; };
    Lv SA[S], SB[S];
    Quad upY[S + 1];                              // level j's M_y at its previous row
#pragma unroll
    for (int j = 0; j < S; ++j) { SA[j] = {zq, zq, zq, zq, zq}; SB[j] = SA[j]; }
#pragma unroll
    for (int j = 0; j <= S; ++j) upY[j] = zq;
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f;

    auto step = [&](const int t, Lv (&Pv)[S], Lv (&Cv)[S]) {
        issue(t + P);       // past t1r: a zero-fill of the slot of row t + P - 8 (no longer read)
        cp_wait<P>();                                            // row t has landed (own lane's copies)
        const float4* s = ring + (t & (kWaveRing - 1)) * (5 * 32);
        float4 Mx = s[0], My = s[32];
        if (last_q) Mx.w = 0.f;                                  // pinned flux components (L3)
        if (t == ny - 1) My = z4;
        // ---- level 0: -K^0 = (r - div M) + f at row t ----
        const float sh0 = __shfl_up_sync(kFull, Mx.w, 1);        // all lanes shuffle, then select
        const Quad qmy = qd(My), qr = qd(s[64]);
        const Quad div0 = qadd(qdiff_left(qd(Mx), left_edge ? 0.f : sh0), qsub(qmy, upY[0]));
        Cv[0].mx = qd(Mx); Cv[0].my = qmy; Cv[0].r = qr; Cv[0].a = qd(s[96]);
        Cv[0].nk = qadd(qsub(qr, div0), qd(s[128]));
        upY[0] = qmy;
#pragma unroll
        for (int j = 1; j <= S; ++j) {
            const int rho = t - j;
            const Lv& p = Pv[j - 1];
            const Quad cA = Cv[j - 1].a;                         // a^{j-1} at rho + 1
            const float2 nt1y = pk_dup((rho == -1 || rho == ny - 1) ? 0.f : -t1);
            // line 3: M^j(rho) = prox(M^{j-1} - tau1 div^* a^{j-1}); a at (rho, i+1) and (rho+1, i)
            const float a5 = __shfl_down_sync(kFull, p.a.l.x, 1);
            const Quad gx = qdiff_right(p.a, a5);
            const Quad gy = qsub(p.a, cA);
            const Quad qx = {pk_fma(nt1, gx.l, p.mx.l), pk_fma(nt1h, gx.h, p.mx.h)};
            const Quad qy = qfma(nt1y, gy, p.my);
            const Quad n2 = qfma(qy, qy, qmul(qx, qx));
            const Quad inv = {make_float2(rsqrt_ftz(n2.l.x), rsqrt_ftz(n2.l.y)),
                              make_float2(rsqrt_ftz(n2.h.x), rsqrt_ftz(n2.h.y))};
            Quad sf = qfma(nt1, inv, qd(make_float4(1.f, 1.f, 1.f, 1.f)));
            sf = {make_float2(fmaxf(sf.l.x, 0.f), fmaxf(sf.l.y, 0.f)), make_float2(fmaxf(sf.h.x, 0.f), fmaxf(sf.h.y, 0.f))};
            const Quad nmx = qmul(sf, qx), nmy = qmul(sf, qy);
            // line 5: r^j = shrink_{alpha tau1}(r^{j-1} + tau1 a^{j-1})
            const Quad q5 = qfma(pk_dup(t1), p.a, p.r);
            Quad rn;
            if constexpr (RM == 0) {
                const Quad cl = {make_float2(fminf(fmaxf(q5.l.x, -at1), at1), fminf(fmaxf(q5.l.y, -at1), at1)),
                                 make_float2(fminf(fmaxf(q5.h.x, -at1), at1), fminf(fmaxf(q5.h.y, -at1), at1))};
                rn = qsub(q5, cl);
            } else if constexpr (RM == 1) {
                rn = qmul(q5, qd(make_float4(rsc, rsc, rsc, rsc)));
            } else {
                rn = zq;
            }
            // lines 6-7: -K^j = (r^j - div M^j) + f;  a^j = a^{j-1} + tau2 (2 K^j - K^{j-1})
            const float shl = __shfl_up_sync(kFull, nmx.h.y, 1);  // all lanes shuffle, then select
            const Quad Fr = qd(ring[(rho & (kWaveRing - 1)) * (5 * 32) + 128]);
            const Quad divn = qadd(qdiff_left(nmx, left_edge ? 0.f : shl), qsub(nmy, upY[j]));
            const Quad nkn = qadd(qsub(rn, divn), Fr);
            const Quad an = qfma(pk_dup(t2), qfma(pk_dup(-2.f), nkn, p.nk), p.a);
            if (RED && j == S) {                                 // branch-free: weight 0 off the output
                // per-quad partial sums (packed where the terms are), then one weighted add per
                // sum and row; the five a6 sums of k_wave in a different association order
                const float wr = (writer && rho >= y0 && rho < y1) ? 1.f : 0.f;
                const Quad ic = {make_float2(fminf(inv.l.x, 1e30f), fminf(inv.l.y, 1e30f)),
                                 make_float2(fminf(inv.h.x, 1e30f), fminf(inv.h.y, 1e30f))};
                Quad nrm = qfma(n2, ic, qd(make_float4(-t1, -t1, -t1, -t1)));          // |M^j| (k_wave)
                nrm = {make_float2(fmaxf(nrm.l.x, 0.f), fmaxf(nrm.l.y, 0.f)), make_float2(fmaxf(nrm.h.x, 0.f), fmaxf(nrm.h.y, 0.f))};
                const float2 tr = pk_add(nrm.l, nrm.h);
                const float2 k2 = pk_fma(nkn.h, nkn.h, pk_mul(nkn.l, nkn.l));
                const Quad dmx = qsub(nmx, p.mx), dmy = qsub(nmy, p.my), dr = qsub(rn, p.r);
                float2 dz = pk_fma(dmx.h, dmx.h, pk_mul(dmx.l, dmx.l));
                dz = pk_fma(dmy.l, dmy.l, dz); dz = pk_fma(dmy.h, dmy.h, dz);
                dz = pk_fma(dr.l, dr.l, dz); dz = pk_fma(dr.h, dr.h, dz);
                const Quad ub = qsub(divn, Fr);
                float gr, ubs;
                if constexpr (RM == 1) {
                    const float2 g2 = pk_fma(rn.h, rn.h, pk_mul(rn.l, rn.l)), u2 = pk_fma(ub.h, ub.h, pk_mul(ub.l, ub.l));
                    gr = g2.x + g2.y; ubs = u2.x + u2.y;
                } else {
                    gr = (fabsf(rn.l.x) + fabsf(rn.l.y)) + (fabsf(rn.h.x) + fabsf(rn.h.y));
                    ubs = (fabsf(ub.l.x) + fabsf(ub.l.y)) + (fabsf(ub.h.x) + fabsf(ub.h.y));
                }
                s_tr = fmaf(wr, tr.x + tr.y, s_tr);
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
                st4_if(mx_out + g, f4(nmx), wp);
                st4_if(my_out + g, f4(nmy), wp);
                st4_if(r_out + g, f4(rn), wp);
                st4_if(a_out + g, f4(an), wp);
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
