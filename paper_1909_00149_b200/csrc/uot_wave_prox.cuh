// uot_wave_prox.cuh -- chain prox (rho < inf, L19): S Algorithm-1 iterations per HBM pass.
//
// Algorithm 1 with frame updates (P:313-317, line 4 = P:314 generalised to the chain, L19):
// the dual a_t of pair t enters the x-update of frames t and t+1, and x_t, x_{t+1} enter K_t,
// so iteration k+1 of pair t needs iteration k of pairs t-1, t, t+1 at the same pixel (the
// coupling across pairs is pointwise; across pixels it is the 5-point stencil of k_wave).
//
// Layout: the register wavefront of k_wave_pk (uot_wave_pk.cuh) runs one warp per pair --
// a 128-column strip marching down H + 2S rows, level j updating row rho - j at step rho --
// and the warps of consecutive pairs advance together.  Level j at step rho needs the
// neighbour pairs' a^{j-1} at row rho - j, which the neighbours produced at step rho - 1:
// each warp PUSHES its a^0 .. a^{S-1} of a step into both neighbours' receive buffers with
// st.async (shared::cluster, completing bytes on the receiver's mbarrier), and a receiver
// waits on its own mbarrier before step rho + 1 reads them.  No cluster-wide barrier and no
// memory fence per step (a release arrive or fence.acq_rel.cluster is a MEMBAR.ALL.GPU on
// sm_100a, which waits for the warp's outstanding global stores): a warp only waits for its
// two neighbours, so neighbours stay within one step of each other and two buffers per side
// suffice for levels 0 .. S-2 (a warp pushes a^{S-1}, which depends on its reads of those
// slots, before a neighbour can start the step that overwrites them); a^{S-1}, read at level S
// after that push, has three.  Every push is unconditional (a predicated st.async becomes a
// branch with convergence barriers): a warp without a neighbour on a side pushes that side's
// bytes into a private dummy slot, completing them on its own mbarrier, and the receive slots
// of a missing neighbour stay zero from the start (a = 0 there: chain end, L19).  The last
// step's pushes are waited for too, so no push reaches a CTA that has exited.  Frames are recomputed by both pairs that use them: the warp of
// pair t carries x_t and x_{t+1} per level (bit-identical to its neighbours' copies: same
// inputs, same operations), so nothing is exchanged within a step.
//
// Pair groups: a cluster of CL CTAs x 8 warps holds CL*8 consecutive pairs of one chain (the
// CTA-boundary neighbours sit in the adjacent CTA's shared memory).  After S levels a pair is
// exact iff its S neighbours on both sides are in the group (the dependency cone), so a group
// writes the middle CL*8 - 2S pairs; pairs outside the chain (t < 0, t >= P) are empty slots
// whose a is the chain end's a_{-1} = a_{T-1} := 0 exactly (L19).  HBM traffic per pass and
// pair-pixel: M, r, a, x_t, p_t read (x_{t+1}, p_{t+1} are the next pair's, L2 hits) and M, r,
// a, x_t written: 44 B per S iterations, plus the 2S halo pairs of each group.
#pragma once
#include "uot_wave_pk.cuh"

namespace uotk {

constexpr int kWpWarps = 8;               // warps (pairs) per CTA
constexpr int kWpStateRing = 3;           // rows of the state ring (M, r, a, x_t, x_{t+1}): current + 2 ahead
constexpr int kWpPRing = 8;               // rows of the p ring (p_t, p_{t+1} at the level rows)
template <int S> struct WpCfg {
    static constexpr int P = kWpStateRing - 1;                    // rows in flight ahead
    static_assert(S + P + 1 <= kWpPRing, "p ring holds rows rho - S .. rho + P");
    static constexpr size_t warp_floats = (size_t)(kWpStateRing * 6 + kWpPRing * 2) * 32 * 4;
    // receive buffers: levels 0 .. S-2 [2 bufs][2 sides][S-1][warp][lane], level S-1 [3 bufs][2 sides][warp][lane],
    // then one dummy slot per warp [warp][lane]
    static constexpr size_t rb_floats = (size_t)(2 * 2 * (S - 1) + 3 * 2 + 1) * kWpWarps * 32 * 4;
    static constexpr size_t smem = (warp_floats * kWpWarps + rb_floats) * sizeof(float) + kWpWarps * 2 * 8;
};

struct WaveProxArgs {
    int nx, ny, strips, segs, H;
    int B, T, P;                    // chains, frames and pairs per chain
    int groups, cl;                 // pair groups per chain, CTAs per cluster
    int own_lo, own_hi;             // pairs [own_lo, own_hi) of each chain are written; the others are
                                    // ghost pairs (a sharded chain's copies of its neighbours' pairs)
    long long N;
    const float* p;                 // [B][T][N] prox centres
    const float* mx_in; const float* my_in; const float* a_in; const float* r_in; const float* x_in;
    float* mx_out; float* my_out; float* a_out; float* r_out; float* x_out;
    float tau1, tau2, atau1, r_scale, c1, c2, c3;
    int fix_first;
    double* partials;               // [B*P][strips * segs][kRec] when reducing
    const int* stop;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned map_rank(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
}
// one arrival that also expects `bytes` of st.async data in the current phase (if p)
__device__ __forceinline__ void mbar_arm(unsigned a, unsigned bytes, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
                 "@q mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n\t}"
                 :: "r"(a), "r"(bytes), "r"((int)p) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned phase) {
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}"
                 :: "r"(a), "r"(phase) : "memory");
}
// 16 bytes into a cluster CTA's shared memory, completing 16 bytes on its mbarrier
__device__ __forceinline__ void st_async4(unsigned addr, float4 v, unsigned bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                 :: "r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ void cluster_sync() {       // once per launch: release / acquire
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int S, int RM, bool RED>
__global__ void __launch_bounds__(kWpWarps * 32, 1) k_wave_prox(const WaveProxArgs A) {
    static_assert(S >= 2 && S <= 3, "levels per pass (S = 4: 255 registers and spills; shared memory)");
    using C = WpCfg<S>;
    constexpr int HL = wave_halo_lanes(S), OUT = wave_out(S), P = C::P;
    extern __shared__ __align__(16) float4 wpsm[];
    pdl_wait();
    const bool stopped = A.stop != nullptr && *reinterpret_cast<const volatile int*>(A.stop);
    // every CTA of the cluster sees the same flag (set before this launch): uniform exit
    if (stopped) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rank = (int)cluster_rank(), CL = A.cl;
    const int grp = blockIdx.x / CL;                              // (chain, group)
    const int b = grp / A.groups, g = grp - b * A.groups;
    const int u = blockIdx.y, sy = u / A.strips, sx = u - sy * A.strips;
    const int Pc = A.P;
    const int own = A.own_hi - A.own_lo;
    const int lo = A.own_lo + (int)((long long)g * own / A.groups), hi = A.own_lo + (int)((long long)(g + 1) * own / A.groups);
    const int q = rank * kWpWarps + w;                            // slot in the group
    const int t = lo - S + q;                                     // pair of this warp
    const bool exists = t >= 0 && t < Pc && t < hi + S;
    const bool out_pair = t >= lo && t < hi;
    const bool has_l = q > 0, has_r = q < CL * kWpWarps - 1;      // neighbour slots in the cluster
    const int nx = A.nx, ny = A.ny;
    const int gs = sx * OUT, gi = gs + 4 * lane;
    const bool lane_in = gi < nx;
    const bool last_q = gi + 3 == nx - 1;
    const bool left_edge = lane == 0 && sx == 0;
    const bool writer = out_pair && lane_in && (lane >= HL || sx == 0) && (lane <= 31 - HL || gs + 128 >= nx);
    const int y0 = sy * A.H, y1 = min(y0 + A.H, ny);
    const int t0 = y0 - S, t1r = y1 - 1 + S;
    const size_t po = ((size_t)b * Pc + (size_t)(exists ? t : 0)) * (size_t)A.N;    // pair planes
    const size_t fo = ((size_t)b * A.T + (size_t)(exists ? t : 0)) * (size_t)A.N;   // frame t
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1, rsc = A.r_scale;
    const float2 c1 = pk_dup(A.c1), c2 = pk_dup(A.c2), nc3 = pk_dup(-A.c3);
    const bool fix0 = A.fix_first && t == 0;                      // constant first frame
    const bool own_last = t == Pc - 1 && A.own_hi == Pc;          // also owns frame T-1 (writes, reductions)
    const float2 nt1 = pk_dup(-t1), nt1h = make_float2(-t1, last_q ? 0.f : -t1);

    float4* sring = wpsm + (size_t)w * (C::warp_floats / 4) + lane;        // [slot][6][lane]
    float4* pring = sring + kWpStateRing * 6 * 32;                          // [slot][2][lane]
    float4* rbuf = wpsm + (size_t)kWpWarps * (C::warp_floats / 4);          // see WpCfg::rb_floats
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(rbuf + C::rb_floats / 4);   // [warp][buf]
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const Quad zq = qd(z4);
    // neighbour slots: the same CTA (warp +- 1) or the adjacent CTA of the cluster; a neighbour
    // that is an empty slot (outside the chain or past the group's halo) sends nothing: its a is 0
    auto slot_exists = [&](int tt) { return tt >= 0 && tt < Pc && tt < hi + S; };
    const bool l_ex = has_l && slot_exists(t - 1), r_ex = has_r && slot_exists(t + 1);
    const unsigned lw = w > 0 ? (unsigned)(w - 1) : (unsigned)(kWpWarps - 1);
    const unsigned rw = w < kWpWarps - 1 ? (unsigned)(w + 1) : 0u;
    const unsigned lrank = w > 0 ? (unsigned)rank : (unsigned)(rank - 1);
    const unsigned rrank = w < kWpWarps - 1 ? (unsigned)rank : (unsigned)(rank + 1);
    // byte offset of (step parity p2 = rel & 1, rel mod 3 = p3, side, level) for warp ww
    auto rboff = [&](int p2, int p3, int side, int lvl, unsigned ww) {
        const int k = lvl < S - 1 ? (p2 * 2 + side) * (S - 1) + lvl : 4 * (S - 1) + p3 * 2 + side;
        return (unsigned)(((k * kWpWarps + (int)ww) * 32 + lane) * 16);
    };
    const unsigned rb_base = smem_u32(rbuf), mb_base = smem_u32(mbar);
    const unsigned my_mb = mb_base + (unsigned)w * 16u;
    const unsigned dummy = rb_base + (unsigned)((((4 * (S - 1) + 6) * kWpWarps + w) * 32 + lane) * 16);
    // pushes to the left neighbour land in its side 1 ("from the right"), to the right one in side 0;
    // a missing side's pushes go to the dummy slot and complete on this warp's own mbarrier
    const unsigned l_rb = l_ex ? map_rank(rb_base, lrank) : 0u, r_rb = r_ex ? map_rank(rb_base, rrank) : 0u;
    const unsigned l_mb = l_ex ? map_rank(mb_base + lw * 16u, lrank) : my_mb;
    const unsigned r_mb = r_ex ? map_rank(mb_base + rw * 16u, rrank) : my_mb;
    const unsigned expect = 2u * S * 32u * 16u;                   // bytes per step and warp: both sides
    const int nsteps = t1r - t0 + 1;                              // data of every step is exchanged

    auto issue = [&](int tr) {                                   // row tr -> state slot, p slot
        const bool ok = lane_in && tr >= 0 && tr < ny && tr <= t1r;
        const size_t ro = ok ? (size_t)tr * nx + gi : 0;
        float4* s = sring + ((tr - t0) % kWpStateRing) * (6 * 32);
        float4* pp = pring + (tr & (kWpPRing - 1)) * (2 * 32);
        cp_async16(reinterpret_cast<float*>(s), A.mx_in + po + ro, ok);
        cp_async16(reinterpret_cast<float*>(s + 32), A.my_in + po + ro, ok);
        cp_async16(reinterpret_cast<float*>(s + 64), A.r_in + po + ro, ok);
        cp_async16(reinterpret_cast<float*>(s + 96), A.a_in + po + ro, ok);
        cp_async16(reinterpret_cast<float*>(s + 128), A.x_in + fo + ro, ok);
        cp_async16(reinterpret_cast<float*>(s + 160), A.x_in + fo + A.N + ro, ok);
        cp_async16(reinterpret_cast<float*>(pp), A.p + fo + ro, ok);
        cp_async16(reinterpret_cast<float*>(pp + 32), A.p + fo + A.N + ro, ok);
        cp_commit();
    };
#pragma unroll
    for (int k = 0; k < kWpStateRing * 6; ++k) sring[k * 32] = z4;
#pragma unroll
    for (int k = 0; k < kWpPRing * 2; ++k) pring[k * 32] = z4;
    if (exists) {
#pragma unroll
        for (int k = 0; k < P; ++k) issue(t0 + k);
    }
    if (lane == 0) {
        mbar_init(my_mb, 1);
        mbar_init(my_mb + 8, 1);
    }
    // receive slots start at zero (step t0's reads; a missing neighbour's side stays zero)
    for (int k = 0; k < 4 * (S - 1) + 6; ++k) rbuf[((size_t)k * kWpWarps + w) * 32 + lane] = z4;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // phase 0 of both buffers: the data of steps t0, t0 + 1
    mbar_arm(my_mb, expect, lane == 0 && exists);
    mbar_arm(my_mb + 8, expect, lane == 0 && exists && nsteps > 1);
    cluster_sync();                                              // zeroed slots and barriers visible cluster-wide
    if (!exists) {                 // an empty slot: its neighbours expect nothing from it
        cp_wait<0>();
        pdl_trigger();
        return;
    }

    struct Lv { Quad mx, my, r, a, nk, x0, x1; };
    Lv SA[S], SB[S];
    Quad upY[S + 1];
#pragma unroll
    for (int j = 0; j < S; ++j) { SA[j] = {zq, zq, zq, zq, zq, zq, zq}; SB[j] = SA[j]; }
#pragma unroll
    for (int j = 0; j <= S; ++j) upY[j] = zq;
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f, s_px = 0.f;

    auto step = [&](const int tr, Lv (&Pv)[S], Lv (&Cv)[S]) {
        const int rel = tr - t0;
        const int ibuf = (rel - 1) & 1, obuf = rel & 1;            // buffers of steps tr - 1 (in), tr (out)
        const int p3 = rel % 3, q3 = (rel + 2) % 3;                // rel and rel - 1 mod 3
        {
            issue(tr + P);
            cp_wait<P>();
            const float4* s = sring + p3 * (6 * 32);            // (kWpStateRing == 3)
            float4 Mx = s[0], My = s[32];
            if (last_q) Mx.w = 0.f;                              // pinned flux components (L3)
            if (tr == ny - 1) My = z4;
            const float sh0 = __shfl_up_sync(kFull, Mx.w, 1);
            const Quad qmy = qd(My), qr = qd(s[64]), x0 = qd(s[128]), x1 = qd(s[160]);
            const Quad div0 = qadd(qdiff_left(qd(Mx), left_edge ? 0.f : sh0), qsub(qmy, upY[0]));
            Cv[0].mx = qd(Mx); Cv[0].my = qmy; Cv[0].r = qr; Cv[0].a = qd(s[96]);
            Cv[0].x0 = x0; Cv[0].x1 = x1;
            Cv[0].nk = qadd(qsub(qr, div0), qsub(x1, x0));       // -K^0 = (r - div M) + (x_{t+1} - x_t)
            upY[0] = qmy;
        }
        // the neighbours' pushes of step tr - 1 have landed; re-arm that buffer for step tr + 1
        if (rel > 0) {
            mbar_wait(my_mb + ibuf * 8, (unsigned)((rel - 1) >> 1) & 1u);
            mbar_arm(my_mb + ibuf * 8, expect, lane == 0 && rel + 1 <= nsteps - 1);
            __syncwarp();
        }
        auto publish = [&](int lvl, const Quad& v) {
            st_async4(l_ex ? l_rb + rboff(obuf, p3, 1, lvl, lw) : dummy, f4(v), l_mb + obuf * 8);
            st_async4(r_ex ? r_rb + rboff(obuf, p3, 0, lvl, rw) : dummy, f4(v), r_mb + obuf * 8);
        };
        {
            publish(0, Cv[0].a);
#pragma unroll
            for (int j = 1; j <= S; ++j) {
                const int rho = tr - j;
                const Lv& p = Pv[j - 1];
                // the neighbours' a^{j-1} at row rho (published at step tr - 1)
                const Quad anl = qd(rbuf[rboff(ibuf, q3, 0, j - 1, w) / 16]);
                const Quad anr = qd(rbuf[rboff(ibuf, q3, 1, j - 1, w) / 16]);
                Quad n2, inv, nmx, nmy, rn;
                {
                    Quad qx, qy;
                    const Quad cA = Cv[j - 1].a;
                    const float2 nt1y = pk_dup((rho == -1 || rho == ny - 1) ? 0.f : -t1);
                    const float a5 = __shfl_down_sync(kFull, p.a.l.x, 1);
                    const Quad gx = qdiff_right(p.a, a5), gy = qsub(p.a, cA);
                    qx = {pk_fma(nt1, gx.l, p.mx.l), pk_fma(nt1h, gx.h, p.mx.h)};
                    qy = qfma(nt1y, gy, p.my);
                    n2 = qfma(qy, qy, qmul(qx, qx));
                    inv = {make_float2(rsqrt_ftz(n2.l.x), rsqrt_ftz(n2.l.y)), make_float2(rsqrt_ftz(n2.h.x), rsqrt_ftz(n2.h.y))};
                    Quad sf = qfma(nt1, inv, qd(make_float4(1.f, 1.f, 1.f, 1.f)));
                    sf = {make_float2(fmaxf(sf.l.x, 0.f), fmaxf(sf.l.y, 0.f)), make_float2(fmaxf(sf.h.x, 0.f), fmaxf(sf.h.y, 0.f))};
                    nmx = qmul(sf, qx); nmy = qmul(sf, qy);
                    const Quad q5 = qfma(pk_dup(t1), p.a, p.r);
                    if constexpr (RM == 0) {
                        const Quad cl = {make_float2(fminf(fmaxf(q5.l.x, -at1), at1), fminf(fmaxf(q5.l.y, -at1), at1)),
                                         make_float2(fminf(fmaxf(q5.h.x, -at1), at1), fminf(fmaxf(q5.h.y, -at1), at1))};
                        rn = qsub(q5, cl);
                    } else if constexpr (RM == 1) {
                        rn = qmul(q5, qd(make_float4(rsc, rsc, rsc, rsc)));
                    } else {
                        rn = zq;
                    }
                }
                // line 4: x_t, x_{t+1} from a_{t-1}, a_t, a_{t+1} of level j-1
                const float4* pr = pring + (rho & (kWpPRing - 1)) * (2 * 32);
                const Quad p0 = qd(pr[0]), p1 = qd(pr[32]);
                Quad x0n = qfma(c1, p0, qfma(c2, p.x0, qmul(qd(make_float4(nc3.x, nc3.x, nc3.x, nc3.x)), qsub(p.a, anl))));
                x0n = {make_float2(fmaxf(x0n.l.x, 0.f), fmaxf(x0n.l.y, 0.f)), make_float2(fmaxf(x0n.h.x, 0.f), fmaxf(x0n.h.y, 0.f))};
                if (fix0) x0n = p.x0;
                Quad x1n = qfma(c1, p1, qfma(c2, p.x1, qmul(qd(make_float4(nc3.x, nc3.x, nc3.x, nc3.x)), qsub(anr, p.a))));
                x1n = {make_float2(fmaxf(x1n.l.x, 0.f), fmaxf(x1n.l.y, 0.f)), make_float2(fmaxf(x1n.h.x, 0.f), fmaxf(x1n.h.y, 0.f))};
                const Quad fn = qsub(x1n, x0n);
                // lines 6-7: -K^j = (r^j - div M^j) + (x_{t+1} - x_t);  a^j = a^{j-1} + tau2 (2 K^j - K^{j-1})
                const float shl = __shfl_up_sync(kFull, nmx.h.y, 1);
                const Quad divn = qadd(qdiff_left(nmx, left_edge ? 0.f : shl), qsub(nmy, upY[j]));
                const Quad nkn = qadd(qsub(rn, divn), fn);
                const Quad an = qfma(pk_dup(t2), qfma(pk_dup(-2.f), nkn, p.nk), p.a);
                if (RED && j == S) {
                    const float wr = (writer && rho >= y0 && rho < y1) ? 1.f : 0.f;
                    const float wl = own_last ? wr : 0.f;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const float n2v = qc(n2, v), invv = qc(inv, v), rv = qc(rn, v), kv = qc(nkn, v);
                        const float nrm = fmaxf(fmaf(n2v, fminf(invv, 1e30f), -t1), 0.f);
                        const float dmx = qc(nmx, v) - qc(p.mx, v), dmy = qc(nmy, v) - qc(p.my, v), dr = rv - qc(p.r, v);
                        const float d0 = qc(x0n, v) - qc(p.x0, v), e0 = qc(x0n, v) - qc(p0, v);
                        const float d1 = qc(x1n, v) - qc(p.x1, v), e1 = qc(x1n, v) - qc(p1, v);
                        s_tr = fmaf(wr, nrm, s_tr);
                        s_gr = fmaf(wr, pw(rv, RM), s_gr);
                        s_k2 = fmaf(wr * kv, kv, s_k2);
                        s_dz = fmaf(wr, dmx * dmx + dmy * dmy + dr * dr + d0 * d0, s_dz);
                        s_dz = fmaf(wl, d1 * d1, s_dz);
                        s_ub = fmaf(wr, pw(qc(divn, v) - qc(fn, v), RM), s_ub);
                        s_px = fmaf(wr, e0 * e0, s_px);
                        s_px = fmaf(wl, e1 * e1, s_px);
                    }
                }
                upY[j] = nmy;
                if (j < S) {
                    Cv[j].mx = nmx; Cv[j].my = nmy; Cv[j].r = rn; Cv[j].a = an; Cv[j].nk = nkn;
                    Cv[j].x0 = x0n; Cv[j].x1 = x1n;
                    publish(j, an);               // a^j depends on this level's reads
                } else {
                    const bool wp = writer && rho >= y0 && rho < y1;
                    const size_t go = (size_t)rho * nx + gi;
                    st4_if(A.mx_out + po + go, f4(nmx), wp);
                    st4_if(A.my_out + po + go, f4(nmy), wp);
                    st4_if(A.r_out + po + go, f4(rn), wp);
                    st4_if(A.a_out + po + go, f4(an), wp);
                    st4_if(A.x_out + fo + go, f4(x0n), wp);
                    st4_if(A.x_out + fo + A.N + go, f4(x1n), wp && own_last);
                }
            }
        }
    };
    int tr = t0;
#pragma unroll 1
    for (; tr + 1 <= t1r; tr += 2) {
        step(tr, SA, SB);
        step(tr + 1, SB, SA);
    }
    if (tr <= t1r) step(tr, SA, SB);
    // the last step's pushes (into this warp's buffers) have landed: no push is in flight to an exited CTA
    mbar_wait(my_mb + ((nsteps - 1) & 1) * 8, (unsigned)((nsteps - 1) >> 1) & 1u);
    cp_wait<0>();
    pdl_trigger();
    if constexpr (RED) {
        if (out_pair) {
            double v[6] = {s_tr, s_gr, s_k2, s_dz, s_ub, s_px};
#pragma unroll
            for (int k = 0; k < 6; ++k) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(kFull, v[k], o);
            }
            if (lane == 0) {
                const int upp = A.strips * A.segs;
                double* Pp = A.partials + (((size_t)b * Pc + t) * upp + u) * kRec;
#pragma unroll
                for (int k = 0; k < 6; ++k) Pp[k] = v[k];
                Pp[6] = 0.0; Pp[7] = 0.0;
            }
        }
    }
}

}  // namespace uotk
