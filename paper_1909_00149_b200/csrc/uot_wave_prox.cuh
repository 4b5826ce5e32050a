// uot_wave_prox.cuh -- chain prox (rho < inf, L19): S Algorithm-1 iterations per HBM pass.
//
// Algorithm 1 with frame updates (P:313-317, line 4 = P:314 generalised to the chain, L19):
// the dual a_t of pair t enters the x-update of frames t and t+1, and x_t, x_{t+1} enter K_t,
// so iteration k+1 of pair t needs iteration k of pairs t-1, t, t+1 at the same pixel (the
// coupling across pairs is pointwise; across pixels it is the 5-point stencil of k_wave).
//
// Layout: the register wavefront of k_wave_pk (uot_wave_pk.cuh) runs one warp per pair --
// a strip of 32 V columns (V = 4 by default: 128 columns; V = 2: 64) marching down H + 2S rows,
// level j updating row rho - j at step rho --
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
// step's pushes are waited for too, so no push reaches a CTA that has exited.  Frames are
// recomputed by both pairs that use them: the warp of
// pair t carries x_t and x_{t+1} per level (bit-identical to its neighbours' copies: same
// inputs, same operations), so nothing is exchanged within a step.
//
// Pair groups: a cluster of CL CTAs x NW warps (NW = 8 at V = 4; 12 or 16 at V = 2) holds CL*NW
// consecutive pairs of one chain (the CTA-boundary neighbours sit in the adjacent CTA's shared
// memory).  After S levels a pair is exact iff its S neighbours on both sides are in the group
// (the dependency cone), so a group writes the middle CL*NW - 2S pairs; pairs outside the chain (t < 0, t >= P) are empty slots
// whose a is the chain end's a_{-1} = a_{T-1} := 0 exactly (L19).  HBM traffic per pass and
// pair-pixel: M, r, a, x_t, p_t read (x_{t+1}, p_{t+1} are the next pair's, L2 hits) and M, r,
// a, x_t written: 44 B per S iterations, plus the 2S halo pairs of each group.
#pragma once
#include "uot_wave_pk.cuh"

namespace uotk {

// Lane layouts: V = 4 columns per lane (one float4 quad, 128-column strips, 8 warps = 8 pairs per
// CTA; the round-2 kernel) or V = 2 (one fp32x2 pair, 64-column strips, 16 warps per CTA: half
// the registers per warp, twice the warps per SM for the latency-bound pass).
// Same arithmetic per pixel either way (the packed ops of k_wave_pk).
struct Duo { float2 l; };                 // columns (c, c+1) of one lane
__device__ __forceinline__ Duo qadd(const Duo& a, const Duo& b) { return {pk_add(a.l, b.l)}; }
__device__ __forceinline__ Duo qsub(const Duo& a, const Duo& b) { return {pk_sub(a.l, b.l)}; }
__device__ __forceinline__ Duo qmul(const Duo& a, const Duo& b) { return {pk_mul(a.l, b.l)}; }
__device__ __forceinline__ Duo qfma(float2 s, const Duo& b, const Duo& c) { return {pk_fma(s, b.l, c.l)}; }
__device__ __forceinline__ Duo qfma(const Duo& a, const Duo& b, const Duo& c) { return {pk_fma(a.l, b.l, c.l)}; }
__device__ __forceinline__ float qc(const Duo& q, int v) { return v == 0 ? q.l.x : q.l.y; }
__device__ __forceinline__ Duo qdiff_right(const Duo& q, float right) { return {make_float2(q.l.x - q.l.y, q.l.y - right)}; }
__device__ __forceinline__ Duo qdiff_left(const Duo& q, float left) { return {make_float2(q.l.x - left, q.l.y - q.l.x)}; }

template <int V> struct WpLane;
template <> struct WpLane<4> {
    using T = Quad; using M = float4;
    __device__ static T ld(const M& m) { return qd(m); }
    __device__ static M st(const T& t) { return f4(t); }
    __device__ static T splat(float v) { return qd(make_float4(v, v, v, v)); }
    __device__ static float first(const T& t) { return t.l.x; }
    __device__ static float last(const T& t) { return t.h.y; }
    __device__ static void zero_last(M& m) { m.w = 0.f; }
    __device__ static T relu(const T& t) {
        return {make_float2(fmaxf(t.l.x, 0.f), fmaxf(t.l.y, 0.f)), make_float2(fmaxf(t.h.x, 0.f), fmaxf(t.h.y, 0.f))};
    }
    __device__ static T clampv(const T& t, float c) {
        return {make_float2(fminf(fmaxf(t.l.x, -c), c), fminf(fmaxf(t.l.y, -c), c)),
                make_float2(fminf(fmaxf(t.h.x, -c), c), fminf(fmaxf(t.h.y, -c), c))};
    }
    __device__ static T rsq(const T& t) {
        return {make_float2(rsqrt_ftz(t.l.x), rsqrt_ftz(t.l.y)), make_float2(rsqrt_ftz(t.h.x), rsqrt_ftz(t.h.y))};
    }
    // -tau1 per column with the pinned column (the lane's last) scaled by 0 when `pin`
    __device__ static T nt1x(float nt1, bool pin) { return {pk_dup(nt1), make_float2(nt1, pin ? 0.f : nt1)}; }
    __device__ static void cp(float* s, const float* g, bool ok) { cp_async16(s, g, ok); }
    __device__ static void st_if(float* g, const T& v, bool p) { st4_if(g, f4(v), p); }
};
template <> struct WpLane<2> {
    using T = Duo; using M = float2;
    __device__ static T ld(const M& m) { return {m}; }
    __device__ static M st(const T& t) { return t.l; }
    __device__ static T splat(float v) { return {make_float2(v, v)}; }
    __device__ static float first(const T& t) { return t.l.x; }
    __device__ static float last(const T& t) { return t.l.y; }
    __device__ static void zero_last(M& m) { m.y = 0.f; }
    __device__ static T relu(const T& t) { return {make_float2(fmaxf(t.l.x, 0.f), fmaxf(t.l.y, 0.f))}; }
    __device__ static T clampv(const T& t, float c) { return {make_float2(fminf(fmaxf(t.l.x, -c), c), fminf(fmaxf(t.l.y, -c), c))}; }
    __device__ static T rsq(const T& t) { return {make_float2(rsqrt_ftz(t.l.x), rsqrt_ftz(t.l.y))}; }
    __device__ static T nt1x(float nt1, bool pin) { return {make_float2(nt1, pin ? 0.f : nt1)}; }
    __device__ static void cp(float* s, const float* g, bool ok) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0) : "memory");
    }
    __device__ static void st_if(float* g, const T& v, bool p) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.f32 [%0], {%1, %2};\n\t}"
                     :: "l"(g), "f"(v.l.x), "f"(v.l.y), "r"((int)p));
    }
};
constexpr int kWpWarps = 8;               // warps (pairs) per CTA of the V = 4 kernel
constexpr int kWpStateRing = 3;           // rows of the state ring (M, r, a, x_t, x_{t+1}): current + 2 ahead
constexpr int kWpPRing = 8;               // rows of the p ring (p_t, p_{t+1} at the level rows)
// halo lanes / written columns / strips of a V-column-per-lane strip (32 V columns)
__host__ __device__ constexpr int wp_halo_lanes(int S, int V) { return (S + V - 1) / V; }
__host__ __device__ constexpr int wp_out(int S, int V) { return 32 * V - 2 * V * wp_halo_lanes(S, V); }
__host__ __device__ constexpr int wp_strips(int nx, int S, int V) {
    return nx <= 32 * V ? 1 : (nx - 32 * V + wp_out(S, V) - 1) / wp_out(S, V) + 1;
}
template <int S, int V = 4, int NW = (V == 4 ? 8 : 16)> struct WpCfg {
    static constexpr int W = NW;                                  // warps (pairs) per CTA
    static constexpr int P = kWpStateRing - 1;                    // rows in flight ahead
    static_assert(S + P + 1 <= kWpPRing, "p ring holds rows rho - S .. rho + P");
    static constexpr size_t warp_floats = (size_t)(kWpStateRing * 6 + kWpPRing * 2) * 32 * V;
    // receive buffers: levels 0 .. S-2 [2 bufs][2 sides][S-1][warp][lane], level S-1 [3 bufs][2 sides][warp][lane],
    // then one dummy slot per warp [warp][lane]
    static constexpr size_t rb_floats = (size_t)(2 * 2 * (S - 1) + 3 * 2 + 1) * W * 32 * V;
#ifndef UOT_PROX_UY
#define UOT_PROX_UY 1
#endif
    // UOT_PROX_UY (default 1): each level's M_y of the previous row (div M's upper neighbour) in
    // shared memory instead of registers -- frees 16 registers per thread at S = 3 (spills 60 / 136
    // -> 48 / 80 B) and measured 1.831e11 vs 1.820e11 px-it/s on C4 chain prox (passes of 2), 1.731e11
    // vs 1.713e11 (3-first), the same on two repeats (scripts/gpu_r02c_ab_uy.sh)
    static constexpr size_t uy_floats = UOT_PROX_UY ? (size_t)(S + 1) * 32 * V : 0;
    static constexpr size_t smem = (warp_floats * W + rb_floats + uy_floats * W) * sizeof(float) + W * 2 * 8;
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

__device__ __forceinline__ void st_async2(unsigned addr, float2 v, unsigned bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                 :: "r"(addr), "f"(v.x), "f"(v.y), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_v(unsigned addr, float4 v, unsigned bar) { st_async4(addr, v, bar); }
__device__ __forceinline__ void st_async_v(unsigned addr, float2 v, unsigned bar) { st_async2(addr, v, bar); }

template <int S, int RM, bool RED, int V = 4, int NWT = (V == 4 ? 8 : 16)>
__global__ void __launch_bounds__(NWT * 32, 1) k_wave_prox(const WaveProxArgs A) {
    static_assert(S >= 2 && S <= 3, "levels per pass (S = 4: 255 registers and spills; shared memory)");
    using C = WpCfg<S, V, NWT>;
    using L = WpLane<V>;
    using T = typename L::T;
    using Mv = typename L::M;
    constexpr int NW = C::W;                                      // warps (pairs) per CTA
    constexpr int HL = wp_halo_lanes(S, V), OUT = wp_out(S, V), P = C::P;
    constexpr int SW = 32 * V;                                    // strip width (columns)
    constexpr unsigned VB = (unsigned)sizeof(Mv);                 // bytes per lane and row
    extern __shared__ __align__(16) float4 wpsm_raw[];
    Mv* const wpsm = reinterpret_cast<Mv*>(wpsm_raw);
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
    const int q = rank * NW + w;                                  // slot in the group
    const int t = lo - S + q;                                     // pair of this warp
    const bool exists = t >= 0 && t < Pc && t < hi + S;
    const bool out_pair = t >= lo && t < hi;
    const bool has_l = q > 0, has_r = q < CL * NW - 1;            // neighbour slots in the cluster
    const int nx = A.nx, ny = A.ny;
    const int gs = sx * OUT, gi = gs + V * lane;
    const bool lane_in = gi < nx;
    const bool last_q = gi + V - 1 == nx - 1;
    const bool left_edge = lane == 0 && sx == 0;
    const bool writer = out_pair && lane_in && (lane >= HL || sx == 0) && (lane <= 31 - HL || gs + SW >= nx);
    const int y0 = sy * A.H, y1 = min(y0 + A.H, ny);
    const int t0 = y0 - S, t1r = y1 - 1 + S;
    const size_t po = ((size_t)b * Pc + (size_t)(exists ? t : 0)) * (size_t)A.N;    // pair planes
    const size_t fo = ((size_t)b * A.T + (size_t)(exists ? t : 0)) * (size_t)A.N;   // frame t
    const float t1 = A.tau1, t2 = A.tau2, at1 = A.atau1, rsc = A.r_scale;
    const float2 c1 = pk_dup(A.c1), c2 = pk_dup(A.c2);
    const T nc3 = L::splat(-A.c3);
    const bool fix0 = A.fix_first && t == 0;                      // constant first frame
    const bool own_last = t == Pc - 1 && A.own_hi == Pc;          // also owns frame T-1 (writes, reductions)
    const float2 nt1 = pk_dup(-t1);
    const T nt1v = L::nt1x(-t1, last_q);                          // the pinned column nx-1 takes 0 (L3)

    Mv* sring = wpsm + (size_t)w * (C::warp_floats / V) + lane;           // [slot][6][lane]
    Mv* pring = sring + kWpStateRing * 6 * 32;                             // [slot][2][lane]
    Mv* rbuf = wpsm + (size_t)NW * (C::warp_floats / V);                   // see WpCfg::rb_floats
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(rbuf + C::rb_floats / V);   // [warp][buf]
    Mv zm;
    if constexpr (V == 4) zm = make_float4(0.f, 0.f, 0.f, 0.f); else zm = make_float2(0.f, 0.f);
    const T zq = L::ld(zm);
    // neighbour slots: the same CTA (warp +- 1) or the adjacent CTA of the cluster; a neighbour
    // that is an empty slot (outside the chain or past the group's halo) sends nothing: its a is 0
    auto slot_exists = [&](int tt) { return tt >= 0 && tt < Pc && tt < hi + S; };
    const bool l_ex = has_l && slot_exists(t - 1), r_ex = has_r && slot_exists(t + 1);
    const unsigned lw = w > 0 ? (unsigned)(w - 1) : (unsigned)(NW - 1);
    const unsigned rw = w < NW - 1 ? (unsigned)(w + 1) : 0u;
    const unsigned lrank = w > 0 ? (unsigned)rank : (unsigned)(rank - 1);
    const unsigned rrank = w < NW - 1 ? (unsigned)rank : (unsigned)(rank + 1);
    // byte offset of (step parity p2 = rel & 1, rel mod 3 = p3, side, level) for warp ww
    auto rboff = [&](int p2, int p3, int side, int lvl, unsigned ww) {
        const int k = lvl < S - 1 ? (p2 * 2 + side) * (S - 1) + lvl : 4 * (S - 1) + p3 * 2 + side;
        return (unsigned)(((k * NW + (int)ww) * 32 + lane) * VB);
    };
    const unsigned rb_base = smem_u32(rbuf), mb_base = smem_u32(mbar);
    const unsigned my_mb = mb_base + (unsigned)w * 16u;
    const unsigned dummy = rb_base + (unsigned)((((4 * (S - 1) + 6) * NW + w) * 32 + lane) * VB);
    // pushes to the left neighbour land in its side 1 ("from the right"), to the right one in side 0;
    // a missing side's pushes go to the dummy slot and complete on this warp's own mbarrier
    const unsigned l_rb = l_ex ? map_rank(rb_base, lrank) : 0u, r_rb = r_ex ? map_rank(rb_base, rrank) : 0u;
    const unsigned l_mb = l_ex ? map_rank(mb_base + lw * 16u, lrank) : my_mb;
    const unsigned r_mb = r_ex ? map_rank(mb_base + rw * 16u, rrank) : my_mb;
    const unsigned expect = 2u * S * 32u * VB;                    // bytes per step and warp: both sides
    const int nsteps = t1r - t0 + 1;                              // data of every step is exchanged

    auto issue = [&](int tr) {                                   // row tr -> state slot, p slot
        const bool ok = lane_in && tr >= 0 && tr < ny && tr <= t1r;
        const size_t ro = ok ? (size_t)tr * nx + gi : 0;
        Mv* s = sring + ((tr - t0) % kWpStateRing) * (6 * 32);
        Mv* pp = pring + (tr & (kWpPRing - 1)) * (2 * 32);
        L::cp(reinterpret_cast<float*>(s), A.mx_in + po + ro, ok);
        L::cp(reinterpret_cast<float*>(s + 32), A.my_in + po + ro, ok);
        L::cp(reinterpret_cast<float*>(s + 64), A.r_in + po + ro, ok);
        L::cp(reinterpret_cast<float*>(s + 96), A.a_in + po + ro, ok);
        L::cp(reinterpret_cast<float*>(s + 128), A.x_in + fo + ro, ok);
        L::cp(reinterpret_cast<float*>(s + 160), A.x_in + fo + A.N + ro, ok);
        L::cp(reinterpret_cast<float*>(pp), A.p + fo + ro, ok);
        L::cp(reinterpret_cast<float*>(pp + 32), A.p + fo + A.N + ro, ok);
        cp_commit();
    };
#pragma unroll
    for (int k = 0; k < kWpStateRing * 6; ++k) sring[k * 32] = zm;
#pragma unroll
    for (int k = 0; k < kWpPRing * 2; ++k) pring[k * 32] = zm;
    if (exists) {
#pragma unroll
        for (int k = 0; k < P; ++k) issue(t0 + k);
    }
    if (lane == 0) {
        mbar_init(my_mb, 1);
        mbar_init(my_mb + 8, 1);
    }
    // receive slots start at zero (step t0's reads; a missing neighbour's side stays zero)
    for (int k = 0; k < 4 * (S - 1) + 6; ++k) rbuf[((size_t)k * NW + w) * 32 + lane] = zm;
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

    struct Lv { T mx, my, r, a, nk, x0, x1; };
    Lv SA[S], SB[S];
    T upY_r[UOT_PROX_UY ? 1 : S + 1];
    Mv* const uyb = reinterpret_cast<Mv*>(mbar + NW * 2) + (size_t)w * (S + 1) * 32 + lane;
    auto upy_get = [&](int j) -> T { if constexpr (UOT_PROX_UY != 0) return L::ld(uyb[j * 32]); else return upY_r[j]; };
    auto upy_set = [&](int j, const T& v) { if constexpr (UOT_PROX_UY != 0) uyb[j * 32] = L::st(v); else upY_r[j] = v; };
#pragma unroll
    for (int j = 0; j < S; ++j) { SA[j] = {zq, zq, zq, zq, zq, zq, zq}; SB[j] = SA[j]; }
#pragma unroll
    for (int j = 0; j <= S; ++j) upy_set(j, zq);
    float s_tr = 0.f, s_gr = 0.f, s_k2 = 0.f, s_dz = 0.f, s_ub = 0.f, s_px = 0.f;

    auto step = [&](const int tr, Lv (&Pv)[S], Lv (&Cv)[S]) {
        const int rel = tr - t0;
        const int ibuf = (rel - 1) & 1, obuf = rel & 1;            // buffers of steps tr - 1 (in), tr (out)
        const int p3 = rel % 3, q3 = (rel + 2) % 3;                // rel and rel - 1 mod 3
        {
            issue(tr + P);
            cp_wait<P>();
            const Mv* s = sring + p3 * (6 * 32);                  // (kWpStateRing == 3)
            Mv Mx = s[0], My = s[32];
            if (last_q) L::zero_last(Mx);                         // pinned flux components (L3)
            if (tr == ny - 1) My = zm;
            const T qmx = L::ld(Mx);
            const float sh0 = __shfl_up_sync(kFull, L::last(qmx), 1);
            const T qmy = L::ld(My), qr = L::ld(s[64]), x0 = L::ld(s[128]), x1 = L::ld(s[160]);
            const T div0 = qadd(qdiff_left(qmx, left_edge ? 0.f : sh0), qsub(qmy, upy_get(0)));
            Cv[0].mx = qmx; Cv[0].my = qmy; Cv[0].r = qr; Cv[0].a = L::ld(s[96]);
            Cv[0].x0 = x0; Cv[0].x1 = x1;
            Cv[0].nk = qadd(qsub(qr, div0), qsub(x1, x0));       // -K^0 = (r - div M) + (x_{t+1} - x_t)
            upy_set(0, qmy);
        }
        // the neighbours' pushes of step tr - 1 have landed; re-arm that buffer for step tr + 1
        if (rel > 0) {
            mbar_wait(my_mb + ibuf * 8, (unsigned)((rel - 1) >> 1) & 1u);
            mbar_arm(my_mb + ibuf * 8, expect, lane == 0 && rel + 1 <= nsteps - 1);
            __syncwarp();
        }
        auto publish = [&](int lvl, const T& v) {
            st_async_v(l_ex ? l_rb + rboff(obuf, p3, 1, lvl, lw) : dummy, L::st(v), l_mb + obuf * 8);
            st_async_v(r_ex ? r_rb + rboff(obuf, p3, 0, lvl, rw) : dummy, L::st(v), r_mb + obuf * 8);
        };
        {
            publish(0, Cv[0].a);
#pragma unroll
            for (int j = 1; j <= S; ++j) {
                const int rho = tr - j;
                const Lv& p = Pv[j - 1];
                // the neighbours' a^{j-1} at row rho (published at step tr - 1)
                const T anl = L::ld(rbuf[rboff(ibuf, q3, 0, j - 1, w) / VB]);
                const T anr = L::ld(rbuf[rboff(ibuf, q3, 1, j - 1, w) / VB]);
                T n2, inv, nmx, nmy, rn;
                {
                    T qx, qy;
                    const T cA = Cv[j - 1].a;
                    const float2 nt1y = pk_dup((rho == -1 || rho == ny - 1) ? 0.f : -t1);
                    const float a5 = __shfl_down_sync(kFull, L::first(p.a), 1);
                    const T gx = qdiff_right(p.a, a5), gy = qsub(p.a, cA);
                    qx = qfma(nt1v, gx, p.mx);
                    qy = qfma(nt1y, gy, p.my);
                    n2 = qfma(qy, qy, qmul(qx, qx));
                    inv = L::rsq(n2);
                    const T sf = L::relu(qfma(nt1, inv, L::splat(1.f)));
                    nmx = qmul(sf, qx); nmy = qmul(sf, qy);
                    const T q5 = qfma(pk_dup(t1), p.a, p.r);
                    if constexpr (RM == 0) {
                        rn = qsub(q5, L::clampv(q5, at1));
                    } else if constexpr (RM == 1) {
                        rn = qmul(q5, L::splat(rsc));
                    } else {
                        rn = zq;
                    }
                }
                // line 4: x_t, x_{t+1} from a_{t-1}, a_t, a_{t+1} of level j-1
                const Mv* pr = pring + (rho & (kWpPRing - 1)) * (2 * 32);
                const T p0 = L::ld(pr[0]), p1 = L::ld(pr[32]);
                T x0n = L::relu(qfma(c1, p0, qfma(c2, p.x0, qmul(nc3, qsub(p.a, anl)))));
                if (fix0) x0n = p.x0;
                const T x1n = L::relu(qfma(c1, p1, qfma(c2, p.x1, qmul(nc3, qsub(anr, p.a)))));
                const T fn = qsub(x1n, x0n);
                // lines 6-7: -K^j = (r^j - div M^j) + (x_{t+1} - x_t);  a^j = a^{j-1} + tau2 (2 K^j - K^{j-1})
                const float shl = __shfl_up_sync(kFull, L::last(nmx), 1);
                const T divn = qadd(qdiff_left(nmx, left_edge ? 0.f : shl), qsub(nmy, upy_get(j)));
                const T nkn = qadd(qsub(rn, divn), fn);
                const T an = qfma(pk_dup(t2), qfma(pk_dup(-2.f), nkn, p.nk), p.a);
                if (RED && j == S) {
                    const float wr = (writer && rho >= y0 && rho < y1) ? 1.f : 0.f;
                    const float wl = own_last ? wr : 0.f;
#pragma unroll
                    for (int v = 0; v < V; ++v) {
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
                upy_set(j, nmy);
                if (j < S) {
                    Cv[j].mx = nmx; Cv[j].my = nmy; Cv[j].r = rn; Cv[j].a = an; Cv[j].nk = nkn;
                    Cv[j].x0 = x0n; Cv[j].x1 = x1n;
                    publish(j, an);               // a^j depends on this level's reads
                } else {
                    const bool wp = writer && rho >= y0 && rho < y1;
                    const size_t go = (size_t)rho * nx + gi;
                    L::st_if(A.mx_out + po + go, nmx, wp);
                    L::st_if(A.my_out + po + go, nmy, wp);
                    L::st_if(A.r_out + po + go, rn, wp);
                    L::st_if(A.a_out + po + go, an, wp);
                    L::st_if(A.x_out + fo + go, x0n, wp);
                    L::st_if(A.x_out + fo + A.N + go, x1n, wp && own_last);
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
