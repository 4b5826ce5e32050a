// uot_api.cu -- C-ABI (include/uot.h) over the sm_100a kernels of the fused
// Algorithm-1 iteration (arXiv 1909.00149).
//
// The library owns no device memory: every buffer, including the fp64
// reduction scratch, is caller-owned (PyTorch tensors in the Python binding).
// Everything is enqueued on the stream bound at uot_create; host synchronisation
// happens only when a host report is requested.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: named ranges for nsys / ncu --nvtx (no-ops without a tool)

#include "uot.h"
#include "uot_kernels.cuh"
#include "uot_persist.cuh"
#include "uot_temporal.cuh"
#include "uot_wave.cuh"
#include "uot_wave_pk.cuh"
#include "uot_wave_n.cuh"
#include "uot_wave_prox.cuh"

using namespace uotk;

// TMA descriptor of a [G][ny][nx] fp32 plane stack, box kRW x rows x 1, zero fill out of bounds
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        else
            cudaGetLastError();
    }
    return fn;
}
static bool encode_plane_map(CUtensorMap* m, const float* base, int nx, int ny, int G, int box_rows) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn || !base) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)G};
    const cuuint64_t strides[2] = {(cuuint64_t)nx * 4, (cuuint64_t)nx * ny * 4};
    const cuuint32_t box[3] = {(cuuint32_t)kRW, (cuuint32_t)box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// One temporally blocked variant (S fused iterations per pass, TH interior rows per tile):
// its kernels (without / with reductions), launch shape and TMA tensor maps.
struct TVar {
    int S, th, tx, ty, rows, threads;
    size_t smem;
    bool ok, tma;
    bool wave;                                 // register wavefront k_wave (tx strips x ty segments of th rows)
    int vn;                                    // wave: columns per lane (4: k_wave_pk / k_wave, 128-column strips;
                                               // 2: k_wave_n, 64-column strips)
    const void* fn[2];
    CUtensorMap mx[2], my[2], a[2], r[2], f;   // [G][ny][nx] views, box 72 x rows
};

template <int TH, int S, int RM>
static bool tvar_fill(TVar& v, bool wide) {
    using namespace uotk;
    v.S = S; v.th = TH; v.rows = TB<TH, S>::RH; v.smem = TB<TH, S>::smem;
    v.threads = wide ? kT2Wide : kT2Threads;
    v.fn[0] = wide ? (const void*)k_iter2<TH, S, false, kT2Wide, RM> : (const void*)k_iter2<TH, S, false, kT2Threads, RM>;
    v.fn[1] = wide ? (const void*)k_iter2<TH, S, true, kT2Wide, RM> : (const void*)k_iter2<TH, S, true, kT2Threads, RM>;
    bool ok = true;
    for (const void* f : v.fn)
        ok = ok && cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem) == cudaSuccess;
    return ok;
}

// pk: the packed fp32x2 instruction stream (k_wave_pk, default) or the scalar k_wave (UOT_WAVE_PK=0)
template <int S, int RM>
static bool wvar_fill(TVar& v, bool pk) {
    using namespace uotk;
    v.S = S; v.wave = true; v.tma = false; v.threads = kWaveWarps * 32; v.smem = kWaveSmem;
    v.fn[0] = pk ? (const void*)k_wave_pk<S, RM, false> : (const void*)k_wave<S, RM, false>;
    v.fn[1] = pk ? (const void*)k_wave_pk<S, RM, true> : (const void*)k_wave<S, RM, true>;
    bool ok = true;
    for (const void* f : v.fn)
        ok = ok && cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem) == cudaSuccess;
    return ok;
}

// narrow strips: k_wave_n (one fp32x2 column pair per lane, 64 columns per warp)
template <int S, int RM>
static bool wvar_fill_n(TVar& v) {
    using namespace uotk;
    v.S = S; v.wave = true; v.tma = false; v.threads = 32; v.smem = kWaveNSmem;
    v.fn[0] = (const void*)k_wave_n<S, RM, false>;
    v.fn[1] = (const void*)k_wave_n<S, RM, true>;
    bool ok = true;
    for (const void* f : v.fn)
        ok = ok && cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem) == cudaSuccess;
    return ok;
}

static bool wvar_select(TVar& v, int S, int rm, bool pk) {
    if (v.vn == 2) {
        if (S == 5) return rm == 1 ? wvar_fill_n<5, 1>(v) : (rm == 2 ? wvar_fill_n<5, 2>(v) : wvar_fill_n<5, 0>(v));
        if (S == 4) return rm == 1 ? wvar_fill_n<4, 1>(v) : (rm == 2 ? wvar_fill_n<4, 2>(v) : wvar_fill_n<4, 0>(v));
        if (S == 3) return rm == 1 ? wvar_fill_n<3, 1>(v) : (rm == 2 ? wvar_fill_n<3, 2>(v) : wvar_fill_n<3, 0>(v));
        return rm == 1 ? wvar_fill_n<2, 1>(v) : (rm == 2 ? wvar_fill_n<2, 2>(v) : wvar_fill_n<2, 0>(v));
    }
    if (S == 5) return rm == 1 ? wvar_fill<5, 1>(v, pk) : (rm == 2 ? wvar_fill<5, 2>(v, pk) : wvar_fill<5, 0>(v, pk));
    if (S == 4) return rm == 1 ? wvar_fill<4, 1>(v, pk) : (rm == 2 ? wvar_fill<4, 2>(v, pk) : wvar_fill<4, 0>(v, pk));
    if (S == 3) return rm == 1 ? wvar_fill<3, 1>(v, pk) : (rm == 2 ? wvar_fill<3, 2>(v, pk) : wvar_fill<3, 0>(v, pk));
    return rm == 1 ? wvar_fill<2, 1>(v, pk) : (rm == 2 ? wvar_fill<2, 2>(v, pk) : wvar_fill<2, 0>(v, pk));
}

template <int TH, int S>
static bool tvar_fill_m(TVar& v, bool wide, int rm) {
    return rm == 1 ? tvar_fill<TH, S, 1>(v, wide) : (rm == 2 ? tvar_fill<TH, S, 2>(v, wide) : tvar_fill<TH, S, 0>(v, wide));
}

// Supported (S, TH): S = 2 with TH = 32; S = 4 with TH in {32, 36}.
static bool tvar_select(TVar& v, int S, int th, bool wide, int rm) {
    if (S == 3 || S == 5) return false;         // SMEM tiles: two or four iterations per pass
    if (S == 4) return th == 32 ? tvar_fill_m<32, 4>(v, wide, rm) : tvar_fill_m<36, 4>(v, wide, rm);
    return tvar_fill_m<32, 2>(v, wide, rm);
}

// ============================================================================ kernels
namespace uotk {

// Fixed-order block reduction of one double (256 threads): warp butterfly, then
// warp 0 over the 8 warp sums.  Same inputs -> same bits.
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(kFull, r, o);
    }
    return r;   // valid in thread 0
}

__device__ __forceinline__ double block_max(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(kFull, r, o));
    }
    return r;
}

__global__ void __launch_bounds__(256) k_setup_f(const SetupArgs S) {
    __shared__ double sh[32];
    const int g = blockIdx.y;
    const int b = g / S.P, t = g % S.P;
    const float* x0 = S.frames + ((size_t)b * S.T + t) * (size_t)S.N;
    const float* x1 = x0 + S.N;
    float* f = S.f ? S.f + (size_t)g * S.N : nullptr;
    double s2 = 0.0, s1 = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < S.N;
         k += (long long)S.bpp * blockDim.x) {
        const float v = x1[k] - x0[k];                    // f = x_{t+1} - x_t (L1)
        if (S.f) f[k] = v;
        s2 += (double)v * v;
        s1 += fabs((double)v);
    }
    s2 = block_sum(s2, sh);
    s1 = block_sum(s1, sh);
    if (threadIdx.x == 0) {
        double* P = S.partials + ((size_t)g * S.bpp + blockIdx.x) * kRec;
        P[0] = s2; P[1] = s1;
        for (int q = 2; q < kRec; ++q) P[q] = 0.0;
    }
}

__global__ void __launch_bounds__(256) k_objective(const ObjArgs O) {
    __shared__ double sh[32];
    const int g = blockIdx.y;
    const int b = g / O.P, t = g % O.P;
    const int nx = O.nx, ny = O.ny;
    const size_t po = (size_t)g * O.N;
    const float* x0 = O.x + ((size_t)b * O.T + t) * (size_t)O.N;
    const float* x1 = x0 + O.N;
    const float* mx = O.mx + po;
    const float* my = O.my + po;
    const float* r = O.r + po;
    const float* a = O.a + po;
    double tr = 0, gr = 0, ub = 0, af = 0, mg = 0, ma = 0, px = 0, a2 = 0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < O.N;
         k += (long long)O.bpp * blockDim.x) {
        const int i = (int)(k % nx), j = (int)(k / nx);
        const double mxk = (i < nx - 1) ? mx[k] : 0.0;
        const double myk = (j < ny - 1) ? my[k] : 0.0;
        const double mxl = (i >= 1) ? mx[k - 1] : 0.0;          // i-1 < nx-1 always
        const double myu = (j >= 1) ? my[k - nx] : 0.0;
        const double dv = (mxk - mxl) + (myk - myu);             // div M
        const double f = (double)(x1[k] - x0[k]);
        const double u = dv - f, rk = (double)r[k];
        tr += sqrt(mxk * mxk + myk * myk);
        gr += O.p2 ? rk * rk : fabs(rk);
        ub += O.p2 ? u * u : fabs(u);
        af += (double)a[k] * f;
        a2 += (double)a[k] * (double)a[k];
        const double gx = (i < nx - 1) ? (double)a[k] - (double)a[k + 1] : 0.0;   // div^* a (L4)
        const double gy = (j < ny - 1) ? (double)a[k] - (double)a[k + nx] : 0.0;
        mg = fmax(mg, sqrt(gx * gx + gy * gy));
        ma = fmax(ma, fabs((double)a[k]));
        if (O.p != nullptr) {
            // frames attributed to pair t; a shard's last frame belongs to the next rank
            const int s_hi = (t == O.P - 1 && !O.next_owns_last) ? t + 1 : t;
            for (int s = t; s <= s_hi; ++s) {
                const size_t fo = ((size_t)b * O.T + s) * (size_t)O.N + k;
                const double d = (double)O.x[fo] - (double)O.p[fo];
                px += d * d;
            }
        }
    }
    tr = block_sum(tr, sh); gr = block_sum(gr, sh); ub = block_sum(ub, sh); af = block_sum(af, sh);
    mg = block_max(mg, sh); ma = block_max(ma, sh); px = block_sum(px, sh); a2 = block_sum(a2, sh);
    if (threadIdx.x == 0) {
        double* P = O.partials + ((size_t)g * O.bpp + blockIdx.x) * kRec;
        P[0] = tr; P[1] = gr; P[2] = ub; P[3] = af; P[4] = mg; P[5] = ma; P[6] = px; P[7] = a2;
    }
}

// glob slots
enum {
    GL_TR = 0, GL_GR = 1, GL_K2 = 2, GL_DZ = 3, GL_UB = 4, GL_PX = 5,
    GL_FSQ = 8, GL_FL1 = 9, GL_CONV = 10, GL_NONF = 11, GL_LASTRED = 12,
    GL_N = 32
};

__global__ void __launch_bounds__(256) k_pair_reduce(const ReduceArgs R) {
    __shared__ double sh[32];
    __shared__ int am_last;
    pdl_wait();
    if (R.is_iteration && R.stop != nullptr && *reinterpret_cast<const volatile int*>(R.stop)) return;
    const int g = blockIdx.x;
    const double* base = R.partials + (size_t)g * R.recs_per_pair * kRec;
    double out[kRec];
#pragma unroll
    for (int q = 0; q < kRec; ++q) {
        const bool mx = (R.max_mask >> q) & 1u;
        double v = 0.0;
        for (int k = threadIdx.x; k < R.recs_per_pair; k += blockDim.x) {
            const double e = base[(size_t)k * kRec + q];
            v = mx ? fmax(v, e) : v + e;
        }
        out[q] = mx ? block_max(v, sh) : block_sum(v, sh);
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < kRec; ++q) R.pair_out[(size_t)g * kRec + q] = out[q];
        __threadfence();
        am_last = (atomicAdd(R.counter, 1) == R.G - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    // last block: sum the pairs' rows in fixed order (thread q < 8 owns field q)
    __shared__ double tot[kRec];
    if (threadIdx.x < kRec) {
        double v = 0.0;
        for (int g2 = 0; g2 < R.G; ++g2) v += __ldcg(R.pair_out + (size_t)g2 * kRec + threadIdx.x);
        tot[threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    *R.counter = 0;
    if (R.is_setup) {
        R.glob[GL_FSQ] = tot[0];
        R.glob[GL_FL1] = tot[1];
        return;
    }
    if (!R.is_iteration) return;
    bool nonfinite = false;
    for (int c = 0; c < 6; ++c) { R.glob[c] = tot[c]; nonfinite |= !isfinite(tot[c]); }
    R.glob[GL_LASTRED] = (double)R.iteration;
    if (nonfinite) {
        R.glob[GL_NONF] = 1.0;
        if (R.stop) *R.stop = 1;
        return;
    }
    if (R.tol > 0.0 && R.stop != nullptr) {
        bool ok;
        if (R.stop_kind == 1) {
            // Alg.2 stopping rule: ||[x-s; z-s]|| < eps and rho ||[dx; dz]|| < eps
            ok = sqrt(tot[3]) < R.tol && R.rho_admm * sqrt(tot[4]) < R.tol;
        } else {
            // L13: primal ||K|| and dual ||dz||/tau1 relative to ||f||
            const double scale = R.tol * fmax(sqrt(R.glob[GL_FSQ]), 1e-30);
            ok = sqrt(tot[2]) <= scale && sqrt(tot[3]) / R.tau1 <= scale;
        }
        if (ok) {
            R.glob[GL_CONV] = (double)R.iteration;
            __threadfence();
            *R.stop = 1;
        }
    }
}

}  // namespace uotk (k_pair_reduce)
#include "uot_tpersist.inc"
#include "uot_single.cuh"
namespace uotk {

// prox cold start (L8): x^0 = 0, or max(p, 0) with UOT_RESET_X_FROM_P
// with UOT_FIX_FIRST_FRAME, frame 0 of each chain is the constant argument s = p_0
__global__ void __launch_bounds__(256) k_init_x(const float* p, float* x, long long n, int from_p,
                                                int fix_first, long long frame_len, int T) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const bool first = fix_first && ((k / frame_len) % T == 0);
        x[k] = first ? p[k] : (from_p ? fmaxf(p[k], 0.f) : 0.f);
    }
}

__global__ void k_init_glob(double* glob, int* stop, int* counter, int reset_all) {
    if (threadIdx.x == 0) {
        if (reset_all) {
            for (int q = 0; q < GL_N; ++q) glob[q] = 0.0;
        }
        glob[GL_CONV] = -1.0;
        glob[GL_NONF] = 0.0;
        *stop = 0;
        *counter = 0;
    }
}

// Cross-rank stopping test (uot_stop_pack / uot_stop_apply): pack this rank's sums of the last
// checked iteration; after the caller's all-reduce, apply the L13 test to the GLOBAL sums.
__global__ void k_stop_pack(const double* glob, double* out) {
    if (threadIdx.x < 6) out[threadIdx.x] = glob[threadIdx.x];     // TR GR K2 DZ UB PX
    if (threadIdx.x == 6) out[6] = glob[GL_FSQ];
    if (threadIdx.x == 7) out[7] = glob[GL_NONF];
}
__global__ void k_stop_apply(const double* sums, double* glob, int* stop, double tol, double tau1) {
    if (threadIdx.x != 0 || *stop) return;
    if (sums[7] != 0.0) { glob[GL_NONF] = 1.0; *stop = 1; return; }
    if (!(tol > 0.0)) return;
    const double scale = tol * fmax(sqrt(sums[6]), 1e-30);
    if (sqrt(sums[2]) <= scale && sqrt(sums[3]) / tau1 <= scale) {
        glob[GL_CONV] = glob[GL_LASTRED];
        __threadfence();
        *stop = 1;
    }
}

}  // namespace uotk

// ============================================================================ host side
struct Geometry {
    int vec, strips, segs, H, items;
};

// Host-side early exit for device-side stopping: after every chunk of launches the
// stop flag is copied (async) to pinned host memory with an event; before
// enqueueing chunk k+2 the host waits for chunk k's event and stops enqueueing if
// the flag was set.  The GPU always has the next chunk queued.
struct StopPoller {
    int* h = nullptr;                 // pinned [2]
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool pending[2] = {false, false};
    int chunk = 0;
    bool init() {
        if (h) return true;
        if (cudaHostAlloc(&h, 2 * sizeof(int), cudaHostAllocDefault) != cudaSuccess) { h = nullptr; return false; }
        for (int q = 0; q < 2; ++q)
            if (cudaEventCreateWithFlags(&ev[q], cudaEventDisableTiming) != cudaSuccess) return false;
        return true;
    }
    void begin() { pending[0] = pending[1] = false; chunk = 0; }
    // after a chunk: snapshot the flag
    void post(const int* dstop, cudaStream_t s) {
        const int q = chunk & 1;
        cudaMemcpyAsync(&h[q], dstop, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ev[q], s);
        pending[q] = true;
        ++chunk;
    }
    // before the next chunk: true if the device already stopped (checks the older snapshot)
    bool stopped() {
        const int q = chunk & 1;           // the slot about to be reused = two chunks ago
        if (!pending[q]) return false;
        cudaEventSynchronize(ev[q]);
        pending[q] = false;
        return h[q] != 0;
    }
    void release() {
        for (int q = 0; q < 2; ++q) if (ev[q]) cudaEventDestroy(ev[q]);
        if (h) cudaFreeHost(h);
        h = nullptr;
    }
};
static const int kPollChunk = 128;

struct uot_ctx {
    uot_params p;
    uot_buffers b;
    cudaStream_t s;
    int B, T, P, G, nx, ny;
    long long N;
    bool prox;
    Geometry geo;
    int bpp;
    float tau1f, tau2f;
    double tau1, tau2;
    int64_t iter;
    int64_t launches;
    double* part;
    double* pair_it;
    double* pair_obj;
    double* glob;
    int* stop;
    int* counter;
    float* pxchg;       // persistent kernel exchange slots
    int* pflags;        // [kMaxPersistCtas] + barrier[2]
    struct { bool ok; int TW, TH, tx, ty, ctas, threads; size_t smem; } pg;
    int64_t persist_launches;
    StopPoller poll;
    int r_mode;          // 0 l1, 1 l2 (p = 2), 2 balanced
    float r_scale;
    int fix_first;
    bool timing;
    bool stop_armed;
    bool ext_stop;       // stop armed by uot_stop_external: the test runs in uot_stop_apply (global sums)
    int slot;            // ping-pong slot of mx/my/a(/x) holding the current iterate
    int rcur;            // 0: r holds the current r, 1: r_alt (after an odd number of k_iter2 passes)
    bool t2ok;           // temporally blocked fixed-marginal kernel available (r_alt given)
    bool t2on;           // ... and enabled (uot_set_temporal)
    int t2vec;           // its 16-byte loads (nx % 4 == 0, aligned planes)
    TVar tv[4];          // its variants: [0] two iterations per pass, [1] four, [2] three, [3] five (k_wave)
    float pass_cost[6];  // relative device time of a pass of S = 1..5 iterations (pass scheduler)
    bool pdl;            // programmatic dependent launch for the pass kernels (UOT_PDL)
    struct {             // persistent temporally blocked passes (k_tpersist, small grids)
        bool ok;
        int th, tx, ty, ctas, nt;
        size_t smem;
        const void* fn;
        CUtensorMap mx[2][2], my[2][2], a[2][2], r[2][2], f[2];   // [S = 4, 2][slot / r buffer]
    } tp;
    bool t4on;           // four-iteration passes enabled (UOT_T4)
    struct {             // chain prox: register wavefront with pair groups (k_wave_prox)
        bool ok;
        int S;               // iterations of the long pass (3); short pass: 2
        bool prefer2;        // split stretches into 2s (+ one 3 when odd) rather than 3s (+ 2s)
        int own_lo, own_hi;  // written pairs (uot_set_own_pairs: a shard's own pairs between ghost pairs)
        int cl, groups;      // CTAs per cluster, pair groups per chain
        int strips, segs, H;
        int strips2;         // strips of the two-iteration pass (its halo: fewer lanes at vn = 2)
        int vn, warps;       // columns per lane (4: 128-column strips, 8 pairs per CTA; 2: 64-column
                             // strips, 16 pairs per CTA) and warps per CTA
        size_t smem[2];      // dynamic shared memory of the long / two-iteration pass
        const void* fn[2][2];  // [long / two-iteration pass][red]
    } pw;
    bool single_on;      // one-CTA k_single for single small pairs (UOT_SINGLE)
    int single_v;        // its pixels per thread: 8 (nx % 8 == 0) or 4 (UOT_SINGLE_V=4 forces 4, =16 tries 16)
    struct LogE { int64_t iter; int slot, rcur; };
    std::vector<LogE> log;           // launches since the stop was armed (device-stop correction)
    std::vector<LogE> persist_base;  // state at the start of each persistent launch since arming
    std::vector<cudaEvent_t> ev;     // event pool, pairs (start, stop)
    size_t ev_used;
    std::vector<int> ev_kind;        // per timed launch: uot_kernel_path code (4: UOT-DF kernel)
    char err[512];
};

static char g_err[512] = "";

static int fail(uot_ctx* c, int code, const char* fmt, ...) {
    char* dst = c ? c->err : g_err;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(dst, 512, fmt, ap);
    va_end(ap);
    return code;
}

static const int kSMs = 148;

// Segment height of the register wavefront: a warp marches H + 2S rows for H output rows, and
// the G x strips x ceil(ny / H) warps run in waves of kSMs x (resident warps per SM).  Time is
// modelled as (waves, rounded up) x (H + 2S): the smallest H that fits one fewer wave wins.
// Measured (C3, 63 x 256^2, S = 5): H = 16 -> 2.55 waves, 2.88e11 px-it/s; H = 43 -> 0.96 wave,
// 4.12e11; H = 37 -> 1.12 waves, 2.52e11.  C4 / C5 keep 512-row segments (the model's pick is
// within 2% there); segments are capped at 512 rows (the measured C4 optimum of round 1).
// UOT_WAVE_H overrides.
static int wave_height(long long G, int strips, int ny, int S, int resident = 0) {
    if (resident <= 0) resident = S >= 4 ? 8 : 10;             // k_wave warps per SM (WaveCfg: registers)
    const long long wave = (long long)kSMs * resident;
    int bestH = 16;
    double best = 1e300;
    for (int n = (ny + 511) / 512; n <= (ny + 15) / 16; ++n) {  // n segments of H = ceil(ny / n) rows
        const int H = (ny + n - 1) / n;
        if (H < 16) break;
        const long long units = G * strips * n;
        const long long waves = (units + wave - 1) / wave;
        const double t = (double)waves * (H + 2 * S) * (1.0 + 1e-9 * n);   // ties: fewer segments
        if (t < best * (1.0 - 1e-12)) { best = t; bestH = H; }
    }
    return std::max(16, bestH);
}

// Relative cost of a wavefront pass with a given strip layout: whole waves x rows marched x the
// pixel columns one SM advances per row step (resident warps x columns per warp) / the layout's
// pixel throughput.  Compares the 128-column strips (k_wave_pk, 8 warps / SM at S >= 4) with the
// 64-column ones (k_wave_n, 16).  Measured on C3 (63 x 256^2, S = 5): k_wave_n computes 0.86x
// the pixel-levels of k_wave_pk (5 x 64 vs 3 x 128 columns, 37- vs 43-row segments) but takes
// 1.13x the time (52.6 vs 46.4 us per pass: twice the cp.async / LDS / SHFL per pixel), so its
// per-pixel throughput is 0.76 of k_wave_pk's (kWaveNEff); it wins only on rows where the quad
// strips waste much more, e.g. 136 columns (2 x 128 vs 3 x 64).
constexpr double kWaveNEff = 0.76;
static double wave_cost(long long G, int strips, int ny, int H, int S, int resident, int cols, double eff) {
    const long long wave = (long long)kSMs * resident;
    const long long units = G * strips * (long long)((ny + H - 1) / H);
    return (double)((units + wave - 1) / wave) * (H + 2 * S) * resident * cols / eff;
}

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

static bool pw_regroup(uot_ctx* c);

// Chain prox (rho < inf) without shard halos: k_wave_prox passes of 3 (and 2) iterations.  A pair
// group is a cluster of cl CTAs x kWpWarps pairs writing the middle cl*8 - 2*3 of them; cl
// (1, 2, 4, 8) minimises the CTAs per (strip, segment), the segment height follows the
// wave-quantisation model with the co-resident clusters the occupancy API reports.
// (l1 growth term only: the p = 2 / balanced variants of chain prox run k_iter.)
static void plan_prox_wave(uot_ctx* c) {
    using namespace uotk;
    memset(&c->pw, 0, sizeof(c->pw));
    if (c->r_mode != 0) return;
    // passes of 3 (fn[0]) and 2 (fn[1]) iterations; groups are planned for 3 (the longest pass).  C4
    // chain prox: passes of 2 with one 3 for odd stretches (default) 1.80e11 px-it/s, 3s with 2s for
    // 3k+1 (UOT_PROX_PASS=3) 1.72e11 -- the S = 3 kernel carries 255 registers with spills, S = 2
    // none; S = 4 (300+ B of spills) 0.97e11
    c->pw.S = 3;
    c->pw.prefer2 = env_int("UOT_PROX_PASS", 2) != 3;
    // lane layout: 128-column strips with 8 pairs per CTA (default) or 64-column strips with 12 / 16
    // (UOT_PROX_V=2, UOT_PROX_W=12 / 16: fewer registers per warp, more warps per SM).  Measured on C4
    // chain prox (passes of 2): V4 x 8 1.79e11 px-it/s, V2 x 12 1.54e11, V2 x 16 (128-register cap,
    // spills) 1.20e11 -- more resident warps do not pay for twice the per-pixel cp.async / LDS /
    // st.async / SHFL traffic
    c->pw.vn = env_int("UOT_PROX_V", 4) == 2 ? 2 : 4;
    const int nw_env = env_int("UOT_PROX_W", 12);
    if (c->pw.vn == 2 && nw_env == 16) {
        c->pw.warps = 16;
        c->pw.fn[0][0] = (const void*)k_wave_prox<3, 0, false, 2, 16>;
        c->pw.fn[0][1] = (const void*)k_wave_prox<3, 0, true, 2, 16>;
        c->pw.fn[1][0] = (const void*)k_wave_prox<2, 0, false, 2, 16>;
        c->pw.fn[1][1] = (const void*)k_wave_prox<2, 0, true, 2, 16>;
        c->pw.smem[0] = WpCfg<3, 2, 16>::smem; c->pw.smem[1] = WpCfg<2, 2, 16>::smem;
    } else if (c->pw.vn == 2) {
        c->pw.warps = 12;
        c->pw.fn[0][0] = (const void*)k_wave_prox<3, 0, false, 2, 12>;
        c->pw.fn[0][1] = (const void*)k_wave_prox<3, 0, true, 2, 12>;
        c->pw.fn[1][0] = (const void*)k_wave_prox<2, 0, false, 2, 12>;
        c->pw.fn[1][1] = (const void*)k_wave_prox<2, 0, true, 2, 12>;
        c->pw.smem[0] = WpCfg<3, 2, 12>::smem; c->pw.smem[1] = WpCfg<2, 2, 12>::smem;
    } else {
        c->pw.warps = 8;
        c->pw.fn[0][0] = (const void*)k_wave_prox<3, 0, false, 4>;
        c->pw.fn[0][1] = (const void*)k_wave_prox<3, 0, true, 4>;
        c->pw.fn[1][0] = (const void*)k_wave_prox<2, 0, false, 4>;
        c->pw.fn[1][1] = (const void*)k_wave_prox<2, 0, true, 4>;
        c->pw.smem[0] = WpCfg<3, 4>::smem; c->pw.smem[1] = WpCfg<2, 4>::smem;
    }
    for (int k = 0; k < 2; ++k)
        for (int red = 0; red < 2; ++red)
            if (cudaFuncSetAttribute(c->pw.fn[k][red], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->pw.smem[k]) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
    const int S = c->pw.S;
    int best_cl = 0;
    long long best = 1LL << 62;
    const int clenv = env_int("UOT_PROX_CL", 0);
    for (int cl = 1; cl <= 8; cl *= 2) {
        if (clenv > 0 && cl != clenv) continue;
        const int V = cl * c->pw.warps - 2 * S;
        if (V <= 0) continue;
        const long long ctas = (long long)c->B * ((c->P + V - 1) / V) * cl;
        if (ctas < best) { best = ctas; best_cl = cl; }
    }
    if (!best_cl) return;
    c->pw.own_lo = 0;
    c->pw.own_hi = c->P;
    // pair slots per pair (halo pairs + idle slots): C4 320 / 255 = 1.25 runs the wave (1.54e11 vs
    // k_iter 1.29e11 px-it/s); C3 96 / 63 = 1.52 is slower than one pass per iteration (0.87e11 vs
    // 1.08e11), so above 1.34 chain prox stays on k_iter (UOT_PROX_WAVE=2 forces the wave)
    if ((double)best * c->pw.warps / ((double)c->B * c->P) > 1.34 && env_int("UOT_PROX_WAVE", 1) != 2) return;
    c->pw.cl = best_cl;
    c->pw.strips = wp_strips(c->nx, S, c->pw.vn);
    c->pw.strips2 = wp_strips(c->nx, 2, c->pw.vn);
    if (!pw_regroup(c)) return;
    c->pw.ok = true;
    if (env_int("UOT_DEBUG", 0))
        fprintf(stderr, "k_wave_prox plan: S %d V %d cl %d groups %d strips %d segs %d H %d\n",
                c->pw.S, c->pw.vn, c->pw.cl, c->pw.groups, c->pw.strips, c->pw.segs, c->pw.H);
}

// Pair groups over the own pairs [own_lo, own_hi) and the segment height (the wave model with the
// co-resident clusters the occupancy API reports).
static bool pw_regroup(uot_ctx* c) {
    using namespace uotk;
    const int S = c->pw.S, best_cl = c->pw.cl;
    const int own = c->pw.own_hi - c->pw.own_lo;
    const int NW = c->pw.warps;
    c->pw.groups = (own + best_cl * NW - 2 * S - 1) / (best_cl * NW - 2 * S);
    // co-resident clusters (one 256-thread CTA per SM; cluster placement may strand SMs)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(best_cl * 64, 1);
    cfg.blockDim = dim3(NW * 32);
    cfg.dynamicSmemBytes = c->pw.smem[0];
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = best_cl; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, c->pw.fn[0][0], &cfg) != cudaSuccess || nclus <= 0) {
        cudaGetLastError();
        return false;
    }
    const long long G = (long long)c->B * c->pw.groups * best_cl;     // CTAs per (strip, segment)
    const int hset = env_int("UOT_PROX_WAVE_H", 0);
    // wave_height with its wave = kSMs x resident: resident = co-resident CTAs / kSMs (rounded)
    int H = 16;
    {
        const long long wave = (long long)nclus * best_cl;
        double bt = 1e300;
        for (int n = (c->ny + 511) / 512; n <= (c->ny + 15) / 16; ++n) {
            const int h = (c->ny + n - 1) / n;
            if (h < 16) break;
            const long long units = G * c->pw.strips * n;
            const double t = (double)((units + wave - 1) / wave) * (h + 2 * S) * (1.0 + 1e-9 * n);
            if (t < bt * (1.0 - 1e-12)) { bt = t; H = h; }
        }
    }
    if (hset > 0) H = std::max(16, hset);               // >= 16: records within uot_scratch_doubles
    if (H > c->ny) H = c->ny;
    c->pw.H = H;
    c->pw.segs = (c->ny + H - 1) / H;
    return true;
}

// Work decomposition of k_iter: strips of
// 32*vec pixels; segment height H chosen so that the warp count fills the
// 148 SMs several times, H in [4, 64].
static Geometry choose_geometry(int nx, int ny, int G, bool vec4_ok) {
    const long long target = (long long)kSMs * 48;   // warps: ~3 waves at 16 resident warps/SM
    Geometry g{};
    g.vec = vec4_ok ? 4 : 1;
    if (vec4_ok) {
        const int strips4 = (nx + 127) / 128;
        const long long max_w = (long long)G * strips4 * ((ny + 3) / 4);
        if (max_w < target && (nx % 4 == 0)) {
            // small grid: narrower strips give more warps
            g.vec = 1;
        }
    }
    const int forced_vec = env_int("UOT_VEC", 0);
    if (forced_vec == 1 || ((forced_vec == 4 || forced_vec == 2) && vec4_ok)) g.vec = forced_vec;
    g.strips = (nx + 32 * g.vec - 1) / (32 * g.vec);
    const long long cols = (long long)G * g.strips;
    long long segs_needed = (target + cols - 1) / cols;
    int H = (int)((ny + segs_needed - 1) / segs_needed);
    if (H > 64) H = 64;
    if (H < (g.vec == 4 ? 8 : 4)) H = (g.vec == 4 ? 8 : 4);   // r01 sweep (profiles/r01_sweep_vec_segH.txt)
    const int forced_h = env_int("UOT_SEG_H", 0);
    if (forced_h > 0) H = forced_h < 4 ? 4 : forced_h;
    if (H > ny) H = ny;
    g.H = H;
    g.segs = (ny + H - 1) / H;
    g.items = G * g.strips * g.segs;
    return g;
}

static int blocks_per_pair(long long N) {
    long long b = (N + 4095) / 4096;
    if (b < 1) b = 1;
    if (b > 256) b = 256;
    return (int)b;
}

static const int kMaxPersistCtas = 148;          // one tile-CTA per SM at most
static const int kMaxTileEdge = 4 * 128 + 4 * 64; // 4*TW + 4*TH for the largest tile
static size_t part_records(const Geometry& g, int G, int bpp) {
    size_t a = (size_t)g.items, b = (size_t)G * bpp;
    size_t m = a > b ? a : b;
    return m > (size_t)kMaxPersistCtas ? m : (size_t)kMaxPersistCtas;
}
// persistent-kernel exchange slots (floats) + flags/barrier (ints), in doubles
static size_t persist_scratch_doubles() {
    return ((size_t)kMaxPersistCtas * 2 * kMaxTileEdge) / 2 + (kMaxPersistCtas + 8) / 2 + 8;
}

static double chain_norm2(int nx, int ny, int T, bool prox, bool fix_first = false) {
    const double pi = 3.14159265358979323846;
    const double lam = (nx >= 2 ? 2.0 + 2.0 * cos(pi / nx) : 0.0) + (ny >= 2 ? 2.0 + 2.0 * cos(pi / ny) : 0.0);
    if (!prox) return lam + 1.0;                        // K = [D, -I]
    if (fix_first && T == 2) return lam + 2.0;          // K = [D, -I, -I] (eq:Prox_UOT_specialcase)
    return lam + 1.0 + 2.0 + 2.0 * cos(pi / T);         // K = [D, -I, A], A path incidence (L12)
}

// Persistent SMEM-resident path (uot_persist.cuh): small grids whose tiles fit
// one CTA per SM; fixed marginals, or prox with T == 2 and no shard halos.
static void plan_persist(uot_ctx* c) {
    c->pg.ok = false;
    const int mode = env_int("UOT_PERSIST", -1);      // -1 auto, 0 off, 1 force when possible
    if (mode == 0) return;
    if (c->prox && (c->T != 2 || c->b.a_prev_halo || c->b.a_next_halo)) return;
    int dev = 0, nsm = kSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (!coop) return;
    const int limit = nsm < kMaxPersistCtas ? nsm : kMaxPersistCtas;
    struct Cand { int TW, TH; };
    const Cand cands[] = {{32, 16}, {32, 32}, {64, 32}, {64, 64}, {128, 64}};
    int TW = 0, TH = 0;
    if ((long long)c->nx * c->ny <= 8192 && c->nx <= 128 && c->ny <= 128 && c->G <= limit) {
        TW = c->nx; TH = c->ny;                           // one tile per pair: no inter-CTA sync
    } else {
        for (const Cand& q : cands) {
            const long long tiles = (long long)((c->nx + q.TW - 1) / q.TW) * ((c->ny + q.TH - 1) / q.TH);
            if (tiles * c->G <= limit) { TW = q.TW; TH = q.TH; break; }
        }
    }
    const char* tenv = getenv("UOT_TILE");            // "WxH" override (tuning)
    if (tenv && *tenv) {
        int w = 0, h = 0;
        if (sscanf(tenv, "%dx%d", &w, &h) == 2 && w > 0 && h > 0 && w <= 128 && h <= 64) { TW = w; TH = h; }
    }
    if (TW == 0) return;
    const PLayout L(TW, TH);
    const size_t smem = L.floats(c->prox) * sizeof(float);
    if (smem > 200 * 1024) return;
    int threads = ((TW * TH / 4 + 31) / 32) * 32;
    if (threads < 128) threads = 128;
    if (threads > 512) threads = 512;
    const void* fn = c->prox ? (const void*)k_persist<true> : (const void*)k_persist<false>;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return;
    }
    const int tx = (c->nx + TW - 1) / TW, ty = (c->ny + TH - 1) / TH;
    const int ctas = tx * ty * c->G;
    if (ctas > per_sm * nsm || ctas > kMaxPersistCtas) return;
    c->pg.ok = true;
    c->pg.TW = TW; c->pg.TH = TH; c->pg.tx = tx; c->pg.ty = ty; c->pg.ctas = ctas;
    c->pg.threads = threads; c->pg.smem = smem;
}

template <int TH, int RM>
static const void* tp_kernel_t(int) {      // 320 threads (640 measured slower on C1 / C2)
    return (const void*)uotk::k_tpersist<TH, RM, uotk::kT2Threads>;
}
static const void* tp_kernel(int th, int rm, int nt) {
    if (th == 36) return rm == 1 ? tp_kernel_t<36, 1>(nt) : (rm == 2 ? tp_kernel_t<36, 2>(nt) : tp_kernel_t<36, 0>(nt));
    return rm == 1 ? tp_kernel_t<16, 1>(nt) : (rm == 2 ? tp_kernel_t<16, 2>(nt) : tp_kernel_t<16, 0>(nt));
}

extern "C" {

size_t uot_scratch_doubles(const uot_params* p) {
    if (!p || p->nx < 1 || p->ny < 1 || p->n_chains < 1 || p->n_frames < 2) return 0;
    const int G = p->n_chains * (p->n_frames - 1);
    const long long N = (long long)p->nx * p->ny;
    const int bpp = blocks_per_pair(N);
    size_t recs = 0;
    for (int v4 = 0; v4 < 2; ++v4) {
        Geometry g = choose_geometry(p->nx, p->ny, G, v4 && (p->nx % 4 == 0));
        size_t r = part_records(g, G, bpp);
        if (r > recs) recs = r;
    }
    // also cover the vec-1 geometry with H = 4 (env overrides)
    Geometry g1{1, (p->nx + 31) / 32, (p->ny + 3) / 4, 4, 0};
    size_t r1 = (size_t)G * g1.strips * g1.segs;
    if (r1 > recs) recs = r1;
    const size_t r2 = (size_t)G * ((p->nx + kTW - 1) / kTW) * ((p->ny + 15) / 16);   // k_iter2 tiles (TH >= 16)
    if (r2 > recs) recs = r2;
    return recs * kRec + 2 * (size_t)G * kRec + GL_N + 4 + persist_scratch_doubles();
}

int uot_default_steps(const uot_params* p, double safety, double* tau1, double* tau2) {
    if (!p || !tau1 || !tau2) return fail(nullptr, UOT_E_INVALID, "null argument");
    if (!(safety > 0.0 && safety < 1.0)) return fail(nullptr, UOT_E_INVALID, "safety must be in (0,1)");
    if (p->nx < 1 || p->ny < 1 || p->n_frames < 2) return fail(nullptr, UOT_E_INVALID, "bad grid");
    const bool prox = isfinite(p->rho);
    const double t = sqrt(safety / chain_norm2(p->nx, p->ny, p->n_frames, prox, (p->flags & UOT_FIX_FIRST_FRAME) != 0));
    *tau1 = t;
    *tau2 = t;
    return UOT_OK;
}

static bool al16(const void* q) { return ((uintptr_t)q & 15u) == 0; }

int uot_create(const uot_params* prm, const uot_buffers* buf, void* stream, uot_ctx** out) {
    if (!out) return fail(nullptr, UOT_E_INVALID, "out is NULL");
    *out = nullptr;
    if (!prm || !buf) return fail(nullptr, UOT_E_INVALID, "params/buffers NULL");
    uot_params p = *prm;
    if (p.nx < 1 || p.ny < 1) return fail(nullptr, UOT_E_INVALID, "nx, ny must be >= 1");
    if (p.n_chains < 1 || p.n_frames < 2) return fail(nullptr, UOT_E_INVALID, "need n_chains >= 1, n_frames >= 2");
    if (!(p.alpha > 0.0)) return fail(nullptr, UOT_E_INVALID, "alpha must be > 0 (+inf = balanced)");
    if (!(p.rho > 0.0)) return fail(nullptr, UOT_E_INVALID, "rho must be > 0 (+inf = fixed marginals)");
    if (!(p.tau1 >= 0.0) || !(p.tau2 >= 0.0) || !isfinite(p.tau1) || !isfinite(p.tau2))
        return fail(nullptr, UOT_E_INVALID, "tau1, tau2 must be finite and >= 0");
    const bool prox = isfinite(p.rho);
    if (p.tau1 == 0.0 || p.tau2 == 0.0) {
        double t1, t2;
        uot_default_steps(&p, 0.99, &t1, &t2);
        if (p.tau1 == 0.0) p.tau1 = t1;
        if (p.tau2 == 0.0) p.tau2 = t2;
    }
    const double bound = 1.0 / chain_norm2(p.nx, p.ny, p.n_frames, prox, (p.flags & UOT_FIX_FIRST_FRAME) != 0);
    if (!(p.flags & UOT_FORCE_STEPS) && !(p.tau1 * p.tau2 < bound))
        return fail(nullptr, UOT_E_INVALID, "tau1*tau2 = %g violates Theorem 1 bound %g (set UOT_FORCE_STEPS)",
                    p.tau1 * p.tau2, bound);
    const uot_buffers& b = *buf;
    if (!b.frames || !b.mx[0] || !b.mx[1] || !b.my[0] || !b.my[1] || !b.r || !b.a[0] || !b.a[1] || !b.scratch)
        return fail(nullptr, UOT_E_INVALID, "a required buffer pointer is NULL");
    if (!prox && !b.f) return fail(nullptr, UOT_E_INVALID, "fixed mode needs buffers.f");
    if (prox && (!b.x[0] || !b.x[1])) return fail(nullptr, UOT_E_INVALID, "prox mode needs buffers.x[0], x[1]");
    if (((uintptr_t)b.scratch & 7u) != 0) return fail(nullptr, UOT_E_INVALID, "scratch must be 8-byte aligned");

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, UOT_E_CUDA, "no CUDA device (%s)", cudaGetErrorString(e));
    }

    uot_ctx* c = new (std::nothrow) uot_ctx();
    if (!c) return fail(nullptr, UOT_E_CUDA, "host allocation failed");
    c->p = p;
    c->b = b;
    c->s = reinterpret_cast<cudaStream_t>(stream);
    c->B = p.n_chains; c->T = p.n_frames; c->P = p.n_frames - 1; c->G = c->B * c->P;
    c->nx = p.nx; c->ny = p.ny; c->N = (long long)p.nx * p.ny;
    c->prox = prox;
    bool vec4_ok = (p.nx % 4 == 0) && al16(b.frames) && al16(b.mx[0]) && al16(b.mx[1]) &&
                   al16(b.my[0]) && al16(b.my[1]) && al16(b.r) && al16(b.a[0]) && al16(b.a[1]);
    if (prox) vec4_ok = vec4_ok && al16(b.x[0]) && al16(b.x[1]) && al16(b.a_prev_halo) && al16(b.a_next_halo);
    else vec4_ok = vec4_ok && al16(b.f);
    c->geo = choose_geometry(p.nx, p.ny, c->G, vec4_ok);
    c->bpp = blocks_per_pair(c->N);
    c->tau1 = p.tau1; c->tau2 = p.tau2;
    c->r_mode = !isfinite(p.alpha) ? 2 : ((p.flags & UOT_RESIDUAL_L2) ? 1 : 0);
    c->r_scale = c->r_mode == 1 ? (float)(1.0 / (1.0 + 2.0 * p.alpha * p.tau1)) : 1.f;
    c->fix_first = (prox && (p.flags & UOT_FIX_FIRST_FRAME)) ? 1 : 0;
    c->tau1f = (float)p.tau1; c->tau2f = (float)p.tau2;
    c->iter = 0;
    c->launches = 0;
    memset(c->tv, 0, sizeof(c->tv));
    c->tv[0].th = 32;
    c->tv[1].th = env_int("UOT_T4_TH", 36) == 32 ? 32 : 36;   // 36: measured best on C4 (3 CTAs / SM)
    c->tv[2].th = 32;                                           // (three- and five-iteration passes: k_wave only)
    c->tv[3].th = 32;
    // register wavefront (k_wave) for 16-byte-aligned planes with nx % 4 == 0 (UOT_WAVE=0: SMEM tiles)
    // Enough independent strips to fill the GPU: segment height 512 (halved down to 16 for
    // smaller problems, >= 2 waves of 8 warps per SM); below one wave at 16 rows the SMEM tiles.
    const long long strips = wave_strips(p.nx, 4);
    const int wave_h_env = env_int("UOT_WAVE_H", 0);
    int wave_h = wave_h_env > 0 ? std::max(16, wave_h_env) : 16;   // >= 16: records within uot_scratch_doubles
    const int wenv_wave = env_int("UOT_WAVE", -1);
    const bool wave = (p.nx % 4 == 0) &&
                      (wenv_wave >= 0 ? wenv_wave != 0
                                      : (long long)c->G * strips * ((p.ny + wave_h - 1) / wave_h) >= (long long)kSMs * 8);
    static const int kVarS[4] = {2, 4, 3, 5};
    const int wave_v = env_int("UOT_WAVE_V", 0);
    const bool wave_pk = env_int("UOT_WAVE_PK", 1) != 0;
    for (int k = 0; k < 4; ++k) {
        TVar& v = c->tv[k];
        v.wave = wave;
        if (wave) {
            const int S = kVarS[k], res4 = S >= 4 ? 8 : 10;
            v.vn = 4;
            v.tx = wave_strips(p.nx, S);
            v.th = wave_h_env > 0 ? wave_h : wave_height(c->G, v.tx, p.ny, S, res4);
            // 64-column strips (k_wave_n) where they save enough computed halo pixels to pay for
            // their lower per-pixel throughput (wave_cost); UOT_WAVE_V = 2 / 4 forces
            const int tx2 = waven_strips(p.nx, S);
            const int th2 = wave_h_env > 0 ? wave_h : wave_height(c->G, tx2, p.ny, S, kWaveNMinB);
            const bool narrow = wave_v == 2 ||
                (wave_v == 0 && wave_pk &&
                 wave_cost(c->G, tx2, p.ny, th2, S, kWaveNMinB, 64, kWaveNEff) <
                     wave_cost(c->G, v.tx, p.ny, v.th, S, res4, 128, 1.0));
            if (narrow) { v.vn = 2; v.tx = tx2; v.th = th2; }
        } else {
            v.tx = (p.nx + kTW - 1) / kTW;
        }
        v.ty = (p.ny + v.th - 1) / v.th;
    }
    memset(&c->pw, 0, sizeof(c->pw));
    if (prox && b.r_alt && !b.a_prev_halo && !b.a_next_halo && p.nx % 4 == 0 && env_int("UOT_PROX_WAVE", 1) != 0 &&
        al16(b.frames) && al16(b.mx[0]) && al16(b.mx[1]) && al16(b.my[0]) && al16(b.my[1]) && al16(b.a[0]) &&
        al16(b.a[1]) && al16(b.r) && al16(b.r_alt) && al16(b.x[0]) && al16(b.x[1]))
        plan_prox_wave(c);
    size_t recs = part_records(c->geo, c->G, c->bpp);
    for (const TVar& v : c->tv)
        if ((size_t)c->G * v.tx * v.ty > recs) recs = (size_t)c->G * v.tx * v.ty;
    // (16-row segments at most: uot_set_own_pairs may regroup the pairs and re-choose the height)
    if (c->pw.ok && (size_t)c->G * c->pw.strips * ((p.ny + 15) / 16) > recs) recs = (size_t)c->G * c->pw.strips * ((p.ny + 15) / 16);
    c->part = b.scratch;
    c->pair_it = c->part + recs * kRec;
    c->pair_obj = c->pair_it + (size_t)c->G * kRec;
    c->glob = c->pair_obj + (size_t)c->G * kRec;
    int* ints = reinterpret_cast<int*>(c->glob + GL_N);
    c->stop = ints;
    c->counter = ints + 1;
    c->pxchg = reinterpret_cast<float*>(c->glob + GL_N + 4);
    c->pflags = reinterpret_cast<int*>(c->pxchg + (size_t)kMaxPersistCtas * 2 * kMaxTileEdge);
    plan_persist(c);
    c->slot = 0;
    c->rcur = 0;
    c->t2ok = !prox && b.r_alt != nullptr && env_int("UOT_TEMPORAL", 1) != 0;
    c->t2on = true;
    c->t2vec = (p.nx % 4 == 0) && al16(b.f) && al16(b.mx[0]) && al16(b.mx[1]) && al16(b.my[0]) && al16(b.my[1]) &&
               al16(b.a[0]) && al16(b.a[1]) && al16(b.r) && al16(b.r_alt);
    c->t4on = env_int("UOT_T4", 1) != 0;
    c->single_on = env_int("UOT_SINGLE", 1) != 0;
    c->single_v = env_int("UOT_SINGLE_V", 8);
    c->pdl = env_int("UOT_PDL", 1) != 0;
    if (c->t2ok) {
        const int wenv = env_int("UOT_T2_WIDE", -1);
        for (int k = 0; k < 4; ++k) {
            TVar& v = c->tv[k];
            const int S = kVarS[k];
            const bool wide = wenv >= 0 ? (wenv != 0) : ((long long)c->G * v.tx * v.ty <= kSMs);
            if (v.wave && !c->t2vec) {          // unaligned planes: SMEM tiles
                v.wave = false;
                v.th = S == 4 ? (env_int("UOT_T4_TH", 36) == 32 ? 32 : 36) : 32;
                v.tx = (p.nx + kTW - 1) / kTW;
                v.ty = (p.ny + v.th - 1) / v.th;
            }
            v.ok = v.wave ? wvar_select(v, S, c->r_mode, env_int("UOT_WAVE_PK", 1) != 0) : tvar_select(v, S, v.th, wide, c->r_mode);
            if (!v.ok) {
                cudaGetLastError();
                continue;
            }
            v.tma = false;
            if (!v.wave && c->t2vec && env_int("UOT_T2_TMA", 1) != 0) {
                bool ok = true;
                for (int q = 0; q < 2; ++q) {
                    ok = ok && encode_plane_map(&v.mx[q], b.mx[q], p.nx, p.ny, c->G, v.rows);
                    ok = ok && encode_plane_map(&v.my[q], b.my[q], p.nx, p.ny, c->G, v.rows);
                    ok = ok && encode_plane_map(&v.a[q], b.a[q], p.nx, p.ny, c->G, v.rows);
                }
                ok = ok && encode_plane_map(&v.r[0], b.r, p.nx, p.ny, c->G, v.rows);
                ok = ok && encode_plane_map(&v.r[1], b.r_alt, p.nx, p.ny, c->G, v.rows);
                ok = ok && encode_plane_map(&v.f, b.f, p.nx, p.ny, c->G, v.rows);
                v.tma = ok;
            }
        }
        if (!c->tv[0].ok) c->t2ok = false;
    }
    // persistent temporally blocked passes for grids of at most one co-resident wave of tiles
    memset(&c->tp, 0, sizeof(c->tp));
    if (c->t2ok && c->t2vec && env_int("UOT_TPERSIST", 1) != 0) {
        // tile rows: 36 (one 76 KB CTA per SM), 16 for tiny grids (more, shorter tiles: C1 1.47e9
        // vs 1.27e9 px-it/s; C2 with 36: 8.0e10 vs 7.8e10)
        const long long t36 = (long long)c->G * ((p.nx + kTW - 1) / kTW) * ((p.ny + 35) / 36);
        const int thenv = env_int("UOT_TP_TH", 0);
        const int TH = thenv == 16 ? 16 : (thenv == 36 ? 36 : (t36 * 2 < kSMs ? 16 : 36));
        c->tp.th = TH;
        c->tp.tx = (p.nx + kTW - 1) / kTW;
        c->tp.ty = (p.ny + TH - 1) / TH;
        c->tp.smem = TH == 36 ? TB<36, 4>::smem : TB<16, 4>::smem;
        c->tp.nt = kT2Threads;
        c->tp.fn = tp_kernel(TH, c->r_mode, c->tp.nt);
        int nb = 0, dev = 0, nsm = kSMs;
        bool ok = cudaFuncSetAttribute(c->tp.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->tp.smem) ==
                      cudaSuccess &&
                  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, c->tp.fn, c->tp.nt, c->tp.smem) == cudaSuccess;
        if (ok && cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const long long ctas = (long long)c->G * c->tp.tx * c->tp.ty;
        // only where a launch per pass is latency-bound: at most one CTA per SM
        const int tpenv = env_int("UOT_TPERSIST", -1);
        ok = ok && nb >= 1 && ctas <= (long long)nb * nsm && (tpenv == 1 || ctas <= 2LL * nsm);
        for (int si = 0; si < 2 && ok; ++si) {
            const int rows = TH + 2 * (si == 0 ? 4 : 2);
            for (int q = 0; q < 2; ++q) {
                ok = ok && encode_plane_map(&c->tp.mx[si][q], b.mx[q], p.nx, p.ny, c->G, rows);
                ok = ok && encode_plane_map(&c->tp.my[si][q], b.my[q], p.nx, p.ny, c->G, rows);
                ok = ok && encode_plane_map(&c->tp.a[si][q], b.a[q], p.nx, p.ny, c->G, rows);
            }
            ok = ok && encode_plane_map(&c->tp.r[si][0], b.r, p.nx, p.ny, c->G, rows);
            ok = ok && encode_plane_map(&c->tp.r[si][1], b.r_alt, p.nx, p.ny, c->G, rows);
            ok = ok && encode_plane_map(&c->tp.f[si], b.f, p.nx, p.ny, c->G, rows);
        }
        c->tp.ctas = (int)ctas;
        c->tp.ok = ok;
        if (!ok) cudaGetLastError();
    }
    {   // relative pass costs (C4 measurements): k_wave 1 : 1.155 : 1.15 : 1.137 : 1.35 (S = 1..5),
        // SMEM tiles 1 : 1.46 : - : 2.19; UOT_PASS_COST="c2,c3,c4" overrides (c1 = 1)
        const bool wv = c->tv[0].wave;
        c->pass_cost[0] = 0.f; c->pass_cost[1] = 1.f;
        c->pass_cost[2] = wv ? 1.155f : 1.46f;
        c->pass_cost[3] = wv ? 1.15f : 1e9f;
        c->pass_cost[4] = wv ? 1.137f : 2.19f;
        c->pass_cost[5] = wv ? 1.35f : 1e9f;
        const char* pc = getenv("UOT_PASS_COST");
        if (pc) {
            float a2, a3, a4, a5 = 1e9f;
            const int got = sscanf(pc, "%f,%f,%f,%f", &a2, &a3, &a4, &a5);
            if (got >= 3) {
                c->pass_cost[2] = a2; c->pass_cost[3] = a3; c->pass_cost[4] = a4;
                if (got == 4) c->pass_cost[5] = a5;
            }
        }
    }
    c->err[0] = 0;
    c->timing = false;
    c->stop_armed = false;
    c->ext_stop = false;
    c->persist_launches = 0;
    c->ev_used = 0;
    *out = c;
    return UOT_OK;
}

static int check_launch(uot_ctx* c, const char* what, bool kernel = true) {
    if (kernel) c->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return UOT_OK;
}

static int launch_setup(uot_ctx* c) {
    SetupArgs S{c->T, c->P, c->N, c->bpp, c->b.frames, c->prox ? nullptr : c->b.f, c->part};
    k_setup_f<<<dim3(c->bpp, c->G), 256, 0, c->s>>>(S);
    int rc = check_launch(c, "k_setup_f");
    if (rc) return rc;
    ReduceArgs R{};
    R.partials = c->part; R.recs_per_pair = c->bpp; R.G = c->G; R.pair_out = c->pair_obj;
    R.glob = c->glob; R.counter = c->counter; R.stop = nullptr; R.max_mask = 0u;
    R.is_iteration = 0; R.is_setup = 1; R.iteration = 0; R.tol = 0; R.tau1 = c->tau1;
    k_pair_reduce<<<c->G, 256, 0, c->s>>>(R);
    return check_launch(c, "k_pair_reduce(setup)");
}

// NVTX range over one C-ABI call (host-side enqueue time; the device work it enqueues follows)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static int resolve_pending(uot_ctx* c);

int uot_reset(uot_ctx* c, uint32_t flags) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    const size_t bytes = (size_t)c->G * c->N * sizeof(float);
    cudaMemsetAsync(c->b.mx[0], 0, bytes, c->s);
    cudaMemsetAsync(c->b.my[0], 0, bytes, c->s);
    cudaMemsetAsync(c->b.r, 0, bytes, c->s);
    cudaMemsetAsync(c->b.a[0], 0, bytes, c->s);
    c->slot = 0;
    c->rcur = 0;
    c->stop_armed = false;          // the cold start supersedes any pending device-side stop
    c->ext_stop = false;
    c->log.clear();
    c->persist_base.clear();
    int rc = check_launch(c, "memset", false);
    if (rc) return rc;
    k_init_glob<<<1, 32, 0, c->s>>>(c->glob, c->stop, c->counter, 1);
    rc = check_launch(c, "k_init_glob");
    if (rc) return rc;
    if (c->prox) {
        const long long n = (long long)c->B * c->T * c->N;
        k_init_x<<<4 * kSMs, 256, 0, c->s>>>(c->b.frames, c->b.x[0], n, (flags & UOT_RESET_X_FROM_P) ? 1 : 0,
                                             (c->p.flags & UOT_FIX_FIRST_FRAME) ? 1 : 0, c->N, c->T);
        rc = check_launch(c, "k_init_x");
        if (rc) return rc;
    }
    c->iter = 0;
    return launch_setup(c);
}

int uot_load_frames(uot_ctx* c, const float* host_frames) {
    if (!c || !host_frames) return fail(c, UOT_E_INVALID, "null argument");
    int prc = resolve_pending(c);       // the setup reduction rewrites the report slots
    if (prc) return prc;
    const size_t bytes = (size_t)c->B * c->T * c->N * sizeof(float);
    cudaError_t e = cudaMemcpyAsync(const_cast<float*>(c->b.frames), host_frames, bytes, cudaMemcpyHostToDevice, c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaMemcpyAsync: %s", cudaGetErrorString(e));
    return launch_setup(c);
}

// Launch with programmatic dependent launch when enabled (UOT_PDL, default on): the kernel
// (k_wave, k_iter2, k_pair_reduce: pdl_wait() first) may be scheduled while its predecessor
// drains, hiding the launch latency of back-to-back passes on small grids.
static cudaError_t launch_k(const uot_ctx* c, const void* fn, dim3 grid, dim3 block, size_t smem, void** args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = c->pdl ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

extern "C++" {
template <int V, bool RED, bool PROX>
static void launch_iter_t(uot_ctx* c, const IterArgs& A) {
    const int blocks = (A.items + kWarps - 1) / kWarps;
    void* args[1] = {(void*)&A};
    launch_k(c, (const void*)k_iter<V, RED, PROX>, dim3(blocks), dim3(kWarps * 32), 0, args);
}
template <int V>
static void launch_iter_v(uot_ctx* c, const IterArgs& A, bool red, bool prox) {
    if (prox) {
        if (red) launch_iter_t<V, true, true>(c, A); else launch_iter_t<V, false, true>(c, A);
    } else {
        if (red) launch_iter_t<V, true, false>(c, A); else launch_iter_t<V, false, false>(c, A);
    }
}
}

// Pairs selected by a launch: all, interior (not adjacent to a shard halo), boundary.
static int pairs_in_part(const uot_ctx* c, int part) {
    if (part == UOT_PART_ALL) return c->G;
    const int nb = c->P >= 2 ? 2 : 1;
    if (part == UOT_PART_BOUNDARY) return c->B * nb;
    return c->B * (c->P - nb);
}

// One kernel launch of iteration c->iter for `part`; part ALL / BOUNDARY completes
// the iteration (slot flip, reductions when `red`).
static float* rbuf(const uot_ctx* c) { return c->rcur ? c->b.r_alt : c->b.r; }
static void log_launch(uot_ctx* c) {
    if (c->stop_armed) c->log.push_back({c->iter, c->slot, c->rcur});
}

static int launch_one(uot_ctx* c, int part, bool red, const int* stop, double tol) {
    const int in = c->slot, o = in ^ 1;
    const int gsel = pairs_in_part(c, part);
    if (gsel > 0) {
        IterArgs A{};
        A.nx = c->nx; A.ny = c->ny;
        A.strips = c->geo.strips; A.segs = c->geo.segs; A.H = c->geo.H;
        A.items = gsel * c->geo.strips * c->geo.segs;
        A.sel = part; A.Gsel = gsel;
        A.N = c->N;
        A.f = c->b.f;
        A.mx_in = c->b.mx[in]; A.my_in = c->b.my[in]; A.a_in = c->b.a[in];
        A.mx_out = c->b.mx[o]; A.my_out = c->b.my[o]; A.a_out = c->b.a[o];
        A.r = rbuf(c);
        A.tau1 = c->tau1f; A.tau2 = c->tau2f; A.atau1 = (float)(c->p.alpha * c->tau1);
        A.r_mode = c->r_mode; A.r_scale = c->r_scale; A.fix_first = c->fix_first;
        A.G = c->G; A.T = c->T; A.P = c->P;
        if (c->prox) {
            const double rt = c->p.rho * c->tau1;
            A.x_in = c->b.x[in]; A.x_out = c->b.x[o]; A.p = c->b.frames;
            A.a_prev_halo = c->b.a_prev_halo; A.a_next_halo = c->b.a_next_halo;
            A.c1 = (float)(rt / (1.0 + rt)); A.c2 = (float)(1.0 / (1.0 + rt)); A.c3 = (float)(c->tau1 / (1.0 + rt));
        }
        A.partials = c->part;
        A.stop = stop;
        cudaEvent_t e1 = nullptr;
        if (c->timing) {
            if (c->ev_used + 2 > c->ev.size()) {
                for (int q = 0; q < 2; ++q) {
                    cudaEvent_t e;
                    if (cudaEventCreate(&e) != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventCreate");
                    c->ev.push_back(e);
                }
            }
            cudaEventRecord(c->ev[c->ev_used], c->s);
            e1 = c->ev[c->ev_used + 1];
            c->ev_used += 2;
            c->ev_kind.push_back(0);
        }
        if (c->geo.vec == 4) launch_iter_v<4>(c, A, red, c->prox);
        else if (c->geo.vec == 2) launch_iter_v<2>(c, A, red, c->prox);
        else launch_iter_v<1>(c, A, red, c->prox);
        if (e1) cudaEventRecord(e1, c->s);
        int rc = check_launch(c, "k_iter");
        if (rc) return rc;
    }
    if (part == UOT_PART_INTERIOR) return UOT_OK;
    c->iter++;
    c->slot ^= 1;
    log_launch(c);
    if (red) {
        ReduceArgs R{};
        R.partials = c->part; R.recs_per_pair = c->geo.strips * c->geo.segs; R.G = c->G;
        R.pair_out = c->pair_it; R.glob = c->glob; R.counter = c->counter;
        R.stop = const_cast<int*>(stop); R.max_mask = 0u; R.is_iteration = 1; R.is_setup = 0;
        R.iteration = c->iter; R.tol = tol; R.tau1 = c->tau1;
        {
            void* rargs[1] = {(void*)&R};
            launch_k(c, (const void*)k_pair_reduce, dim3(c->G), dim3(256), 0, rargs);
        }
        int rc = check_launch(c, "k_pair_reduce(iter)");
        if (rc) return rc;
    }
    return UOT_OK;
}

static int launch_persist(uot_ctx* c, int n, int reduce_every, bool reduce_last, const int* stop, double tol) {
    cudaError_t e = cudaMemsetAsync(c->pflags, 0, sizeof(int) * (kMaxPersistCtas + 2), c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "memset flags: %s", cudaGetErrorString(e));
    PersistArgs A{};
    A.nx = c->nx; A.ny = c->ny; A.G = c->G; A.T = c->T; A.P = c->P; A.N = c->N;
    A.TW = c->pg.TW; A.TH = c->pg.TH; A.tiles_x = c->pg.tx; A.tiles_y = c->pg.ty;
    A.n_iters = n; A.red_every = reduce_every; A.red_last = reduce_last ? 1 : 0;
    A.iter0 = c->iter; A.slot0 = c->slot; A.prox = c->prox;
    A.f = c->b.f;
    for (int q = 0; q < 2; ++q) {
        A.mxb[q] = c->b.mx[q]; A.myb[q] = c->b.my[q]; A.ab[q] = c->b.a[q]; A.xb[q] = c->b.x[q];
    }
    A.r = rbuf(c); A.p = c->b.frames;
    A.tau1 = c->tau1f; A.tau2 = c->tau2f; A.atau1 = (float)(c->p.alpha * c->tau1);
    A.r_mode = c->r_mode; A.r_scale = c->r_scale; A.fix_first = c->fix_first;
    if (c->prox) {
        const double rt = c->p.rho * c->tau1;
        A.c1 = (float)(rt / (1.0 + rt)); A.c2 = (float)(1.0 / (1.0 + rt)); A.c3 = (float)(c->tau1 / (1.0 + rt));
    }
    A.xchg = c->pxchg; A.flags = c->pflags; A.bar = c->pflags + kMaxPersistCtas;
    A.partials = c->part; A.pair_out = c->pair_it; A.glob = c->glob;
    A.stop = const_cast<int*>(stop); A.tol = tol; A.tau1d = c->tau1;
    void* args[] = {&A};
    cudaEvent_t e1 = nullptr;
    if (c->timing) {
        while (c->ev_used + 2 > c->ev.size()) {
            cudaEvent_t ev;
            if (cudaEventCreate(&ev) != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventCreate");
            c->ev.push_back(ev);
        }
        cudaEventRecord(c->ev[c->ev_used], c->s);
        e1 = c->ev[c->ev_used + 1];
        c->ev_used += 2;
        c->ev_kind.push_back(2);
    }
    const void* fn = c->prox ? (const void*)k_persist<true> : (const void*)k_persist<false>;
    e = cudaLaunchCooperativeKernel(fn, dim3(c->pg.ctas), dim3(c->pg.threads), args, c->pg.smem, c->s);
    if (e1) cudaEventRecord(e1, c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "k_persist launch: %s", cudaGetErrorString(e));
    int rc = check_launch(c, "k_persist");
    if (rc) return rc;
    const int slot0 = c->slot;
    c->slot = slot0 ^ (n & 1);            // the kernel writes iterate iter0 + done to slot slot0 ^ (done & 1)
    if (c->stop_armed) c->persist_base.push_back({c->iter, slot0, c->rcur});   // (device-stop correction)
    c->iter += n;            // uot_get_report corrects it if the device stopped early
    c->persist_launches++;
    return UOT_OK;
}

// Small single-pair fixed-marginal grids (C1): all n iterations in ONE CTA (k_single,
// uot_single.cuh), reductions and stopping test in-kernel.
static bool use_single(const uot_ctx* c) {
    return !c->prox && c->G == 1 && c->t2vec && c->single_on && (c->nx / 4) * c->ny <= kSingleThreads;
}

static int launch_single(uot_ctx* c, int n, int reduce_every, bool reduce_last, const int* stop, double tol) {
    SingleArgs A{};
    A.nx = c->nx; A.ny = c->ny; A.f = c->b.f;
    A.slot0 = c->slot;
    A.mx_in = c->b.mx[c->slot]; A.my_in = c->b.my[c->slot]; A.a_in = c->b.a[c->slot];
    for (int q = 0; q < 2; ++q) { A.mxb[q] = c->b.mx[q]; A.myb[q] = c->b.my[q]; A.ab[q] = c->b.a[q]; }
    A.r = rbuf(c);
    A.tau1 = c->tau1f; A.tau2 = c->tau2f; A.atau1 = (float)(c->p.alpha * c->tau1); A.r_scale = c->r_scale;
    A.n_iters = n; A.red_every = reduce_every; A.red_last = reduce_last ? 1 : 0;
    A.iter0 = c->iter;
    A.pair_out = c->pair_it; A.glob = c->glob;
    A.stop = const_cast<int*>(stop); A.tol = tol; A.tau1d = c->tau1;
    void* args[1] = {(void*)&A};
    cudaEvent_t e1 = nullptr;
    if (c->timing) {
        while (c->ev_used + 2 > c->ev.size()) {
            cudaEvent_t ev;
            if (cudaEventCreate(&ev) != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventCreate");
            c->ev.push_back(ev);
        }
        cudaEventRecord(c->ev[c->ev_used], c->s);
        e1 = c->ev[c->ev_used + 1];
        c->ev_used += 2;
        c->ev_kind.push_back(10);
    }
    // pixels per thread: 16 (UOT_SINGLE_V=16, nx % 16 == 0), 8 (nx % 8 == 0, default) or 4
    const int V = (c->single_v == 16 && c->nx % 16 == 0) ? 16 : ((c->nx % 8 == 0 && c->single_v != 4) ? 8 : 4);
    const void* fn = V == 16 ? (c->r_mode == 0 ? (const void*)k_single<0, 16>
                                               : (c->r_mode == 1 ? (const void*)k_single<1, 16> : (const void*)k_single<2, 16>))
                   : V == 8 ? (c->r_mode == 0 ? (const void*)k_single<0, 8>
                                              : (c->r_mode == 1 ? (const void*)k_single<1, 8> : (const void*)k_single<2, 8>))
                            : (c->r_mode == 0 ? (const void*)k_single<0, 4>
                                              : (c->r_mode == 1 ? (const void*)k_single<1, 4> : (const void*)k_single<2, 4>));
    const int threads = ((c->nx / V) * c->ny + 31) / 32 * 32;
    launch_k(c, fn, dim3(1), dim3(threads), 0, args);
    if (e1) cudaEventRecord(e1, c->s);
    int rc = check_launch(c, "k_single");
    if (rc) return rc;
    const int slot0 = c->slot;
    c->slot = slot0 ^ (n & 1);            // iterate iter0 + done is written to slot slot0 ^ (done & 1)
    if (c->stop_armed) c->persist_base.push_back({c->iter, slot0, c->rcur});   // (device-stop correction)
    c->iter += n;
    c->persist_launches++;
    return UOT_OK;
}

// All n iterations in one cooperative launch of k_tpersist (uot_tpersist.inc): passes of 4 (2
// before a checked iteration) on SMEM tiles, one grid barrier per pass.  Requires every run up
// to a check to be even (use_tpersist).  The host replays the pass plan for the slot / r-buffer
// bookkeeping and the device-stop log.
static bool use_tpersist(const uot_ctx* c, int n, int reduce_every) {
    return c->tp.ok && c->t2ok && c->t2on && n >= 2 && (n % 2 == 0) && (reduce_every % 2 == 0);
}

static int launch_tpersist(uot_ctx* c, int n, int reduce_every, bool reduce_last, const int* stop, double tol) {
    cudaError_t e = cudaMemsetAsync(c->pflags + kMaxPersistCtas, 0, 2 * sizeof(int), c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "memset barrier: %s", cudaGetErrorString(e));
    TPArgs P{};
    Iter2Args& A = P.A;
    A.nx = c->nx; A.ny = c->ny; A.tiles_x = c->tp.tx; A.tiles_y = c->tp.ty; A.N = c->N;
    A.f = c->b.f;
    A.tau1 = c->tau1f; A.tau2 = c->tau2f; A.atau1 = (float)(c->p.alpha * c->tau1);
    A.r_mode = c->r_mode; A.r_scale = c->r_scale;
    A.vec = 1; A.tma = 1;
    A.partials = c->part;
    for (int q = 0; q < 2; ++q) { P.mxb[q] = c->b.mx[q]; P.myb[q] = c->b.my[q]; P.ab[q] = c->b.a[q]; }
    P.rb[0] = c->b.r; P.rb[1] = c->b.r_alt;
    P.slot0 = c->slot; P.rcur0 = c->rcur;
    P.n_iters = n; P.red_every = reduce_every; P.red_last = reduce_last ? 1 : 0;
    P.iter0 = c->iter;
    P.bar = c->pflags + kMaxPersistCtas;
    P.stop = const_cast<int*>(stop);
    P.pair_out = c->pair_it; P.glob = c->glob; P.tol = tol; P.tau1d = c->tau1;
    TPMaps M;
    memset(&M, 0, sizeof(M));
    for (int si = 0; si < 2; ++si)
        for (int par = 0; par < 2; ++par) {
            const int sl = c->slot ^ par, rb = c->rcur ^ par;
            M.m[si][par][0] = c->tp.mx[si][sl]; M.m[si][par][1] = c->tp.my[si][sl];
            M.m[si][par][2] = c->tp.r[si][rb]; M.m[si][par][3] = c->tp.a[si][sl]; M.m[si][par][4] = c->tp.f[si];
        }
    void* args[2] = {(void*)&P, (void*)&M};
    cudaEvent_t e1 = nullptr;
    if (c->timing) {
        while (c->ev_used + 2 > c->ev.size()) {
            cudaEvent_t ev;
            if (cudaEventCreate(&ev) != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventCreate");
            c->ev.push_back(ev);
        }
        cudaEventRecord(c->ev[c->ev_used], c->s);
        e1 = c->ev[c->ev_used + 1];
        c->ev_used += 2;
        c->ev_kind.push_back(8);
    }
    e = cudaLaunchCooperativeKernel(c->tp.fn, dim3(c->tp.ctas), dim3(c->tp.nt), args, c->tp.smem, c->s);
    if (e1) cudaEventRecord(e1, c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "k_tpersist launch: %s", cudaGetErrorString(e));
    int rc = check_launch(c, "k_tpersist");
    if (rc) return rc;
    // replay the device's pass plan: slots, r buffer and the device-stop log per pass
    for (int k = 0; k < n;) {
        int d = n - k;
        if (reduce_every > 0) d = std::min(d, reduce_every - (k % reduce_every));
        const int S = d >= 4 ? 4 : 2;
        k += S;
        c->iter += S;
        c->slot ^= 1;
        c->rcur ^= 1;
        log_launch(c);
    }
    c->persist_launches++;
    return UOT_OK;
}

// S fixed-marginal iterations in one HBM pass (k_iter2<TH, S>, uot_temporal.cuh): iterations
// iter+1 .. iter+S; reductions (red) for iteration iter+S.
static int launch_pass(uot_ctx* c, int vi, bool red, const int* stop, double tol) {
    const TVar& v = c->tv[vi];
    const int in = c->slot, o = in ^ 1;
    Iter2Args A{};
    A.nx = c->nx; A.ny = c->ny; A.tiles_x = v.tx; A.tiles_y = v.ty; A.N = c->N;
    A.f = c->b.f;
    A.mx_in = c->b.mx[in]; A.my_in = c->b.my[in]; A.a_in = c->b.a[in]; A.r_in = rbuf(c);
    A.mx_out = c->b.mx[o]; A.my_out = c->b.my[o]; A.a_out = c->b.a[o];
    A.r_out = c->rcur ? c->b.r : c->b.r_alt;
    A.tau1 = c->tau1f; A.tau2 = c->tau2f; A.atau1 = (float)(c->p.alpha * c->tau1);
    A.r_mode = c->r_mode; A.r_scale = c->r_scale;
    A.vec = c->t2vec;
    A.tma = v.tma ? 1 : 0;
    Iter2Maps Mp;
    memset(&Mp, 0, sizeof(Mp));
    if (v.tma) {
        Mp.tmap[0] = v.mx[in]; Mp.tmap[1] = v.my[in]; Mp.tmap[2] = v.r[c->rcur];
        Mp.tmap[3] = v.a[in]; Mp.tmap[4] = v.f;
    }
    A.partials = c->part; A.stop = stop;
    WaveArgs W{};
    if (v.wave) {
        W.nx = c->nx; W.ny = c->ny; W.strips = v.tx; W.segs = v.ty; W.H = v.th; W.G = c->G; W.N = c->N;
        W.f = A.f; W.mx_in = A.mx_in; W.my_in = A.my_in; W.a_in = A.a_in; W.r_in = A.r_in;
        W.mx_out = A.mx_out; W.my_out = A.my_out; W.a_out = A.a_out; W.r_out = A.r_out;
        W.tau1 = A.tau1; W.tau2 = A.tau2; W.atau1 = A.atau1; W.r_scale = A.r_scale;
        W.partials = c->part; W.stop = stop;
    }
    const long long units = (long long)c->G * v.tx * v.ty;
    const unsigned blocks = (unsigned)(v.wave ? (units + kWaveWarps - 1) / kWaveWarps : units);
    cudaEvent_t e1 = nullptr;
    if (c->timing) {
        while (c->ev_used + 2 > c->ev.size()) {
            cudaEvent_t ev;
            if (cudaEventCreate(&ev) != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventCreate");
            c->ev.push_back(ev);
        }
        cudaEventRecord(c->ev[c->ev_used], c->s);
        e1 = c->ev[c->ev_used + 1];
        c->ev_used += 2;
        c->ev_kind.push_back(v.wave ? (v.S == 5 ? 9 : (v.S == 4 ? 6 : (v.S == 3 ? 7 : 5))) : (v.S == 4 ? 3 : 1));
    }
    if (v.wave) {
        void* kargs[1] = {(void*)&W};
        launch_k(c, v.fn[red ? 1 : 0], dim3(blocks), dim3(v.threads), v.smem, kargs);
    } else {
        void* kargs[2] = {(void*)&A, (void*)&Mp};
        launch_k(c, v.fn[red ? 1 : 0], dim3(blocks), dim3(v.threads), v.smem, kargs);
    }
    if (e1) cudaEventRecord(e1, c->s);
    int rc = check_launch(c, "k_iter2");
    if (rc) return rc;
    c->iter += v.S;
    c->slot ^= 1;
    c->rcur ^= 1;
    log_launch(c);
    if (red) {
        ReduceArgs R{};
        R.partials = c->part; R.recs_per_pair = v.tx * v.ty; R.G = c->G;
        R.pair_out = c->pair_it; R.glob = c->glob; R.counter = c->counter;
        R.stop = const_cast<int*>(stop); R.max_mask = 0u; R.is_iteration = 1; R.is_setup = 0;
        R.iteration = c->iter; R.tol = tol; R.tau1 = c->tau1;
        {
            void* rargs[1] = {(void*)&R};
            launch_k(c, (const void*)k_pair_reduce, dim3(c->G), dim3(256), 0, rargs);
        }
        rc = check_launch(c, "k_pair_reduce(iter2)");
        if (rc) return rc;
    }
    return UOT_OK;
}

// Chain prox: S (4 or 2) iterations in one pass of k_wave_prox (uot_wave_prox.cuh), launched as
// clusters of pw.cl CTAs; iterations iter+1 .. iter+S, reductions (red) for iteration iter+S.
static int launch_prox_pass(uot_ctx* c, int S, bool red, const int* stop, double tol) {
    const int in = c->slot, o = in ^ 1;
    const int strips = S == 2 ? c->pw.strips2 : c->pw.strips;    // the pass's own halo (lanes per side)
    uotk::WaveProxArgs W{};
    W.nx = c->nx; W.ny = c->ny; W.strips = strips; W.segs = c->pw.segs; W.H = c->pw.H;
    W.B = c->B; W.T = c->T; W.P = c->P; W.groups = c->pw.groups; W.cl = c->pw.cl; W.N = c->N;
    W.own_lo = c->pw.own_lo; W.own_hi = c->pw.own_hi;
    W.p = c->b.frames;
    W.mx_in = c->b.mx[in]; W.my_in = c->b.my[in]; W.a_in = c->b.a[in]; W.r_in = rbuf(c); W.x_in = c->b.x[in];
    W.mx_out = c->b.mx[o]; W.my_out = c->b.my[o]; W.a_out = c->b.a[o];
    W.r_out = c->rcur ? c->b.r : c->b.r_alt; W.x_out = c->b.x[o];
    const double rt = c->p.rho * c->tau1;
    W.tau1 = c->tau1f; W.tau2 = c->tau2f; W.atau1 = (float)(c->p.alpha * c->tau1); W.r_scale = c->r_scale;
    W.c1 = (float)(rt / (1.0 + rt)); W.c2 = (float)(1.0 / (1.0 + rt)); W.c3 = (float)(c->tau1 / (1.0 + rt));
    W.fix_first = c->fix_first;
    W.partials = c->part; W.stop = stop;
    cudaEvent_t e1 = nullptr;
    if (c->timing) {
        while (c->ev_used + 2 > c->ev.size()) {
            cudaEvent_t ev;
            if (cudaEventCreate(&ev) != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventCreate");
            c->ev.push_back(ev);
        }
        cudaEventRecord(c->ev[c->ev_used], c->s);
        e1 = c->ev[c->ev_used + 1];
        c->ev_used += 2;
        c->ev_kind.push_back(11);
    }
    if (red && (c->pw.own_lo > 0 || c->pw.own_hi < c->P)) {
        // ghost pairs are not reduced: zero their records ([pair][strips * segs][kRec], contiguous
        // per pair), which the kernel leaves untouched
        const size_t per = (size_t)strips * c->pw.segs * kRec * sizeof(double);
        for (int b = 0; b < c->B; ++b) {
            double* base = c->part + (size_t)b * c->P * strips * c->pw.segs * kRec;
            cudaError_t me = cudaSuccess;
            if (c->pw.own_lo > 0) me = cudaMemsetAsync(base, 0, per * c->pw.own_lo, c->s);
            if (me == cudaSuccess && c->pw.own_hi < c->P)
                me = cudaMemsetAsync(base + (size_t)c->pw.own_hi * strips * c->pw.segs * kRec, 0,
                                     per * (c->P - c->pw.own_hi), c->s);
            if (me != cudaSuccess) return fail(c, UOT_E_CUDA, "ghost records: %s", cudaGetErrorString(me));
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(c->B * c->pw.groups * c->pw.cl), (unsigned)(strips * c->pw.segs));
    cfg.blockDim = dim3(c->pw.warps * 32);
    cfg.dynamicSmemBytes = c->pw.smem[S == 2 ? 1 : 0];
    cfg.stream = c->s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c->pw.cl; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = c->pdl ? 2 : 1;
    void* kargs[1] = {(void*)&W};
    cudaError_t e = cudaLaunchKernelExC(&cfg, c->pw.fn[S == 2 ? 1 : 0][red ? 1 : 0], kargs);
    if (e1) cudaEventRecord(e1, c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "k_wave_prox launch: %s", cudaGetErrorString(e));
    int rc = check_launch(c, "k_wave_prox");
    if (rc) return rc;
    c->iter += S;
    c->slot ^= 1;
    c->rcur ^= 1;
    log_launch(c);
    if (red) {
        ReduceArgs R{};
        R.partials = c->part; R.recs_per_pair = strips * c->pw.segs; R.G = c->G;
        R.pair_out = c->pair_it; R.glob = c->glob; R.counter = c->counter;
        R.stop = const_cast<int*>(stop); R.max_mask = 0u; R.is_iteration = 1; R.is_setup = 0;
        R.iteration = c->iter; R.tol = tol; R.tau1 = c->tau1;
        {
            void* rargs[1] = {(void*)&R};
            launch_k(c, (const void*)k_pair_reduce, dim3(c->G), dim3(256), 0, rargs);
        }
        rc = check_launch(c, "k_pair_reduce(prox wave)");
        if (rc) return rc;
    }
    return UOT_OK;
}

// Small grids: the SMEM-resident persistent kernel, unless k_iter2 serves the fixed-
// marginal problem and it has more than kPersistMaxPx pair-pixels (measured: C2, 512^2,
// 5.5 us/iteration with k_iter2 vs 8.8 with k_persist; C1, 64^2: k_persist 2x faster).
static const long long kPersistMaxPx = 65536;
static bool use_persist(const uot_ctx* c) {
    if (!c->pg.ok) return false;
    return !(c->t2ok && c->t2on && (long long)c->G * c->N > kPersistMaxPx);
}

// Temporally blocked pass of S iterations available in this context: its variant index, or -1.
static int pass_variant(const uot_ctx* c, int S) {
    if (!(c->t2ok && c->t2on)) return -1;
    if (S == 2) return c->tv[0].ok ? 0 : -1;
    if (!c->t4on) return -1;
    if (S == 4) return c->tv[1].ok ? 1 : -1;
    if (S == 3) return c->tv[2].ok ? 2 : -1;
    if (S == 5) return c->tv[3].ok ? 3 : -1;
    return -1;
}

// Iterations of the first pass of the cheapest split of d iterations into passes of the
// available S (a reduction may only follow the last pass; order is immaterial to the cost).
static int pick_pass(const uot_ctx* c, int d) {
    bool av[6] = {false, true, pass_variant(c, 2) >= 0, pass_variant(c, 3) >= 0, pass_variant(c, 4) >= 0,
                  pass_variant(c, 5) >= 0};
    if (d > 12) {                       // long runs: the best cost per iteration
        int b = 1;
        for (int S = 2; S <= 5; ++S)
            if (av[S] && c->pass_cost[S] / S < c->pass_cost[b] / b) b = S;
        return b;
    }
    float best[13];
    int first[13];
    best[0] = 0.f;
    first[0] = 0;
    for (int x = 1; x <= d; ++x) {
        best[x] = 1e30f;
        first[x] = 1;
        for (int S = 1; S <= 5; ++S)            // ties: the short pass first (the checked pass is a long one)
            if (av[S] && S <= x && c->pass_cost[S] + best[x - S] < best[x]) {
                best[x] = c->pass_cost[S] + best[x - S];
                first[x] = S;
            }
    }
    return first[d];
}

static int launch_iters(uot_ctx* c, int n, int reduce_every, bool reduce_last, const int* stop, double tol) {
    if (n >= 1 && use_single(c)) return launch_single(c, n, reduce_every, reduce_last, stop, tol);
    if (use_tpersist(c, n, reduce_every)) return launch_tpersist(c, n, reduce_every, reduce_last, stop, tol);
    if (use_persist(c) && n >= 2) return launch_persist(c, n, reduce_every, reduce_last, stop, tol);
    const bool poll = stop != nullptr && n > 2 * kPollChunk && c->poll.init();
    if (poll) c->poll.begin();
    auto need_red = [&](int k) {
        return (reduce_last && k == n - 1) || (reduce_every > 0 && ((k + 1) % reduce_every == 0));
    };
    int next_poll = kPollChunk;
    for (int k = 0; k < n;) {
        if (poll && k >= next_poll) {
            next_poll += kPollChunk;
            c->poll.post(stop, c->s);
            if (c->poll.stopped()) {            // the device stopped >= one chunk ago: skip the rest
                c->iter += n - k;               // uot_get_report corrects the count from the device
                return UOT_OK;
            }
        }
        // iterations up to and including the next reduction (or the end of the call)
        int d = n - k;
        if (reduce_every > 0) d = std::min(d, reduce_every - (k % reduce_every));
        if (c->pw.ok) {                 // chain prox: passes of 3 and 2 (one k_iter only for a single iteration)
            const int L = c->pw.S;         // (never a one-iteration pass unless d == 1)
            const int S = c->pw.prefer2 ? ((d % 2 == 1 && d >= 3) ? 3 : (d >= 2 ? 2 : 1))
                                        : (d == L + 1 ? 2 : (d >= L ? L : (d >= 2 ? 2 : 1)));
            if (S == 1 && (c->pw.own_lo > 0 || c->pw.own_hi < c->P))   // k_iter would update the ghost pairs
                return fail(c, UOT_E_INVALID, "ghost pairs set (uot_set_own_pairs): iterate in runs of 2..%d between checks", L);
            const int rc = S == 1 ? launch_one(c, UOT_PART_ALL, need_red(k), stop, tol)
                                  : launch_prox_pass(c, S, need_red(k + S - 1), stop, tol);
            k += S;
            if (rc) return rc;
            continue;
        }
        const int S = pick_pass(c, d);
        const int rc = S == 1 ? launch_one(c, UOT_PART_ALL, need_red(k), stop, tol)
                              : launch_pass(c, pass_variant(c, S), need_red(k + S - 1), stop, tol);
        k += S;
        if (rc) return rc;
    }
    return UOT_OK;
}

static int read_glob(uot_ctx* c, double* h) {
    cudaError_t e = cudaMemcpyAsync(h, c->glob, GL_N * sizeof(double), cudaMemcpyDeviceToHost, c->s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "reading reductions: %s", cudaGetErrorString(e));
    return UOT_OK;
}

static void fill_report(const uot_ctx* c, const double* h, uot_report* out) {
    memset(out, 0, sizeof(*out));
    const double a = c->p.alpha;
    out->transport = h[GL_TR];
    const bool bal = c->r_mode == 2;
    out->growth = bal ? 0.0 : a * h[GL_GR];
    out->prox_term = c->prox ? 0.5 * c->p.rho * h[GL_PX] : 0.0;
    out->objective = out->transport + out->growth + out->prox_term;
    out->primal_res = sqrt(h[GL_K2]);
    out->dual_res = sqrt(h[GL_DZ]) / c->tau1;
    out->upper_bound = bal ? (h[GL_UB] == 0.0 ? out->transport : INFINITY) : out->transport + a * h[GL_UB];
    out->lower_bound = NAN;
    out->f_norm = sqrt(h[GL_FSQ]);
    out->iterations = c->iter;
    out->converged = h[GL_CONV] >= 0.0;
    out->nonfinite = h[GL_NONF] != 0.0;
}

int uot_iterate(uot_ctx* c, int32_t n, int32_t check_every, double tol) {
    NvtxRange nvtx_("uot_iterate");
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    if (n < 0 || check_every < 0) return fail(c, UOT_E_INVALID, "n_iters and check_every must be >= 0");
    if (c->ext_stop) {                   // one chunk of a cross-rank stopped run: no local test
        if (tol > 0.0) return fail(c, UOT_E_INVALID, "external stop armed: pass tol = 0 and test with uot_stop_apply");
        return launch_iters(c, n, check_every, n > 0, c->stop, 0.0);
    }
    int prc = resolve_pending(c);
    if (prc) return prc;
    const int* stop = nullptr;
    if (tol > 0.0) {
        k_init_glob<<<1, 32, 0, c->s>>>(c->glob, c->stop, c->counter, 0);
        int rc = check_launch(c, "k_init_glob");
        if (rc) return rc;
        stop = c->stop;
        c->stop_armed = true;
        c->log.clear();
        c->persist_base.clear();
        c->log.push_back({c->iter, c->slot, c->rcur});
    }
    return launch_iters(c, n, check_every, n > 0, stop, tol);
}

int uot_iterate_part(uot_ctx* c, int32_t part, int32_t reduce) {
    NvtxRange nvtx_("uot_iterate_part");
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    if (part != UOT_PART_ALL && part != UOT_PART_INTERIOR && part != UOT_PART_BOUNDARY)
        return fail(c, UOT_E_INVALID, "bad part %d", part);
    if (c->ext_stop) return launch_one(c, part, reduce != 0, c->stop, 0.0);
    int prc = resolve_pending(c);
    if (prc) return prc;
    return launch_one(c, part, reduce != 0, nullptr, 0.0);
}

// Apply a device-side stop armed by uot_iterate(tol > 0) / uot_solve: the launches after
// the stopping iteration exited without writing, so the host's iteration count, slot and r
// buffer are rewound to the stop entry of the launch log.
static void apply_stop(uot_ctx* c, const double* h) {
    if (!c->stop_armed) return;
    const int64_t planned = c->iter;
    if (h[GL_CONV] >= 0.0) c->iter = (int64_t)h[GL_CONV];             // later launches exited early
    else if (h[GL_NONF] != 0.0 && h[GL_LASTRED] > 0) c->iter = (int64_t)h[GL_LASTRED];
    if (c->iter != planned) {
        // slot / r buffer of the iterate the device stopped at: replay the launch log
        // (a k_iter2 pass advances 2 iterations but flips the slots once)
        bool found = false;
        for (const auto& e : c->log)
            if (e.iter == c->iter) { c->slot = e.slot; c->rcur = e.rcur; found = true; break; }
        if (!found)                                                   // stopped inside a persistent launch
            for (const auto& e : c->persist_base)
                if (e.iter <= c->iter) { c->slot = e.slot ^ (int)((c->iter - e.iter) & 1); c->rcur = e.rcur; }
    }
    c->stop_armed = false;
    c->ext_stop = false;
    c->log.clear();
    c->persist_base.clear();
}

static bool capturing(const uot_ctx* c) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(c->s, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusActive;
}

// Every entry point that enqueues work on the iterate first resolves a stop armed by an
// earlier asynchronous uot_iterate(tol > 0): otherwise it would read a slot the device may
// never have written, and a later report would rewind past its work.  Resolving needs one
// stream synchronisation, which a graph capture cannot contain.
static int resolve_pending(uot_ctx* c) {
    if (!c->stop_armed) return UOT_OK;
    if (capturing(c))
        return fail(c, UOT_E_INVALID, "a device-side stop is pending: call uot_get_report before capturing");
    double h[GL_N];
    int rc = read_glob(c, h);
    if (rc) return rc;
    apply_stop(c, h);
    return UOT_OK;
}

int uot_get_report(uot_ctx* c, uot_report* out) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    double h[GL_N];
    int rc = read_glob(c, h);
    if (rc) return rc;
    apply_stop(c, h);
    uot_report rep;
    fill_report(c, h, &rep);
    if (out) *out = rep;
    if (rep.nonfinite) return fail(c, UOT_E_NONFINITE, "non-finite value in the reductions");
    return UOT_OK;
}

int uot_prox_step(uot_ctx* c, int32_t n, uot_report* out) {
    NvtxRange nvtx_("uot_prox_step");
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    if (n < 0) return fail(c, UOT_E_INVALID, "n_iters < 0");
    const bool cap = capturing(c);
    if (cap && out) return fail(c, UOT_E_INVALID, "a host report needs a stream synchronisation: pass out = NULL under graph capture");
    int rc = resolve_pending(c);
    if (rc) return rc;
    const int slot0 = c->slot, rcur0 = c->rcur;
    rc = launch_iters(c, n, 0, out != nullptr && n > 0, nullptr, 0.0);
    if (rc) return rc;
    // Under CUDA-graph capture every replay re-runs the captured launches with the captured
    // buffer pointers, so the call must end in the slots it started from: copy the iterate
    // back when the passes flipped them an odd number of times.
    if (cap && (c->slot != slot0 || c->rcur != rcur0)) {
        const size_t plane = (size_t)c->G * c->N * sizeof(float);
        cudaError_t e = cudaSuccess;
        if (c->slot != slot0) {
            e = cudaMemcpyAsync(c->b.mx[slot0], c->b.mx[c->slot], plane, cudaMemcpyDeviceToDevice, c->s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(c->b.my[slot0], c->b.my[c->slot], plane, cudaMemcpyDeviceToDevice, c->s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(c->b.a[slot0], c->b.a[c->slot], plane, cudaMemcpyDeviceToDevice, c->s);
            if (e == cudaSuccess && c->prox && c->b.x[0] && c->b.x[1])
                e = cudaMemcpyAsync(c->b.x[slot0], c->b.x[c->slot], (size_t)c->B * c->T * c->N * sizeof(float),
                                    cudaMemcpyDeviceToDevice, c->s);
        }
        if (e == cudaSuccess && c->rcur != rcur0)
            e = cudaMemcpyAsync(rcur0 ? c->b.r_alt : c->b.r, rbuf(c), plane, cudaMemcpyDeviceToDevice, c->s);
        if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "graph slot restore: %s", cudaGetErrorString(e));
        c->slot = slot0;
        c->rcur = rcur0;
    }
    return out ? uot_get_report(c, out) : UOT_OK;
}

int uot_solve(uot_ctx* c, int32_t max_iters, double tol, int32_t check_every, uot_report* out) {
    NvtxRange nvtx_("uot_solve");
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    if (max_iters < 0 || check_every < 1) return fail(c, UOT_E_INVALID, "max_iters >= 0 and check_every >= 1 required");
    int prc = resolve_pending(c);
    if (prc) return prc;
    // always arm the device-side stop (tol <= 0 never triggers it, but non-finite values do)
    k_init_glob<<<1, 32, 0, c->s>>>(c->glob, c->stop, c->counter, 0);
    int rc = check_launch(c, "k_init_glob");
    if (rc) return rc;
    c->stop_armed = true;
    c->log.clear();
    c->persist_base.clear();
    c->log.push_back({c->iter, c->slot, c->rcur});
    rc = launch_iters(c, max_iters, check_every, max_iters > 0, c->stop, tol);
    if (rc) return rc;
    uot_report rep;
    rc = uot_get_report(c, &rep);
    if (out) *out = rep;
    if (rc) return rc;
    if (tol > 0.0 && !rep.converged) return fail(c, UOT_E_NOT_CONVERGED, "not converged after %d iterations", max_iters);
    return UOT_OK;
}

int uot_objective(uot_ctx* c, double* per_pair, uot_report* out) {
    NvtxRange nvtx_("uot_objective");
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    int prc = resolve_pending(c);
    if (prc) return prc;
    const int slot = c->slot;
    ObjArgs O{};
    O.nx = c->nx; O.ny = c->ny; O.T = c->T; O.P = c->P; O.N = c->N; O.bpp = c->bpp;
    O.x = c->prox ? c->b.x[slot] : c->b.frames;
    O.p = c->prox ? c->b.frames : nullptr;
    O.next_owns_last = c->b.a_next_halo != nullptr;
    O.mx = c->b.mx[slot]; O.my = c->b.my[slot]; O.r = rbuf(c); O.a = c->b.a[slot];
    O.partials = c->part;
    O.p2 = c->r_mode == 1;
    k_objective<<<dim3(c->bpp, c->G), 256, 0, c->s>>>(O);
    int rc = check_launch(c, "k_objective");
    if (rc) return rc;
    ReduceArgs R{};
    R.partials = c->part; R.recs_per_pair = c->bpp; R.G = c->G; R.pair_out = c->pair_obj;
    R.glob = c->glob; R.counter = c->counter; R.stop = nullptr; R.max_mask = (1u << 4) | (1u << 5);
    R.is_iteration = 0; R.is_setup = 0; R.tau1 = c->tau1;
    k_pair_reduce<<<c->G, 256, 0, c->s>>>(R);
    rc = check_launch(c, "k_pair_reduce(objective)");
    if (rc) return rc;
    double* rows = (double*)malloc(sizeof(double) * c->G * kRec);
    double h[GL_N];
    cudaError_t e = cudaMemcpyAsync(rows, c->pair_obj, sizeof(double) * c->G * kRec, cudaMemcpyDeviceToHost, c->s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, c->glob, GL_N * sizeof(double), cudaMemcpyDeviceToHost, c->s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->s);
    if (e != cudaSuccess) { free(rows); return fail(c, UOT_E_CUDA, "objective readback: %s", cudaGetErrorString(e)); }
    const double a = c->p.alpha;
    double tr = 0, gr = 0, ub = 0, lb = 0, px = 0;
    bool nonfinite = false;
    for (int g = 0; g < c->G; ++g) {
        const double* q = rows + (size_t)g * kRec;
        // weak duality; c scales a into the dual-feasible set
        const bool bal = c->r_mode == 2, p2 = c->r_mode == 1;
        double cc = 1.0;
        if (q[4] > cc) cc = q[4];
        if (!bal && !p2 && q[5] / a > cc) cc = q[5] / a;
        const double U = bal ? (q[2] == 0.0 ? q[0] : INFINITY) : q[0] + a * q[2];
        const double L = p2 ? -q[3] / cc - q[7] / (4.0 * a * cc * cc) : -q[3] / cc;
        const double obj = bal ? q[0] : q[0] + a * q[1];
        if (per_pair) {
            double* P = per_pair + (size_t)g * 8;
            P[0] = q[0]; P[1] = q[1]; P[2] = U; P[3] = q[3]; P[4] = q[4]; P[5] = q[5]; P[6] = L;
            P[7] = obj;
        }
        tr += q[0]; gr += bal ? 0.0 : q[1]; ub += U; lb += L; px += q[6];
        for (int k = 0; k < 8; ++k) if (k != 2) nonfinite |= !isfinite(q[k]);
    }
    free(rows);
    if (out) {
        memset(out, 0, sizeof(*out));
        out->transport = tr;
        out->growth = a * gr;
        out->prox_term = c->prox ? 0.5 * c->p.rho * px : 0.0;
        out->objective = tr + a * gr + out->prox_term;
        out->primal_res = NAN;
        out->dual_res = NAN;
        out->upper_bound = ub;
        out->lower_bound = lb;
        out->f_norm = sqrt(h[GL_FSQ]);
        out->iterations = c->iter;
        out->nonfinite = nonfinite;
    }
    if (nonfinite) return fail(c, UOT_E_NONFINITE, "non-finite state");
    return UOT_OK;
}

int uot_set_timing(uot_ctx* c, int enable) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    c->timing = enable != 0;
    return UOT_OK;
}

int uot_get_timing(uot_ctx* c, double* ms_total, int64_t* n) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    cudaError_t e = cudaStreamSynchronize(c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "sync: %s", cudaGetErrorString(e));
    double tot = 0.0;
    for (size_t q = 0; q + 1 < c->ev_used; q += 2) {
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, c->ev[q], c->ev[q + 1]);
        if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventElapsedTime: %s", cudaGetErrorString(e));
        tot += ms;
    }
    if (ms_total) *ms_total = tot;
    if (n) *n = (int64_t)(c->ev_used / 2);
    c->ev_used = 0;
    c->ev_kind.clear();
    return UOT_OK;
}

int uot_get_timing_paths(uot_ctx* c, double* ms, int64_t* n) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    if (!ms || !n) return fail(c, UOT_E_INVALID, "ms and n must be non-NULL");
    cudaError_t e = cudaStreamSynchronize(c->s);
    if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "sync: %s", cudaGetErrorString(e));
    for (int k = 0; k < UOT_N_PATHS; ++k) { ms[k] = 0.0; n[k] = 0; }
    for (size_t q = 0; q + 1 < c->ev_used; q += 2) {
        float t = 0.f;
        e = cudaEventElapsedTime(&t, c->ev[q], c->ev[q + 1]);
        if (e != cudaSuccess) return fail(c, UOT_E_CUDA, "cudaEventElapsedTime: %s", cudaGetErrorString(e));
        const int k = q / 2 < c->ev_kind.size() ? c->ev_kind[q / 2] : 0;
        ms[k] += t;
        n[k] += 1;
    }
    c->ev_used = 0;
    c->ev_kind.clear();
    return UOT_OK;
}

int uot_wave_cols(const uot_ctx* c) {
    if (!c) return -1;
    const TVar& v = c->tv[3];                 // the five-iteration pass (all wave variants share the layout rule)
    return (c->t2ok && v.ok && v.wave) ? 32 * v.vn : 0;
}

int uot_state_slot(const uot_ctx* c) { return c ? c->slot : -1; }
int uot_r_slot(const uot_ctx* c) { return c ? c->rcur : -1; }

int uot_kernel_path(const uot_ctx* c) {
    if (!c) return -1;
    if (use_single(c)) return 10;
    if (c->tp.ok && c->t2ok && c->t2on) return 8;
    if (use_persist(c)) return 2;
    if (c->pw.ok) return 11;
    if (!(c->t2ok && c->t2on)) return 0;
    const bool four = c->t4on && c->tv[1].ok;
    const TVar& v = c->tv[four ? 1 : 0];
    if (v.wave && four && c->tv[3].ok) return 9;        // the pass kind of long runs: five per pass
    return v.wave ? (four ? 6 : 5) : (four ? 3 : 1);
}

int uot_set_own_pairs(uot_ctx* c, int32_t lo, int32_t hi) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    if (!c->pw.ok) return fail(c, UOT_E_INVALID, "ghost pairs need the chain-prox wave path (uot_kernel_path 11)");
    if (!(0 <= lo && lo < hi && hi <= c->P)) return fail(c, UOT_E_INVALID, "own pairs [%d, %d) outside [0, %d)", lo, hi, c->P);
    int prc = resolve_pending(c);
    if (prc) return prc;
    const int olo = c->pw.own_lo, ohi = c->pw.own_hi;
    c->pw.own_lo = lo;
    c->pw.own_hi = hi;
    if (!pw_regroup(c)) {
        c->pw.own_lo = olo; c->pw.own_hi = ohi;
        pw_regroup(c);
        return fail(c, UOT_E_CUDA, "k_wave_prox regroup failed");
    }
    return UOT_OK;
}

int uot_set_temporal(uot_ctx* c, int enable) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    if (enable && !c->t2ok) return fail(c, UOT_E_INVALID, "k_iter2 unavailable (prox mode, no r_alt, or UOT_TEMPORAL=0)");
    c->t2on = enable != 0;
    return UOT_OK;
}

int uot_stop_external(uot_ctx* c) {
    if (!c) return fail(nullptr, UOT_E_INVALID, "ctx is NULL");
    int rc = resolve_pending(c);
    if (rc) return rc;
    k_init_glob<<<1, 32, 0, c->s>>>(c->glob, c->stop, c->counter, 0);
    rc = check_launch(c, "k_init_glob");
    if (rc) return rc;
    c->stop_armed = true;
    c->ext_stop = true;
    c->log.clear();
    c->persist_base.clear();
    c->log.push_back({c->iter, c->slot, c->rcur});
    return UOT_OK;
}

int uot_stop_pack(uot_ctx* c, double* sums8) {
    if (!c || !sums8) return fail(c, UOT_E_INVALID, "null argument");
    k_stop_pack<<<1, 32, 0, c->s>>>(c->glob, sums8);
    return check_launch(c, "k_stop_pack");
}

int uot_stop_apply(uot_ctx* c, const double* sums8, double tol) {
    if (!c || !sums8) return fail(c, UOT_E_INVALID, "null argument");
    if (!c->ext_stop) return fail(c, UOT_E_INVALID, "uot_stop_external was not called");
    k_stop_apply<<<1, 32, 0, c->s>>>(sums8, c->glob, c->stop, tol, c->tau1);
    return check_launch(c, "k_stop_apply");
}

int64_t uot_launch_count(const uot_ctx* c) { return c ? c->launches : -1; }

void uot_destroy(uot_ctx* c) {
    if (!c) return;
    c->poll.release();
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    delete c;
}

const char* uot_last_error(const uot_ctx* c) { return c ? c->err : g_err; }

}  // extern "C"

// UOT-DF ADMM (Algorithm 2) on top of the kernels above
#include "uot_df.inc"
#include "uot_rpca.inc"
