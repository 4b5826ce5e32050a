/*
 * uot.h -- C-ABI of the B200 (sm_100a) hot path of arXiv 1909.00149:
 * the per-iteration Chambolle-Pock update of Algorithm 1
 * that evaluates / proxes the unbalanced Beckmann OT regulariser
 * eq:Unbal_OT_beckman on pixel grids.
 *
 * Library: paper_1909_00149_b200/libuot_b200.so (extern "C", no C++ types,
 * no exceptions across the ABI).  All compute runs in the library's CUDA
 * kernels; there is no CPU fallback: without a CUDA device every compute
 * entry point returns UOT_E_CUDA.
 *
 * Readings of the paper (sign of the constraint, rho convention, boundary,
 * stopping rule, ...) are DESIGN.md L1..L30 and are cited as "Lnn".
 *
 * ---------------------------------------------------------------------------
 * Problem.  A context holds B independent chains of T frames x_t (fp32,
 * [B][T][ny][nx], C-contiguous, i = contiguous axis = paper index i, P:152,
 * L5).  Each adjacent pair (t, t+1) carries one UOT term (eq:RPCA_UOTDF
 * P:746-756, "T-1 OT problems"), pair g = b*(T-1) + t, with the
 * constraint (L1)
 *        div(M_g) - r_g = x_{t+1} - x_t          (north star: psi = -r)
 * and the objective ||M_g||_{2,1} + alpha ||r_g||_1 (p = 1).
 * Per pair the state is the flux M = (Mx, My) (Mx[:, nx-1] and
 * My[ny-1, :] are pinned to 0, L3), the transport residual r and the
 * dual a.  In prox mode (rho finite) the frames become variables x
 * with centres p = frames (eq:Prox_UOT P:218-226, Alg.1 line 4 P:314, L2, L19).
 *
 * One iteration (Alg.1 lines 3-7), every right-hand side at
 * iteration k (Jacobi, L10):
 *   m_i <- shrink^{l2}_{tau1}(m_i - tau1 div^*(a)_i)
 *   x   <- Pi_+((rho tau1 p + x - tau1 A^T a)/(1 + rho tau1))  (prox only)
 *   r   <- shrink^{l1}_{alpha tau1}(r + tau1 a)
 *   a   <- a + tau2 (2 K(M',r',x') - K(M,r,x)),  K = div M - r - x_{t+1} + x_t
 *
 * ---------------------------------------------------------------------------
 */
#ifndef UOT_B200_H
#define UOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  0/2/3 mirror the exit codes of SPEC.md S:477. */
#define UOT_OK              0
#define UOT_E_INVALID       2  /* bad argument; nothing was enqueued            */
#define UOT_E_NOT_CONVERGED 3  /* uot_solve hit max_iters with tol > 0; state and report valid */
#define UOT_E_NONFINITE     4  /* NaN/Inf seen in the reductions         */
#define UOT_E_CUDA          5  /* CUDA error (incl. no device); see uot_last_error */

/* uot_params.flags */
#define UOT_FORCE_STEPS     1u /* accept tau1*tau2 >= 1/||K||^2 (Theorem 1 not satisfied) */
#define UOT_FIX_FIRST_FRAME 2u /* prox mode: frame 0 of each chain is a constant argument s
                                  (eq:Prox_UOT_specialcase); x_0 stays = frames[b][0] */
#define UOT_RESIDUAL_L2     4u /* p = 2: growth penalty alpha ||r||_2^2, r-update
                                  r <- (r + tau1 a)/(1 + 2 alpha tau1) ("averaging update") */
/* uot_reset flags */
#define UOT_RESET_X_FROM_P  1u /* prox mode: x^0 = max(p, 0) instead of 0 (L8)   */

typedef struct uot_ctx uot_ctx;   /* opaque, host-side */

typedef struct {
    int32_t  nx, ny;       /* grid, >= 1 each; nx = contiguous axis            */
    int32_t  n_chains;     /* B >= 1 independent chains (batched pairs: T = 2)                 */
    int32_t  n_frames;     /* T >= 2 frames per chain held by this context (a shard's frames
                              include the shared boundary frame)        */
    double   alpha;        /* paper mu > 0; p = 1 (or 2 with UOT_RESIDUAL_L2);
                              +INFINITY = balanced Beckmann eq:OT_beckman (r dropped, footnote P:609) */
    double   rho;          /* weight of (rho/2)||x - p||^2 as printed in Alg.1 line 4 (L2);
                              +INFINITY = fixed marginals (x == frames, evaluation of eq:Unbal_OT_beckman) */
    double   tau1, tau2;   /* primal / dual steps > 0; 0 = Theorem-1 default (uot_default_steps,
                              safety 0.99)                                                      */
    uint32_t flags;        /* UOT_FORCE_STEPS | UOT_FIX_FIRST_FRAME | UOT_RESIDUAL_L2          */
} uot_params;

/* Device buffers.  ALL are CALLER-OWNED device pointers (e.g. torch tensors),
 * fp32 unless noted, C-contiguous; the library stores the pointers (they must
 * outlive the context) and allocates nothing on the device.  P = T-1.
 * 16-byte alignment and nx % 4 == 0 select the float4 kernels; otherwise a
 * scalar-lane variant runs (same results up to fp32 rounding order).       */
typedef struct {
    const float* frames;   /* [B][T][ny][nx] x_t (fixed) or prox centres p_t                   */
    float*  f;             /* [B][P][ny][nx] scratch: x_{t+1} - x_t (fixed mode)               */
    float*  mx[2];         /* [B][P][ny][nx] ping-pong flux x-component                         */
    float*  my[2];         /* [B][P][ny][nx] ping-pong flux y-component                         */
    float*  r;             /* [B][P][ny][nx] transport residual (updated in place)              */
    float*  a[2];          /* [B][P][ny][nx] ping-pong dual                                      */
    float*  x[2];          /* [B][T][ny][nx] ping-pong frames (prox mode), NULL when rho = inf  */
    const float* a_prev_halo; /* [B][ny][nx] dual of the pair preceding frame 0 (chain prox shard), or NULL = 0 */
    const float* a_next_halo; /* [B][ny][nx] dual of the pair following frame T-1, or NULL = 0; non-NULL
                                 also means frame T-1 is the next shard's first frame: it is updated
                                 here bit-identically but its terms are reduced by its owner       */
    double* scratch;       /* uot_scratch_doubles(&params) doubles (reduction partials, flags)  */
    float*  r_alt;         /* [B][P][ny][nx] second r buffer, or NULL.  Enables the temporally
                              blocked kernels (several iterations per HBM pass: k_wave / k_iter2
                              with fixed marginals, k_wave_prox in chain prox without halos),
                              which cannot update r in place.  Which of r / r_alt holds the
                              current r: uot_r_slot().                                         */
} uot_buffers;

/* Reductions (fp64) summed over this context's pairs, DESIGN.md "Reductions". */
typedef struct {
    double objective;      /* sum ||M||_{2,1} + alpha ||r||_1 (+ (rho/2)||x - p||^2 in prox mode) */
    double transport;      /* sum ||M||_{2,1}                                      */
    double growth;         /* sum alpha ||r||_p^p (0 when balanced)                              */
    double prox_term;      /* (rho/2) sum ||x - p||^2 (0 in fixed mode)                         */
    double primal_res;     /* ||K^{k+1}||_2, constraint violation (L13)                         */
    double dual_res;       /* ||z^{k+1} - z^k||_2 / tau1, z = (M, r[, x]) (L13)                 */
    double upper_bound;    /* sum ||M||_{2,1} + alpha ||div M - f||_p^p >= V (feasible repair;
                              balanced: ||M|| if div M = f exactly, else +inf)                 */
    double lower_bound;    /* weak-duality bound <= V (uot_objective only, else NaN)           */
    double f_norm;         /* ||x_{t+1} - x_t||_2 over all pairs (stopping scale)               */
    int64_t iterations;    /* executions of Alg.1 lines 3-7 since the last uot_reset (L9)      */
    int32_t converged;     /* uot_solve: 1 if the tol test passed                               */
    int32_t nonfinite;     /* 1 if a NaN/Inf was seen                                           */
} uot_report;

/* Number of doubles the caller must provide in buffers.scratch. */
size_t uot_scratch_doubles(const uot_params* params);

/* Theorem-1 steps (L11/L12): tau1 = tau2 = sqrt(safety / ||K||^2),
 * ||K||^2 = lambda_max(div div^*) + 1 (fixed), + 3 (pair prox, the paper's
 * bound), + 3 + 2cos(pi/T) (chain prox of T frames), + 2 (pair prox with
 * UOT_FIX_FIRST_FRAME: K = [D, -I, -I]); lambda_max =
 * g(nx) + g(ny), g(n) = 2 + 2cos(pi/n) (n >= 2), g(1) = 0.  0 < safety < 1.
 * Host-only, no device needed.  Returns UOT_OK or UOT_E_INVALID. */
int uot_default_steps(const uot_params* params, double safety, double* tau1, double* tau2);

/* Validate params/buffers, bind the stream (a cudaStream_t, NULL = legacy
 * default stream) and create a context.  Enqueues nothing; call uot_reset.
 * On error *out = NULL and a message is available from uot_last_error(NULL). */
int uot_create(const uot_params* params, const uot_buffers* buffers, void* cuda_stream, uot_ctx** out);

/* Cold start ("initialized to 0"): M = r = a = 0, x = 0 (or max(p,0)
 * with UOT_RESET_X_FROM_P), f = x_{t+1} - x_t; iteration count 0.  Async. */
int uot_reset(uot_ctx* ctx, uint32_t flags);

/* Copy frames from HOST memory (pinned for async) into buffers.frames's
 * device storage on the context stream and recompute f; the state is kept
 * (warm start across outer iterations).  host_frames holds
 * B*T*ny*nx floats in the same layout.  Async w.r.t. the host if pinned. */
int uot_load_frames(uot_ctx* ctx, const float* host_frames);

/* Asynchronous iterations: enqueue n_iters >= 0 iterations with the residual
 * reductions every check_every-th iteration (0 = none) and on the last one;
 * tol > 0 arms the device-side stopping test (L13) -- later launches exit
 * immediately once it passes.  No host synchronisation; read the result with
 * uot_get_report.  A stop armed this way stays pending until uot_get_report, or until
 * the next entry point that enqueues work on the iterate (uot_iterate, _part,
 * uot_prox_step, uot_solve, uot_objective, uot_load_frames), which first synchronises
 * the stream once and applies it; under graph capture such a call returns
 * UOT_E_INVALID instead.  uot_reset discards it. */
int uot_iterate(uot_ctx* ctx, int32_t n_iters, int32_t check_every, double tol);

/* One iteration restricted to a part of the pairs, for overlapping the shard
 * halo exchange: UOT_PART_INTERIOR runs the pairs that
 * do not read a_prev_halo / a_next_halo (first / last pair of each chain) and
 * does NOT complete the iteration; UOT_PART_BOUNDARY runs the others and
 * completes it (slot flip, reductions if reduce != 0).  UOT_PART_ALL = both.
 * Async. */
#define UOT_PART_ALL       0
#define UOT_PART_INTERIOR  1
#define UOT_PART_BOUNDARY  2
int uot_iterate_part(uot_ctx* ctx, int32_t part, int32_t reduce);

/* Synchronise the context stream and return the reductions of the last
 * reducing iteration (and the iteration count, corrected if the device
 * stopped early). */
int uot_get_report(uot_ctx* ctx, uot_report* out);

/* Run n_iters >= 0 iterations (Alg.1 lines 3-7).  out == NULL: fully async
 * (graph-capturable, no host sync; under capture the call ends in the buffer slots it
 * started from -- device copies are appended when the passes flipped them -- so every
 * replay continues from the previous one; replays do not advance the context's
 * iteration count); out != NULL: the last iteration also computes the reductions and
 * the call synchronises the stream to fill *out (UOT_E_INVALID under graph capture). */
int uot_prox_step(uot_ctx* ctx, int32_t n_iters, uot_report* out);

/* Iterate until primal_res <= tol*max(f_norm, 1e-30) and dual_res <= the same
 * (L13), checking every check_every iterations ON THE DEVICE (no host sync in
 * the loop: later launches exit immediately once converged), or until
 * max_iters.  tol <= 0: run exactly max_iters.  Fills *out (may be NULL).
 * Returns UOT_OK, UOT_E_NOT_CONVERGED (tol > 0 and not met), UOT_E_NONFINITE. */
int uot_solve(uot_ctx* ctx, int32_t max_iters, double tol, int32_t check_every, uot_report* out);

/* Objective and weak-duality certificate of the CURRENT state, per pair
 * (DESIGN.md "Certificate"):  per_pair[g*8 + .] = {transport, sum|r|^p, U,
 * <a,f>, max ||div^* a||, max |a|, L, objective}, L <= V_alpha <= U
 * (p = 2: L = -<a,f>/c - ||a||^2/(4 alpha c^2), c = max(1, max||div^*a||)).
 * per_pair may be NULL; out may be NULL.  Synchronises the stream. */
int uot_objective(uot_ctx* ctx, double* per_pair, uot_report* out);

/* Kernel timing for the roofline report (bench.py): enable != 0 brackets every
 * fused-iteration kernel launch with a CUDA event pair on the context stream.
 * uot_get_timing synchronises, returns the summed device time (ms) and the
 * number of timed launches since the last call, and clears the record. */
int uot_set_timing(uot_ctx* ctx, int enable);
int uot_get_timing(uot_ctx* ctx, double* ms_total, int64_t* n_launches);
/* As uot_get_timing, split by kernel: ms[k], n[k] for k = uot_kernel_path codes (0 k_iter,
 * 1 / 3 two- / four-iteration k_iter2 pass, 2 k_persist, 5 / 7 / 6 / 9 two- / three- / four- /
 * five-iteration k_wave pass, 8 k_tpersist, 10 k_single, 11 chain-prox k_wave_prox pass) and 4 =
 * the UOT-DF ADMM kernel; both arrays hold UOT_N_PATHS entries.  Clears the record. */
#define UOT_N_PATHS 12
int uot_get_timing_paths(uot_ctx* ctx, double* ms, int64_t* n);

/* Which ping-pong slot (0/1) of mx/my/a/x holds the current iterate. */
int uot_state_slot(const uot_ctx* ctx);
/* Which r buffer holds the current r: 0 = buffers.r, 1 = buffers.r_alt. */
int uot_r_slot(const uot_ctx* ctx);
/* Fixed marginals with buffers.r_alt: enable (1, the default) or disable (0) the two-iterations-
 * per-pass kernel k_iter2; disabled, every iteration is one pass of k_iter (for A/B timing).
 * Returns UOT_E_INVALID if k_iter2 is unavailable and enable != 0. */
int uot_set_temporal(uot_ctx* ctx, int enable);
/* Kernel that runs the iterations of this context: 0 = k_iter (one pass per iteration),
 * 1 = k_iter2 (SMEM tiles, two iterations per pass, fixed marginals), 2 = k_persist (all
 * iterations of a call in one cooperative launch, small grids), 3 = k_iter2 with
 * four-iteration passes, 5 / 6 / 9 = k_wave (register wavefront, 16-byte-aligned planes
 * with nx % 4 == 0) with two / four / five iterations per pass, 8 = k_tpersist (small grids: all
 * iterations of a call in one cooperative launch of SMEM-tile passes, when every run up to a
 * check has even length; otherwise the per-pass kernels), 10 = k_single (one small pair with
 * nx % 4 == 0 and nx/4 * ny <= 1024, fixed marginals: every iteration of a call in ONE CTA with the
 * state in registers, reductions and stopping test in-kernel; UOT_SINGLE=0 disables it), 11 =
 * k_wave_prox (chain prox, rho < inf, with buffers.r_alt, aligned planes, nx % 4 == 0 and no
 * shard halos, when its pair groups waste at most 1.34 pair slots per pair: three (two)
 * iterations per pass, pairs of a group in clusters of CTAs exchanging duals by st.async;
 * UOT_PROX_WAVE=0 disables it, =2 forces it).  Four-iteration contexts fill in
 * with two-iteration passes / k_iter where a reduction falls inside four iterations. */
int uot_kernel_path(const uot_ctx* ctx);

/* Strip width of the register-wavefront passes (kernel paths 5 / 6 / 7 / 9; the five-iteration
 * pass's layout): 128 = k_wave_pk / k_wave (one float4 column quad per lane), 64 = k_wave_n (one
 * fp32x2 column pair per lane, twice the resident warps; chosen per grid where the narrower
 * strips compute fewer halo pixels, e.g. 256-column rows -- DESIGN.md §6; UOT_WAVE_V = 2 / 4
 * forces either), 0 when the context has no wavefront passes, -1 for a NULL context.  Iterates
 * are equal either way (same arithmetic per pixel). */
int uot_wave_cols(const uot_ctx* ctx);

/* Ghost pairs of a chain-prox shard: only pairs [lo, hi) of each chain are written
 * and reduced by k_wave_prox passes; pairs outside are read-only copies of the neighbouring
 * shards' pairs (with their frames), which the caller refreshes after every pass -- S
 * iterations per exchange instead of one.  The context's first / last pair is treated as a
 * chain end (a = 0 beyond it), so a side whose ghost pairs do not reach the chain's end needs
 * >= S = 3 of them (the dependency cone of one pass; dist.ghost_range).  Requires
 * uot_kernel_path == 11; afterwards every run between checks must be >= 2 iterations (passes
 * of 3 and 2; UOT_E_INVALID for a single iteration, which would be a k_iter pass updating the
 * ghosts); the iteration reports sum the own pairs
 * only (uot_objective still covers every pair of the context: use its per-pair rows).
 * lo = 0, hi = P restores the whole chain. */
int uot_set_own_pairs(uot_ctx* ctx, int32_t lo, int32_t hi);

/* Cross-rank stopping test for a chain sharded over ranks: the
 * L13 test must use the residuals and ||f|| summed over ALL shards, so no rank may stop on
 * its own sums.  Stream-ordered, no host synchronisation:
 *   uot_stop_external(ctx)            arm the stop flag (launches exit once it is set) with
 *                                     the local test disabled, until uot_get_report;
 *   uot_iterate(ctx, d, d, 0.0)       a chunk of d iterations, reductions on its last;
 *   uot_stop_pack(ctx, sums8)         sums8 (8 device doubles, caller-owned) <- this rank's
 *                                     [transport, growth, ||K||^2, ||dz||^2, ub, prox, ||f||^2,
 *                                     nonfinite] of the last checked iteration;
 *   (caller: all-reduce sums8 over the ranks, e.g. ncclAllReduce sum, same stream order)
 *   uot_stop_apply(ctx, sums8, tol)   set the stop if the GLOBAL sums pass the L13 test
 *                                     (or any rank saw a non-finite value).
 * Every rank takes the same decision at the same iteration; uot_get_report rewinds to it.
 * UOT_E_INVALID: NULL pointers, uot_stop_apply without uot_stop_external, or
 * uot_iterate(tol > 0) while armed. */
int uot_stop_external(uot_ctx* ctx);
int uot_stop_pack(uot_ctx* ctx, double* sums8);
int uot_stop_apply(uot_ctx* ctx, const double* sums8, double tol);

/* CUDA kernels launched by this context since creation (for accounting). */
int64_t uot_launch_count(const uot_ctx* ctx);

void uot_destroy(uot_ctx* ctx);

/* Last error message of ctx (or of the last failed uot_create if ctx == NULL). */
const char* uot_last_error(const uot_ctx* ctx);

/* ===========================================================================
 * UOT-DF ADMM: Algorithm 2 for eq:UOT-DF
 * with Phi = I and R = 0 -- the denoising setting of the paper's
 * runtime experiment (Fig. 1) -- on B independent problems:
 *     min_{s >= 0} 1/2 ||y - s||^2 + kappa V_mu(s0, s)
 * Per ADMM iteration (readings L22, L23 in DESIGN.md):
 *   s <- Pi_+((x + a + z + b)/2)   (minimiser of the printed augmented
 *                                    Lagrangian P:479-484; L23)
 *   x <- (y + rho (s - a))/(1 + rho)                          (line 5, Phi = I)
 *   z <- inner_iters warm-started Alg.1 iterations of the fixed-first-argument
 *        prox (eq:Prox_UOT_specialcase) of V_{s0} with weight rho/kappa (L2)
 *        and centre s - b                                      (line 6)
 *   a <- a + x - s;  b <- b + z - s                            (lines 7-8)
 * inner_iters = 1 (the paper's setting) runs as ONE fused streaming
 * kernel per ADMM iteration; inner_iters > 1 composes a pointwise kernel, the
 * prox kernels above and a pointwise dual update.
 * Stopping: ||[x-s; z-s]||_2 < eps and rho ||[dx; dz]||_2 < eps,
 * tested on the device every check_every iterations.
 * ======================================================================== */
typedef struct uot_df_ctx uot_df_ctx;

typedef struct {
    int32_t  nx, ny, n_problems;   /* grid, B >= 1                                            */
    double   mu;                   /* UOT unbalance weight (alpha elsewhere), > 0 or +inf (balanced) */
    double   kappa;                /* dynamics weight kappa > 0                       */
    double   rho;                  /* ADMM penalty rho > 0                            */
    double   tau1, tau2;           /* inner Alg.1 steps; 0 = Theorem-1 default for K = [D,-I,-I] */
    int32_t  inner_iters;          /* Alg.1 iterations per ADMM iteration, >= 1 (1)     */
    uint32_t flags;                /* UOT_RESIDUAL_L2, UOT_FORCE_STEPS                        */
} uot_df_params;

typedef struct {                   /* caller-owned device buffers, fp32, [B][ny][nx] unless noted */
    const float* y;                /* measurements (Phi = I)                                   */
    const float* s0;               /* prior s~, the constant first argument            */
    float* s;                      /* estimate s^k (output; written on checked iterations)     */
    float* x; float* a; float* b;  /* ADMM split variable and scaled duals        */
    float* pf;                     /* [B][2][ny][nx] inner prox frames (s0, centre)            */
    float* xz[2];                  /* [B][2][ny][nx] inner frames (s0, z), ping-pong           */
    float* mx[2]; float* my[2];    /* inner flux, ping-pong                                    */
    float* r;                      /* inner transport residual                                 */
    float* ain[2];                 /* inner dual, ping-pong                                    */
    float* tmp[2];                 /* scratch planes (inner_iters > 1 only; may be NULL otherwise) */
    double* scratch;               /* uot_df_scratch_doubles(&params) doubles                  */
} uot_df_buffers;

typedef struct {
    double primal_res;             /* ||[x - s; z - s]||_2                                      */
    double dual_res;               /* rho ||[x - x_prev; z - z_prev]||_2                        */
    double data_term;              /* 1/2 ||y - s||^2                                           */
    double transport, growth;      /* inner ||M||_{2,1}, mu ||r||_p^p (fused path; NaN otherwise) */
    double objective;              /* data_term + kappa (transport + growth) (estimate)        */
    int64_t iterations;            /* ADMM iterations since uot_df_reset                       */
    int32_t converged, nonfinite;
} uot_df_report;

size_t uot_df_scratch_doubles(const uot_df_params* params);
int uot_df_create(const uot_df_params* params, const uot_df_buffers* buffers, void* cuda_stream, uot_df_ctx** out);
/* cold start (Alg.2 line 2: s = x = z = a = b = 0; inner state 0). Async. */
int uot_df_reset(uot_df_ctx* ctx);
/* up to max_iters ADMM iterations; eps <= 0 runs exactly max_iters. Fills *out (may be NULL).
 * Returns UOT_OK, UOT_E_NOT_CONVERGED (eps > 0 not met), UOT_E_NONFINITE, ... */
int uot_df_solve(uot_df_ctx* ctx, int32_t max_iters, double eps, int32_t check_every, uot_df_report* out);
int uot_df_set_timing(uot_df_ctx* ctx, int enable);
int uot_df_get_timing(uot_df_ctx* ctx, double* ms_total, int64_t* n_launches);
int64_t uot_df_launch_count(const uot_df_ctx* ctx);
void uot_df_destroy(uot_df_ctx* ctx);
const char* uot_df_last_error(const uot_df_ctx* ctx);

/* ===========================================================================
 * RPCA+UOT-DF ADMM: Algorithm 3 for
 * eq:RPCA_UOTDF on one video of T frames y_t (ny x nx):
 *   min_{S, L >= 0} 1/2 sum_t ||y_t - Phi_t(s_t + l_t)||^2 + lambda ||S||_1
 *                   + gamma ||L||_* + kappa sum_{t<T-1} V_mu(s_t, s_{t+1})
 * with Phi_t DIAGONAL (per-pixel weights phi_t >= 0, e.g. masks; NULL = I),
 * the O(TN) case of P:861-862.  Per ADMM iteration, in the paper's order:
 *   lines 5-9 + 12 : one pointwise kernel: s (one-sided shrink, L25), L, x
 *                    (rho restored, L26), A <- A + X - S - L (L27), and the
 *                    prox centres (s_t - b_t, s_{t+1} - c_{t+1}) of line 11
 *   line 10        : T <- svt_{gamma/rho}(L + D) by the Gram route: G = M^T M
 *                    (fp64, M = L + D is N x T), eigen-decomposition of the
 *                    T x T matrix G by a warm-started parallel Jacobi solver in
 *                    one CTA, W = V diag(max(1 - tau/sqrt(lambda), 0)) V^T,
 *                    T = M W; fused with line 13 (D <- D + L - T)
 *   line 11        : inner_iters warm-started iterations of Algorithm 1 on the
 *                    T-1 independent pair proxes (weight rho/kappa, L2)
 *   lines 14-15    : b_t <- b_t + z_t - s_t, c_{t+1} <- c_{t+1} + w_{t+1} - s_{t+1}
 * Residuals (L28): primal ||[X-S-L; L-T; z-s; w-s]||, dual rho||[dX; dT; dz; dw]||;
 * stop when both < eps, tested on the device every check_every iterations.
 * Line 10 for T > 128 (the T x T Jacobi solver no longer fits one CTA): the partial SVD of P:861
 * by subspace iteration -- Gram matrix in 128-frame blocks, one CholeskyQR2-orthonormalised step
 * of width k = min(T, 64) (UOT_RPCA_K, <= 128) per ADMM iteration, warm-started from the previous Ritz vectors, the
 * k x k Rayleigh quotient by the same Jacobi solver; exact when the k Ritz vectors span every
 * eigenvector of G with lambda > (gamma/rho)^2 (UOT_RPCA_SVT=1 forces it at any T, UOT_RPCA_K
 * sets k).  Limits: 2 <= T <= UOT_RPCA_MAX_T.
 * ======================================================================== */
#define UOT_RPCA_MAX_T 512
/* Signed split eq:RPCA_UOTDF_PN: S = S+ - S-, S+/- >= 0,
 * each with its own l1 term and its own chain of UOT terms (reading L30: the split of
 * Algorithm 3 extended with z+/-, w+/-, b+/-, c+/-; s+ and s- updated jointly, exactly, per
 * pixel).  buffers.S holds S+, buffers.Sm S-; every per-pair buffer then has 2(T-1) pairs:
 * the S+ chain's T-1 pairs first, then the S- chain's. */
#define UOT_RPCA_SIGNED 8u
typedef struct uot_rpca_ctx uot_rpca_ctx;

typedef struct {
    int32_t  nx, ny, n_frames;     /* grid and T                                                */
    double   lambda, gamma;        /* sparsity and low-rank weights, > 0             */
    double   kappa, mu;            /* OT weight kappa > 0 and unbalance weight mu > 0 (or +inf)  */
    double   rho;                  /* ADMM penalty > 0                                           */
    double   tau1, tau2;           /* inner Alg.1 steps; 0 = Theorem-1 default (pair prox)       */
    int32_t  inner_iters;          /* Alg.1 iterations per ADMM iteration, >= 1      */
    uint32_t flags;                /* UOT_RESIDUAL_L2, UOT_FORCE_STEPS, UOT_RPCA_SIGNED          */
    /* Frame-range shard of a video of n_frames_total frames (line 11's
     * T-1 pair proxes, "simultaneously solved", split by frame range).  The
     * context holds frames [frame0, frame0 + n_frames) of the video and their n_frames - 1
     * pairs; with UOT_RPCA_HAS_NEXT its last frame is the next shard's first (a halo frame:
     * updated here bit-identically, reduced by its owner).  0 / 0 = the whole video.        */
    int32_t  frame0, n_frames_total;
    uint32_t shard_flags;          /* UOT_RPCA_HAS_PREV | UOT_RPCA_HAS_NEXT                      */
} uot_rpca_params;
#define UOT_RPCA_HAS_PREV 1u
#define UOT_RPCA_HAS_NEXT 2u

typedef struct {                   /* caller-owned device buffers, fp32, 16-B aligned           */
    const float* y;                /* [T][ny][nx] observations                                   */
    const float* phi;              /* [T][ny][nx] diagonal of Phi_t, or NULL (Phi = I)            */
    float *S, *L, *X, *Tm, *A, *D; /* [T][ny][nx] ADMM state (Tm = the paper's T; S = S+ if signed) */
    float* Sm;                     /* [T][ny][nx] S- (UOT_RPCA_SIGNED only, else NULL)           */
    /* per-pair buffers: Q = T-1 pairs, or 2(T-1) with UOT_RPCA_SIGNED                           */
    float* pc;                     /* [Q][2][ny][nx] prox centres (inner frames)                 */
    float* zw[2];                  /* [Q][2][ny][nx] (z_t, w_{t+1}) = inner x, ping-pong         */
    float* bc;                     /* [Q][2][ny][nx] (b_t, c_{t+1})                              */
    float* zprev;                  /* [Q][2][ny][nx] scratch (inner_iters > 1 only, else NULL)   */
    float* mx[2]; float* my[2];    /* [Q][ny][nx] inner flux, ping-pong                          */
    float* r;                      /* [Q][ny][nx] inner residual                                 */
    float* ain[2];                 /* [Q][ny][nx] inner dual, ping-pong                          */
    double* scratch;               /* uot_rpca_scratch_doubles(&params) doubles                  */
    /* sharded contexts only (else NULL):                                                        */
    float* mgather;                /* [n_frames_total][ny][nx]: M = L + D of EVERY frame (line 10); uot_rpca_iterate_pre
                                    * writes this shard's owned frames and zeros the others, the caller sums the
                                    * buffers of all shards (all-reduce: exactly one nonzero term per element)  */
    float* halo_prev;              /* [chains][2][ny][nx] (w, c) of the pair left of frame0 (HAS_PREV), received */
    float* halo_next;              /* [chains][2][ny][nx] (z, b) of the pair right of the last frame (HAS_NEXT)   */
} uot_rpca_buffers;

typedef struct {
    double primal_res, dual_res;   /* L28                                                        */
    double data_term;              /* 1/2 sum ||y - Phi(s + l)||^2                               */
    double l1_term;                /* lambda ||S||_1 (signed: lambda (||S+||_1 + ||S-||_1))       */
    double nuclear;                /* ||T||_* after line 10 (from the eigenvalues)               */
    double transport, growth;      /* inner ||M||_{2,1}, mu ||r||_p^p summed over pairs          */
    double objective;              /* data + l1 + gamma nuclear + kappa (transport + growth)     */
    int64_t iterations;            /* ADMM iterations since uot_rpca_reset                      */
    int32_t converged, nonfinite;
    int32_t jacobi_sweeps;         /* sweeps of the last eigen-decomposition                     */
    double svt_min_ritz;           /* T > 128 (partial SVD): smallest Ritz value of the k-wide subspace; the
                                    * SVT is exact only while it is < (gamma/rho)^2 (else raise UOT_RPCA_K);
                                    * -1 on the exact T <= 128 path                                */
} uot_rpca_report;

size_t uot_rpca_scratch_doubles(const uot_rpca_params* params);
/* Validates params/buffers (UOT_E_INVALID) and builds the inner Alg.1 context. */
int uot_rpca_create(const uot_rpca_params* params, const uot_rpca_buffers* buffers, void* cuda_stream,
                    uot_rpca_ctx** out);
/* Cold start (Alg.3 line 2: every variable 0; inner states 0; no eigenvector warm start). Async. */
int uot_rpca_reset(uot_rpca_ctx* ctx);
/* Up to max_iters ADMM iterations; eps <= 0 runs exactly max_iters.  Fills *out (may be NULL;
 * then the call is fully asynchronous).  Returns UOT_OK, UOT_E_NOT_CONVERGED, UOT_E_NONFINITE, ... */
int uot_rpca_solve(uot_rpca_ctx* ctx, int32_t max_iters, double eps, int32_t check_every, uot_rpca_report* out);
/* Per-launch CUDA-event timing of the line-1..15 kernels (summed ms, launches), as uot_set_timing. */
int uot_rpca_set_timing(uot_rpca_ctx* ctx, int enable);
int uot_rpca_get_timing(uot_rpca_ctx* ctx, double* ms_by_kernel /*[6]: pre, gram, eig, apply, prox, post*/,
                        int64_t* n_iters);
/* Sharded ADMM iteration, split where the shards exchange (DESIGN.md 6a "Sharded"); the caller
 * owns the collectives (NCCL over NVLink, same stream order):
 *   uot_rpca_stop_external(ctx)          arm the device stop, local test disabled
 *   loop: uot_rpca_iterate_pre(ctx, red) lines 5-9, 12, line-11 centres; mgather <- own M
 *         (caller) all-reduce(sum) mgather over the shards
 *         uot_rpca_iterate_post(ctx, red) lines 10 (Gram of all frames, eigen, T for this
 *                                       shard's frames), 11, 13-15; residual partial sums
 *         (caller) send (z, b) of the first pair to the previous shard's halo_next and
 *                  (w, c) of the last pair to the next shard's halo_prev
 *         if red: uot_rpca_stop_pack(ctx, sums8) -> (caller) all-reduce(sum) ->
 *                 uot_rpca_stop_apply(ctx, sums8, eps)
 *   uot_rpca_get_report(ctx, out)        sync; this shard's sums (nuclear norm is global);
 *                                        iteration count rewound to a device stop
 * sums8 = [primal^2, dual^2/rho^2, data, l1, transport, growth, nonfinite, 0] (device doubles).
 * An unsharded context may use the same calls (mgather then unused). */
int uot_rpca_iterate_pre(uot_rpca_ctx* ctx, int32_t reduce);
int uot_rpca_iterate_post(uot_rpca_ctx* ctx, int32_t reduce);
int uot_rpca_stop_external(uot_rpca_ctx* ctx);
int uot_rpca_stop_pack(uot_rpca_ctx* ctx, double* sums8);
int uot_rpca_stop_apply(uot_rpca_ctx* ctx, const double* sums8, double eps);
int uot_rpca_get_report(uot_rpca_ctx* ctx, uot_rpca_report* out);
int uot_rpca_state_slot(const uot_rpca_ctx* ctx);   /* ping-pong slot of zw/mx/my/ain holding the iterate */
int64_t uot_rpca_launch_count(const uot_rpca_ctx* ctx);
void uot_rpca_destroy(uot_rpca_ctx* ctx);
const char* uot_rpca_last_error(const uot_rpca_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* UOT_B200_H */
