/*
 * uot_oracle.c -- plain, slow, float64 CPU oracle for the hot path of
 * arXiv 1909.00149 (Lee, Bertrand, Rozell), Algorithm 1.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path under
 * paper_1909_00149_b200/csrc; neither side includes or links the other.
 *
 * Every function follows the paper step by step with materialised arrays
 * (no fusion, no halo tricks, no reordering).  Citations are PAPER.md line
 * numbers ("P:nnn") plus the equation / algorithm label they fall in; the
 * readings of the paper taken where it is silent or inconsistent are listed
 * in DESIGN.md section "Readings" (L1..L21) and cited here as "Lnn".
 *
 * Conventions (L1, L3, L5):
 *   - a plane is [ny][nx] C-contiguous, index k = j*nx + i, i (paper i,
 *     P:152) is the contiguous axis;
 *   - flux components Mx[j][nx-1] and My[ny-1][i] do not exist (closed grid,
 *     L3): they are read as 0 and written as 0;
 *   - constraint of eq:Unbal_OT_beckman with p = x_t,
 *     q = x_{t+1}:  div(M) - r = x_{t+1} - x_t  (L1), so the constraint
 *     value is K(M, r, x) = div(M) - r - x_{t+1} + x_t  (P:276 with A = [I,-I]);
 *   - p = 1; rho = +inf means fixed marginals x == frames (L2).
 *
 * Parity of this file is pinned by tests/test_oracle_pins.py (P1..P20, DF1..DF4
 * of DESIGN.md) -- closed forms, invariants, brute-force LPs, duality bounds --
 * and its stopping-rule / report reductions by tests/test_oracle_residual_pins.py
 * (P21..P23: recomputed from consecutive states).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

typedef struct {
    int32_t nx, ny;       /* grid */
    int32_t n_chains;     /* B independent sequences */
    int32_t n_frames;     /* T >= 2 frames per chain; pairs P = T-1 */
    double alpha;         /* paper mu > 0; +INFINITY = balanced Beckmann (eq:OT_beckman,
                             r dropped: footnote P:609) */
    double rho;           /* weight of (rho/2)||x-p||^2 as printed in Alg.1 line 4; INFINITY = fixed */
    double tau1, tau2;    /* primal / dual steps */
    int32_t p_norm;       /* 1 or 2 (mu ||r||_2^2, the "averaging update" of P:297, L14) */
    int32_t fix_first;    /* prox mode: frame 0 of each chain held at p_0 (eq:Prox_UOT_specialcase,
                             P:337-349: "A := I, K := div(M) - s + x - r") */
} uot_ref_params;

#define REP_STRIDE 8

/* ---- flux accessors implementing the zero-flux boundary of P:158 (L3) ---- */
static double MXv(const double* mx, int nx, int ny, int i, int j) {
    (void)ny;
    if (i < 0 || j < 0 || i >= nx - 1) return 0.0;   /* Mx[j][nx-1] pinned */
    return mx[(size_t)j * nx + i];
}
static double MYv(const double* my, int nx, int ny, int i, int j) {
    if (i < 0 || j < 0 || j >= ny - 1) return 0.0;   /* My[ny-1][i] pinned */
    return my[(size_t)j * nx + i];
}

/* div(M)[i,j] = (Mx[i,j]-Mx[i-1,j]) + (My[i,j]-My[i,j-1]), zero flux outside
 * the support.  P:153-158. */
void uot_ref_div(int nx, int ny, const double* mx, const double* my, double* out) {
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            out[(size_t)j * nx + i] =
                (MXv(mx, nx, ny, i, j) - MXv(mx, nx, ny, i - 1, j)) +
                (MYv(my, nx, ny, i, j) - MYv(my, nx, ny, i, j - 1));
}

/* div^*(a): the adjoint of div (formula not printed -> L4):
 * (div^* a)_x[i,j] = a[i,j] - a[i+1,j] for i < nx-1, 0 on the pinned column;
 * (div^* a)_y[i,j] = a[i,j] - a[i,j+1] for j < ny-1, 0 on the pinned row.
 * Pinned by the adjoint identity (test P1), not by this comment. */
void uot_ref_div_adj(int nx, int ny, const double* a, double* gx, double* gy) {
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t k = (size_t)j * nx + i;
            gx[k] = (i < nx - 1) ? a[k] - a[k + 1] : 0.0;
            gy[k] = (j < ny - 1) ? a[k] - a[k + (size_t)nx] : 0.0;
        }
}

/* shrink^{l2}_sigma(q) = max(||q||_2 - sigma, 0) * q / ||q||_2, applied per
 * row m_i in R^2 (eq:Prox_UOT_M_prox); 0/0 := 0 (L7). */
void uot_ref_shrink_l2(int64_t n, const double* qx, const double* qy, double sigma,
                       double* ox, double* oy) {
    for (int64_t k = 0; k < n; ++k) {
        double nrm = sqrt(qx[k] * qx[k] + qy[k] * qy[k]);
        double s = (nrm > sigma) ? (nrm - sigma) / nrm : 0.0;
        ox[k] = s * qx[k];
        oy[k] = s * qy[k];
    }
}

/* shrink^{l1}_sigma(q) = sign(q) * max(|q| - sigma, 0); sign(0)=0 (L7). */
void uot_ref_shrink_l1(int64_t n, const double* q, double sigma, double* out) {
    for (int64_t k = 0; k < n; ++k) {
        double m = fabs(q[k]) - sigma;
        double sg = (q[k] > 0) ? 1.0 : ((q[k] < 0) ? -1.0 : 0.0);
        out[k] = (m > 0) ? sg * m : 0.0;
    }
}

/* lambda_max of the discrete Laplacian div o div^* on an nx x ny grid with the
 * zero-flux boundary (Theorem 1).  Closed form: the 1-D path
 * Laplacian on n nodes has spectrum 2-2cos(pi k/n), k=0..n-1, so
 * lambda_max = g(nx) + g(ny), g(n) = 2+2cos(pi/n) for n >= 2, g(1) = 0.
 * Pinned against power iteration on uot_ref_div/uot_ref_div_adj (test P5). */
double uot_ref_lambda_max(int nx, int ny) {
    const double pi = 3.14159265358979323846;
    double gx = nx >= 2 ? 2.0 + 2.0 * cos(pi / nx) : 0.0;
    double gy = ny >= 2 ? 2.0 + 2.0 * cos(pi / ny) : 0.0;
    return gx + gy;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1 on B chains of T frames, one UOT term per adjacent
 * pair (t, t+1) (eq:RPCA_UOTDF P:746-756: "T-1 OT problems").
 *
 * rho = +inf (fixed marginals, L2): x == frames, only M, r, a iterate; this is
 *   Alg.1 with line 4 removed -- the evaluation of eq:Unbal_OT_beckman.
 * rho finite (prox mode, L19): x iterates; frame s enters K_s with +1 and
 *   K_{s-1} with -1, so (A^T a)_s = a_s - a_{s-1} (a_{-1} = a_{T-1} := 0);
 *   for T = 2 this is exactly Alg.1 line 4 with A = [I, -I] (L1).
 *
 * The state is updated in place; K^k is recomputed from the incoming state
 * (L8/L9: K^0 from the initial state).  All right-hand sides of lines 3-5 read
 * iteration-k values (Jacobi, L10).
 *
 * rep[g*8 + .] (pair g = b*P + t) receives the reductions of the LAST executed
 * iteration:
 *   0: sum_k ||m_k^{k+1}||_2                (transport, ||M||_{2,1} P:146-151)
 *   1: sum_k |r_k^{k+1}|^p                  (growth, ||r||_p^p; objective adds alpha*)
 *   2: sum_k (K^{k+1}_k)^2                  (primal residual^2, L13)
 *   3: sum ||z^{k+1}-z^k||^2, z=(M,r[,x])   (dual residual^2 * tau1^2, L13)
 *   4: sum_k |div(M^{k+1}) - (x_{t+1}-x_t)|^p (repaired upper-bound growth term)
 *   5: sum_k (x^{k+1}-p)^2                  (prox term / (rho/2); 0 in fixed mode)
 *   6: sum_k f_k^2, f = x_{t+1}-x_t at k+1  (for relative stopping)
 *   7: number of pixels N
 * In prox mode the per-frame terms (3: x part, 5) of frame s are attributed
 * to pair min(s, P-1) of its chain.
 * Returns 0, or 4 if a non-finite value was produced.
 */
int uot_ref_iterate(const uot_ref_params* prm, const double* frames,
                    double* mx, double* my, double* r, double* a, double* x,
                    int n_iters, double* rep) {
    const int nx = prm->nx, ny = prm->ny, B = prm->n_chains, T = prm->n_frames;
    const int P = T - 1;
    const size_t N = (size_t)nx * ny;
    const int G = B * P;
    const int prox = isfinite(prm->rho);
    const double tau1 = prm->tau1, tau2 = prm->tau2, alpha = prm->alpha, rho = prm->rho;
    if (nx < 1 || ny < 1 || B < 1 || T < 2) return 2;

    double* gx = malloc(sizeof(double) * N * G);
    double* gy = malloc(sizeof(double) * N * G);
    double* mxn = malloc(sizeof(double) * N * G);
    double* myn = malloc(sizeof(double) * N * G);
    double* rn = malloc(sizeof(double) * N * G);
    double* an = malloc(sizeof(double) * N * G);
    double* Kold = malloc(sizeof(double) * N * G);
    double* Knew = malloc(sizeof(double) * N * G);
    double* dv = malloc(sizeof(double) * N * G);
    double* xn = prox ? malloc(sizeof(double) * N * B * T) : NULL;
    int status = 0;

    /* frame-valued variable of frame s of chain b: x in prox mode, the given
     * frame in fixed mode (x == p, L2) */
#define XV(arr, b, s) ((arr) + ((size_t)(b) * T + (s)) * N)
    const double* xcur_base = prox ? x : frames;

    /* K^k from the incoming state: div(M) - r - x_{t+1} + x_t */
    #pragma omp parallel for schedule(static)
    for (int g = 0; g < G; ++g) {
        int b = g / P, t = g % P;
        size_t o = (size_t)g * N;
        uot_ref_div(nx, ny, mx + o, my + o, dv + o);
        const double* x0 = XV(xcur_base, b, t);
        const double* x1 = XV(xcur_base, b, t + 1);
        for (size_t k = 0; k < N; ++k)
            Kold[o + k] = dv[o + k] - r[o + k] - x1[k] + x0[k];
    }

    for (int it = 0; it < n_iters; ++it) {
        const int last = (it == n_iters - 1);
        /* Alg.1 line 3: m_i <- shrink^{l2}_{tau1}(m_i - tau1 div^*(a^k)_i) */
        #pragma omp parallel for schedule(static)
        for (int g = 0; g < G; ++g) {
            size_t o = (size_t)g * N;
            uot_ref_div_adj(nx, ny, a + o, gx + o, gy + o);
            for (size_t k = 0; k < N; ++k) {
                int i = (int)(k % nx), j = (int)(k / nx);
                gx[o + k] = MXv(mx + o, nx, ny, i, j) - tau1 * gx[o + k];  /* q_x */
                gy[o + k] = MYv(my + o, nx, ny, i, j) - tau1 * gy[o + k];  /* q_y */
            }
            uot_ref_shrink_l2((int64_t)N, gx + o, gy + o, tau1, mxn + o, myn + o);
            /* Alg.1 line 5: r <- shrink^{l1}_{mu tau1}(r^k + tau1 a^k);
             * p = 2: r <- argmin mu r^2 - a r + (r - r^k)^2/(2 tau1) = (r^k + tau1 a^k)/(1 + 2 mu tau1)
             * ("averaging update"; derived); balanced (mu = inf): r = 0 */
            for (size_t k = 0; k < N; ++k) gx[o + k] = r[o + k] + tau1 * a[o + k];
            if (!isfinite(alpha))
                for (size_t k = 0; k < N; ++k) rn[o + k] = 0.0;
            else if (prm->p_norm == 2)
                for (size_t k = 0; k < N; ++k) rn[o + k] = gx[o + k] / (1.0 + 2.0 * alpha * tau1);
            else
                uot_ref_shrink_l1((int64_t)N, gx + o, alpha * tau1, rn + o);
        }
        /* Alg.1 line 4 (prox mode): x <- Pi_+((rho tau1 p + x^k - tau1 A^T a^k)/(1+rho tau1)) */
        if (prox) {
            #pragma omp parallel for schedule(static)
            for (int bs = 0; bs < B * T; ++bs) {
                int b = bs / T, s = bs % T;
                const double* p = XV(frames, b, s);
                const double* xs = XV(x, b, s);
                double* xo = XV(xn, b, s);
                const double* a_s = (s < P) ? a + ((size_t)b * P + s) * N : NULL;       /* a_s, s <= P-1 */
                const double* a_sm = (s >= 1) ? a + ((size_t)b * P + s - 1) * N : NULL; /* a_{s-1} */
                if (s == 0 && prm->fix_first) {          /* constant first argument s */
                    for (size_t k = 0; k < N; ++k) xo[k] = p[k];
                    continue;
                }
                for (size_t k = 0; k < N; ++k) {
                    double ATa = (a_s ? a_s[k] : 0.0) - (a_sm ? a_sm[k] : 0.0);
                    double v = (rho * tau1 * p[k] + xs[k] - tau1 * ATa) / (1.0 + rho * tau1);
                    xo[k] = v > 0.0 ? v : 0.0;
                }
            }
        }
        const double* xnew_base = prox ? xn : frames;
        /* Alg.1 lines 6-7: b = 2K^{k+1} - K^k, a <- a^k + tau2 b */
        #pragma omp parallel for schedule(static)
        for (int g = 0; g < G; ++g) {
            int b = g / P, t = g % P;
            size_t o = (size_t)g * N;
            uot_ref_div(nx, ny, mxn + o, myn + o, dv + o);
            const double* x0 = XV(xnew_base, b, t);
            const double* x1 = XV(xnew_base, b, t + 1);
            for (size_t k = 0; k < N; ++k) {
                Knew[o + k] = dv[o + k] - rn[o + k] - x1[k] + x0[k];
                double bb = 2.0 * Knew[o + k] - Kold[o + k];
                an[o + k] = a[o + k] + tau2 * bb;
            }
            if (last && rep) {
                double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0;
                for (size_t k = 0; k < N; ++k) {
                    int i = (int)(k % nx), j = (int)(k / nx);
                    double dmx = mxn[o + k] - MXv(mx + o, nx, ny, i, j);
                    double dmy = myn[o + k] - MYv(my + o, nx, ny, i, j);
                    double dr = rn[o + k] - r[o + k];
                    double f = x1[k] - x0[k];
                    const double u = dv[o + k] - f;
                    s0 += sqrt(mxn[o + k] * mxn[o + k] + myn[o + k] * myn[o + k]);
                    s1 += (prm->p_norm == 2) ? rn[o + k] * rn[o + k] : fabs(rn[o + k]);
                    s2 += Knew[o + k] * Knew[o + k];
                    s3 += dmx * dmx + dmy * dmy + dr * dr;
                    s4 += (prm->p_norm == 2) ? u * u : fabs(u);
                    s6 += f * f;
                }
                if (prox) {
                    /* frames attributed to this pair: t, plus T-1 for the last pair */
                    for (int s = t; s <= (t == P - 1 ? t + 1 : t); ++s) {
                        const double* p = XV(frames, b, s);
                        const double* xs = XV(x, b, s);
                        const double* xo = XV(xn, b, s);
                        for (size_t k = 0; k < N; ++k) {
                            double dx = xo[k] - xs[k];
                            double dp = xo[k] - p[k];
                            s3 += dx * dx;
                            s5 += dp * dp;
                        }
                    }
                }
                double* R = rep + (size_t)g * REP_STRIDE;
                R[0] = s0; R[1] = s1; R[2] = s2; R[3] = s3; R[4] = s4; R[5] = s5; R[6] = s6;
                R[7] = (double)N;
            }
        }
        /* commit: (M, r, x, a, K^k) <- (M^{k+1}, r^{k+1}, x^{k+1}, a^{k+1}, K^{k+1}) */
        for (size_t k = 0; k < N * G; ++k) {
            int i = (int)((k % N) % nx), j = (int)((k % N) / nx);
            mx[k] = (i < nx - 1) ? mxn[k] : 0.0;
            my[k] = (j < ny - 1) ? myn[k] : 0.0;
            r[k] = rn[k];
            a[k] = an[k];
            Kold[k] = Knew[k];
            if (!isfinite(a[k]) || !isfinite(mx[k]) || !isfinite(my[k]) || !isfinite(r[k])) status = 4;
        }
        if (prox) memcpy(x, xn, sizeof(double) * N * B * T);
    }
#undef XV
    free(gx); free(gy); free(mxn); free(myn); free(rn); free(an);
    free(Kold); free(Knew); free(dv); free(xn);
    return status;
}

/* Objective and weak-duality certificate of eq:Unbal_OT_beckman at the given
 * state (derived from the Lagrangian P:235-242):
 * the dual of min ||M||_{2,1} + alpha||r||_1 s.t. div M - r = f is
 *   max -<a, f>  s.t. ||(div^* a)_k||_2 <= 1, |a_k| <= alpha,
 * so for ANY a, with c = max(1, max_k ||(div^*a)_k||, max_k |a_k|/alpha),
 *   L = -<a, f>/c  <=  V_alpha(x_t, x_{t+1})  <=  U = ||M||_{2,1} + alpha ||div M - f||_1.
 * p = 2 (alpha ||r||_2^2): dual max -<a,f> - ||a||^2/(4 alpha) s.t. ||div^*a|| <= 1:
 *   c = max(1, max||div^*a||), L = -<a,f>/c - ||a||^2/(4 alpha c^2), U = ||M|| + alpha||div M - f||^2.
 * balanced (alpha = inf, eq:OT_beckman): c = max(1, max||div^*a||), L = -<a,f>/c,
 *   U = ||M|| if div M = f exactly, else +inf.
 * f = x_{t+1} - x_t uses x (prox mode) or the frames (fixed mode).
 * cert[g*8 + .]: 0 transport, 1 sum|r|^p, 2 U, 3 <a,f>, 4 max||div^*a||,
 * 5 max|a|, 6 L, 7 objective ||M||_{2,1} + alpha||r||_p^p. */
int uot_ref_certificate(const uot_ref_params* prm, const double* frames,
                        const double* mx, const double* my, const double* r,
                        const double* a, const double* x, double* cert) {
    const int nx = prm->nx, ny = prm->ny, B = prm->n_chains, T = prm->n_frames;
    const int P = T - 1;
    const size_t N = (size_t)nx * ny;
    const int prox = isfinite(prm->rho);
    const double alpha = prm->alpha;
    double* dv = malloc(sizeof(double) * N);
    double* gx = malloc(sizeof(double) * N);
    double* gy = malloc(sizeof(double) * N);
    for (int g = 0; g < B * P; ++g) {
        int b = g / P, t = g % P;
        size_t o = (size_t)g * N;
        const double* base = prox ? x : frames;
        const double* x0 = base + ((size_t)b * T + t) * N;
        const double* x1 = base + ((size_t)b * T + t + 1) * N;
        uot_ref_div(nx, ny, mx + o, my + o, dv);
        uot_ref_div_adj(nx, ny, a + o, gx, gy);
        const int p2 = prm->p_norm == 2;
        double tr = 0, gr = 0, ub = 0, af = 0, mg = 0, ma = 0, a2 = 0;
        for (size_t k = 0; k < N; ++k) {
            int i = (int)(k % nx), j = (int)(k / nx);
            double mxk = MXv(mx + o, nx, ny, i, j), myk = MYv(my + o, nx, ny, i, j);
            double f = x1[k] - x0[k];
            double u = dv[k] - f;
            tr += sqrt(mxk * mxk + myk * myk);
            gr += p2 ? r[o + k] * r[o + k] : fabs(r[o + k]);
            ub += p2 ? u * u : fabs(u);
            af += a[o + k] * f;
            a2 += a[o + k] * a[o + k];
            double gn = sqrt(gx[k] * gx[k] + gy[k] * gy[k]);
            if (gn > mg) mg = gn;
            if (fabs(a[o + k]) > ma) ma = fabs(a[o + k]);
        }
        double c = 1.0;
        if (mg > c) c = mg;
        const int bal = !isfinite(alpha);
        if (!bal && !p2 && ma / alpha > c) c = ma / alpha;
        double* C = cert + (size_t)g * REP_STRIDE;
        C[0] = tr; C[1] = gr; C[3] = af; C[4] = mg; C[5] = ma;
        if (bal) {
            C[2] = (ub == 0.0) ? tr : INFINITY;
            C[6] = -af / c;
            C[7] = tr;
        } else {
            C[2] = tr + alpha * ub;
            C[6] = p2 ? -af / c - a2 / (4.0 * alpha * c * c) : -af / c;
            C[7] = tr + alpha * gr;
        }
    }
    free(dv); free(gx); free(gy);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 2 (UOT-DF ADMM) for eq:UOT-DF with
 * Phi = I and R = 0 (the denoising setting of Fig. 1), on B
 * independent problems (y_b, s0_b):
 *   min_{s >= 0} 1/2 ||y - s||^2 + kappa V_mu(s0, s)
 * (V is symmetric, P13, so the prior is the constant FIRST argument of the
 * prox as in Alg. 2 line 6 / eq:Prox_UOT_specialcase, reading L22).
 * Per outer iteration, in the paper's order:
 *   line 4: s <- Pi_+((x + a + z + b)/2): the minimiser over s of the printed
 *           augmented Lagrangian; the printed line 4 / P:487-492
 *           "prox(x + a)" drops the (z - s + b) term, with which the UOT term
 *           could never reach s (reading L23, pinned by DF3's KKT check)
 *   line 5: x <- (y + rho (s - a)) / (1 + rho)                (Phi = I)
 *   line 6: z <- prox^mu_{kappa/rho V_{s0}}(s - b): inner_iters warm-started
 *           iterations of Alg. 1 with the first argument fixed (A := I,
 *           P:343-349); in the L2 rho convention its weight is rho/kappa (L2)
 *   line 7: a <- a + x - s;  line 8: b <- b + z - s
 * res[it*2 + 0/1] = primal ||[x - s; z - s]||_2, dual rho ||[x - x_prev; z - z_prev]||_2
 * (stopping criterion of P:562-567).  State arrays [B][N]; inner state
 * mx, my, r, ain [B][N] (the inner "pair" of each problem).  Returns 0 or 4. */
typedef struct {
    int32_t nx, ny, n_problems;
    double mu, kappa, rho, tau1, tau2;
    int32_t inner_iters, p_norm;
} uot_ref_df_params;

int uot_ref_df_admm(const uot_ref_df_params* prm, const double* y, const double* s0,
                    double* s, double* x, double* z, double* a, double* b,
                    double* mx, double* my, double* r, double* ain, int n_outer, double* res) {
    const int B = prm->n_problems;
    const size_t N = (size_t)prm->nx * prm->ny;
    double* fr = malloc(sizeof(double) * N * 2 * B);    /* inner frames [B][2][N]: (s0, v) */
    double* xin = malloc(sizeof(double) * N * 2 * B);   /* inner x [B][2][N]: (s0, z)      */
    double* xn = malloc(sizeof(double) * N * B);
    uot_ref_params ip;
    ip.nx = prm->nx; ip.ny = prm->ny; ip.n_chains = B; ip.n_frames = 2;
    ip.alpha = prm->mu; ip.rho = prm->rho / prm->kappa; ip.tau1 = prm->tau1; ip.tau2 = prm->tau2;
    ip.p_norm = prm->p_norm; ip.fix_first = 1;
    int status = 0;
    for (int it = 0; it < n_outer; ++it) {
        double pr = 0.0, du = 0.0;
        for (size_t k = 0; k < N * B; ++k) {
            double v = 0.5 * (x[k] + a[k] + z[k] + b[k]);
            s[k] = v > 0.0 ? v : 0.0;                                  /* line 4 (L23) */
            xn[k] = (y[k] + prm->rho * (s[k] - a[k])) / (1.0 + prm->rho);   /* line 5 */
        }
        for (int bb = 0; bb < B; ++bb)
            for (size_t k = 0; k < N; ++k) {
                size_t q = (size_t)bb * N + k;
                fr[((size_t)bb * 2) * N + k] = s0[q];
                fr[((size_t)bb * 2 + 1) * N + k] = s[q] - b[q];        /* prox centre v = s - b */
                xin[((size_t)bb * 2) * N + k] = s0[q];
                xin[((size_t)bb * 2 + 1) * N + k] = z[q];
            }
        int rc = uot_ref_iterate(&ip, fr, mx, my, r, ain, xin, prm->inner_iters, NULL);   /* line 6 */
        if (rc) status = rc;
        for (int bb = 0; bb < B; ++bb)
            for (size_t k = 0; k < N; ++k) {
                size_t q = (size_t)bb * N + k;
                double zn = xin[((size_t)bb * 2 + 1) * N + k];
                a[q] += xn[q] - s[q];                                  /* line 7 */
                b[q] += zn - s[q];                                     /* line 8 */
                pr += (xn[q] - s[q]) * (xn[q] - s[q]) + (zn - s[q]) * (zn - s[q]);
                du += (xn[q] - x[q]) * (xn[q] - x[q]) + (zn - z[q]) * (zn - z[q]);
                x[q] = xn[q];
                z[q] = zn;
            }
        if (res) { res[2 * it] = sqrt(pr); res[2 * it + 1] = prm->rho * sqrt(du); }
    }
    free(fr); free(xin); free(xn);
    return status;
}
