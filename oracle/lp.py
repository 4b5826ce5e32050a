"""Independent ground truths used to PIN the oracle (TEST INFRASTRUCTURE ONLY).

None of these calls Algorithm 1: they are closed forms and brute-force linear
programs for cases where eq:Unbal_OT_beckman has an exact
solution by other means.  Citations: P:nnn = PAPER.md line, S:nnn = SPEC.md line.
"""
from __future__ import annotations

import itertools

import numpy as np


def w1_1d(p, q):
    """Balanced 1-D Beckmann (eq:OT_beckman) on a 1 x n grid:
    div M = M_i - M_{i-1} = q_i - p_i fixes M uniquely as a prefix sum, so
    W = sum_i |sum_{j<=i} (q_j - p_j)|."""
    p, q = np.asarray(p, float), np.asarray(q, float)
    if abs(p.sum() - q.sum()) > 1e-9 * max(1.0, abs(p.sum())):
        raise ValueError("unbalanced input")
    return float(np.abs(np.cumsum(q - p)[:-1]).sum())


def two_delta(m_p, m_q, d, alpha):
    """Two axis-aligned deltas at grid distance d: transport the
    common mass min(m_p, m_q) at cost min(d, 2 alpha) per unit (moving costs d,
    destroy+create costs 2 alpha) and pay alpha per unit of surplus."""
    return min(m_p, m_q) * min(d, 2.0 * alpha) + alpha * abs(m_p - m_q)


def uot_1d_enum(p, q, alpha):
    """Exact optimum of eq:Unbal_OT_beckman on a 1 x n grid (p = 1, L6 unit
    spacing) by exhaustive vertex enumeration, n <= 7.

    Eliminating r = div M - f (f = q - p) leaves the convex piecewise-linear
        F(M) = sum_{i<n-1} |M_i| + alpha sum_i |M_i - M_{i-1} - f_i|
    in M in R^{n-1} (M_{-1} = M_{n-1} = 0).  A minimiser exists at a point where
    n-1 linearly independent pieces vanish; enumerate all such choices."""
    p, q = np.asarray(p, float), np.asarray(q, float)
    n = p.size
    f = q - p
    m = n - 1
    if m == 0:
        return alpha * abs(f[0])
    rows, rhs = [], []
    for i in range(m):                       # |M_i| = 0
        e = np.zeros(m); e[i] = 1.0
        rows.append(e); rhs.append(0.0)
    for i in range(n):                       # M_i - M_{i-1} - f_i = 0
        e = np.zeros(m)
        if i < m:
            e[i] += 1.0
        if i - 1 >= 0:
            e[i - 1] -= 1.0
        rows.append(e); rhs.append(f[i])
    rows, rhs = np.array(rows), np.array(rhs)

    def F(M):
        Mf = np.concatenate([M, [0.0]])
        Mp = np.concatenate([[0.0], M])
        return np.abs(M).sum() + alpha * np.abs(Mf - Mp - f).sum()

    best = np.inf
    for S in itertools.combinations(range(len(rows)), m):
        A = rows[list(S)]
        if abs(np.linalg.det(A)) < 1e-12:
            continue
        M = np.linalg.solve(A, rhs[list(S)])
        best = min(best, F(M))
    return float(best)


def uot_1d_linprog(p, q, alpha):
    """Same LP as uot_1d_enum solved by scipy HiGHS (any n): variables
    M = M+ - M-, r = r+ - r- >= 0;  min sum(M+ + M-) + alpha sum(r+ + r-)
    s.t. M_i - M_{i-1} - r_i = q_i - p_i (eq:Unbal_OT_beckman with L1)."""
    from scipy.optimize import linprog
    p, q = np.asarray(p, float), np.asarray(q, float)
    n = p.size
    m = n - 1
    nv = 2 * m + 2 * n
    c = np.concatenate([np.ones(2 * m), alpha * np.ones(2 * n)])
    A = np.zeros((n, nv))
    for i in range(n):
        if i < m:
            A[i, i] += 1.0; A[i, m + i] -= 1.0
        if i - 1 >= 0:
            A[i, i - 1] -= 1.0; A[i, m + i - 1] += 1.0
        A[i, 2 * m + i] -= 1.0; A[i, 2 * m + n + i] += 1.0
    res = linprog(c, A_eq=A, b_eq=q - p, bounds=(0, None), method="highs")
    assert res.status == 0, res.message
    return float(res.fun)


def laplacian_matrix(nx, ny):
    """Explicit matrix of div o div^* built column by column from the
    DEFINITION of div and its adjoint as the matrix transpose --
    independent of the oracle's stencil code (used by pin P5)."""
    N = nx * ny
    nmx = [(j, i) for j in range(ny) for i in range(nx - 1)]   # existing Mx (L3)
    nmy = [(j, i) for j in range(ny - 1) for i in range(nx)]   # existing My
    D = np.zeros((N, len(nmx) + len(nmy)))
    for c, (j, i) in enumerate(nmx):       # unit Mx[j,i]: +1 at (j,i), -1 at (j,i+1)
        D[j * nx + i, c] += 1.0
        D[j * nx + i + 1, c] -= 1.0
    for c, (j, i) in enumerate(nmy):       # unit My[j,i]: +1 at (j,i), -1 at (j+1,i)
        D[j * nx + i, len(nmx) + c] += 1.0
        D[(j + 1) * nx + i, len(nmx) + c] -= 1.0
    return D @ D.T, D


def uot_1d_p2_enum(p, q, alpha):
    """Exact optimum of the p = 2 variant (alpha ||r||_2^2) on a 1 x n grid,
    n <= 7, by enumerating sign patterns of M: eliminating r = div M - f gives
        F(M) = sum_i |M_i| + alpha sum_i (M_i - M_{i-1} - f_i)^2,
    convex piecewise quadratic; on the piece with signs s (s_i = 0 -> M_i = 0)
    F is a quadratic whose stationary point solves a linear system; the global
    minimum is the best sign-consistent stationary point over all 3^(n-1) pieces."""
    p, q = np.asarray(p, float), np.asarray(q, float)
    n = p.size
    f = q - p
    m = n - 1
    if m == 0:
        return alpha * f[0] ** 2
    D = np.zeros((n, m))                 # (D M)_i = M_i - M_{i-1}
    for i in range(n):
        if i < m:
            D[i, i] += 1.0
        if i - 1 >= 0:
            D[i, i - 1] -= 1.0

    def F(M):
        return np.abs(M).sum() + alpha * ((D @ M - f) ** 2).sum()

    best = F(np.zeros(m))
    for signs in itertools.product((-1, 0, 1), repeat=m):
        s = np.array(signs, float)
        free = np.nonzero(s)[0]
        if free.size == 0:
            continue
        Df = D[:, free]
        # grad: s_free + 2 alpha Df^T (Df M - f) = 0
        H = 2 * alpha * Df.T @ Df
        g = 2 * alpha * Df.T @ f - s[free]
        try:
            Mf = np.linalg.solve(H, g)
        except np.linalg.LinAlgError:
            continue
        if np.all(s[free] * Mf >= -1e-12):
            M = np.zeros(m)
            M[free] = Mf
            best = min(best, F(M))
    return float(best)


def uot_df_1d_qp(y, s0, kappa, mu):
    """Exact optimum of eq:UOT-DF with Phi = I on a 1 x n grid,
        min_{s >= 0} 1/2 ||y - s||^2 + kappa V_mu(s0, s),
    written as one QP in (s, M+, M-, r+, r-) >= 0 with the Beckmann constraint
    M_i - M_{i-1} - r_i = s_i - s0_i (L1) and solved by scipy SLSQP (independent
    of Algorithms 1-2).  Returns (value, s)."""
    from scipy.optimize import minimize
    y, s0 = np.asarray(y, float), np.asarray(s0, float)
    n = y.size
    m = n - 1
    nv = n + 2 * m + 2 * n

    def unpack(v):
        return v[:n], v[n:n + m] - v[n + m:n + 2 * m], v[n + 2 * m:n + 2 * m + n] - v[n + 2 * m + n:]

    def obj(v):
        s = v[:n]
        return 0.5 * ((y - s) ** 2).sum() + kappa * (v[n:n + 2 * m].sum() + mu * v[n + 2 * m:].sum())

    def grad(v):
        g = np.empty(nv)
        g[:n] = v[:n] - y
        g[n:n + 2 * m] = kappa
        g[n + 2 * m:] = kappa * mu
        return g

    A = np.zeros((n, nv))
    for i in range(n):
        A[i, i] = -1.0                                        # - s_i
        if i < m:
            A[i, n + i] += 1.0; A[i, n + m + i] -= 1.0        # + M_i
        if i >= 1:
            A[i, n + i - 1] -= 1.0; A[i, n + m + i - 1] += 1.0   # - M_{i-1}
        A[i, n + 2 * m + i] -= 1.0; A[i, n + 2 * m + n + i] += 1.0   # - r_i
    cons = {"type": "eq", "fun": lambda v: A @ v + s0, "jac": lambda v: A}
    x0 = np.concatenate([np.maximum(y, 0), np.zeros(2 * m + 2 * n)])
    best = None
    for start in (x0, np.concatenate([np.maximum(s0, 0), np.zeros(2 * m + 2 * n)])):
        res = minimize(obj, start, jac=grad, constraints=[cons], bounds=[(0, None)] * nv, method="SLSQP",
                       options={"ftol": 1e-15, "maxiter": 2000})
        if best is None or res.fun < best.fun:
            best = res
    return float(best.fun), unpack(best.x)[0]


def rpca_pair_1d_qp(y0, y1, lam, kappa, mu):
    """Exact optimum of eq:RPCA_UOTDF on a 1 x n grid with T = 2, Phi = I and
    the low-rank part absent (L = 0, the gamma -> infinity limit):
        min_{s0, s1 >= 0} 1/2||y0 - s0||^2 + 1/2||y1 - s1||^2 + lam (|s0|_1 + |s1|_1)
                          + kappa V_mu(s0, s1),
    one QP in (s0, s1, M+, M-, r+, r-) >= 0 with the Beckmann constraint
    M_i - M_{i-1} - r_i = s1_i - s0_i (L1), solved by scipy SLSQP (independent of
    Algorithms 1 and 3).  Returns (value, s0, s1)."""
    from scipy.optimize import minimize
    y0, y1 = np.asarray(y0, float), np.asarray(y1, float)
    n = y0.size
    m = n - 1
    o_m = 2 * n
    o_r = 2 * n + 2 * m
    nv = o_r + 2 * n

    def obj(v):
        s0, s1 = v[:n], v[n:2 * n]
        return (0.5 * ((y0 - s0) ** 2).sum() + 0.5 * ((y1 - s1) ** 2).sum() + lam * (s0.sum() + s1.sum())
                + kappa * (v[o_m:o_r].sum() + mu * v[o_r:].sum()))

    def grad(v):
        g = np.empty(nv)
        g[:n] = v[:n] - y0 + lam
        g[n:2 * n] = v[n:2 * n] - y1 + lam
        g[o_m:o_r] = kappa
        g[o_r:] = kappa * mu
        return g

    A = np.zeros((n, nv))
    for i in range(n):
        A[i, i] = 1.0                                                # + s0_i
        A[i, n + i] = -1.0                                           # - s1_i
        if i < m:
            A[i, o_m + i] += 1.0; A[i, o_m + m + i] -= 1.0           # + M_i
        if i >= 1:
            A[i, o_m + i - 1] -= 1.0; A[i, o_m + m + i - 1] += 1.0   # - M_{i-1}
        A[i, o_r + i] -= 1.0; A[i, o_r + n + i] += 1.0               # - r_i
    cons = {"type": "eq", "fun": lambda v: A @ v, "jac": lambda v: A}
    best = None
    for s0i, s1i in ((np.maximum(y0 - lam, 0), np.maximum(y1 - lam, 0)), (np.zeros(n), np.zeros(n))):
        x0 = np.concatenate([s0i, s1i, np.zeros(2 * m + 2 * n)])
        # start feasible: r = s0 - s1 (pure creation / destruction)
        d = s1i - s0i
        x0[o_r:o_r + n] = np.maximum(-d, 0)
        x0[o_r + n:] = np.maximum(d, 0)
        res = minimize(obj, x0, jac=grad, constraints=[cons], bounds=[(0, None)] * nv, method="SLSQP",
                       options={"ftol": 1e-15, "maxiter": 3000})
        if best is None or res.fun < best.fun:
            best = res
    return float(best.fun), best.x[:n].copy(), best.x[n:2 * n].copy()
