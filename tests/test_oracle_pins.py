"""Pins of the float64 oracle against things other than itself (P1..P17).

Each test names the pin id, the PAPER.md passage (P:nnn) or SPEC.md line (S:nnn)
it comes from, and what independent truth it checks: a hand example, a closed
form, an explicitly assembled matrix, a brute-force LP, a duality bound, or an
invariant.  No expected value here comes from the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import lp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _pinned(mx, my):
    mx = mx.copy(); my = my.copy()
    mx[..., :, -1] = 0.0
    my[..., -1, :] = 0.0
    return mx, my


# ----------------------------------------------------------------------------- P1-P5 operators
@pytest.mark.parametrize("ny,nx", [(1, 8), (8, 8), (16, 16), (31, 17), (17, 31)])
def test_P1_adjoint_identity(ny, nx):
    """P1: <div m, a> = <m, div* a> on 100 random pairs, rel <= 1e-10."""
    g = np.random.default_rng(ny * 100 + nx)
    for _ in range(100):
        mx, my = _pinned(g.normal(size=(ny, nx)), g.normal(size=(ny, nx)))
        a = g.normal(size=(ny, nx))
        lhs = np.sum(oracle.div(mx, my) * a)
        gx, gy = oracle.div_adj(a)
        rhs = np.sum(mx * gx) + np.sum(my * gy)
        scale = np.sqrt(np.sum(mx**2) + np.sum(my**2)) * np.linalg.norm(a)
        assert abs(lhs - rhs) <= 1e-10 * scale


@pytest.mark.parametrize("ny,nx", [(1, 5), (3, 4), (5, 3), (6, 6)])
def test_P1b_div_matches_definition_matrix(ny, nx):
    """P1b: the oracle's div / div* equal the matrix D assembled column by column
    from the definition P:153-158 (oracle/lp.py laplacian_matrix) and D^T."""
    _, D = lp.laplacian_matrix(nx, ny)
    nmx = ny * (nx - 1)
    g = np.random.default_rng(7)
    mx, my = _pinned(g.normal(size=(ny, nx)), g.normal(size=(ny, nx)))
    vec = np.concatenate([mx[:, : nx - 1].ravel(), my[: ny - 1, :].ravel()])
    np.testing.assert_allclose(oracle.div(mx, my).ravel(), D @ vec, atol=1e-13)
    a = g.normal(size=(ny, nx))
    gx, gy = oracle.div_adj(a)
    t = D.T @ a.ravel()
    np.testing.assert_allclose(gx[:, : nx - 1].ravel(), t[:nmx], atol=1e-13)
    np.testing.assert_allclose(gy[: ny - 1, :].ravel(), t[nmx:], atol=1e-13)
    assert np.all(gx[:, -1] == 0) and np.all(gy[-1, :] == 0)


def test_P2_closed_grid_sum_div_zero():
    """P2: sum div(M) = 0 for any flux (zero-flux boundary P:158)."""
    g = np.random.default_rng(3)
    for shape in [(8, 8), (1, 13), (13, 1), (9, 31)]:
        mx, my = g.normal(size=shape), g.normal(size=shape)   # pinned entries are ignored by div
        assert abs(oracle.div(mx, my).sum()) < 1e-11


def test_P2b_pinned_flux_stays_zero():
    """P2b: Mx[:, nx-1] and My[ny-1, :] stay exactly 0 through the iteration (L3)."""
    fr = np.random.default_rng(4).random((1, 2, 7, 9))
    st, _ = oracle.iterate(fr, 1.5, math.inf, 0.3, 0.3, 40)
    assert np.all(st.mx[..., :, -1] == 0) and np.all(st.my[..., -1, :] == 0)
    assert np.abs(st.mx).max() > 0 and np.abs(st.my).max() > 0


def test_P3_hand_examples():
    """P3: 2x2 hand evaluations of div and div* (S:48)."""
    for key in ("divergence_2x2", "divergence_2x2_y"):
        e = GOLD[key]
        np.testing.assert_array_equal(oracle.div(np.array(e["mx"], float), np.array(e["my"], float)),
                                      np.array(e["div"], float))
    e = GOLD["adjoint_2x2"]
    gx, gy = oracle.div_adj(np.array(e["a"], float))
    np.testing.assert_array_equal(gx, np.array(e["gx"], float))
    np.testing.assert_array_equal(gy, np.array(e["gy"], float))
    c = np.full((4, 5), 2.5)                       # constant a -> zero flux
    gx, gy = oracle.div_adj(c)
    assert np.all(gx == 0) and np.all(gy == 0)


def test_P4_shrink_examples():
    """P4: shrink^{l2} and shrink^{l1} fixtures."""
    for e in GOLD["shrink_l2"]:
        ox, oy = oracle.shrink_l2(np.array([e["q"][0]]), np.array([e["q"][1]]), e["sigma"])
        np.testing.assert_allclose([ox[0], oy[0]], e["out"], rtol=0, atol=1e-15)
    for e in GOLD["shrink_l1"]:
        np.testing.assert_allclose(oracle.shrink_l1(np.array(e["q"], float), e["sigma"]), e["out"], atol=1e-15)
    g = np.random.default_rng(5)                   # nonexpansive
    u, v = g.normal(size=(2, 1000)), g.normal(size=(2, 1000))
    su, sv = oracle.shrink_l2(u[0], u[1], 0.7), oracle.shrink_l2(v[0], v[1], 0.7)
    d_out = np.hypot(su[0] - sv[0], su[1] - sv[1])
    assert np.all(d_out <= np.hypot(u[0] - v[0], u[1] - v[1]) + 1e-15)
    assert np.all(np.abs(oracle.shrink_l1(u[0], 0.3) - oracle.shrink_l1(v[0], 0.3)) <= np.abs(u[0] - v[0]) + 1e-15)


@pytest.mark.parametrize("e", GOLD["lambda_max"])
def test_P5_lambda_max_fixtures(e):
    """P5: lambda_max(nabla^2) (Theorem 1) fixtures (S:91 + derived)."""
    assert oracle.lambda_max(e["nx"], e["ny"]) == pytest.approx(e["value"], abs=1e-12)


@pytest.mark.parametrize("ny,nx", [(1, 2), (2, 1), (3, 5), (6, 6), (4, 9), (1, 17)])
def test_P5b_lambda_max_vs_dense_eigensolver(ny, nx):
    """P5b: the closed form equals the top eigenvalue of the explicitly
    assembled D D^T (matrix from the definition), and is < 8."""
    L, _ = lp.laplacian_matrix(nx, ny)
    lam = np.linalg.eigvalsh(L).max()
    assert oracle.lambda_max(nx, ny) == pytest.approx(lam, rel=1e-12)
    assert lam < 8.0


def test_P5c_default_steps_and_chain_norm():
    """P5c: Theorem-1 default steps (product 0.99/11 with lambda bound 8)
    and ||K||^2 of the fixed / pair / chain operators (L12) vs dense SVD."""
    e = GOLD["default_steps"][0]
    assert e["safety"] / (e["lambda"] + e["extra"]) == pytest.approx(e["tau_product"], rel=1e-12)
    nx, ny = 4, 3
    _, D = lp.laplacian_matrix(nx, ny)
    N = nx * ny
    I = np.eye(N)
    # fixed mode: K = [D, -I];  pair prox: K = [D, -I, I, -I];  chain of T frames
    Kf = np.hstack([D, -I])
    assert np.linalg.norm(Kf, 2) ** 2 == pytest.approx(oracle.lambda_max(nx, ny) + 1, rel=1e-10)
    Kp = np.hstack([D, -I, I, -I])
    assert np.linalg.norm(Kp, 2) ** 2 == pytest.approx(oracle.lambda_max(nx, ny) + 3, rel=1e-10)
    for T in (3, 4, 6):
        P = T - 1
        Kc = np.zeros((P * N, P * D.shape[1] + P * N + T * N))
        for t in range(P):
            Kc[t * N:(t + 1) * N, t * D.shape[1]:(t + 1) * D.shape[1]] = D
            c0 = P * D.shape[1]
            Kc[t * N:(t + 1) * N, c0 + t * N:c0 + (t + 1) * N] = -I
            c1 = c0 + P * N
            Kc[t * N:(t + 1) * N, c1 + t * N:c1 + (t + 1) * N] = I            # +x_t
            Kc[t * N:(t + 1) * N, c1 + (t + 1) * N:c1 + (t + 2) * N] = -I     # -x_{t+1}
        lam = np.linalg.norm(Kc, 2) ** 2
        t1, t2 = oracle.default_steps(nx, ny, prox=True, n_frames=T, safety=1.0)
        assert 1.0 / (t1 * t2) == pytest.approx(lam, rel=1e-10)


# ----------------------------------------------------------------------------- P6 worked iterations
def test_P6_first_two_iterations_closed_form():
    """P6: from a zero start, iteration 1 gives M = 0, r = 0, a = -tau2 f;
    iteration 2 gives r = -tau1 sign(f) max(tau2|f| - alpha, 0) and
    M = tau1 shrink_1(tau2 div* f)  (Alg.1 lines 3-7, by hand)."""
    g = np.random.default_rng(11)
    fr = g.normal(size=(1, 2, 6, 7))
    f = fr[0, 1] - fr[0, 0]
    alpha, t1, t2 = 0.4, 0.31, 0.27
    st, _ = oracle.iterate(fr, alpha, math.inf, t1, t2, 1)
    assert np.all(st.mx == 0) and np.all(st.my == 0) and np.all(st.r == 0)
    np.testing.assert_allclose(st.a[0, 0], -t2 * f, rtol=1e-14, atol=1e-15)
    st, _ = oracle.iterate(fr, alpha, math.inf, t1, t2, 2)
    np.testing.assert_allclose(st.r[0, 0], -t1 * np.sign(f) * np.maximum(t2 * np.abs(f) - alpha, 0), atol=1e-14)
    fx, fy = oracle.div_adj(f)
    qx, qy = t2 * fx, t2 * fy
    n = np.hypot(qx, qy)
    s = np.where(n > 1.0, (n - 1.0) / np.where(n > 0, n, 1), 0.0)
    np.testing.assert_allclose(st.mx[0, 0], t1 * s * qx, atol=1e-14)
    np.testing.assert_allclose(st.my[0, 0], t1 * s * qy, atol=1e-14)
    # a^2 = a^1 + tau2 (2 K^2 - K^1) with K^1 = -f, a^1 = -tau2 f  =>  a^2 = 2 tau2 K^2
    K2 = oracle.div(st.mx[0, 0], st.my[0, 0]) - st.r[0, 0] - f
    np.testing.assert_allclose(st.a[0, 0], 2 * t2 * K2, atol=1e-14)


# ----------------------------------------------------------------------------- P7-P14 values
def test_P7_certificate_brackets_every_iterate_and_closes():
    """P7: weak duality (from the Lagrangian P:235-242): L_k <= V <= U_k at
    every iterate, and the gap closes as Theorem 1 promises."""
    g = np.random.default_rng(12)
    fr = g.random((1, 2, 8, 8)) * (g.random((1, 2, 8, 8)) < 0.3)
    alpha = 1.3
    st = None
    Ls, Us = [], []
    for _ in range(30):
        st, _ = oracle.iterate(fr, alpha, math.inf, 0.32, 0.32, 500, st)
        c = oracle.certificate(fr, st, alpha)
        Ls.append(c[0, 6]); Us.append(c[0, 2])
    assert max(Ls) <= min(Us) + 1e-12
    assert (Us[-1] - Ls[-1]) <= 1e-8 * Us[-1]


@pytest.mark.parametrize("alpha", [0.05, 0.2, 0.3, 1 / (2 * math.sqrt(2))])
def test_P8_small_alpha_closed_form(alpha):
    """P8: for alpha <= 1/(2 sqrt 2), a = -alpha sign(f) is dual feasible
    (||div* a|| <= 2 sqrt2 alpha <= 1), so V = alpha ||x1 - x0||_1 exactly
    (L6; pins the converged values of C2 / C5)."""
    g = np.random.default_rng(int(alpha * 1000))
    fr = g.random((1, 2, 9, 8))
    f = fr[0, 1] - fr[0, 0]
    U, L, obj = oracle.evaluate(fr[0, 0], fr[0, 1], alpha, iters=40000, tol=1e-10)
    v = alpha * np.abs(f).sum()
    assert L <= v * (1 + 1e-12) and U >= v * (1 - 1e-12)
    assert U == pytest.approx(v, rel=1e-7) and L == pytest.approx(v, rel=1e-7)


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("alpha", [0.5, 1.0, 2.0, 5.0])
def test_P9_two_delta(d, alpha):
    """P9: two axis-aligned deltas on 8x8:
    V = min(mp,mq) min(d, 2 alpha) + alpha |mp - mq|."""
    fr = np.zeros((1, 2, 8, 8))
    fr[0, 0, 3, 1] = 1.0
    fr[0, 1, 3, 1 + d] = 1.0
    U, L, _ = oracle.evaluate(fr[0, 0], fr[0, 1], alpha, iters=300000, tol=1e-9)
    v = lp.two_delta(1.0, 1.0, d, alpha)
    assert L - 1e-9 <= v <= U + 1e-9
    assert U == pytest.approx(v, rel=2e-5, abs=1e-8)


@pytest.mark.parametrize("e", GOLD["two_delta"])
def test_P9b_two_delta_fixtures(e):
    """P9b: SPEC fixtures S:362-364 through the closed form AND the oracle (vertical placement)."""
    assert lp.two_delta(e["m_p"], e["m_q"], e["d"], e["alpha"]) == pytest.approx(e["value"])
    fr = np.zeros((1, 2, 8, 8))
    fr[0, 0, 1, 4] = e["m_p"]
    fr[0, 1, 1 + e["d"], 4] = e["m_q"]
    U, L, _ = oracle.evaluate(fr[0, 0], fr[0, 1], e["alpha"], iters=300000, tol=1e-9)
    assert U == pytest.approx(e["value"], rel=2e-5) and L <= e["value"] + 1e-9


def test_P10_P11_balanced_1d_closed_form():
    """P10/P11: 1-D balanced W1 = sum |cumsum(q - p)| is reached by
    the unbalanced model at finite alpha >= (nx+ny-2)/2 (limit of P:208)."""
    for e in GOLD["w1_1d"]:
        assert lp.w1_1d(e["p"], e["q"]) == pytest.approx(e["value"])
    g = np.random.default_rng(13)
    for trial in range(5):
        p = g.random(16); q = g.random(16); q *= p.sum() / q.sum()
        w = lp.w1_1d(p, q)
        U, L, _ = oracle.evaluate(p, q, alpha=(16 + 1 - 2) / 2.0, iters=200000, tol=1e-8)
        assert L - 1e-7 <= w <= U + 1e-7
        assert U == pytest.approx(w, rel=1e-6)


def test_P12_unbalanced_1d_bruteforce_lp():
    """P12: 1-D unbalanced optimum by vertex enumeration (n <= 6) and
    by HiGHS (n = 16); the oracle's certified bracket must contain it."""
    for e in GOLD["uot_1d"]:
        assert lp.uot_1d_enum(e["p"], e["q"], e["alpha"]) == pytest.approx(e["value"])
    g = np.random.default_rng(14)
    for alpha in (0.1, 1.0, 10.0):
        for trial in range(4):
            p, q = g.random(5), g.random(5)
            v_enum = lp.uot_1d_enum(p, q, alpha)
            v_lp = lp.uot_1d_linprog(p, q, alpha)
            assert v_enum == pytest.approx(v_lp, rel=1e-9, abs=1e-12)
            U, L, _ = oracle.evaluate(p, q, alpha, iters=200000, tol=1e-9)
            assert L - 1e-8 <= v_enum <= U + 1e-8
            assert U == pytest.approx(v_enum, rel=1e-6, abs=1e-9)
    p, q = g.random(16), g.random(16)
    v = lp.uot_1d_linprog(p, q, 1.7)
    U, L, _ = oracle.evaluate(p, q, 1.7, iters=200000, tol=1e-9)
    assert U == pytest.approx(v, rel=1e-6) and L <= v + 1e-8


def test_P13_structural_properties():
    """P13: symmetry V(p,q) = V(q,p), monotone in alpha,
    positive homogeneity V(cp, cq) = c V(p, q) (derived)."""
    g = np.random.default_rng(15)
    p = g.random((6, 7)) * (g.random((6, 7)) < 0.4)
    q = g.random((6, 7)) * (g.random((6, 7)) < 0.4)
    v = lambda a, b, al: oracle.evaluate(a, b, al, iters=80000, tol=1e-9)[0]
    assert v(p, q, 1.1) == pytest.approx(v(q, p, 1.1), rel=1e-6)
    vals = [v(p, q, al) for al in (0.1, 0.5, 1.0, 2.0, 10.0)]
    assert all(vals[k] <= vals[k + 1] * (1 + 1e-7) for k in range(len(vals) - 1))
    assert v(3.0 * p, 3.0 * q, 1.1) == pytest.approx(3.0 * v(p, q, 1.1), rel=1e-6)


def test_P14_mass_balance():
    """P14: sum div M = 0 (closed grid) so at convergence sum r = sum x0 - sum x1
    (constraint of eq:Unbal_OT_beckman)."""
    g = np.random.default_rng(16)
    fr = g.random((1, 2, 8, 8))
    fr[0, 1] *= 1.4
    st, rep = oracle.iterate(fr, 0.8, math.inf, 0.32, 0.32, 30000)
    assert st.r.sum() == pytest.approx(fr[0, 0].sum() - fr[0, 1].sum(), rel=1e-8)
    assert rep[0, 2] < 1e-16      # primal residual ||K||^2 ~ 0


# ----------------------------------------------------------------------------- P15-P17 prox mode
def _kkt_prox(fr, st, alpha, rho):
    """Optimality conditions of eq:Prox_UOT from the Lagrangian P:234-242 (our
    sign convention L1, rho convention L2), chain generalisation L19:
      K(M, r, x) = 0;  |a| <= alpha, a = alpha sign(r) where r != 0;
      ||div* a|| <= 1, div* a = -M/||M|| where M != 0;  x = Pi_+(p - A^T a / rho)."""
    B, T, ny, nx = fr.shape
    P = T - 1
    out = {}
    K = np.zeros_like(st.a)
    for b in range(B):
        for t in range(P):
            K[b, t] = oracle.div(st.mx[b, t], st.my[b, t]) - st.r[b, t] - st.x[b, t + 1] + st.x[b, t]
    out["K"] = np.abs(K).max()
    out["a_box"] = max(0.0, np.abs(st.a).max() - alpha)
    nz = np.abs(st.r) > 1e-6
    out["a_sign"] = np.abs(st.a[nz] - alpha * np.sign(st.r[nz])).max() if nz.any() else 0.0
    worst_g = 0.0
    worst_dir = 0.0
    for b in range(B):
        for t in range(P):
            gx, gy = oracle.div_adj(st.a[b, t])
            worst_g = max(worst_g, np.hypot(gx, gy).max() - 1.0)
            n = np.hypot(st.mx[b, t], st.my[b, t])
            m = n > 1e-6
            if m.any():
                worst_dir = max(worst_dir, np.abs(gx[m] + st.mx[b, t][m] / n[m]).max(),
                                np.abs(gy[m] + st.my[b, t][m] / n[m]).max())
    out["divadj_box"] = max(0.0, worst_g)
    out["divadj_dir"] = worst_dir
    ATa = np.zeros_like(fr)
    for b in range(B):
        for s in range(T):
            ATa[b, s] = (st.a[b, s] if s < P else 0) - (st.a[b, s - 1] if s >= 1 else 0)
    out["x"] = np.abs(st.x - np.maximum(fr - ATa / rho, 0.0)).max()
    return out


@pytest.mark.parametrize("T", [2, 4])
def test_P15_prox_kkt_at_convergence(T):
    """P15a: the prox-mode fixed point satisfies the optimality conditions of
    eq:Prox_UOT (pair, T=2, exactly Alg.1 line 4) and of its chain form (L19)."""
    g = np.random.default_rng(17 + T)
    fr = g.random((1, T, 6, 6)) * (g.random((1, T, 6, 6)) < 0.5)
    alpha, rho = 0.9, 2.0
    t1, t2 = oracle.default_steps(6, 6, prox=True, n_frames=T, safety=0.9)
    st, _ = oracle.iterate(fr, alpha, rho, t1, t2, 60000)
    k = _kkt_prox(fr, st, alpha, rho)
    for key, val in k.items():
        assert val < 1e-7, (key, val)


def test_P15b_prox_limits():
    """P15b: p0 = p1 >= 0 -> x = p; alpha -> 0 -> x = Pi_+(p);
    rho -> inf with x^0 = p reproduces fixed-marginal iterates (L2, L8)."""
    g = np.random.default_rng(18)
    p = g.random((6, 6))
    fr = np.stack([p, p])[None]
    st, _ = oracle.iterate(fr, 1.0, 3.0, 0.28, 0.28, 20000)
    np.testing.assert_allclose(st.x[0], fr[0], atol=1e-8)
    fr2 = g.normal(size=(1, 2, 6, 6))
    st, _ = oracle.iterate(fr2, 1e-9, 3.0, 0.28, 0.28, 20000)
    np.testing.assert_allclose(st.x, np.maximum(fr2, 0), atol=1e-6)
    fr3 = g.random((1, 2, 6, 6))
    s0 = oracle.zero_state(fr3, prox=True, x_from_p=True)
    sp, _ = oracle.iterate(fr3, 0.7, 1e12, 0.28, 0.28, 50, s0)
    sf, _ = oracle.iterate(fr3, 0.7, math.inf, 0.28, 0.28, 50)
    for u, v in ((sp.mx, sf.mx), (sp.my, sf.my), (sp.r, sf.r), (sp.a, sf.a)):
        np.testing.assert_allclose(u, v, atol=1e-9)


def test_P16_mode_equivalences():
    """P16: a fixed-marginal chain of T frames is T-1 independent pair problems
    (pairs couple only through x, which is fixed) -- P:765 'simultaneously solved';
    B chains are independent."""
    g = np.random.default_rng(19)
    fr = g.random((2, 4, 5, 6))
    st, rep = oracle.iterate(fr, 1.2, math.inf, 0.3, 0.3, 200)
    for b in range(2):
        for t in range(3):
            s1, r1 = oracle.iterate(fr[b:b + 1, t:t + 2], 1.2, math.inf, 0.3, 0.3, 200)
            np.testing.assert_array_equal(s1.a[0, 0], st.a[b, t])
            np.testing.assert_array_equal(s1.mx[0, 0], st.mx[b, t])
            np.testing.assert_array_equal(r1[0], rep[b * 3 + t])


def test_P17_theorem1_convergence():
    """P17: Theorem 1: with tau1 tau2 = 0.9/11 the pair-prox iterates
    reach a fixed point (relative change < 1e-6) within 5e4 iterations
     on 20 random 8x8 instances."""
    g = np.random.default_rng(20)
    tau = math.sqrt(0.9 / 11.0)
    for trial in range(20):
        fr = g.random((1, 2, 8, 8))
        st = None
        ok = False
        for chunk in range(50):
            st, _ = oracle.iterate(fr, 0.6, 1.5, tau, tau, 1000, st)
            nxt, _ = oracle.iterate(fr, 0.6, 1.5, tau, tau, 1, st)
            ch = max(np.abs(nxt.a - st.a).max(), np.abs(nxt.mx - st.mx).max(),
                     np.abs(nxt.r - st.r).max(), np.abs(nxt.x - st.x).max())
            sc = max(np.abs(st.a).max(), np.abs(st.x).max(), 1.0)
            if ch / sc < 1e-6:
                ok = True
                break
        assert ok, trial


def test_oracle_deterministic_and_nonfinite():
    """Bitwise reruns; a NaN input is reported as non-finite."""
    fr = np.random.default_rng(21).random((3, 2, 9, 9))
    s1, r1 = oracle.iterate(fr, 0.9, math.inf, 0.3, 0.3, 50)
    s2, r2 = oracle.iterate(fr, 0.9, math.inf, 0.3, 0.3, 50)
    assert np.array_equal(s1.a, s2.a) and np.array_equal(r1, r2)
    fr[0, 0, 2, 2] = np.nan
    with pytest.raises(FloatingPointError):
        oracle.iterate(fr, 0.9, math.inf, 0.3, 0.3, 3)


# ----------------------------------------------------------------------------- P18-P20 NEXT(2) variants
def test_P18_balanced_beckmann():
    """P18: alpha = inf is balanced Beckmann eq:OT_beckman (r dropped, footnote P:609):
    1-D value = sum |cumsum(q - p)|, two deltas cost d, and the
    unbalanced value is <= balanced for every alpha."""
    g = np.random.default_rng(30)
    for trial in range(4):
        p = g.random(12); q = g.random(12); q *= p.sum() / q.sum()
        w = lp.w1_1d(p, q)
        U, L, obj = oracle.evaluate(p, q, math.inf, iters=300000, tol=1e-9)
        assert L - 1e-8 <= w and obj == pytest.approx(w, rel=1e-6)
        assert oracle.evaluate(p, q, 0.7, iters=100000, tol=1e-8)[0] <= w + 1e-7
    fr = np.zeros((1, 2, 8, 8)); fr[0, 0, 2, 1] = 1.0; fr[0, 1, 2, 5] = 1.0
    U, L, obj = oracle.evaluate(fr[0, 0], fr[0, 1], math.inf, iters=300000, tol=1e-9)
    assert obj == pytest.approx(4.0, rel=1e-3) and 4.0 * (1 - 1e-3) <= L <= 4.0 + 1e-9
    st, _ = oracle.iterate(fr, math.inf, math.inf, 0.3, 0.3, 200)
    assert np.all(st.r == 0)


@pytest.mark.parametrize("alpha", [0.2, 1.0, 5.0])
def test_P19_p2_residual_bruteforce_and_kkt(alpha):
    """P19: p = 2 ("averaging update"; r = (r + tau1 a)/(1 + 2 alpha tau1))
    vs exact sign-pattern enumeration of the 1-D problem; at the fixed point the
    r-stationarity a = 2 alpha r holds (Lagrangian P:235-242)."""
    g = np.random.default_rng(int(alpha * 10))
    for trial in range(4):
        p, q = g.random(5), g.random(5)
        v = lp.uot_1d_p2_enum(p, q, alpha)
        U, L, obj = oracle.evaluate(p, q, alpha, iters=300000, tol=1e-10, p_norm=2)
        assert L - 1e-8 <= v <= U + 1e-8
        assert U == pytest.approx(v, rel=1e-6, abs=1e-9)
    fr = g.random((1, 2, 6, 7))
    st, rep = oracle.iterate(fr, alpha, math.inf, 0.3, 0.3, 60000, p_norm=2)
    np.testing.assert_allclose(st.a, 2 * alpha * st.r, atol=1e-8)
    assert rep[0, 2] < 1e-18


def test_P20_fixed_first_argument_prox():
    """P20: eq:Prox_UOT_specialcase: frame 0 fixed at s, x = frame 1 with
    A := I.  Fixed point satisfies x = Pi_+(p + a/rho), K = 0, |a| <= alpha,
    ||div* a|| <= 1; s = p >= 0 gives x = p; a far-away delta prior barely
    moves a strongly attached x."""
    g = np.random.default_rng(31)
    fr = g.random((2, 2, 7, 6)) * (g.random((2, 2, 7, 6)) < 0.5)
    alpha, rho = 0.8, 1.5
    t = oracle.default_steps(6, 7, prox=True, fix_first=True, safety=0.95)[0]
    st, _ = oracle.iterate(fr, alpha, rho, t, t, 60000, fix_first=True)
    np.testing.assert_array_equal(st.x[:, 0], fr[:, 0])
    np.testing.assert_allclose(st.x[:, 1], np.maximum(fr[:, 1] + st.a[:, 0] / rho, 0), atol=1e-7)
    for b in range(2):
        K = oracle.div(st.mx[b, 0], st.my[b, 0]) - st.r[b, 0] - st.x[b, 1] + st.x[b, 0]
        assert np.abs(K).max() < 1e-8
        gx, gy = oracle.div_adj(st.a[b, 0])
        assert np.hypot(gx, gy).max() <= 1 + 1e-8 and np.abs(st.a).max() <= alpha + 1e-8
    p = g.random((6, 6))
    st, _ = oracle.iterate(np.stack([p, p])[None], 1.0, 2.0, t, t, 5000, fix_first=True)
    np.testing.assert_allclose(st.x[0, 1], p, atol=1e-9)
    fr = np.zeros((1, 2, 8, 8)); fr[0, 0, 1, 1] = 1.0; fr[0, 1, 1, 4] = 1.0
    t = oracle.default_steps(8, 8, prox=True, fix_first=True, safety=0.95)[0]
    st, _ = oracle.iterate(fr, 10.0, 100.0, t, t, 60000, fix_first=True)
    assert np.abs(st.x[0, 1] - fr[0, 1]).max() < 0.035          # |x - p| <= |a|/rho, |a| <= 3
    c = oracle.certificate(np.stack([fr[0, 0], st.x[0, 1]])[None], st, 10.0)
    assert c[0, 0] == pytest.approx(3.0, rel=3e-2)                    # transport ~ 3
    # prox optimality vs the candidate x = p (value V(s, p) = 3 by P9): F(x*) <= F(p)
    assert c[0, 7] + 0.5 * 100.0 * ((st.x[0, 1] - fr[0, 1]) ** 2).sum() <= 3.0 + 1e-7


def test_P5d_fixed_first_step_norm():
    """P5d: ||K||^2 = lambda_max + 2 for K = [D, -I, -I] (fixed-first pair prox)."""
    nx, ny = 5, 3
    _, D = lp.laplacian_matrix(nx, ny)
    I = np.eye(nx * ny)
    K = np.hstack([D, -I, -I])
    t1, t2 = oracle.default_steps(nx, ny, prox=True, fix_first=True, safety=1.0)
    assert 1.0 / (t1 * t2) == pytest.approx(np.linalg.norm(K, 2) ** 2, rel=1e-10)


# ----------------------------------------------------------------------------- DF1-DF4 Algorithm 2
def _df_tau(nx, ny):
    return oracle.default_steps(nx, ny, prox=True, fix_first=True, safety=0.95)[0]


def test_DF1_DF2_limits():
    """DF1: kappa -> 0 gives s = Pi_+(y); DF2: noiseless y = s0 >= 0 gives s = y."""
    g = np.random.default_rng(40)
    y = g.normal(size=(2, 6, 7))
    s0 = g.random((2, 6, 7))
    t = _df_tau(7, 6)
    st, res = oracle.df_admm(y, s0, 1.0, 1e-9, 1.0, t, t, 400)
    np.testing.assert_allclose(st["s"], np.maximum(y, 0), atol=1e-6)
    st, res = oracle.df_admm(s0, s0, 1.0, 2.0, 1.0, t, t, 3000)
    np.testing.assert_allclose(st["s"], s0, atol=1e-6)


def test_DF3_kkt_of_uot_df():
    """DF3: the ADMM fixed point solves eq:UOT-DF: s = x = z (splitting) and
    s = Pi_+(y + kappa a*) with a* a dual certificate of V(s0, s): K = 0, |a*| <= mu,
    ||div* a*|| <= 1 (Lagrangian P:235-242, subgradient of V in its argument is -a*)."""
    g = np.random.default_rng(41)
    s0 = g.random((1, 8, 8)) * (g.random((1, 8, 8)) < 0.3)
    y = np.roll(s0, 1, axis=2) * 1.3 + 0.02 * g.normal(size=(1, 8, 8))
    mu, kappa, rho = 0.8, 0.6, 1.0
    t = _df_tau(8, 8)
    st, res = oracle.df_admm(y, s0, mu, kappa, rho, t, t, 20000)
    assert res[-1, 0] < 1e-9 and res[-1, 1] < 1e-9
    np.testing.assert_allclose(st["x"], st["s"], atol=1e-8)
    np.testing.assert_allclose(st["z"], st["s"], atol=1e-8)
    np.testing.assert_allclose(st["s"], np.maximum(y + kappa * st["ain"], 0), atol=1e-7)
    K = oracle.div(st["mx"][0], st["my"][0]) - st["r"][0] - st["z"][0] + s0[0]
    assert np.abs(K).max() < 1e-8
    assert np.abs(st["ain"]).max() <= mu + 1e-8
    gx, gy = oracle.div_adj(st["ain"][0])
    assert np.hypot(gx, gy).max() <= 1 + 1e-8


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_DF4_uot_df_1d_bruteforce_qp(seed):
    """DF4: 1-D eq:UOT-DF optimum by an independent QP (SLSQP over (s, M, r)) equals the
    value at the ADMM limit; V evaluated by the HiGHS LP of P12."""
    g = np.random.default_rng(50 + seed)
    s0 = g.random(6) * (g.random(6) < 0.6)
    y = np.roll(s0, 1) + 0.1 * g.normal(size=6)
    mu, kappa = 0.7, 0.9
    v_qp, s_qp = lp.uot_df_1d_qp(y, s0, kappa, mu)
    t = _df_tau(6, 1)
    st, res = oracle.df_admm(y[None, None, :], s0[None, None, :], mu, kappa, 1.0, t, t, 30000)
    s = st["s"][0, 0]
    v_admm = 0.5 * ((y - s) ** 2).sum() + kappa * lp.uot_1d_linprog(s0, s, mu)
    assert v_admm == pytest.approx(v_qp, rel=1e-6, abs=1e-9)
    np.testing.assert_allclose(s, s_qp, atol=1e-4)
