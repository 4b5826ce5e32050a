"""Pins of the Algorithm-3 oracle (oracle/rpca.py, RPCA+UOT-DF ADMM) against
things other than itself (R1..R7).

Independent truths used: SVT fixtures and the prox optimality of SVT (S:284-290,
P:838-840), closed forms of the two limits of eq:RPCA_UOTDF (lambda -> inf: the SVT of a
rank-1 nonnegative Y; gamma, 1/kappa -> inf: the nonnegative soft threshold), an
independent 1-D QP (SLSQP over (s0, s1, M, r)) for T = 2, the KKT conditions of
eq:RPCA_UOTDF at the ADMM limit (with V evaluated by the certified Algorithm-1 solve of
P7), and the first two iterations from the cold start derived by hand.  Every reading
(L25..L27) is shown to be needed: the literal printed line fails a pin.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import lp, rpca


def _tau(nx, ny):
    return oracle.default_steps(nx, ny, prox=True)[0]


def _instance(seed, T=4, ny=6, nx=6, neg=0.0, mask=True):
    """Sparse movers + rank-1 background (the paper's synthetic protocol, at
    desk size), diagonal Phi with ~20% zero (masked) pixels, small noise."""
    g = np.random.default_rng(seed)
    S = np.zeros((T, ny, nx))
    for t in range(T):
        S[t, 2, (1 + t) % nx] = 1.0
        S[t, 4, (4 - t % 2) % nx] = 0.7
    U, V = g.random((ny * nx, 1)), g.random((T, 1))
    L = (U @ V.T).T.reshape(T, ny, nx) / 4.0
    phi = np.where(g.random((T, ny, nx)) < 0.2, 0.0, g.uniform(0.5, 1.5, (T, ny, nx))) if mask else np.ones((T, ny, nx))
    Y = phi * (S + L) + 0.01 * g.normal(size=(T, ny, nx))
    Y[:, 0, :] -= neg
    return Y, phi


# ----------------------------------------------------------------------------- R1 SVT
def test_R1_svt_fixtures():
    """R1: S:286-290 fixtures: diag(3,1), sigma 2 -> diag(1,0); sigma 0 -> identity;
    rank-1 u v^T with ||u|| ||v|| = 5 at sigma 5 -> 0."""
    np.testing.assert_allclose(rpca.svt(np.diag([3.0, 1.0]), 2.0), np.diag([1.0, 0.0]), atol=1e-14)
    X = np.random.default_rng(0).normal(size=(7, 4))
    np.testing.assert_allclose(rpca.svt(X, 0.0), X, atol=1e-12)
    u, v = np.array([3.0, 4.0, 0.0]), np.array([0.6, 0.8])        # ||u|| = 5, ||v|| = 1
    np.testing.assert_allclose(rpca.svt(np.outer(u, v), 5.0), 0.0, atol=1e-13)


@pytest.mark.parametrize("shape,sigma", [((9, 4), 0.7), ((30, 6), 2.0), ((5, 5), 0.1)])
def test_R1b_svt_is_the_nuclear_prox(shape, sigma):
    """R1b: svt(X, s) minimises s||Y||_* + 1/2||Y - X||_F^2: no random
    perturbation lowers the objective, and the norm-subgradient test holds:
    G = (X - Y)/s has spectral norm <= 1 and <G, Y> = ||Y||_*."""
    g = np.random.default_rng(hash(shape) % 1000)
    X = g.normal(size=shape)
    Y = rpca.svt(X, sigma)
    F = lambda Z: sigma * rpca.nuclear_norm(Z) + 0.5 * ((Z - X) ** 2).sum()
    f0 = F(Y)
    for _ in range(200):
        assert F(Y + 1e-3 * g.normal(size=shape)) >= f0 - 1e-12
    G = (X - Y) / sigma
    assert np.linalg.norm(G, 2) <= 1 + 1e-10
    assert np.sum(G * Y) == pytest.approx(rpca.nuclear_norm(Y), rel=1e-10, abs=1e-12)


# ----------------------------------------------------------------------------- R2, R3 limits
def test_R2_large_lambda_gives_svt_of_rank1():
    """R2: lambda -> inf forces S = 0; with Phi = I and a rank-1 nonnegative Y the
    remaining problem min 1/2||Y - L||^2 + gamma||L||_*, L >= 0 has the closed form
    L = (1 - gamma/sigma_1) Y (the SVT is already nonnegative)."""
    g = np.random.default_rng(2)
    T, ny, nx = 5, 4, 6
    Y = np.outer(g.random(T), g.random(ny * nx)).reshape(T, ny, nx)
    gamma = 0.3
    t = _tau(nx, ny)
    st, res, nuc = rpca.admm(Y, 1e6, gamma, 0.5, 1.0, 1.0, t, t, 3000)
    s1 = np.linalg.svd(Y.reshape(T, -1), compute_uv=False)[0]
    assert np.abs(st["S"]).max() == 0.0
    np.testing.assert_allclose(st["L"], (1 - gamma / s1) * Y, atol=1e-10)
    assert nuc[-1] == pytest.approx(s1 - gamma, rel=1e-10)


def test_R3_large_gamma_small_kappa_gives_soft_threshold():
    """R3: gamma -> inf forces L = 0 and kappa -> 0 removes the OT coupling, so
    s_t = argmin_{s >= 0} 1/2||y - phi s||^2 + lambda||s||_1 = max((phi y - lambda)/phi^2, 0)
    (closed form, diagonal Phi with phi > 0)."""
    g = np.random.default_rng(3)
    T, ny, nx = 3, 5, 4
    Y = g.normal(size=(T, ny, nx))
    phi = g.uniform(0.5, 1.5, (T, ny, nx))
    lam = 0.2
    t = _tau(nx, ny)
    st, res, _ = rpca.admm(Y, lam, 1e6, 1e-9, 1.0, 1.0, t, t, 4000, phi=phi)
    np.testing.assert_allclose(st["S"], np.maximum((phi * Y - lam) / phi**2, 0.0), atol=1e-7)
    assert np.abs(st["L"]).max() < 1e-12


# ----------------------------------------------------------------------------- R4 1-D QP
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_R4_pair_1d_bruteforce_qp(seed):
    """R4: T = 2, 1 x 6 grid, gamma -> inf (L = 0): the ADMM limit equals the optimum of
    an independent QP over (s0, s1, M, r) (oracle/lp.py rpca_pair_1d_qp)."""
    g = np.random.default_rng(10 + seed)
    n = 6
    s0 = g.random(n) * (g.random(n) < 0.6)
    y0 = s0 + 0.05 * g.normal(size=n)
    y1 = np.roll(s0, 1) * 1.2 + 0.05 * g.normal(size=n)
    lam, kappa, mu = 0.05, 0.8, 0.7
    v, q0, q1 = lp.rpca_pair_1d_qp(y0, y1, lam, kappa, mu)
    t = _tau(n, 1)
    st, res, _ = rpca.admm(np.stack([y0, y1])[:, None, :], lam, 1e6, kappa, mu, 1.0, t, t, 20000)
    np.testing.assert_allclose(st["S"][0, 0], q0, atol=1e-5)
    np.testing.assert_allclose(st["S"][1, 0], q1, atol=1e-5)
    s = st["S"][:, 0]
    val = 0.5 * ((y0 - s[0]) ** 2).sum() + 0.5 * ((y1 - s[1]) ** 2).sum() + lam * s.sum() \
        + kappa * lp.uot_1d_linprog(s[0], s[1], mu)
    assert val == pytest.approx(v, rel=1e-7, abs=1e-10)


# ----------------------------------------------------------------------------- R5 KKT
def _kkt(Y, phi, st, lam, gamma, kappa, mu, rho):
    """Optimality conditions of eq:RPCA_UOTDF at an ADMM fixed point (derived from the
    augmented Lagrangian P:796-802): returns the max violation of each."""
    S, L, X, Tm, A, D = (st[k] for k in ("S", "L", "X", "Tm", "A", "D"))
    T = S.shape[0]
    z = np.zeros((1,) + S.shape[1:])
    out = {}
    out["feasibility"] = max(np.abs(X - S - L).max(), np.abs(L - Tm).max(),
                             np.abs(st["Z"] - S[:-1]).max(), np.abs(st["W"] - S[1:]).max())
    # x: Phi^T(Phi x - y) + rho A = 0
    out["x"] = np.abs(rho * A - phi * (Y - phi * X)).max()
    # s: rho(a + b + c) in lambda + N_+(s): = lambda where s > 0, <= lambda where s = 0
    G = rho * (A + np.concatenate([st["Bd"], z]) + np.concatenate([z, st["Cd"]]))
    pos = S > 1e-9
    out["s"] = max(np.abs(G - lam)[pos].max(initial=0), np.maximum(G - lam, 0)[~pos].max(initial=0))
    out["s_nonneg"] = max(-S.min(), 0.0)
    # L: A - D in -N_+(L)
    pos = L > 1e-9
    out["L"] = max(np.abs(A - D)[pos].max(initial=0), np.maximum(A - D, 0)[~pos].max(initial=0))
    # T: rho D in gamma d||L||_* <=> ||rho D||_2 <= gamma and <rho D, L> = gamma ||L||_*
    Lm, Dm = L.reshape(T, -1).T, rho * D.reshape(T, -1).T
    out["nuclear"] = max(np.linalg.norm(Dm, 2) - gamma, 0.0) + abs(np.sum(Dm * Lm) - gamma * rpca.nuclear_norm(Lm))
    # (z, w): -rho (b, c)/kappa in dV(z, w) + N_+ => <-rho(b,c)/kappa, (z,w)> = V(z, w)
    viol = 0.0
    for p in range(T - 1):
        U_, L_, _ = oracle.evaluate(st["Z"][p], st["W"][p], mu, iters=200000, tol=1e-10)
        hom = -(rho / kappa) * ((st["Bd"][p] * st["Z"][p]).sum() + (st["Cd"][p] * st["W"][p]).sum())
        viol = max(viol, abs(hom - 0.5 * (U_ + L_)) - 0.5 * (U_ - L_))
    out["ot"] = viol
    return out


@pytest.fixture(scope="module")
def kkt_instance():
    Y, phi = _instance(3, neg=0.5)
    prm = dict(lam=0.05, gamma=0.4, kappa=0.3, mu=1.5, rho=2.0)
    return Y, phi, prm


def test_R5_kkt_at_the_limit(kkt_instance):
    """R5: the Algorithm-3 limit on a general instance (all four terms active, masked
    diagonal Phi, rho != 1) satisfies every optimality condition of eq:RPCA_UOTDF."""
    Y, phi, prm = kkt_instance
    t = _tau(6, 6)
    st, res, _ = rpca.admm(Y, prm["lam"], prm["gamma"], prm["kappa"], prm["mu"], prm["rho"], t, t, 20000,
                           inner_iters=3, phi=phi)
    assert res[-1, 0] < 1e-12 and res[-1, 1] < 1e-12
    k = _kkt(Y, phi, st, **prm)
    for name, v in k.items():
        assert v < 1e-8, (name, v)
    assert np.abs(st["S"]).max() > 0.1 and np.abs(st["L"]).max() > 0.05     # both parts active
    # objective at the output <= objective at the cold start
    assert rpca.objective(Y, st["S"], st["L"], prm["lam"], prm["gamma"], prm["kappa"], prm["mu"], phi) \
        < 0.5 * (Y**2).sum()


def test_R5b_literal_line9_fails_kkt(kkt_instance):
    """R5b (reading L26): the printed line 9 (no rho on k_t) converges to a point that
    violates x-stationarity when rho != 1."""
    Y, phi, prm = kkt_instance
    t = _tau(6, 6)
    st, res, _ = rpca.admm(Y, prm["lam"], prm["gamma"], prm["kappa"], prm["mu"], prm["rho"], t, t, 5000,
                           inner_iters=3, phi=phi, literal=("L26",))
    assert _kkt(Y, phi, st, **prm)["x"] > 1e-2


def test_R5c_literal_dual_sign_diverges(kkt_instance):
    """R5c (reading L27): the printed line 12 (A + X - S + L) has no fixed point with
    X = S + L and L != 0: the iteration blows up or stays infeasible."""
    Y, phi, prm = kkt_instance
    t = _tau(6, 6)
    try:
        st, res, _ = rpca.admm(Y, prm["lam"], prm["gamma"], prm["kappa"], prm["mu"], prm["rho"], t, t, 5000,
                               inner_iters=3, phi=phi, literal=("L27",))
        assert _kkt(Y, phi, st, **prm)["feasibility"] > 1e-2
    except FloatingPointError:
        pass


# ----------------------------------------------------------------------------- R6 hand iterations
def test_R6_first_two_iterations_closed_form():
    """R6: from the cold start (line 2), derived by hand from lines 5-15:
    iteration 1: s = 0, L = 0, x = phi y/(phi^2 + rho), T = 0, z = w = 0, A = x, D = b = c = 0;
    iteration 2: s_t = max((2 x1_t - lambda/rho)/sigma_t, 0), L = Pi_+(x1 - s/2),
    x = (phi y + rho (s + L - x1))/(phi^2 + rho), A = x1 + x - s - L.
    The literal printed lines (L25 two-sided shrink, L26, L27) each break one of these."""
    Y, phi = _instance(4, T=5, neg=0.5)
    lam, gamma, kappa, mu, rho = 0.05, 0.4, 0.3, 1.5, 2.0
    t = _tau(6, 6)
    run = lambda n, lit=(): rpca.admm(Y, lam, gamma, kappa, mu, rho, t, t, n, phi=phi, literal=lit)[0]
    st1 = run(1)
    x1 = phi * Y / (phi**2 + rho)
    for k in ("S", "L", "Tm", "D", "Z", "W", "Bd", "Cd"):
        assert np.abs(st1[k]).max() == 0.0, k
    np.testing.assert_allclose(st1["X"], x1, atol=1e-15)
    np.testing.assert_allclose(st1["A"], x1, atol=1e-15)
    sig = np.array([2.0, 3.0, 3.0, 3.0, 2.0])[:, None, None]
    s2 = np.maximum((2 * x1 - lam / rho) / sig, 0.0)
    L2 = np.maximum(x1 - s2 / 2, 0.0)
    X2 = (phi * Y + rho * (s2 + L2 - x1)) / (phi**2 + rho)
    st2 = run(2)
    np.testing.assert_allclose(st2["S"], s2, atol=1e-14)
    np.testing.assert_allclose(st2["L"], L2, atol=1e-14)
    np.testing.assert_allclose(st2["X"], X2, atol=1e-14)
    np.testing.assert_allclose(st2["A"], x1 + X2 - s2 - L2, atol=1e-14)
    assert (2 * x1 - lam / rho < -lam / rho * 2).any()         # some pixel where L25 matters
    assert np.abs(run(2, ("L25",))["S"] - s2).max() > 1e-3
    assert np.abs(run(2, ("L26",))["X"] - X2).max() > 1e-3
    assert np.abs(run(2, ("L27",))["A"] - (x1 + X2 - s2 - L2)).max() > 1e-3


# ----------------------------------------------------------------------------- R7 structure
def test_R7_kappa_couples_frames_and_inner_iters_converge_to_same_limit():
    """R7: (a) the limit does not depend on inner_iters (warm-started inexact prox,
    P:891-900: only the path changes); (b) a larger kappa lowers the total OT cost
    sum_t V(s_t, s_{t+1}) of the solution (the regulariser acts)."""
    Y, phi = _instance(5, T=3, neg=0.0)
    t = _tau(6, 6)
    lam, gamma, mu, rho = 0.05, 0.4, 1.5, 2.0
    a1 = rpca.admm(Y, lam, gamma, 0.3, mu, rho, t, t, 8000, inner_iters=1, phi=phi)[0]
    a5 = rpca.admm(Y, lam, gamma, 0.3, mu, rho, t, t, 8000, inner_iters=5, phi=phi)[0]
    np.testing.assert_allclose(a1["S"], a5["S"], atol=1e-7)
    np.testing.assert_allclose(a1["L"], a5["L"], atol=1e-7)

    def ot(st):
        return sum(oracle.evaluate(st["S"][p], st["S"][p + 1], mu, iters=100000, tol=1e-9)[0] for p in range(2))
    lo = rpca.admm(Y, lam, gamma, 0.05, mu, rho, t, t, 8000, inner_iters=3, phi=phi)[0]
    hi = rpca.admm(Y, lam, gamma, 1.0, mu, rho, t, t, 8000, inner_iters=3, phi=phi)[0]
    assert ot(hi) < ot(lo)


# ----------------------------------------------------------------------------- signed split (NEXT(4))
def test_SG0_signed_s_update_bruteforce():
    """SG0 (reading L30): the joint (s+, s-) update is the exact minimiser over the quadrant
    (checked against a 601 x 601 grid search on random scalar instances)."""
    g = np.random.default_rng(0)
    grid = np.linspace(0, 6, 601)
    A_, B_ = np.meshgrid(grid, grid)
    for _ in range(300):
        u, kp, km = g.normal(size=3) * 2
        m = int(g.integers(1, 3))
        lr = abs(g.normal()) * 0.5
        sp, sm = rpca.signed_s_update(np.array(u), np.array(kp), np.array(km), m, lr)
        F = lambda a, b: lr * (a + b) + 0.5 * (u - a + b) ** 2 + 0.5 * (m * a * a - 2 * kp * a) + 0.5 * (m * b * b - 2 * km * b)
        assert sp >= 0 and sm >= 0
        assert F(sp, sm) <= F(A_, B_).min() + 1e-12


def test_SG1_signed_soft_threshold_limit():
    """SG1: gamma -> inf (L = 0), kappa -> 0: s+ - s- solves the signed lasso
    min 1/2||y - phi s||^2 + lambda||s||_1: s+ = max(phi y - lambda, 0)/phi^2, s- = max(-phi y - lambda, 0)/phi^2."""
    g = np.random.default_rng(31)
    T, ny, nx = 3, 5, 4
    Y = g.normal(size=(T, ny, nx))
    phi = g.uniform(0.5, 1.5, (T, ny, nx))
    lam = 0.2
    t = _tau(nx, ny)
    st, res, _ = rpca.admm_signed(Y, lam, 1e6, 1e-9, 1.0, 1.0, t, t, 4000, phi=phi)
    np.testing.assert_allclose(st["Sp"], np.maximum(phi * Y - lam, 0) / phi**2, atol=1e-7)
    np.testing.assert_allclose(st["Sm"], np.maximum(-phi * Y - lam, 0) / phi**2, atol=1e-7)


def test_SG2_sign_flip_symmetry():
    """SG2 (S:306 'sign-flipped data swaps the roles of S+ and S-'): with L = 0 (gamma -> inf)
    eq:RPCA_UOTDF_PN is symmetric under Y -> -Y, (S+, S-) -> (S-, S+) (compared at the
    limits: L >= 0 makes the transients differ)."""
    Y, phi = _instance(9, T=4, mask=True)
    Y = Y - 0.4
    t = _tau(6, 6)
    a = rpca.admm_signed(Y, 0.05, 1e6, 0.3, 1.5, 2.0, t, t, 6000, inner_iters=3, phi=phi)[0]
    b = rpca.admm_signed(-Y, 0.05, 1e6, 0.3, 1.5, 2.0, t, t, 6000, inner_iters=3, phi=phi)[0]
    np.testing.assert_allclose(a["Sp"], b["Sm"], atol=1e-8)
    np.testing.assert_allclose(a["Sm"], b["Sp"], atol=1e-8)


def _signed_instance():
    Y, phi = _instance(12, T=4, neg=0.0)
    Y[:, 3, 2] -= 0.8                                     # a dark target: needs S-
    return Y, phi


def test_SG3_signed_kkt_at_the_limit():
    """SG3: the limit of the signed split satisfies the optimality conditions of
    eq:RPCA_UOTDF_PN: feasibility of every split, x-stationarity, rho(a + b+ + c+) and
    rho(-a + b- + c-) in lambda + N_+(s+/-), the L and nuclear-norm conditions, and the
    OT subgradient identity for each sign's chain."""
    Y, phi = _signed_instance()
    lam, gamma, kappa, mu, rho = 0.05, 0.4, 0.3, 1.5, 2.0
    t = _tau(6, 6)
    st, res, _ = rpca.admm_signed(Y, lam, gamma, kappa, mu, rho, t, t, 20000, inner_iters=3, phi=phi)
    assert res[-1, 0] < 5e-8 and res[-1, 1] < 5e-8     # slow tail: L16-type non-uniqueness
    Sp, Sm, L, X, Tm, A, D = (st[k] for k in ("Sp", "Sm", "L", "X", "Tm", "A", "D"))
    assert Sm.max() > 0.1 and Sp.max() > 0.1                # both signs active
    z = np.zeros((1, 6, 6))
    assert np.abs(X - (Sp - Sm) - L).max() < 1e-6 and np.abs(L - Tm).max() < 1e-6
    for zk, wk, s in (("Zp", "Wp", Sp), ("Zm", "Wm", Sm)):
        assert np.abs(st[zk] - s[:-1]).max() < 1e-6 and np.abs(st[wk] - s[1:]).max() < 1e-6
    assert np.abs(rho * A - phi * (Y - phi * X)).max() < 1e-6
    for sgn, s, bk, ck in ((1.0, Sp, "Bp", "Cp"), (-1.0, Sm, "Bm", "Cm")):
        G = rho * (sgn * A + np.concatenate([st[bk], z]) + np.concatenate([z, st[ck]]))
        pos = s > 1e-9
        assert np.abs(G - lam)[pos].max() < 1e-6
        assert (G - lam)[~pos].max() < 1e-6
    pos = L > 1e-9
    assert np.abs(A - D)[pos].max(initial=0) < 1e-6 and (A - D)[~pos].max(initial=-1) < 1e-6
    Lm, Dm = L.reshape(4, -1).T, rho * D.reshape(4, -1).T
    assert np.linalg.norm(Dm, 2) <= gamma + 1e-6
    assert abs(np.sum(Dm * Lm) - gamma * rpca.nuclear_norm(Lm)) < 1e-6
    for zk, wk, bk, ck in (("Zp", "Wp", "Bp", "Cp"), ("Zm", "Wm", "Bm", "Cm")):
        for p in range(3):
            U_, L_, _ = oracle.evaluate(st[zk][p], st[wk][p], mu, iters=200000, tol=1e-10)
            hom = -(rho / kappa) * ((st[bk][p] * st[zk][p]).sum() + (st[ck][p] * st[wk][p]).sum())
            assert abs(hom - 0.5 * (U_ + L_)) <= 0.5 * (U_ - L_) + 1e-6


def test_SG4_signed_objective_not_above_unsigned():
    """SG4: S- = 0 is feasible for eq:RPCA_UOTDF_PN, so at the limits its objective
    is <= that of eq:RPCA_UOTDF; on data with a dark target it is strictly lower."""
    Y, phi = _signed_instance()
    lam, gamma, kappa, mu, rho = 0.05, 0.4, 0.3, 1.5, 2.0
    t = _tau(6, 6)
    su = rpca.admm(Y, lam, gamma, kappa, mu, rho, t, t, 6000, inner_iters=3, phi=phi)[0]
    ss = rpca.admm_signed(Y, lam, gamma, kappa, mu, rho, t, t, 6000, inner_iters=3, phi=phi)[0]

    def V(s):
        return sum(oracle.evaluate(s[p], s[p + 1], mu, iters=100000, tol=1e-9)[0] for p in range(3))
    fu = rpca.objective(Y, su["S"], su["L"], lam, gamma, kappa, mu, phi) + kappa * V(su["S"])
    S = ss["Sp"] - ss["Sm"]
    data = 0.5 * ((Y - phi * (S + ss["L"])) ** 2).sum()
    fs = data + lam * (ss["Sp"].sum() + ss["Sm"].sum()) + gamma * rpca.nuclear_norm(ss["L"].reshape(4, -1).T) \
        + kappa * (V(ss["Sp"]) + V(ss["Sm"]))
    assert fs < fu - 1e-3


def test_SG5_signed_second_iteration_closed_form():
    """SG5: from the cold start, iteration 1 gives x1 = phi y/(phi^2 + rho) = A1, all else 0;
    iteration 2 gives s+ = max((2 x1 - lambda/rho)/sigma, 0), s- = max((-2 x1 - lambda/rho)/sigma, 0)
    (sigma = 1 + number of pair terms), L = Pi_+(x1 - (s+ - s-)/2)."""
    Y, phi = _instance(4, T=5, neg=0.5)
    lam, gamma, kappa, mu, rho = 0.05, 0.4, 0.3, 1.5, 2.0
    t = _tau(6, 6)
    st = rpca.admm_signed(Y, lam, gamma, kappa, mu, rho, t, t, 2, phi=phi)[0]
    x1 = phi * Y / (phi**2 + rho)
    sig = np.array([2.0, 3.0, 3.0, 3.0, 2.0])[:, None, None]
    sp = np.maximum((2 * x1 - lam / rho) / sig, 0.0)
    sm = np.maximum((-2 * x1 - lam / rho) / sig, 0.0)
    assert sm.max() > 1e-3
    np.testing.assert_allclose(st["Sp"], sp, atol=1e-14)
    np.testing.assert_allclose(st["Sm"], sm, atol=1e-14)
    np.testing.assert_allclose(st["L"], np.maximum(x1 - (sp - sm) / 2, 0.0), atol=1e-14)
