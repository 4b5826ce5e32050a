"""Pins of the oracle's stopping-rule and report reductions (P21-P23).

Algorithm 1 prints no stopping rule ("while not converged"), so reading L13
defines the residuals the oracle reduces in the same sweep as the iteration:
    rep[2] = sum (K^{k+1})^2,  K = div M - r - x_{t+1} + x_t   (P:276 with L1)
    rep[3] = sum ||z^{k+1} - z^k||^2,  z = (M, r[, x])
and Algorithm 2's stopping criterion is printed at P:562-567:
    primal ||[x^{k+1} - s^{k+1}; z^{k+1} - s^{k+1}]||_2,
    dual   rho ||[x^{k+1} - x^k; z^{k+1} - z^k]||_2.

Each test recomputes these quantities in numpy from CONSECUTIVE oracle states (run k
iterations, then one more from the returned state), with its own numpy divergence
(slicing, not the oracle's loops), so a reduction taken from the wrong iterate
(K^k for K^{k+1}), a dropped term (the r part of z, the x part in prox mode) or a
dropped factor (rho) fails here.  tests/oracle_mutation_check.sh applies those
mistakes.  No expected value comes from the CUDA path.
"""
import math

import numpy as np
import pytest

import oracle


def np_div(mx, my):
    """div(M) of P:153-158 with the closed grid of L3, by array slicing."""
    mx = mx.copy(); my = my.copy()
    mx[..., :, -1] = 0.0
    my[..., -1, :] = 0.0
    d = mx.copy()
    d[..., :, 1:] -= mx[..., :, :-1]
    d += my
    d[..., 1:, :] -= my[..., :-1, :]
    return d


def _frames(B, T, ny, nx, seed, nonneg=False):
    g = np.random.default_rng(seed)
    fr = g.normal(size=(B, T, ny, nx))
    fr *= g.random(size=fr.shape) < 0.4
    return np.abs(fr) if nonneg else fr


def _pair_x(fr_or_x, P):
    """(x_t, x_{t+1}) of every pair, [B][P][ny][nx] each."""
    return fr_or_x[:, :P], fr_or_x[:, 1:P + 1]


@pytest.mark.parametrize("p_norm", [1, 2])
@pytest.mark.parametrize("ny,nx,T", [(9, 11, 2), (6, 13, 4)])
def test_P21_fixed_mode_reductions_from_consecutive_states(ny, nx, T, p_norm):
    """P21 (L13): with fixed marginals every report field of the last
    iteration equals its definition evaluated on the states after k and k+1 iterations."""
    B, k, alpha = 2, 7, 0.8
    fr = _frames(B, T, ny, nx, seed=ny * nx + T)
    tau = oracle.default_steps(nx, ny, prox=False)[0]
    s0, _ = oracle.iterate(fr, alpha, math.inf, tau, tau, k, p_norm=p_norm)
    s1, rep = oracle.iterate(fr, alpha, math.inf, tau, tau, 1, state=s0, p_norm=p_norm)
    P = T - 1
    x0, x1 = _pair_x(fr, P)
    f = x1 - x0
    dv1 = np_div(s1.mx, s1.my)
    K1 = dv1 - s1.r - f
    K0 = np_div(s0.mx, s0.my) - s0.r - f
    dz2 = (s1.mx - s0.mx) ** 2 + (s1.my - s0.my) ** 2 + (s1.r - s0.r) ** 2
    pw = (lambda v: v * v) if p_norm == 2 else np.abs
    want = np.stack([
        np.sqrt(s1.mx ** 2 + s1.my ** 2).sum(axis=(2, 3)).ravel(),
        pw(s1.r).sum(axis=(2, 3)).ravel(),
        (K1 ** 2).sum(axis=(2, 3)).ravel(),
        dz2.sum(axis=(2, 3)).ravel(),
        pw(dv1 - f).sum(axis=(2, 3)).ravel(),
        np.zeros(B * P),
        (f ** 2).sum(axis=(2, 3)).ravel(),
        np.full(B * P, float(nx * ny)),
    ], axis=1)
    np.testing.assert_allclose(rep, want, rtol=1e-12, atol=1e-13)
    # the pin must separate K^{k+1} from K^k and the r part of z from none: both differ here
    assert np.all(np.abs((K0 ** 2).sum(axis=(2, 3)).ravel() - want[:, 2]) > 1e-6 * want[:, 2])
    assert np.all(((s1.r - s0.r) ** 2).sum(axis=(2, 3)).ravel() > 1e-12)


@pytest.mark.parametrize("ny,nx,T", [(7, 10, 2), (5, 12, 5)])
def test_P22_prox_mode_reductions_from_consecutive_states(ny, nx, T):
    """P22 (L13, L19): in (chain) prox mode rep[2] uses K^{k+1} with the NEW
    x, rep[3] adds ||x^{k+1} - x^k||^2 and rep[5] = ||x^{k+1} - p||^2, each frame s
    attributed to pair min(s, P-1) of its chain (oracle header)."""
    B, k, alpha, rho = 2, 6, 0.9, 3.0
    fr = _frames(B, T, ny, nx, seed=100 + ny * nx + T, nonneg=True)
    tau = oracle.default_steps(nx, ny, prox=True, n_frames=T)[0]
    s0, _ = oracle.iterate(fr, alpha, rho, tau, tau, k)
    s1, rep = oracle.iterate(fr, alpha, rho, tau, tau, 1, state=s0)
    P = T - 1
    x0, x1 = _pair_x(s1.x, P)
    dv1 = np_div(s1.mx, s1.my)
    K1 = dv1 - s1.r - (x1 - x0)
    dz2 = ((s1.mx - s0.mx) ** 2 + (s1.my - s0.my) ** 2 + (s1.r - s0.r) ** 2).sum(axis=(2, 3))
    dx2 = ((s1.x - s0.x) ** 2).sum(axis=(2, 3))          # [B][T]
    dp2 = ((s1.x - fr) ** 2).sum(axis=(2, 3))
    own = lambda v: np.concatenate([v[:, :P - 1], (v[:, P - 1] + v[:, P])[:, None]], axis=1)
    np.testing.assert_allclose(rep[:, 2], (K1 ** 2).sum(axis=(2, 3)).ravel(), rtol=1e-12)
    np.testing.assert_allclose(rep[:, 3], (dz2 + own(dx2)).ravel(), rtol=1e-12)
    np.testing.assert_allclose(rep[:, 5], own(dp2).ravel(), rtol=1e-12)
    np.testing.assert_allclose(rep[:, 6], ((x1 - x0) ** 2).sum(axis=(2, 3)).ravel(), rtol=1e-12)
    assert np.all(own(dx2).ravel() > 1e-10)                # the x part is not negligible


@pytest.mark.parametrize("inner", [1, 3])
def test_P23_df_admm_residuals_from_consecutive_states(inner):
    """P23: Algorithm 2's reported residuals of the last outer iteration
    equal ||[x - s; z - s]|| and rho ||[x - x_prev; z - z_prev]|| of consecutive states."""
    g = np.random.default_rng(11 + inner)
    B, ny, nx = 2, 9, 12
    y = np.abs(g.normal(size=(B, ny, nx)))
    s0 = np.abs(g.normal(size=(B, ny, nx)))
    mu, kappa, rho = 0.7, 0.5, 2.5
    tau = oracle.default_steps(nx, ny, prox=True, fix_first=True)[0]
    st0, _ = oracle.df_admm(y, s0, mu, kappa, rho, tau, tau, 5, inner_iters=inner)
    st1, res = oracle.df_admm(y, s0, mu, kappa, rho, tau, tau, 1, inner_iters=inner, state=st0)
    s, x, z = st1["s"], st1["x"], st1["z"]
    pr = math.sqrt(((x - s) ** 2).sum() + ((z - s) ** 2).sum())
    du = rho * math.sqrt(((x - st0["x"]) ** 2).sum() + ((z - st0["z"]) ** 2).sum())
    assert res[0, 0] == pytest.approx(pr, rel=1e-12)
    assert res[0, 1] == pytest.approx(du, rel=1e-12)
    # the scaled duals also follow lines 7-8 from the same states
    np.testing.assert_allclose(st1["a"], st0["a"] + x - s, rtol=0, atol=1e-13)
    np.testing.assert_allclose(st1["b"], st0["b"] + z - s, rtol=0, atol=1e-13)
    assert du > 1e-6 and abs(du / rho - du) > 1e-6         # rho != 1 is visible
