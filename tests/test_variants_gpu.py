"""GPU parity of the SURVEY §8(f) NEXT(2) kernel variants vs the oracle:
balanced Beckmann (alpha = +inf, eq:OT_beckman / footnote P:609), the p = 2
residual ("averaging update") and the fixed-first-argument prox
(eq:Prox_UOT_specialcase), on both execution paths."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem

pytestmark = pytest.mark.gpu
# one-pass k_iter ("stream"), register-wavefront passes (four / two iterations per pass;
# prox contexts run k_iter there), SMEM-tile passes, SMEM-resident persistent kernel
PATHS = ["stream", "temporal", "temporal2", "tiles", "persist", "single"]


def _run(monkeypatch, path, fr, alpha, rho, tau, n, **kw):
    monkeypatch.setenv("UOT_PERSIST", "1" if path == "persist" else "0")
    monkeypatch.setenv("UOT_SINGLE", "1" if path == "single" else "0")      # one-CTA k_single (G = 1)
    monkeypatch.setenv("UOT_TEMPORAL", "0" if path == "stream" else "1")
    monkeypatch.setenv("UOT_T4", "0" if path == "temporal2" else "1")
    monkeypatch.setenv("UOT_WAVE", "0" if path == "tiles" else "1")
    prob = Problem(torch.from_numpy(fr).cuda(), alpha, rho=rho, tau1=tau, tau2=tau, **kw)
    rep = prob.step(n, report=True)
    st = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    return prob, st, rep


def _cmp(fr, st, ref, names=("mx", "my", "r", "a"), tol=1e-3):
    f = np.abs(fr[:, 1:].astype(np.float64) - fr[:, :-1]).max()
    for name in names:
        rv = getattr(ref, name)
        scale = max(np.abs(rv).max(), f, np.abs(fr).max() if name == "x" else 0.0)
        e = np.abs(st[name] - rv).max() / scale
        assert e <= tol, (name, e)


def _balanced(B, T, ny, nx, seed):
    fr = inputs.gen_random(B, T, ny, nx, seed=seed, kind="sparse").astype(np.float64)
    fr = fr / fr.sum(axis=(2, 3), keepdims=True) * 10.0      # equal mass in every frame
    return fr.astype(np.float32)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", [(1, 2, 24, 32), (2, 3, 17, 20), (1, 2, 64, 64)])
def test_balanced_fixed(monkeypatch, path, shape):
    fr = _balanced(*shape, seed=sum(shape))
    B, T, ny, nx = shape
    tau = oracle.default_steps(nx, ny, prox=False)[0]
    n = 120
    prob, st, rep = _run(monkeypatch, path, fr, math.inf, math.inf, tau, n)
    ref, rrep = oracle.iterate(fr, math.inf, math.inf, tau, tau, n)
    _cmp(fr, st, ref)
    assert np.all(st["r"] == 0)
    assert rep["growth"] == 0.0
    assert rep["objective"] == pytest.approx(rrep[:, 0].sum(), rel=1e-4)
    _, rows = prob.objective(per_pair=True)
    cert = oracle.certificate(fr, ref, math.inf)
    np.testing.assert_allclose(rows[:, 7], cert[:, 7], rtol=1e-4)
    np.testing.assert_allclose(rows[:, 6], cert[:, 6], rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("rho", [math.inf, 2.0])
@pytest.mark.parametrize("alpha", [0.3, 2.0])
def test_p2_residual(monkeypatch, path, rho, alpha):
    fr = inputs.gen_random(2, 2, 21, 36, seed=5, kind="uniform")
    tau = oracle.default_steps(36, 21, prox=math.isfinite(rho), safety=0.95)[0]
    n = 90
    prob, st, rep = _run(monkeypatch, path, fr, alpha, rho, tau, n, p_norm=2)
    ref, rrep = oracle.iterate(fr, alpha, rho, tau, tau, n, p_norm=2)
    _cmp(fr, st, ref, ("mx", "my", "r", "a") + (("x",) if math.isfinite(rho) else ()))
    obj = rrep[:, 0].sum() + alpha * rrep[:, 1].sum() + (0.5 * rho * rrep[:, 5].sum() if math.isfinite(rho) else 0)
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)
    _, rows = prob.objective(per_pair=True)
    cert = oracle.certificate(fr, ref, alpha, rho, p_norm=2)
    for col in (0, 1, 2, 7):
        np.testing.assert_allclose(rows[:, col], cert[:, col], rtol=1e-4, atol=1e-7)
    np.testing.assert_allclose(rows[:, 6], cert[:, 6], rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("T", [2, 4])
def test_fixed_first_argument_prox(monkeypatch, path, T):
    if path == "persist" and T > 2:
        pytest.skip("persistent path is T = 2 only (falls back to streaming)")
    fr = inputs.gen_random(2, T, 19, 28, seed=T, kind="sparse")
    rho, alpha = 3.0, 0.9
    tau = oracle.default_steps(28, 19, prox=True, n_frames=T, fix_first=True, safety=0.95)[0]
    n = 80
    prob, st, rep = _run(monkeypatch, path, fr, alpha, rho, tau, n, fix_first=True)
    ref, rrep = oracle.iterate(fr, alpha, rho, tau, tau, n, fix_first=True)
    _cmp(fr, st, ref, ("mx", "my", "r", "a", "x"))
    assert np.array_equal(st["x"][:, 0], fr[:, 0].astype(np.float64))        # constant s
    obj = rrep[:, 0].sum() + alpha * rrep[:, 1].sum() + 0.5 * rho * rrep[:, 5].sum()
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)
