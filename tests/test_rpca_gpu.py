"""GPU parity of Algorithm 3 (RPCA+UOT-DF ADMM) through the C-ABI
(uot_rpca_*) against the float64 oracle (oracle/rpca.py) on the same seeded inputs.

Tolerances (north star): every state array within 1e-3 normalised max-abs
(L17: max|g - r| / max(max|r|, max|y|)), objective within 1e-4 relative.
"""
import math
import os

import numpy as np
import pytest

import oracle
from oracle import rpca

pytestmark = pytest.mark.gpu

KEYS = ("S", "L", "X", "Tm", "A", "D", "Z", "W", "Bd", "Cd")


def _tau(nx, ny):
    return oracle.default_steps(nx, ny, prox=True)[0]


def _gpu(Y, phi, prm, n, inner=1, persist=None, eps=0.0, check_every=None):
    import torch
    from paper_1909_00149_b200.uot import RPCAProblem
    old = os.environ.get("UOT_PERSIST")
    if persist is not None:
        os.environ["UOT_PERSIST"] = str(persist)
    try:
        t = _tau(Y.shape[2], Y.shape[1])
        prob = RPCAProblem(torch.from_numpy(Y).cuda(), prm["lam"], prm["gamma"], prm["kappa"], prm["mu"], prm["rho"],
                           phi=None if phi is None else torch.from_numpy(phi).cuda(), tau1=t, tau2=t,
                           inner_iters=inner)
    finally:
        if persist is not None:
            if old is None:
                os.environ.pop("UOT_PERSIST", None)
            else:
                os.environ["UOT_PERSIST"] = old
    rep = prob.solve(n, eps, check_every or n)
    st = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    return prob, rep, st


def _oracle(Y, phi, prm, n, inner=1):
    t = _tau(Y.shape[2], Y.shape[1])
    return rpca.admm(Y.astype(np.float64), prm["lam"], prm["gamma"], prm["kappa"], prm["mu"], prm["rho"], t, t, n,
                     inner_iters=inner, phi=None if phi is None else phi.astype(np.float64))


def _oracle_objective(Y, phi, st, nuc, prm):
    phi = np.ones_like(Y, dtype=np.float64) if phi is None else phi.astype(np.float64)
    S, L = st["S"], st["L"]
    data = 0.5 * ((Y - phi * (S + L)) ** 2).sum()
    mx, my = st["mx"].copy(), st["my"].copy()
    mx[..., :, -1] = 0.0
    my[..., -1, :] = 0.0
    transport = np.sqrt(mx**2 + my**2).sum()
    growth = prm["mu"] * np.abs(st["r"]).sum()
    return data + prm["lam"] * S.sum() + prm["gamma"] * nuc + prm["kappa"] * (transport + growth)


def _compare(Y, st_g, st_o, tol=1e-3):
    scale = max(np.abs(Y).max(), 1e-30)
    out = {}
    for k in KEYS:
        r = st_o[k]
        e = np.abs(st_g[k] - r).max() / max(np.abs(r).max(), scale)
        out[k] = e
        assert e <= tol, (k, e)
    return out


PRM = dict(lam=0.05, gamma=0.4, kappa=0.3, mu=1.5, rho=2.0)


@pytest.mark.parametrize("T,ny,nx,n,inner,persist,masked", [
    (6, 10, 10, 40, 1, None, True),        # the paper's 10x10x6 instance size
    (8, 37, 52, 30, 1, None, True),        # ragged rows, float4 columns
    (8, 37, 52, 30, 1, 0, False),          # streaming inner prox path
    (5, 24, 21, 25, 3, None, True),        # odd T (Jacobi dummy index), inner_iters > 1 (zprev)
    (2, 16, 16, 30, 1, None, False),       # minimal T
    (70, 12, 16, 12, 1, None, True),       # T > 64: 8x8 register tiles of the Gram kernel
])
def test_rpca_parity_fixed_iterations(T, ny, nx, n, inner, persist, masked):
    from paper_1909_00149_b200 import inputs
    Y, phi, _, _ = inputs.gen_rpca(T, ny, nx, seed=T * 1000 + nx, K=max(2, nx // 4), observed=0.7)
    if not masked:
        phi = None
    prob, rep, st_g = _gpu(Y, phi, PRM, n, inner, persist)
    st_o, res, nuc = _oracle(Y, phi, PRM, n, inner)
    _compare(Y, st_g, st_o)
    assert rep["iterations"] == n
    obj = _oracle_objective(Y.astype(np.float64), phi, st_o, nuc[-1], PRM)
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)
    assert rep["nuclear"] == pytest.approx(nuc[-1], rel=1e-4, abs=1e-6)
    assert rep["primal_res"] == pytest.approx(res[-1, 0], rel=2e-2, abs=1e-5)
    assert rep["dual_res"] == pytest.approx(res[-1, 1], rel=2e-2, abs=1e-5)
    assert prob.launches > 6 * n // 2


def test_rpca_parity_growth_term_active():
    """Small mu (0.2 < the 1-px transport cost): the inner prox creates/destroys mass (r != 0),
    exercising the l1 soft threshold of the growth term inside Algorithm 3."""
    from paper_1909_00149_b200 import inputs
    prm = dict(PRM, mu=0.2, kappa=1.0)
    Y, phi, _, _ = inputs.gen_rpca(6, 20, 24, seed=11, K=6, observed=0.8)
    prob, rep, st_g = _gpu(Y, phi, prm, 30)
    st_o, res, nuc = _oracle(Y, phi, prm, 30)
    _compare(Y, st_g, st_o)
    assert np.abs(st_o["r"]).sum() > 1e-3
    obj = _oracle_objective(Y.astype(np.float64), phi, st_o, nuc[-1], prm)
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)


def test_rpca_converges_to_oracle_limit():
    """Converged comparison on the R5 KKT instance: the device-side stopping test fires and
    the fp32 limit matches the fp64 limit (pinned by the KKT conditions, R5)."""
    g = np.random.default_rng(3)
    T, ny, nx = 4, 6, 6
    S = np.zeros((T, ny, nx))
    for t in range(T):
        S[t, 2, 1 + t] = 1.0
        S[t, 4, 4 - t % 2] = 0.7
    L = (g.random((ny * nx, 1)) @ g.random((T, 1)).T).T.reshape(T, ny, nx) / 4
    phi = np.where(g.random((T, ny, nx)) < 0.2, 0.0, g.uniform(0.5, 1.5, (T, ny, nx)))
    Y = (phi * (S + L) + 0.01 * g.normal(size=(T, ny, nx))).astype(np.float32)
    phi = phi.astype(np.float32)
    prob, rep, st_g = _gpu(Y, phi, PRM, 20000, inner=3, eps=2e-6, check_every=20)
    assert rep["converged"] == 1 and rep["iterations"] < 20000
    st_o, res, nuc = _oracle(Y, phi, PRM, 20000, inner=3)
    scale = np.abs(Y).max()
    for k in ("S", "L", "X"):
        assert np.abs(st_g[k] - st_o[k]).max() / scale < 1e-3, k


def test_rpca_c3_full_size_sampled():
    """BASELINE configs[2] shape (T = 64 frames of 256^2, the RPCA video workload of
    bench --mode rpca): 6 ADMM iterations against the oracle on the full arrays."""
    from paper_1909_00149_b200 import inputs
    Y = inputs.gen_c3()[0]
    prm = dict(lam=0.05, gamma=0.05 * 256, kappa=0.5, mu=2.0, rho=1.0)
    prob, rep, st_g = _gpu(Y, None, prm, 6)
    st_o, res, nuc = _oracle(Y, None, prm, 6)
    _compare(Y, st_g, st_o)
    obj = _oracle_objective(Y.astype(np.float64), None, st_o, nuc[-1], prm)
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)


def test_rpca_deterministic_and_reset():
    from paper_1909_00149_b200 import inputs
    Y, phi, _, _ = inputs.gen_rpca(7, 20, 24, seed=5)
    _, r1, s1 = _gpu(Y, phi, PRM, 20)
    prob, r2, s2 = _gpu(Y, phi, PRM, 20)
    for k in KEYS:
        assert np.array_equal(s1[k], s2[k]), k
    prob.reset()
    r3 = prob.solve(20, 0.0, 20)
    s3 = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    for k in KEYS:
        assert np.array_equal(s1[k], s3[k]), k
    assert r3["objective"] == r1["objective"]


def test_rpca_invalid_arguments():
    import torch
    from paper_1909_00149_b200._lib import UotError
    from paper_1909_00149_b200.uot import RPCAProblem
    Y = torch.zeros(4, 8, 8, device="cuda")
    with pytest.raises(UotError):
        RPCAProblem(Y, -1.0, 1.0, 1.0, 1.0)
    with pytest.raises(UotError):
        RPCAProblem(Y, 1.0, 1.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        RPCAProblem(torch.zeros(600, 4, 4, device="cuda"), 1.0, 1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        RPCAProblem(torch.zeros(1, 4, 4, device="cuda"), 1.0, 1.0, 1.0, 1.0)


SKEYS = ("Sp", "Sm", "L", "X", "Tm", "A", "D", "Zp", "Wp", "Bp", "Cp", "Zm", "Wm", "Bm", "Cm")


@pytest.mark.parametrize("T,ny,nx,n,inner", [(6, 10, 10, 40, 1), (7, 37, 52, 30, 3), (2, 16, 16, 30, 1)])
def test_rpca_signed_parity(T, ny, nx, n, inner):
    """Signed split (eq:RPCA_UOTDF_PN) against oracle.rpca.admm_signed:
    data with bright and dark targets so both S+ and S- are active."""
    import torch
    from paper_1909_00149_b200 import inputs
    from paper_1909_00149_b200.uot import RPCAProblem
    Y, phi, S, L = inputs.gen_rpca(T, ny, nx, seed=T * 100 + nx, K=max(2, nx // 4), observed=0.7)
    Y = (Y - 0.8 * phi * np.roll(S, 3, axis=2)).astype(np.float32)          # dark copies of the targets
    t = _tau(nx, ny)
    prob = RPCAProblem(torch.from_numpy(Y).cuda(), PRM["lam"], PRM["gamma"], PRM["kappa"], PRM["mu"], PRM["rho"],
                       phi=torch.from_numpy(phi).cuda(), tau1=t, tau2=t, inner_iters=inner, signed=True)
    rep = prob.solve(n, 0.0, n)
    st_g = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    st_o, res, nuc = rpca.admm_signed(Y.astype(np.float64), PRM["lam"], PRM["gamma"], PRM["kappa"], PRM["mu"],
                                      PRM["rho"], t, t, n, inner_iters=inner, phi=phi.astype(np.float64))
    assert st_o["Sm"].max() > 1e-3 and st_o["Sp"].max() > 1e-3
    scale = np.abs(Y).max()
    for k in SKEYS:
        r = st_o[k]
        e = np.abs(st_g[k] - r).max() / max(np.abs(r).max(), scale)
        assert e <= 1e-3, (k, e)
    Sd = st_o["Sp"] - st_o["Sm"]
    mx, my = st_o["mx"].copy(), st_o["my"].copy()
    mx[..., :, -1] = 0.0
    my[..., -1, :] = 0.0
    obj = 0.5 * ((Y - phi * (Sd + st_o["L"])) ** 2).sum() + PRM["lam"] * (st_o["Sp"].sum() + st_o["Sm"].sum()) \
        + PRM["gamma"] * nuc[-1] + PRM["kappa"] * (np.sqrt(mx**2 + my**2).sum() + PRM["mu"] * np.abs(st_o["r"]).sum())
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)
    assert rep["primal_res"] == pytest.approx(res[-1, 0], rel=2e-2, abs=1e-5)
