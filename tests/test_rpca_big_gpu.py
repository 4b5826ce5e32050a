"""Algorithm 3 on videos of more than 128 frames: line 10 by the partial SVD of P:861 (subspace
iteration on the Gram matrix, uot_rpca_big.inc) against the fp64 oracle's exact SVT
(oracle/rpca.py, numpy SVD), and sharded (emulated shards) bitwise against the unsharded run.

Where the k = 64 Ritz vectors span the whole range of G (rank(M) <= 64: grids of <= 64 pixels,
or T <= 64 with the subspace forced), the subspace SVT is exact and the north-star bars apply
(1e-3 normalised state, 1e-4 objective).  Beyond that the SVT is exact while the k-wide subspace
holds every singular value above tau (certified by the report's smallest Ritz value < tau^2),
and the report flags a subspace that is too small.
"""
import numpy as np
import pytest

import oracle
from oracle import rpca

from test_rpca_gpu import PRM, _compare, _oracle, _oracle_objective

pytestmark = pytest.mark.gpu


def _gpu(Y, phi, prm, n, eps=0.0, check=None, shard=None):
    import torch
    from paper_1909_00149_b200.uot import RPCAProblem
    t = oracle.default_steps(Y.shape[2], Y.shape[1], prox=True)[0]
    prob = RPCAProblem(torch.from_numpy(np.ascontiguousarray(Y)).cuda(), prm["lam"], prm["gamma"], prm["kappa"],
                       prm["mu"], prm["rho"], phi=None if phi is None else torch.from_numpy(np.ascontiguousarray(phi)).cuda(),
                       tau1=t, tau2=t, shard=shard)
    rep = prob.solve(n, eps, check or n) if shard is None else None
    return prob, rep


@pytest.mark.parametrize("T,ny,nx,masked", [(160, 8, 8, True), (200, 4, 16, False), (129, 6, 8, True), (140, 5, 7, True)])
def test_rpca_long_video_exact_subspace(T, ny, nx, masked):
    """T > 128 (the one-CTA Jacobi limit), rank(M) <= N <= 64 = k: the subspace SVT is exact.
    (5 x 7: N % 4 != 0 -- the unpipelined Gram, the lane-per-pixel apply and the scalar line 13.)"""
    from paper_1909_00149_b200 import inputs
    Y, phi, _, _ = inputs.gen_rpca(T, ny, nx, seed=T + nx, K=2, observed=0.8)
    if not masked:
        phi = None
    n = 12
    prob, rep = _gpu(Y, phi, PRM, n)
    st_g = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    st_o, res, nuc = _oracle(Y, phi, PRM, n)
    _compare(Y, st_g, st_o)
    obj = _oracle_objective(Y.astype(np.float64), phi, st_o, nuc[-1], PRM)
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)
    assert rep["nuclear"] == pytest.approx(nuc[-1], rel=1e-4, abs=1e-6)


def test_rpca_forced_subspace_matches_jacobi_path(monkeypatch):
    """UOT_RPCA_SVT=1 at T = 40 (k = T: the full basis): the subspace route gives the Jacobi
    route's iterates (both against the oracle)."""
    from paper_1909_00149_b200 import inputs
    Y, phi, _, _ = inputs.gen_rpca(40, 16, 16, seed=5, K=3, observed=0.7)
    n = 20
    monkeypatch.setenv("UOT_RPCA_SVT", "1")
    prob, rep = _gpu(Y, phi, PRM, n)
    st_g = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    st_o, _, nuc = _oracle(Y, phi, PRM, n)
    _compare(Y, st_g, st_o)
    assert rep["nuclear"] == pytest.approx(nuc[-1], rel=1e-4, abs=1e-6)


def test_rpca_long_video_partial_svd():
    """T = 192 frames of 16 x 16 (rank(M) up to 192 > k = 64): the warm-started subspace holds
    the few singular values above tau = gamma/rho (27 at iteration 5, 1 from iteration ~50 on),
    so the partial SVD follows the exact SVT -- checked against the oracle at 50 iterations at
    the north-star bars, with the report's smallest Ritz value below tau^2 (the certificate that
    the k-wide subspace covers the SVT)."""
    from paper_1909_00149_b200 import inputs
    Y, phi, _, _ = inputs.gen_rpca(192, 16, 16, seed=8, K=3, observed=0.9)
    prm = dict(PRM, gamma=2.0)
    n = 50
    prob, rep = _gpu(Y, phi, prm, n, check=10)
    tau = prm["gamma"] / prm["rho"]
    assert 0.0 <= rep["svt_min_ritz"] < tau * tau
    st_o, res, nuc = _oracle(Y, phi, prm, n)
    st_g = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    _compare(Y, st_g, st_o)
    obj = _oracle_objective(Y.astype(np.float64), phi, st_o, nuc[-1], prm)
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)


def test_rpca_partial_svd_flags_a_too_small_subspace(monkeypatch):
    """gamma = 0.4: ~125 singular values exceed tau, more than k = 16 Ritz vectors can hold;
    the report says so (smallest Ritz value > tau^2) instead of silently truncating."""
    from paper_1909_00149_b200 import inputs
    monkeypatch.setenv("UOT_RPCA_K", "16")
    Y, phi, _, _ = inputs.gen_rpca(192, 16, 16, seed=8, K=3, observed=0.9)
    prob, rep = _gpu(Y, phi, PRM, 20, check=10)
    tau = PRM["gamma"] / PRM["rho"]
    assert rep["svt_min_ritz"] > tau * tau


def test_rpca_long_video_sharded_bitwise():
    """A 150-frame video in 3 frame-range shards (subspace SVT of all 150 frames on every
    shard) is bitwise equal to the unsharded run."""
    import os
    from test_rpca_shard_gpu import _check_bitwise, _emulated
    os.environ["UOT_PERSIST"] = "0"
    try:
        from paper_1909_00149_b200 import inputs
        Y, phi, _, _ = inputs.gen_rpca(150, 8, 8, seed=21, K=2, observed=0.8)
        from test_rpca_shard_gpu import _make
        full = _make(Y, phi)
        full.solve(10, 0.0, 5)
        sh, ranges, _ = _emulated(Y, phi, (0, 50, 100), 10, 5, 0.0)
        _check_bitwise(full, sh, ranges, signed=False)
    finally:
        os.environ.pop("UOT_PERSIST", None)


@pytest.mark.parametrize("ny,nx", [(8, 8), (128, 128)], ids=["8x8", "128x128"])
def test_rpca_long_video_sharded_bitwise_frames(ny, nx):
    """The sharded runs read M from the gathered plane, the unsharded one from L + D: at 128 x 128
    (3 frame blocks x 512 pixel chunks of the line-10 apply, more CTAs than fit the GPU at once)
    the two stay bitwise equal only if line 13 (D = M - T) waits for every block's reads of M
    (k_rp_dupdate after the apply; writing D inside the apply raced with the other blocks)."""
    import os
    from test_rpca_shard_gpu import _check_bitwise, _emulated, _make
    os.environ["UOT_PERSIST"] = "0"
    try:
        from paper_1909_00149_b200 import inputs
        Y, phi, _, _ = inputs.gen_rpca(150, ny, nx, seed=23, K=2, observed=0.8)
        full = _make(Y, phi)
        full.solve(6, 0.0, 3)
        sh, ranges, _ = _emulated(Y, phi, (0, 50, 100), 6, 3, 0.0)
        _check_bitwise(full, sh, ranges, signed=False)
    finally:
        os.environ.pop("UOT_PERSIST", None)


def test_rpca_long_video_large_frames_multiwave(monkeypatch):
    """T = 160 frames of 128 x 128: the line-10 apply runs 3 frame blocks x 512 pixel chunks, more
    CTAs than fit the GPU at once, so the blocks of one pixel chunk run at different times.  Line 13
    (D = M - T) must not overwrite D before every block has read M = L + D (k_rp_dupdate runs after
    the apply); checked against the oracle's exact SVT with the subspace certificate holding."""
    from paper_1909_00149_b200 import inputs
    monkeypatch.setenv("UOT_RPCA_K", "128")      # (the noisy 128 x 128 frames keep ~100 singular values above tau)
    Y, phi, _, _ = inputs.gen_rpca(160, 128, 128, seed=12, K=3, observed=0.9)
    prm = dict(PRM, gamma=2.0)
    n = 50                     # (the one-step-per-iteration subspace tracks the SVT after the first tens)
    prob, rep = _gpu(Y, phi, prm, n, check=10)
    tau = prm["gamma"] / prm["rho"]
    assert 0.0 <= rep["svt_min_ritz"] < tau * tau
    st_o, res, nuc = _oracle(Y, phi, prm, n)
    st_g = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    _compare(Y, st_g, st_o)
    obj = _oracle_objective(Y.astype(np.float64), phi, st_o, nuc[-1], prm)
    assert rep["objective"] == pytest.approx(obj, rel=1e-4)
