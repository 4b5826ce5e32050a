"""Chain prox (rho < inf) on the temporally blocked path k_wave_prox (uot_wave_prox.cuh): S
Algorithm-1 iterations per HBM pass with the pairs of a group in lockstep (P:313-317, line 4 =
P:314 on the chain, L19).  Against the oracle at the north-star tolerances (L17), and against the
one-pass kernel k_iter<PROX> (same arithmetic per pixel and iteration) to fp32 rounding, over
pair groups of 1..8 CTAs (distributed-shared-memory neighbours), several groups per chain,
ragged strips and segments, fix_first, misaligned checks and the device-side stop."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem

pytestmark = pytest.mark.gpu

NO_WAVE = {"UOT_PROX_WAVE": "0"}
WAVE = {"UOT_PROX_WAVE": "2"}       # force the wave (small test chains waste more pair slots than the size rule allows)


def _run(fr, alpha, rho, tau, n, env, monkeypatch, check=0, fix_first=False, x_from_p=False):
    with monkeypatch.context() as m:
        for k, v in env.items():
            m.setenv(k, str(v))
        prob = Problem(torch.from_numpy(fr).cuda(), alpha, rho=rho, tau1=tau, tau2=tau, fix_first=fix_first,
                       reset=False)
    prob.reset(x_from_p=x_from_p)
    prob.iterate(n, check_every=check)
    rep = prob.report() if n > 0 else None
    return prob, rep


def _norm_err(fr, st, ref):
    f = np.abs(fr[:, 1:].astype(np.float64) - fr[:, :-1]).max()
    out = {}
    for name in ("mx", "my", "r", "a", "x"):
        rv = getattr(ref, name)
        scale = max(np.abs(rv).max(), f, np.abs(fr).max() if name == "x" else 0.0)
        out[name] = np.abs(st[name].double().cpu().numpy() - rv).max() / scale
    return out


# (B, T, ny, nx, alpha, rho, env): group sizes 1..8 CTAs, several groups per chain, ragged
# strips (116, 228, 240 columns) and 16-row segments
CASES = [
    (1, 2, 20, 64, 1.2, 2.0, {"UOT_PERSIST": 0}),
    (2, 6, 33, 116, 0.9, 4.0, {"UOT_PROX_CL": 2}),
    (1, 20, 24, 228, 1.5, 10.0, {"UOT_PROX_CL": 2, "UOT_PROX_WAVE_H": 16}),
    (1, 40, 18, 128, 0.8, 1.0, {"UOT_PROX_CL": 4}),
    (2, 30, 17, 240, 2.0, 3.0, {"UOT_PROX_CL": 8, "UOT_PROX_WAVE_H": 16}),
    (1, 9, 40, 36, 1.1, 5.0, {"UOT_PROX_CL": 1}),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[:4])) + "-" + "-".join(
    f"{k[4:]}{v}" for k, v in c[6].items()))
@pytest.mark.parametrize("n,check", [(41, 10), (30, 7)])
@pytest.mark.parametrize("layout", [{}, {"UOT_PROX_V": 2}, {"UOT_PROX_V": 2, "UOT_PROX_W": 16}],
                         ids=["V4W8", "V2W12", "V2W16"])
def test_prox_wave_matches_k_iter_and_oracle(case, n, check, layout, monkeypatch):
    """Every lane layout of k_wave_prox: 128-column strips with 8 pairs per CTA (default),
    64-column strips with 12 or 16."""
    B, T, ny, nx, alpha, rho, env = case
    fr = inputs.gen_random(B, T, ny, nx, seed=T * 13 + nx, kind="sparse")
    tau = oracle.default_steps(nx, ny, prox=True, n_frames=T, safety=0.95)[0]
    pw, rw = _run(fr, alpha, rho, tau, n, {**WAVE, **env, **layout}, monkeypatch, check)
    assert pw.kernel_path == "k_wave_prox"
    pi, ri = _run(fr, alpha, rho, tau, n, {**NO_WAVE, "UOT_PERSIST": 0}, monkeypatch, check)
    assert pi.kernel_path == "k_iter"
    sw, si = pw.state(), pi.state()
    for k in ("mx", "my", "r", "a", "x"):                # same arithmetic: equal up to rounding (isolated
        scale = max(float(si[k].abs().max()), 1e-30)    # 1-ulp differences at segment-edge rows)
        assert float((sw[k] - si[k]).abs().max()) <= 1e-5 * scale, k
    assert rw["iterations"] == ri["iterations"] == n
    for key in ("objective", "transport", "growth", "prox_term", "primal_res", "dual_res", "upper_bound"):
        assert rw[key] == pytest.approx(ri[key], rel=1e-5, abs=1e-9), key
    ref, rrep = oracle.iterate(fr, alpha, rho, tau, tau, n)
    errs = _norm_err(fr, sw, ref)
    assert all(v <= 1e-3 for v in errs.values()), errs
    obj = rrep[:, 0].sum() + alpha * rrep[:, 1].sum() + 0.5 * rho * rrep[:, 5].sum()
    assert rw["objective"] == pytest.approx(obj, rel=1e-4, abs=1e-6)


@pytest.mark.parametrize("T", [2, 5])
def test_prox_wave_fix_first_and_warm_x(T, monkeypatch):
    """Constant first frame and the x^0 = max(p, 0) warm start (L8)."""
    fr = inputs.gen_random(1, T, 21, 64, seed=T, kind="uniform")
    tau = oracle.default_steps(64, 21, prox=True, n_frames=T, safety=0.95, fix_first=True)[0]
    pw, rw = _run(fr, 1.3, 2.5, tau, 26, {**WAVE, "UOT_PROX_CL": 2}, monkeypatch, 10, fix_first=True, x_from_p=True)
    pi, ri = _run(fr, 1.3, 2.5, tau, 26, NO_WAVE, monkeypatch, 10, fix_first=True, x_from_p=True)
    for k in ("mx", "my", "r", "a", "x"):
        scale = max(float(pi.state()[k].abs().max()), 1e-30)
        assert float((pw.state()[k] - pi.state()[k]).abs().max()) <= 1e-5 * scale, k
    s0 = oracle.zero_state(fr, prox=True, x_from_p=True, fix_first=True)
    ref, _ = oracle.iterate(fr, 1.3, 2.5, tau, tau, 26, s0, fix_first=True)
    errs = _norm_err(fr, pw.state(), ref)
    assert all(v <= 1e-3 for v in errs.values()), errs


def test_prox_wave_device_stop(monkeypatch):
    """uot_solve with tol > 0 on the wave path stops on the device at a checked iteration and
    returns that iterate (the log replays slots and r buffers of the 4/2-iteration passes)."""
    fr = inputs.gen_random(1, 4, 12, 32, seed=4, kind="uniform")
    tau = oracle.default_steps(32, 12, prox=True, n_frames=4, safety=0.95)[0]
    with monkeypatch.context() as m:
        m.setenv("UOT_PROX_CL", "2")
        m.setenv("UOT_PROX_WAVE", "2")
        prob = Problem(torch.from_numpy(fr).cuda(), 0.9, rho=3.0, tau1=tau, tau2=tau)
    assert prob.kernel_path == "k_wave_prox"
    rep = prob.solve(20000, tol=1e-4, check_every=10)
    assert rep["converged"] == 1 and rep["status"] == 0
    kc = rep["iterations"]
    assert kc % 10 == 0 and 0 < kc < 20000
    ref, _ = oracle.iterate(fr, 0.9, 3.0, tau, tau, kc)
    errs = _norm_err(fr, prob.state(), ref)
    assert all(v <= 1e-3 for v in errs.values()), errs


def test_prox_wave_graph_capture(monkeypatch):
    """The cluster launches are graph-capturable: warm up 8 iterations, capture 8 (two
    four-iteration passes: an even number of slot flips), replay 3 times -> iterate 32."""
    fr = inputs.gen_random(1, 6, 16, 64, seed=8, kind="sparse")
    tau = oracle.default_steps(64, 16, prox=True, n_frames=6, safety=0.95)[0]
    s = torch.cuda.Stream()
    with monkeypatch.context() as m:
        m.setenv("UOT_PROX_CL", "2")
        m.setenv("UOT_PROX_WAVE", "2")
        prob = Problem(torch.from_numpy(fr).cuda(), 1.0, rho=4.0, tau1=tau, tau2=tau, stream=s)
    assert prob.kernel_path == "k_wave_prox"
    torch.cuda.synchronize()
    prob.step(8)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        prob.step(8)
    for _ in range(3):
        g.replay()
    s.synchronize()
    ref, _ = oracle.iterate(fr, 1.0, 4.0, tau, tau, 32)
    errs = _norm_err(fr, prob.state(), ref)
    assert all(v <= 1e-3 for v in errs.values()), errs


# ----------------------------------------------------------------------------- ghost pairs
def _ghost_exchange(shards):
    """What dist.GhostChain.exchange moves between neighbouring ranks, as device copies between the
    shards' Problems (one GPU): own boundary pairs (M, r, a) and frames into the neighbours' ghosts."""
    from paper_1909_00149_b200.dist import ghost_planes
    for (A, ra), (Bp, rb) in zip(shards[:-1], shards[1:]):
        S = 3
        pa, xa = ghost_planes(A)
        pb, xb = ghost_planes(Bp)
        hi = ra[1] - ra[2]                      # A's own end, local
        lo = rb[0] - rb[2]                      # B's own start, local (= S)
        for ta, tb in zip(pa, pb):
            tb[:, 0:S].copy_(ta[:, hi - S:hi])
            ta[:, hi:hi + S].copy_(tb[:, lo:lo + S])
        xb[:, 0:S].copy_(xa[:, hi - S:hi])
        xa[:, hi:hi + S + 1].copy_(xb[:, lo:lo + S + 1])


@pytest.mark.parametrize("world,B,T", [(2, 1, 20), (3, 2, 26)])
def test_ghost_pair_shards_equal_unsharded(world, B, T, monkeypatch):
    """A chain sharded by frame range with 3 ghost pairs per shared side (uot_set_own_pairs),
    passes of 3 iterations, boundary pairs' state swapped after every pass (dist.GhostChain's
    exchange, emulated by device copies): every own pair and frame equals the unsharded chain's
    bitwise, and the shards' reports add up to the unsharded one."""
    from paper_1909_00149_b200.dist import ghost_range
    fr = inputs.gen_random(B, T, 20, 128, seed=T, kind="sparse")
    tau = oracle.default_steps(128, 20, prox=True, n_frames=T, safety=0.95)[0]
    alpha, rho, passes = 1.1, 4.0, 7
    monkeypatch.setenv("UOT_PROX_WAVE", "2")
    monkeypatch.setenv("UOT_PROX_CL", "2")
    t = torch.from_numpy(fr).cuda()
    full = Problem(t, alpha, rho=rho, tau1=tau, tau2=tau)
    shards = []
    for r in range(world):
        p0, p1, q0, q1 = ghost_range(T - 1, world, r)
        pr = Problem(t[:, q0:q1 + 1].contiguous(), alpha, rho=rho, tau1=tau, tau2=tau)
        pr.set_own_pairs(p0 - q0, p1 - q0)
        shards.append((pr, (p0, p1, q0, q1)))
    for k in range(passes):
        full.iterate(3, check_every=3)
        for pr, _ in shards:
            pr.iterate(3, check_every=3)
        _ghost_exchange(shards)
    fs = full.state()
    reps = [pr.report() for pr, _ in shards]
    for (pr, (p0, p1, q0, q1)) in shards:
        st = pr.state()
        for key in ("mx", "my", "r", "a"):
            assert torch.equal(st[key][:, p0 - q0:p1 - q0], fs[key][:, p0:p1]), (key, p0, p1)
        last = p1 + (1 if p1 == T - 1 else 0)
        assert torch.equal(st["x"][:, p0 - q0:last - q0], fs["x"][:, p0:last]), ("x", p0, p1)
    rf = full.report()
    for key in ("objective", "transport", "growth", "prox_term", "upper_bound"):
        assert sum(r[key] for r in reps) == pytest.approx(rf[key], rel=1e-12), key
    for key in ("primal_res", "dual_res"):
        assert math.sqrt(sum(r[key] ** 2 for r in reps)) == pytest.approx(rf[key], rel=1e-10), key
    assert all(r["iterations"] == rf["iterations"] == 3 * passes for r in reps)


def test_ghost_pairs_reject_single_iteration_runs(monkeypatch):
    fr = inputs.gen_random(1, 14, 12, 64, seed=2, kind="sparse")
    monkeypatch.setenv("UOT_PROX_WAVE", "2")
    p = Problem(torch.from_numpy(fr).cuda(), 1.0, rho=2.0)
    p.set_own_pairs(3, 10)
    from paper_1909_00149_b200._lib import UotError
    with pytest.raises(UotError):
        p.iterate(1, check_every=0)        # a single iteration would be a k_iter pass
    with pytest.raises(UotError):
        p.set_own_pairs(5, 14)             # outside the context's 13 pairs
