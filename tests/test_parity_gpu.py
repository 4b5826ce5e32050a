"""GPU parity: the CUDA path (through the C-ABI) vs the float64 oracle.

Bar (BASELINE.json north star): after a fixed iteration count the objective
matches within 1e-4 relative and every iterate plane F in {Mx, My, r, a}
within 1e-3 max-abs after normalisation (L17):
    e_F = max|F_gpu - F_ref| / max(max|F_ref|, max|f|).
Both sides get the same fp32 frames (the oracle reads them as fp64) and the
same step sizes.  Expected values come only from oracle/.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem

pytestmark = pytest.mark.gpu

OBJ_RTOL = 1e-4
ITER_TOL = 1e-3


def gpu_run(frames_np, alpha, n, tau, env=None, report=True, check_every=0, p_norm=1):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = str(v)
    try:
        fr = torch.from_numpy(frames_np).cuda()
        prob = Problem(fr, alpha, tau1=tau, tau2=tau, p_norm=p_norm)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    if check_every:
        prob.iterate(n, check_every=check_every)
        rep = prob.report()
    else:
        rep = prob.step(n, report=report)
    st = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    return prob, st, rep


def compare(frames_np, st_gpu, st_ref, pairs=None, tol=ITER_TOL):
    """Normalised max-abs error per plane (L17); pairs = indices into the GPU planes."""
    B, T, ny, nx = frames_np.shape
    fr = frames_np.astype(np.float64)
    f = (fr[:, 1:] - fr[:, :-1]).reshape(-1, ny, nx)
    errs = {}
    for name in ("mx", "my", "r", "a"):
        g = st_gpu[name].reshape(-1, ny, nx)
        ref = getattr(st_ref, name).reshape(-1, ny, nx)
        if pairs is not None:
            g = g[pairs]
            f_sel = f[pairs]
        else:
            f_sel = f
        scale = max(np.abs(ref).max(), np.abs(f_sel).max())
        errs[name] = np.abs(g - ref).max() / scale
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, errs
    return errs


def _l2(st_gpu, st_ref, names):
    return math.sqrt(sum(((st_gpu[k].ravel() - getattr(st_ref, k).ravel()) ** 2).sum() for k in names))


def check_residuals(frames_np, st_n, ref_n, rep, rrep, tau, st_prev, ref_prev):
    """Primal / dual residuals of the last iteration (L13; oracle reductions pinned by P21)
    against the oracle's, within a bound DERIVED from the measured iterate error
    e = z_gpu - z_ref (not a fitted tolerance):
      primal: K_gpu - K_ref = div(e_M) - e_r - (fl32(f) - f), ||div|| <= sqrt(8)
              => |P_gpu - P_ref| <= sqrt(8)||e_M|| + ||e_r|| + 2^-24 ||f||;
      dual:   dz_gpu - dz_ref = e^n - e^(n-1) => |D_gpu - D_ref| <= (||e^n|| + ||e^(n-1)||)/tau1,
              with e^(n-1) measured on a separate (n-1)-iteration GPU run (zero at n = 1);
    plus 1e-4 relative for the GPU's fp32 partial sums (<= 512 terms per lane before fp64)."""
    fr = frames_np.astype(np.float64)
    f_norm = math.sqrt(((fr[:, 1:] - fr[:, :-1]) ** 2).sum())
    p_ref = math.sqrt(rrep[:, 2].sum())
    bound = (math.sqrt(8) * _l2(st_n, ref_n, ("mx", "my")) + _l2(st_n, ref_n, ("r",)) + 2.0 ** -24 * f_norm
             + 1e-4 * p_ref + 1e-12)
    assert abs(rep["primal_res"] - p_ref) <= bound, (rep["primal_res"], p_ref, bound)
    d_ref = math.sqrt(rrep[:, 3].sum()) / tau
    e_prev = 0.0 if st_prev is None else _l2(st_prev, ref_prev, ("mx", "my", "r"))
    bound = (_l2(st_n, ref_n, ("mx", "my", "r")) + e_prev) / tau + 1e-4 * d_ref + 1e-12
    assert abs(rep["dual_res"] - d_ref) <= bound, (rep["dual_res"], d_ref, bound)


def tau_for(ny, nx):
    return oracle.default_steps(nx, ny, prox=False, safety=0.99)[0]


# ------------------------------------------------------------------------- small / ragged / edge cases
CASES = [
    # B, T, ny, nx, alpha, iters, kind
    (1, 2, 1, 8, 0.7, 40, "uniform"),
    (1, 2, 8, 1, 0.7, 40, "uniform"),
    (1, 2, 1, 1, 0.7, 10, "uniform"),
    (1, 2, 7, 9, 1.3, 60, "sparse"),
    (2, 3, 37, 130, 2.0, 80, "sparse"),
    (1, 4, 65, 260, 0.5, 80, "uniform"),
    (3, 2, 33, 132, 1.0, 50, "signed"),
    (1, 2, 130, 516, 5.0, 60, "sparse"),
]


# path variants: one-iteration streaming kernel with lane width V and segment height H
# (UOT_PERSIST=0, UOT_TEMPORAL=0), the two-iterations-per-pass SMEM-tiled kernel k_iter2
# (UOT_TEMPORAL=1; odd tails run the streaming kernel), or the SMEM-resident persistent
# kernel (UOT_PERSIST=1, used when the grid fits)
PATHS = [dict(UOT_SINGLE=0, UOT_VEC=1, UOT_SEG_H=0, UOT_PERSIST=0, UOT_TEMPORAL=0),
         dict(UOT_SINGLE=0, UOT_VEC=1, UOT_SEG_H=4, UOT_PERSIST=0, UOT_TEMPORAL=0),
         dict(UOT_SINGLE=0, UOT_VEC=4, UOT_SEG_H=7, UOT_PERSIST=0, UOT_TEMPORAL=0),
         dict(UOT_SINGLE=0, UOT_VEC=4, UOT_SEG_H=0, UOT_PERSIST=0, UOT_TEMPORAL=0),
         dict(UOT_SINGLE=0, UOT_VEC=2, UOT_SEG_H=5, UOT_PERSIST=0, UOT_TEMPORAL=0),
         dict(UOT_SINGLE=0, UOT_PERSIST=0, UOT_TEMPORAL=1), dict(UOT_SINGLE=0, UOT_PERSIST=0, UOT_TEMPORAL=1, UOT_WAVE=1),
         dict(UOT_SINGLE=0, UOT_PERSIST=0, UOT_TEMPORAL=1, UOT_WAVE=1, UOT_T4=0),
         dict(UOT_SINGLE=0, UOT_PERSIST=0, UOT_TEMPORAL=1, UOT_WAVE=0),
         dict(UOT_SINGLE=0, UOT_PERSIST=0, UOT_TEMPORAL=1, UOT_WAVE=0, UOT_T4_TH=32, UOT_T2_WIDE=0), dict(UOT_SINGLE=0, UOT_PERSIST=1),
         dict(UOT_SINGLE=1)]


@pytest.mark.parametrize("env", PATHS, ids=lambda e: "-".join(f"{k[4:]}{v}" for k, v in e.items()))
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[:4])) + f"-a{c[4]}")
def test_parity_small(case, env):
    B, T, ny, nx, alpha, n, kind = case
    fr = inputs.gen_random(B, T, ny, nx, seed=100 + ny + nx, kind=kind)
    tau = tau_for(ny, nx)
    prob, st, rep = gpu_run(fr, alpha, n, tau, env)
    ref, rrep = oracle.iterate(fr, alpha, math.inf, tau, tau, n)
    compare(fr, st, ref)
    obj_ref = rrep[:, 0].sum() + alpha * rrep[:, 1].sum()
    assert rep["objective"] == pytest.approx(obj_ref, rel=OBJ_RTOL, abs=1e-6)
    assert rep["upper_bound"] == pytest.approx(rrep[:, 0].sum() + alpha * rrep[:, 4].sum(), rel=OBJ_RTOL, abs=1e-6)
    check_residuals(fr, st, ref, rep, rrep, tau, gpu_run(fr, alpha, n - 1, tau, env)[1] if n > 1 else None,
                    oracle.iterate(fr, alpha, math.inf, tau, tau, n - 1)[0] if n > 1 else None)
    # pinned flux components are exactly zero (L3)
    assert np.all(st["mx"][..., -1] == 0) and np.all(st["my"][..., -1, :] == 0)
    # per-pair certificate vs the oracle's
    _, rows = prob.objective(per_pair=True)
    cert = oracle.certificate(fr, ref, alpha)
    for col in (0, 2, 7):
        np.testing.assert_allclose(rows[:, col], cert[:, col], rtol=OBJ_RTOL, atol=1e-6)
    np.testing.assert_allclose(rows[:, 6], cert[:, 6], rtol=1e-3, atol=1e-5)


def test_two_delta_converges_to_closed_form():
    """alpha=2, d=3 two-delta case: GPU iterate at 4000 its matches the oracle; its
    certified bracket contains the closed form 3."""
    fr = inputs.gen_two_delta(8, 8, (3, 1), (3, 4))
    tau = tau_for(8, 8)
    prob, st, rep = gpu_run(fr, 2.0, 4000, tau)
    ref, _ = oracle.iterate(fr, 2.0, math.inf, tau, tau, 4000)
    compare(fr, st, ref)
    r, rows = prob.objective(per_pair=True)
    assert rows[0, 6] - 1e-4 <= 3.0 <= rows[0, 2] + 1e-4


# ------------------------------------------------------------------------- BASELINE configs
def _config_parity(name, frames, pairs_ref, n_iters=None):
    cfg = inputs.CONFIGS[name]
    n = n_iters or cfg.iters
    B, T, ny, nx = frames.shape
    tau = tau_for(ny, nx)
    prob, st, rep = gpu_run(frames, cfg.alpha, n, tau)
    G = B * (T - 1)
    errs = []
    obj_g = prob.objective(per_pair=True)[1]
    for g in pairs_ref:
        b, t = divmod(g, T - 1)
        sub = np.ascontiguousarray(frames[b:b + 1, t:t + 2])
        ref, rrep = oracle.iterate(sub, cfg.alpha, math.inf, tau, tau, n)
        sg = {k: v.reshape(G, ny, nx)[g:g + 1] for k, v in st.items()}
        errs.append(compare(sub, sg, ref))
        cert = oracle.certificate(sub, ref, cfg.alpha)
        assert obj_g[g, 7] == pytest.approx(cert[0, 7], rel=OBJ_RTOL), (g, obj_g[g], cert[0])
        assert obj_g[g, 2] == pytest.approx(cert[0, 2], rel=OBJ_RTOL)
    return prob, errs


def test_parity_C1():
    fr = inputs.gen_c1()
    prob, errs = _config_parity("C1", fr, [0])


def test_parity_C2():
    fr = inputs.gen_c2()
    prob, errs = _config_parity("C2", fr, [0])


def test_parity_C3_subset():
    """Full C3 launch (63 pairs, 1000 its); pairs are independent in fixed mode,
    so an oracle run on a subset of pairs is an exact check."""
    fr = inputs.gen_c3()
    prob, errs = _config_parity("C3", fr, [0, 31, 62])


@pytest.mark.slow
def test_parity_C4_subset():
    """Full C4 launch (255 pairs of 1024^2, 500 its) on one GPU; 2 pairs vs oracle."""
    fr = inputs.gen_c4()
    prob, errs = _config_parity("C4", fr, [0, 200])


def test_parity_C5_windows():
    """C5 (4096^2 pairs, 300 its) at full size: each pixel after k iterations
    depends only on inputs within Chebyshev distance k (one stencil ring per
    iteration), so the oracle on a (2k+3)^2 window (clipped at the grid edge)
    gives that pixel exactly.  Sampled pixels vs those windows."""
    cfg = inputs.CONFIGS["C5"]
    fr = inputs.gen_c5(pairs=range(2))                 # 2 pairs of the config (pairs are independent)
    B, T, ny, nx = fr.shape
    n = cfg.iters
    tau = tau_for(ny, nx)
    prob, st, rep = gpu_run(fr, cfg.alpha, n, tau)
    R = n + 2
    for (b, j, i) in [(0, 2048, 1000), (1, 5, 4090), (0, 4095, 0)]:
        j0, j1 = max(0, j - R), min(ny, j + R + 1)
        i0, i1 = max(0, i - R), min(nx, i + R + 1)
        sub = np.ascontiguousarray(fr[b:b + 1, :, j0:j1, i0:i1])
        ref, _ = oracle.iterate(sub, cfg.alpha, math.inf, tau, tau, n)
        fwin = (sub[0, 1].astype(np.float64) - sub[0, 0])
        for name in ("mx", "my", "r", "a"):
            gv = st[name][b, 0, j, i]
            rv = getattr(ref, name)[0, 0, j - j0, i - i0]
            scale = max(np.abs(getattr(ref, name)).max(), np.abs(fwin).max())
            assert abs(gv - rv) / scale <= ITER_TOL, (name, b, j, i, gv, rv)


def test_parity_C5_objective_full_grid():
    """Objective of one full 4096^2 C5 pair after 20 iterations (same launch config)."""
    cfg = inputs.CONFIGS["C5"]
    fr = inputs.gen_c5(pairs=[0])
    tau = tau_for(4096, 4096)
    prob, st, rep = gpu_run(fr, cfg.alpha, 20, tau)
    ref, rrep = oracle.iterate(fr, cfg.alpha, math.inf, tau, tau, 20)
    compare(fr, st, ref)
    assert rep["objective"] == pytest.approx(rrep[0, 0] + cfg.alpha * rrep[0, 1], rel=OBJ_RTOL)


# ------------------------------------------------------------------------- API semantics
def test_warm_start_and_determinism():
    fr = inputs.gen_random(2, 3, 40, 64, seed=5, kind="sparse")
    t = torch.from_numpy(fr).cuda()
    p1 = Problem(t, 1.5)
    p1.step(30)
    p1.step(45)
    p2 = Problem(t, 1.5)
    p2.step(75)
    for k in ("mx", "my", "r", "a"):
        assert torch.equal(p1.state()[k], p2.state()[k])
    r1 = p1.step(0, report=True)
    assert r1["iterations"] == 75


def test_solve_device_side_stop_matches_oracle():
    """uot_solve stops on the device (L13); the returned state is iterate k_c,
    and the oracle run for k_c iterations satisfies the same stopping test."""
    fr = inputs.gen_random(1, 2, 12, 16, seed=9, kind="uniform")
    tau = tau_for(12, 16)
    prob = Problem(torch.from_numpy(fr).cuda(), 0.8, tau1=tau, tau2=tau)
    tol = 1e-4
    rep = prob.solve(20000, tol=tol, check_every=10)
    assert rep["converged"] == 1 and rep["status"] == 0
    kc = rep["iterations"]
    assert kc % 10 == 0 and 0 < kc < 20000
    ref, rrep = oracle.iterate(fr, 0.8, math.inf, tau, tau, kc)
    st = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    compare(fr, st, ref)
    fn = math.sqrt(rrep[0, 6])
    assert math.sqrt(rrep[0, 2]) <= 1.5 * tol * fn
    # a solve that cannot converge reports NOT_CONVERGED with a valid state
    prob.reset()
    rep = prob.solve(20, tol=1e-12, check_every=5)
    assert rep["status"] == 3 and rep["iterations"] == 20


def test_nonfinite_is_reported():
    fr = inputs.gen_random(1, 2, 8, 8, seed=1)
    fr[0, 1, 3, 3] = np.nan
    prob = Problem(torch.from_numpy(fr).cuda(), 1.0)
    from paper_1909_00149_b200._lib import UotError
    with pytest.raises(UotError) as ei:
        prob.step(3, report=True)
    assert ei.value.code == 4


def test_load_frames_host_matches_device_frames():
    fr = inputs.gen_random(1, 3, 16, 32, seed=3)
    fr2 = inputs.gen_random(1, 3, 16, 32, seed=4)
    a = Problem(torch.from_numpy(fr).cuda(), 1.0)
    a.load_frames_host(torch.from_numpy(fr2).pin_memory())
    a.reset()
    a.step(25)
    b = Problem(torch.from_numpy(fr2).cuda(), 1.0)
    b.step(25)
    assert torch.equal(a.state()["a"], b.state()["a"])


@pytest.mark.parametrize("persist", [0, 1])
def test_persistent_and_streaming_agree_with_checks(persist):
    """Both execution paths with in-loop reductions every 7 iterations (grid barrier in
    the persistent kernel) give the oracle's iterate and last-check reductions."""
    fr = inputs.gen_random(1, 2, 96, 160, seed=77, kind="sparse")
    tau = tau_for(96, 160)
    n = 63
    prob, st, rep = gpu_run(fr, 1.7, n, tau, env={"UOT_PERSIST": persist}, check_every=7)
    ref, rrep = oracle.iterate(fr, 1.7, math.inf, tau, tau, n)
    compare(fr, st, ref)
    assert rep["iterations"] == n
    assert rep["objective"] == pytest.approx(rrep[0, 0] + 1.7 * rrep[0, 1], rel=OBJ_RTOL)


def test_persistent_solve_stops_on_device():
    fr = inputs.gen_random(1, 2, 40, 48, seed=78, kind="uniform")
    tau = tau_for(40, 48)
    old = os.environ.get("UOT_PERSIST")
    os.environ["UOT_PERSIST"] = "1"
    try:
        prob = Problem(torch.from_numpy(fr).cuda(), 0.9, tau1=tau, tau2=tau)
    finally:
        if old is None:
            os.environ.pop("UOT_PERSIST")
        else:
            os.environ["UOT_PERSIST"] = old
    rep = prob.solve(30000, tol=1e-4, check_every=10)
    assert rep["converged"] == 1
    kc = rep["iterations"]
    assert kc % 10 == 0 and kc < 30000
    ref, rrep = oracle.iterate(fr, 0.9, math.inf, tau, tau, kc)
    st = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    compare(fr, st, ref)


# ------------------------------------------------------------------------- temporal blocking (k_iter2)
# temporal variants: register wavefront (k_wave; segments of 128 / 16 / 24 rows) or SMEM
# tiles (UOT_WAVE=0; tile rows 36 / 32, 320- or 640-thread CTAs), four- or two-iteration passes
TVARS = [dict(UOT_WAVE=1, UOT_T4=1), dict(UOT_WAVE=1, UOT_T4=1, UOT_WAVE_H=16),
         dict(UOT_WAVE=1, UOT_T4=0), dict(UOT_WAVE=1, UOT_T4=0, UOT_WAVE_H=24),
         dict(UOT_WAVE=1, UOT_T4=1, UOT_PASS_COST="9,0.1,9,9"), dict(UOT_WAVE=1, UOT_T4=1, UOT_PASS_COST="1.2,9,1.26,9"),
         dict(UOT_WAVE=1, UOT_T4=1, UOT_PASS_COST="9,9,9,0.1"), dict(UOT_WAVE=1, UOT_T4=1, UOT_PASS_COST="1.2,1.2,1.3,0.1",
                                                                  UOT_WAVE_H=16),
         dict(UOT_WAVE=0, UOT_T4=1), dict(UOT_WAVE=0, UOT_T4=1, UOT_T4_TH=32, UOT_T2_WIDE=0),
         dict(UOT_WAVE=0, UOT_T4=1, UOT_T2_WIDE=1), dict(UOT_WAVE=0, UOT_T4=0), dict(UOT_WAVE=0, UOT_T4=0, UOT_T2_WIDE=0)]


@pytest.mark.parametrize("tvar", TVARS, ids=lambda e: "-".join(f"{k[4:]}{v}" for k, v in e.items()))
@pytest.mark.parametrize("n,check", [(40, 10), (41, 10), (35, 7), (12, 0), (23, 12)])
def test_temporal_matches_streaming_and_oracle(n, check, tvar):
    """S iterations per HBM pass (k_iter2<TH, S>, S = 4 and 2) give the one-iteration
    kernel's iterates (to fp32 rounding; same arithmetic per iteration) and the oracle's,
    with reductions on aligned (every 10: 4 + 4 + 2) and misaligned (every 7: two-iteration
    passes and single launches fill in) iterations and odd tails; tiles ragged in both
    directions (150 x 200 = 2.3 x 4.7 .. 12.5 tiles)."""
    fr = inputs.gen_random(2, 3, 150, 200, seed=91, kind="sparse")
    tau = tau_for(150, 200)
    _, st_s, rep_s = gpu_run(fr, 1.4, n, tau, env={"UOT_PERSIST": 0, "UOT_TEMPORAL": 0}, check_every=check)
    prob, st_t, rep_t = gpu_run(fr, 1.4, n, tau, env={"UOT_PERSIST": 0, "UOT_TEMPORAL": 1, "UOT_TPERSIST": 0, **tvar},
                                check_every=check)
    if tvar.get("UOT_WAVE", 0) == 1:
        assert prob.kernel_path == ("k_wave5" if tvar["UOT_T4"] else "k_wave2")
    else:
        assert prob.kernel_path == ("k_iter4" if tvar["UOT_T4"] else "k_iter2")
    for k in ("mx", "my", "r", "a"):
        scale = max(np.abs(st_s[k]).max(), 1e-30)
        assert np.abs(st_t[k] - st_s[k]).max() <= 1e-5 * scale, k
    ref, rrep = oracle.iterate(fr, 1.4, math.inf, tau, tau, n)
    compare(fr, st_t, ref)
    assert rep_t["iterations"] == n
    assert rep_t["objective"] == pytest.approx(rrep[:, 0].sum() + 1.4 * rrep[:, 1].sum(), rel=OBJ_RTOL)
    _, st_q, _ = gpu_run(fr, 1.4, n - 1, tau, env={"UOT_PERSIST": 0, "UOT_TEMPORAL": 1, "UOT_TPERSIST": 0, **tvar},
                         check_every=check)
    check_residuals(fr, st_t, ref, rep_t, rrep, tau, st_q, oracle.iterate(fr, 1.4, math.inf, tau, tau, n - 1)[0])
    assert rep_t["dual_res"] == pytest.approx(rep_s["dual_res"], rel=1e-3, abs=1e-6)
    assert np.all(st_t["mx"][..., -1] == 0) and np.all(st_t["my"][..., -1, :] == 0)


@pytest.mark.parametrize("check", [10, 7, 12])
def test_temporal_device_stop_replays_slots(check):
    """A device-side stop inside a run of k_iter2 passes: the returned state is iterate
    k_c (the r buffer and ping-pong slot are recovered from the launch log)."""
    fr = inputs.gen_random(1, 2, 96, 130, seed=93, kind="uniform")
    tau = tau_for(96, 130)
    old = {k: os.environ.get(k) for k in ("UOT_PERSIST", "UOT_TEMPORAL")}
    os.environ["UOT_PERSIST"], os.environ["UOT_TEMPORAL"] = "0", "1"
    try:
        prob = Problem(torch.from_numpy(fr).cuda(), 0.8, tau1=tau, tau2=tau)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    rep = prob.solve(20000, tol=1e-4, check_every=check)
    assert rep["converged"] == 1
    kc = rep["iterations"]
    assert kc % check == 0 and 0 < kc < 20000
    ref, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, kc)
    st = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    compare(fr, st, ref)
    # continuing from the recovered state (warm start) matches a fresh run of kc + 9 iterations
    prob.step(9)
    ref2, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, kc + 9)
    compare(fr, {k: v.double().cpu().numpy() for k, v in prob.state().items()}, ref2)


@pytest.mark.parametrize("follow", ["iterate", "prox_step", "objective", "solve"])
def test_pending_device_stop_is_resolved_by_the_next_call(follow):
    """uot_iterate(tol > 0) arms a device-side stop and returns without a sync; a following
    call that enqueues work (here without a uot_get_report in between) first applies the
    stop, so it continues from iterate k_c, not from the slot the host planned for n."""
    fr = inputs.gen_random(1, 2, 96, 130, seed=93, kind="uniform")
    tau = tau_for(96, 130)
    prob = Problem(torch.from_numpy(fr).cuda(), 0.8, tau1=tau, tau2=tau)
    ref_stop = Problem(torch.from_numpy(fr).cuda(), 0.8, tau1=tau, tau2=tau)
    kc = ref_stop.solve(20000, tol=1e-4, check_every=10)["iterations"]
    assert 0 < kc < 20000
    prob.iterate(20000, check_every=10, tol=1e-4)          # async: stops at kc on the device
    if follow == "iterate":
        prob.iterate(9, check_every=0)
        n_end = kc + 9
    elif follow == "prox_step":
        prob.step(9)
        n_end = kc + 9
    elif follow == "solve":
        prob.solve(9, tol=0.0, check_every=9)
        n_end = kc + 9
    else:
        prob.objective()
        n_end = kc
    rep = prob.report()
    assert rep["iterations"] == n_end
    ref, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, n_end)
    compare(fr, {k: v.double().cpu().numpy() for k, v in prob.state().items()}, ref)


def test_prox_step_report_rejected_under_capture():
    """uot_prox_step(out != NULL) needs a stream sync: refused while the stream is captured."""
    fr = inputs.gen_random(1, 2, 32, 64, seed=5, kind="uniform")
    tau = tau_for(32, 64)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        prob = Problem(torch.from_numpy(fr).cuda(), 0.8, tau1=tau, tau2=tau)
        prob.step(2)
        torch.cuda.synchronize()
        from paper_1909_00149_b200._lib import UotError
        g = torch.cuda.CUDAGraph()
        caught = []
        try:
            with torch.cuda.graph(g, stream=st):
                try:
                    prob.step(2, report=True)
                except UotError as e:
                    caught.append(e.code)
                prob.step(2)                               # the async form is capturable
        except RuntimeError:
            pass
        assert caught == [2]


def test_path_switching_keeps_the_iterate():
    """Mixing k_iter2 passes, one-pass launches and (small grid) the persistent kernel in one
    context: the ping-pong slot / r buffer bookkeeping keeps the iterate the oracle's."""
    fr = inputs.gen_random(1, 2, 100, 120, seed=95, kind="sparse")
    tau = tau_for(100, 120)
    old = os.environ.get("UOT_PERSIST")
    os.environ["UOT_PERSIST"] = "1"
    try:
        prob = Problem(torch.from_numpy(fr).cuda(), 1.2, tau1=tau, tau2=tau)
    finally:
        if old is None:
            os.environ.pop("UOT_PERSIST", None)
        else:
            os.environ["UOT_PERSIST"] = old
    assert prob.kernel_path in ("k_iter2", "k_iter4", "k_wave2", "k_wave4", "k_wave5", "k_persist", "k_tpersist")
    prob.step(7)                       # passes + an odd tail
    prob.set_temporal(False)
    path_off = prob.kernel_path
    prob.step(6)                       # persistent (the grid fits) or one-pass launches
    prob.set_temporal(True)
    prob.step(9)
    ref, _ = oracle.iterate(fr, 1.2, math.inf, tau, tau, 22)
    st = {k: v.double().cpu().numpy() for k, v in prob.state().items()}
    compare(fr, st, ref)
    assert path_off in ("k_iter", "k_persist")


# ------------------------------------------------------------------ persistent tile passes (k_tpersist)
@pytest.mark.parametrize("shape", [(1, 2, 64, 64), (2, 3, 150, 200), (1, 2, 37, 260)])
@pytest.mark.parametrize("n,check", [(40, 10), (36, 6), (20, 0), (41, 10), (30, 7)])
def test_tpersist_matches_oracle(shape, n, check):
    """All passes of a call in one cooperative launch (4-iteration passes, 2 before a check;
    even runs only -- odd ones fall back to the per-pass kernels), parity with the oracle and
    with the one-pass kernel, reductions of the checked iterations."""
    B, T, ny, nx = shape
    fr = inputs.gen_random(B, T, ny, nx, seed=7 + nx, kind="sparse")
    tau = tau_for(ny, nx)
    _, st_s, rep_s = gpu_run(fr, 1.1, n, tau, env={"UOT_PERSIST": 0, "UOT_TEMPORAL": 0}, check_every=check)
    prob, st_t, rep_t = gpu_run(fr, 1.1, n, tau, env={"UOT_SINGLE": 0, "UOT_PERSIST": 0, "UOT_TEMPORAL": 1, "UOT_TPERSIST": 1,
                                                     "UOT_WAVE": 0}, check_every=check)
    assert prob.kernel_path == "k_tpersist"
    l0 = prob.launches
    prob.iterate(8)                        # 8 iterations, reductions on the last: ONE launch
    assert prob.launches - l0 == 1
    prob.iterate(7)                        # odd: per-pass kernels
    assert prob.launches - l0 > 2
    for k in ("mx", "my", "r", "a"):
        scale = max(np.abs(st_s[k]).max(), 1e-30)
        assert np.abs(st_t[k] - st_s[k]).max() <= 1e-5 * scale, k
    ref, rrep = oracle.iterate(fr, 1.1, math.inf, tau, tau, n)
    compare(fr, st_t, ref)
    assert rep_t["iterations"] == n
    assert rep_t["objective"] == pytest.approx(rrep[:, 0].sum() + 1.1 * rrep[:, 1].sum(), rel=OBJ_RTOL)
    _, st_q, _ = gpu_run(fr, 1.1, n - 1, tau, env={"UOT_SINGLE": 0, "UOT_PERSIST": 0, "UOT_TEMPORAL": 1, "UOT_TPERSIST": 1,
                                                  "UOT_WAVE": 0}, check_every=check)
    check_residuals(fr, st_t, ref, rep_t, rrep, tau, st_q, oracle.iterate(fr, 1.1, math.inf, tau, tau, n - 1)[0])
    assert rep_t["dual_res"] == pytest.approx(rep_s["dual_res"], rel=1e-3, abs=1e-6)


@pytest.mark.parametrize("check", [10, 4])
def test_tpersist_device_stop(check):
    """Device-side stop inside a persistent launch: the stop iteration's slots are recovered
    from the replayed pass plan; a warm continuation matches a fresh run."""
    fr = inputs.gen_random(1, 2, 96, 128, seed=97, kind="uniform")
    tau = tau_for(96, 128)
    old = {k: os.environ.get(k) for k in ("UOT_PERSIST", "UOT_TPERSIST", "UOT_WAVE")}
    os.environ.update({"UOT_PERSIST": "0", "UOT_TPERSIST": "1", "UOT_WAVE": "0"})
    try:
        prob = Problem(torch.from_numpy(fr).cuda(), 0.8, tau1=tau, tau2=tau)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert prob.kernel_path == "k_tpersist"
    rep = prob.solve(20000, tol=1e-4, check_every=check)
    assert rep["converged"] == 1
    kc = rep["iterations"]
    assert kc % check == 0 and 0 < kc < 20000
    ref, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, kc)
    compare(fr, {k: v.double().cpu().numpy() for k, v in prob.state().items()}, ref)
    prob.step(10)
    ref2, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, kc + 10)
    compare(fr, {k: v.double().cpu().numpy() for k, v in prob.state().items()}, ref2)


# ------------------------------------------------------------------------- CUDA graph capture
@pytest.mark.parametrize("env", [dict(UOT_WAVE=1, UOT_TPERSIST=0, UOT_PERSIST=0),
                                 dict(UOT_WAVE=0, UOT_TPERSIST=1, UOT_PERSIST=0),
                                 dict(UOT_TEMPORAL=0, UOT_PERSIST=0)],
                         ids=["k_wave", "k_tpersist", "k_iter"])
def test_graph_capture_replays_iterations(env):
    """uot_prox_step without a report is graph-capturable (include/uot.h): capture 10
    iterations (an even number of slot flips for every pass split), replay 3 times, and the
    state is the oracle's iterate 10 + 30 (the warm-up step runs 10 before the capture)."""
    fr = inputs.gen_random(1, 3, 48, 136, seed=31, kind="sparse")
    tau = tau_for(48, 136)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        s = torch.cuda.Stream()
        prob = Problem(torch.from_numpy(fr).cuda(), 0.9, tau1=tau, tau2=tau, stream=s)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    torch.cuda.synchronize()
    prob.step(10)                                   # warm-up outside the capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        prob.step(10)
    for _ in range(3):
        g.replay()
    s.synchronize()
    ref, _ = oracle.iterate(fr, 0.9, math.inf, tau, tau, 40)
    compare(fr, {k: v.double().cpu().numpy() for k, v in prob.state().items()}, ref)


# ------------------------------------------------------------------ k_wave edge shapes
@pytest.mark.parametrize("shape", [(1, 2, 1, 8), (1, 2, 3, 4), (2, 3, 5, 116), (1, 2, 130, 228), (3, 2, 17, 240),
                                   (1, 2, 9, 56), (1, 2, 21, 60), (2, 2, 7, 64), (1, 2, 19, 68), (1, 3, 33, 256)],
                         ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("costs", ["1.155,1.15,1.137,1.35", "9,9,9,0.1"], ids=["default", "S5"])
@pytest.mark.parametrize("pk", [1, 0, "narrow"], ids=["packed", "scalar", "narrow"])
def test_wave_edge_shapes(shape, costs, pk):
    """The register wavefront on degenerate / ragged grids: one row, rows < S, one quad per
    row, widths just under / over one 112- or 120-column strip (52 / 56 / 60 for the 64-column
    strips), with 16-row segments and reductions every 10 and 7 iterations; the packed fp32x2
    kernel (k_wave_pk), the scalar k_wave and the narrow-strip k_wave_n."""
    B, T, ny, nx = shape
    fr = inputs.gen_random(B, T, ny, nx, seed=3 + ny + nx, kind="uniform")
    tau = tau_for(ny, nx)
    env = {"UOT_SINGLE": 0, "UOT_WAVE": 1, "UOT_TPERSIST": 0, "UOT_PERSIST": 0, "UOT_WAVE_H": 16, "UOT_PASS_COST": costs}
    env.update({"UOT_WAVE_PK": 1, "UOT_WAVE_V": 2} if pk == "narrow" else {"UOT_WAVE_PK": pk, "UOT_WAVE_V": 4})
    for n, check in ((30, 10), (23, 7)):
        prob, st, rep = gpu_run(fr, 1.2, n, tau, env=env, check_every=check)
        assert prob.kernel_path.startswith("k_wave")
        assert prob.wave_cols == (64 if pk == "narrow" else 128)
        ref, rrep = oracle.iterate(fr, 1.2, math.inf, tau, tau, n)
        compare(fr, st, ref)
        assert rep["iterations"] == n and np.isfinite(rep["objective"])
        assert rep["objective"] == pytest.approx(rrep[:, 0].sum() + 1.2 * rrep[:, 1].sum(), rel=OBJ_RTOL, abs=1e-6)


@pytest.mark.parametrize("shape", [(2, 3, 150, 200), (1, 3, 77, 256), (1, 2, 40, 1024)], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("costs", ["1.155,1.15,1.137,1.35", "9,9,9,0.1", "1.2,9,1.26,9", "9,0.1,9,9"],
                         ids=["default", "S5", "S3", "S4"])
def test_narrow_strips_equal_quad_strips(shape, costs):
    """k_wave_n (64-column strips, one fp32x2 pair per lane) runs k_wave_pk's arithmetic per
    pixel op for op: the iterates are EQUAL (bitwise up to the sign of zero) for every pass
    length, with reductions every 10 iterations; the reductions agree to fp32 rounding."""
    B, T, ny, nx = shape
    fr = inputs.gen_random(B, T, ny, nx, seed=11 + nx, kind="sparse")
    tau = tau_for(ny, nx)
    base = {"UOT_SINGLE": 0, "UOT_WAVE": 1, "UOT_TPERSIST": 0, "UOT_PERSIST": 0, "UOT_PASS_COST": costs}
    p4, st4, rep4 = gpu_run(fr, 0.8, 40, tau, env={**base, "UOT_WAVE_V": 4}, check_every=10)
    p2, st2, rep2 = gpu_run(fr, 0.8, 40, tau, env={**base, "UOT_WAVE_V": 2}, check_every=10)
    assert (p4.wave_cols, p2.wave_cols) == (128, 64)
    for k in ("mx", "my", "r", "a"):
        assert np.array_equal(st4[k], st2[k]), (k, np.abs(st4[k] - st2[k]).max())
    for k in ("objective", "primal_res", "dual_res"):
        assert rep2[k] == pytest.approx(rep4[k], rel=1e-5, abs=1e-9), k


def test_wave_strip_width_model():
    """The host's strip-width model (wave_cost with the measured per-pixel throughput of the
    narrow strips, 0.76 of k_wave_pk's): C3's 256-column rows and C4's 1024-column rows keep the
    128-column strips (5 x 64 computed columns vs 3 x 128 does not pay; 20 x 64 vs 9 x 128),
    136-column rows take the narrow ones (3 x 64 vs 2 x 128); include/uot.h uot_wave_cols."""
    p3 = Problem(torch.zeros((1, 64, 256, 256), device="cuda"), 0.3, tau1=0.1, tau2=0.1)
    assert p3.wave_cols == 128
    del p3
    p4 = Problem(torch.zeros((1, 256, 1024, 1024), device="cuda"), 0.3, tau1=0.1, tau2=0.1)
    assert p4.wave_cols == 128
    del p4
    p5 = Problem(torch.zeros((1, 128, 512, 136), device="cuda"), 0.3, tau1=0.1, tau2=0.1)
    assert p5.wave_cols == 64


# ------------------------------------------------------------------ randomized differential test
def test_random_pass_schedules_match_one_pass_kernel():
    """Seeded random shapes, iteration counts, check intervals, segment heights, pass splits
    and residual models (l1, p = 2, balanced): the multi-iteration passes (k_wave S = 2..5,
    SMEM tiles, persistent tiles) give the one-pass kernel's iterates to fp32 rounding and
    the same residuals."""
    rng = np.random.default_rng(int(os.environ.get("UOT_RANDOM_SEED", 2024)))
    for case in range(int(os.environ.get("UOT_RANDOM_CASES", 24))):
        B, T = int(rng.integers(1, 3)), int(rng.integers(2, 4))
        ny = int(rng.integers(1, 160))
        nx = 4 * int(rng.integers(1, 90))
        n = int(rng.integers(1, 37))
        check = int(rng.choice([0, 2, 3, 7, 10]))
        variant = int(rng.integers(0, 4))       # residual: l1 (0, 1), p = 2 (2), balanced alpha = inf (3)
        alpha = math.inf if variant == 3 else float(rng.uniform(0.3, 3.0))
        p_norm = 2 if variant == 2 else 1
        path = rng.choice(["wave", "tiles", "tpersist"])
        env = {"UOT_PERSIST": 0}
        if path == "wave":
            env.update(UOT_WAVE=1, UOT_TPERSIST=0, UOT_WAVE_H=int(rng.choice([16, 32, 64, 128])),
                       UOT_WAVE_V=int(rng.choice([0, 2, 4])),
                       UOT_PASS_COST=",".join(f"{c:.2f}" for c in rng.uniform(0.5, 2.0, 4)))
        elif path == "tiles":
            env.update(UOT_WAVE=0, UOT_TPERSIST=0)
        else:
            env.update(UOT_WAVE=0, UOT_TPERSIST=1)
        fr = inputs.gen_random(B, T, ny, nx, seed=1000 + case, kind=str(rng.choice(["uniform", "sparse"])))
        tau = tau_for(ny, nx)
        _, st_s, rep_s = gpu_run(fr, alpha, n, tau, env={"UOT_PERSIST": 0, "UOT_TEMPORAL": 0}, check_every=check,
                                 p_norm=p_norm)
        _, st_t, rep_t = gpu_run(fr, alpha, n, tau, env=env, check_every=check, p_norm=p_norm)
        for k in ("mx", "my", "r", "a"):
            scale = max(np.abs(st_s[k]).max(), 1e-30)
            err = np.abs(st_t[k] - st_s[k]).max() / scale
            assert err <= 3e-5, (case, path, env, (B, T, ny, nx, n, check), k, err)   # fp32 rounding
        assert rep_t["iterations"] == n
        if math.isfinite(rep_s["objective"]):
            assert rep_t["objective"] == pytest.approx(rep_s["objective"], rel=1e-5, abs=1e-7), (case, path, env)
        assert rep_t["primal_res"] == pytest.approx(rep_s["primal_res"], rel=1e-4, abs=1e-7), (case, path, env)
    print(f"random pass schedules: {case + 1} cases")


def test_external_stop_contract():
    """uot_stop_external / _pack / _apply (include/uot.h): apply without arming and a local
    tol while armed are refused; an armed run honours a stop set from outside (the sums of
    another 'rank' are added) at exactly the checked iteration, and uot_get_report rewinds to it."""
    from paper_1909_00149_b200._lib import UotError
    fr = inputs.gen_random(1, 3, 40, 64, seed=12, kind="uniform")
    tau = tau_for(40, 64)
    prob = Problem(torch.from_numpy(fr).cuda(), 0.8, tau1=tau, tau2=tau)
    sums = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(UotError) as e:
        prob.stop_apply(sums, 1e-3)
    assert e.value.code == 2
    prob.stop_external()
    with pytest.raises(UotError) as e:
        prob.iterate(10, check_every=10, tol=1e-3)
    assert e.value.code == 2
    # chunks of 10 with the global test; a huge tol makes the first check stop the run
    for k in range(5):
        prob.iterate(10, check_every=10, tol=0.0)
        prob.stop_pack(sums)
        sums.mul_(2.0)                                  # "all-reduce" over two identical shards
        prob.stop_apply(sums, 1e30)
    rep = prob.report()
    assert rep["converged"] == 1 and rep["iterations"] == 10
    ref, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, 10)
    compare(fr, {k: v.double().cpu().numpy() for k, v in prob.state().items()}, ref)
    rep2 = prob.solve(7, tol=0.0, check_every=7)           # disarmed: an ordinary solve continues
    assert rep2["iterations"] == 17


@pytest.mark.parametrize("env", [dict(UOT_SINGLE=0), dict(UOT_SINGLE=0, UOT_TEMPORAL=0), dict(UOT_SINGLE=1)],
                         ids=["default", "k_iter", "k_single"])
def test_checkpoint_resume_bitwise(env):
    """state_dict() after 23 iterations, load_state_dict() into a fresh problem, 17 more
    iterations == 40 uninterrupted iterations, bitwise (K^k is recomputed from the state at
    the start of every call, L8)."""
    fr = inputs.gen_random(1, 2, 48, 64, seed=41, kind="sparse")
    tau = tau_for(48, 64)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        a = Problem(torch.from_numpy(fr).cuda(), 1.2, tau1=tau, tau2=tau)
        b = Problem(torch.from_numpy(fr).cuda(), 1.2, tau1=tau, tau2=tau)
        c = Problem(torch.from_numpy(fr).cuda(), 1.2, tau1=tau, tau2=tau)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    a.step(40)
    b.step(23)
    ck = b.state_dict()
    c.load_state_dict(ck)
    c.step(17)
    for k in ("mx", "my", "r", "a"):
        assert torch.equal(a.state()[k], c.state()[k]), k
