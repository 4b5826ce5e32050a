"""k_single (uot_single.cuh): every iteration of a call on one small fixed-marginal pair in
ONE CTA, state in registers, reductions and the stopping test in-kernel (SURVEY 8(d) "K2",
config C1).  Parity against the fp64 oracle (north-star bars: 1e-3 normalised iterates, 1e-4
objective), reductions within the derived bound of test_parity_gpu.check_residuals, the
device-side stop, warm continuation, graph capture, and one launch per call."""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem

from test_parity_gpu import OBJ_RTOL, check_residuals, compare, tau_for

pytestmark = pytest.mark.gpu


def _prob(fr, alpha, tau, p_norm=1, stream=None):
    old = os.environ.get("UOT_SINGLE")
    os.environ["UOT_SINGLE"] = "1"
    try:
        return Problem(torch.from_numpy(fr).cuda(), alpha, tau1=tau, tau2=tau, p_norm=p_norm, stream=stream)
    finally:
        if old is None:
            os.environ.pop("UOT_SINGLE", None)
        else:
            os.environ["UOT_SINGLE"] = old


def _st(prob):
    return {k: v.double().cpu().numpy() for k, v in prob.state().items()}


@pytest.mark.parametrize("shape", [(64, 64), (33, 60), (1, 8), (128, 32), (7, 4), (16, 256)],
                         ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("n,check", [(40, 10), (23, 7), (1, 0)])
@pytest.mark.parametrize("alpha,p_norm", [(0.9, 1), (0.6, 2), (math.inf, 1)])
@pytest.mark.parametrize("v", ["8", "4"])
def test_single_parity(shape, n, check, alpha, p_norm, v, monkeypatch):
    monkeypatch.setenv("UOT_SINGLE_V", v)                        # 8 (nx % 8 == 0) or 4 pixels per thread
    ny, nx = shape
    fr = inputs.gen_random(1, 2, ny, nx, seed=ny * 7 + nx, kind="sparse")
    if not math.isfinite(alpha):                               # balanced: equal masses
        fr = (fr.astype(np.float64) / fr.sum(axis=(2, 3), keepdims=True) * 5.0).astype(np.float32)
    tau = tau_for(ny, nx)
    prob = _prob(fr, alpha, tau, p_norm)
    assert prob.kernel_path == "k_single"
    l0 = prob.launches
    prob.iterate(n, check_every=check)
    assert prob.launches - l0 == 1                              # one launch for the whole call
    rep = prob.report()
    ref, rrep = oracle.iterate(fr, alpha, math.inf, tau, tau, n, p_norm=p_norm)
    compare(fr, _st(prob), ref)
    obj = rrep[:, 0].sum() + (0.0 if not math.isfinite(alpha) else alpha * rrep[:, 1].sum())
    assert rep["objective"] == pytest.approx(obj, rel=OBJ_RTOL, abs=1e-6)
    assert rep["iterations"] == n
    if p_norm == 1 and math.isfinite(alpha):
        prv = _prob(fr, alpha, tau)
        prv.iterate(n - 1, check_every=check)
        st_prev = _st(prv) if n > 1 else None
        ref_prev = oracle.iterate(fr, alpha, math.inf, tau, tau, n - 1)[0] if n > 1 else None
        check_residuals(fr, _st(prob), ref, rep, rrep, tau, st_prev, ref_prev)


@pytest.mark.parametrize("check", [10, 7])
def test_single_device_stop_and_warm_continuation(check):
    fr = inputs.gen_random(1, 2, 48, 64, seed=93, kind="uniform")
    tau = tau_for(48, 64)
    prob = _prob(fr, 0.8, tau)
    rep = prob.solve(20000, tol=1e-4, check_every=check)
    assert rep["converged"] == 1
    kc = rep["iterations"]
    assert kc % check == 0 and 0 < kc < 20000
    ref, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, kc)
    compare(fr, _st(prob), ref)
    prob.step(9)
    ref2, _ = oracle.iterate(fr, 0.8, math.inf, tau, tau, kc + 9)
    compare(fr, _st(prob), ref2)


def test_single_graph_capture():
    fr = inputs.gen_random(1, 2, 40, 64, seed=8, kind="uniform")
    tau = tau_for(40, 64)
    s = torch.cuda.Stream()
    prob = _prob(fr, 1.1, tau, stream=s)
    torch.cuda.synchronize()
    prob.step(7)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        prob.step(5)                                            # odd: the capture restores the slots
    for _ in range(3):
        g.replay()
    s.synchronize()
    ref, _ = oracle.iterate(fr, 1.1, math.inf, tau, tau, 7 + 15)
    compare(fr, _st(prob), ref)


def test_single_C1_matches_other_paths():
    """C1 (configs[0]) at its 500 iterations: k_single vs the oracle and vs the one-pass kernel."""
    fr = inputs.gen_c1()
    tau = tau_for(64, 64)
    prob = _prob(fr, 0.5, tau)
    rep = prob.solve(500, tol=0.0, check_every=10)
    ref, rrep = oracle.iterate(fr, 0.5, math.inf, tau, tau, 500)
    compare(fr, _st(prob), ref)
    assert rep["objective"] == pytest.approx(rrep[0, 0] + 0.5 * rrep[0, 1], rel=OBJ_RTOL)
