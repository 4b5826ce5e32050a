"""Debug: which path differs?  k_iter V=1/2/4 vs each other, wave S=3/S=2-only, determinism."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem

def run(fr, alpha, rho, tau, n, env, step=False):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        p = Problem(torch.from_numpy(fr).cuda(), alpha, rho=rho, tau1=tau, tau2=tau)
    finally:
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
    if step:
        for _ in range(n): p.iterate(1)
    else:
        p.iterate(n)
    torch.cuda.synchronize()
    return p, p.kernel_path

def diff(p, q):
    return max(float((p.state()[k] - q.state()[k]).abs().max()) for k in ("mx", "my", "r", "a", "x"))

B, T, ny, nx, alpha, rho = 2, 6, 33, 116, 0.9, 4.0
fr = inputs.gen_random(B, T, ny, nx, seed=T * 13 + nx, kind="sparse")
tau = oracle.default_steps(nx, ny, prox=True, n_frames=T, safety=0.95)[0]
for n in (2, 3, 6, 8, 12):
    base = {"UOT_PROX_WAVE": 0, "UOT_PERSIST": 0}
    k1, _ = run(fr, alpha, rho, tau, n, {**base, "UOT_VEC": 1})
    k2, _ = run(fr, alpha, rho, tau, n, {**base, "UOT_VEC": 2})
    k4, _ = run(fr, alpha, rho, tau, n, {**base, "UOT_VEC": 4})
    kd, pd = run(fr, alpha, rho, tau, n, base)
    w3, p3 = run(fr, alpha, rho, tau, n, {"UOT_PROX_CL": 2})
    w3b, _ = run(fr, alpha, rho, tau, n, {"UOT_PROX_CL": 2})
    w1, _ = run(fr, alpha, rho, tau, n, {"UOT_PROX_CL": 1})
    ws, _ = run(fr, alpha, rho, tau, n, {"UOT_PROX_CL": 2}, step=True)     # single iterations only: k_iter
    print(f"n={n} default k_iter path {pd}: V1-V4 {diff(k1,k4):.2e} V2-V4 {diff(k2,k4):.2e} def-V4 {diff(kd,k4):.2e} | "
          f"wave {p3}: w-V4 {diff(w3,k4):.2e} w-V1 {diff(w3,k1):.2e} w-w {diff(w3,w3b):.2e} cl1-cl2 {diff(w1,w3):.2e} steps-V4 {diff(ws,k4):.2e}")
