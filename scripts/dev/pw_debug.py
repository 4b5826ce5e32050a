"""Debug: k_wave_prox vs k_iter<PROX> vs the oracle on small chains (max |diff| per plane / pair)."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem

def run(fr, alpha, rho, tau, n, env, check):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        p = Problem(torch.from_numpy(fr).cuda(), alpha, rho=rho, tau1=tau, tau2=tau)
    finally:
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
    p.iterate(n, check_every=check)
    torch.cuda.synchronize()
    return p

for (B, T, ny, nx, alpha, rho, env) in [(2, 6, 33, 116, 0.9, 4.0, {"UOT_PROX_CL": 2}), (1, 6, 33, 116, 0.9, 4.0, {"UOT_PROX_CL": 2}),
                                        (1, 6, 8, 16, 0.9, 4.0, {"UOT_PROX_CL": 2}), (1, 3, 8, 16, 0.9, 4.0, {"UOT_PROX_CL": 2})]:
    fr = inputs.gen_random(B, T, ny, nx, seed=T * 13 + nx, kind="sparse")
    tau = oracle.default_steps(nx, ny, prox=True, n_frames=T, safety=0.95)[0]
    for n in (1, 2, 4, 8, 41):
        pw = run(fr, alpha, rho, tau, n, env, 0)
        pi = run(fr, alpha, rho, tau, n, {"UOT_PROX_WAVE": 0, "UOT_PERSIST": 0}, 0)
        ref, _ = oracle.iterate(fr, alpha, rho, tau, tau, n)
        out = []
        for k in ("mx", "my", "r", "a", "x"):
            a = pw.state()[k].double().cpu().numpy(); b = pi.state()[k].double().cpu().numpy()
            d = np.abs(a - b)
            ax = tuple(range(2, d.ndim))
            per = d.max(axis=ax)
            out.append(f"{k}: {d.max():.2e} oracle(w/i) {np.abs(a - getattr(ref, k)).max():.1e}/{np.abs(b - getattr(ref, k)).max():.1e} per-pair {np.array2string(per.max(axis=0), precision=1)}")
        print((B, T, ny, nx), pw.kernel_path, "n", n)
        for o in out: print("   ", o)
        if n == 1:
            d = np.abs(pw.state()["a"].double().cpu().numpy() - pi.state()["a"].double().cpu().numpy())[0]
            idx = np.argwhere(d > 0)
            print("    first a diffs (pair,row,col):", idx[:8].tolist())
