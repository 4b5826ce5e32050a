"""Debug: values at the first differing pixel (chain 0, pair 0, row 16, col 77) for k_iter / wave H=17 / H=64 / oracle."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem

def run(fr, alpha, rho, tau, chunks, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        p = Problem(torch.from_numpy(fr).cuda(), alpha, rho=rho, tau1=tau, tau2=tau)
    finally:
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
    for c in chunks: p.iterate(c)
    torch.cuda.synchronize()
    return {k: v.double().cpu().numpy() for k, v in p.state().items()}

B, T, ny, nx, alpha, rho = 2, 6, 33, 116, 0.9, 4.0
fr = inputs.gen_random(B, T, ny, nx, seed=T * 13 + nx, kind="sparse")
tau = oracle.default_steps(nx, ny, prox=True, n_frames=T, safety=0.95)[0]
np.set_printoptions(precision=10, linewidth=200)
for n in (4, 5, 6):
    k = run(fr, alpha, rho, tau, [n], {"UOT_PROX_WAVE": 0, "UOT_PERSIST": 0})
    w17 = run(fr, alpha, rho, tau, [3, n - 3], {"UOT_PROX_CL": 2, "UOT_PROX_WAVE_H": 17})
    w64 = run(fr, alpha, rho, tau, [3, n - 3], {"UOT_PROX_CL": 2, "UOT_PROX_WAVE_H": 64})
    ref, _ = oracle.iterate(fr, alpha, rho, tau, tau, n)
    print("n", n)
    for key in ("mx", "my", "a", "r"):
        sl = (0, 0, 16, slice(75, 80))
        print(f"  {key} k  ", k[key][sl]); print(f"  {key} w17", w17[key][sl]); print(f"  {key} w64", w64[key][sl]); print(f"  {key} ref", getattr(ref, key)[sl])
    d = np.abs(w17["a"] - k["a"]); print("  a diffs", np.argwhere(d > 0)[:6].tolist())
    d = np.abs(w17["mx"] - k["mx"]); print("  mx diffs", np.argwhere(d > 0)[:6].tolist())
    d = np.abs(w17["x"] - k["x"]); print("  x diffs", np.argwhere(d > 0)[:6].tolist())
