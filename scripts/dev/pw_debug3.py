"""Debug: where does the wave first differ from k_iter (pass combinations)."""
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
    return p

B, T, ny, nx, alpha, rho = 2, 6, 33, 116, 0.9, 4.0
fr = inputs.gen_random(B, T, ny, nx, seed=T * 13 + nx, kind="sparse")
tau = oracle.default_steps(nx, ny, prox=True, n_frames=T, safety=0.95)[0]
base = {"UOT_PROX_WAVE": 0, "UOT_PERSIST": 0}
for chunks in ([3], [4], [5], [2, 2], [3, 1], [1, 3], [3, 2], [2, 3], [3, 3], [2, 2, 2]):
    n = sum(chunks)
    k = run(fr, alpha, rho, tau, [n], base)
    w = run(fr, alpha, rho, tau, chunks, {"UOT_PROX_CL": 2})
    msg = []
    for key in ("mx", "my", "r", "a", "x"):
        d = (w.state()[key] - k.state()[key]).abs().double().cpu().numpy()
        if d.max() > 0:
            idx = np.argwhere(d > 0)
            msg.append(f"{key}: {len(idx)} diffs max {d.max():.1e} first {idx[:4].tolist()}")
    print(chunks, "; ".join(msg) if msg else "equal")
