"""Debug: [3,3] vs k_iter for segment heights / B / the first-differing pixel's values."""
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

for (B, T, ny, nx) in [(2, 6, 33, 116), (1, 6, 33, 116), (1, 6, 40, 64), (1, 3, 64, 128)]:
    alpha, rho = 0.9, 4.0
    fr = inputs.gen_random(B, T, ny, nx, seed=T * 13 + nx, kind="sparse")
    tau = oracle.default_steps(nx, ny, prox=True, n_frames=T, safety=0.95)[0]
    for env in ({"UOT_PROX_CL": 2, "UOT_DEBUG": 1}, {"UOT_PROX_CL": 2, "UOT_PROX_WAVE_H": 64}, {"UOT_PROX_CL": 2, "UOT_PROX_WAVE_H": 16}):
        for chunks in ([3, 3], [3, 3, 3, 3], [12], [30]):
            k = run(fr, alpha, rho, tau, [sum(chunks)], {"UOT_PROX_WAVE": 0, "UOT_PERSIST": 0})
            w = run(fr, alpha, rho, tau, chunks, env)
            msg = []
            for key in ("mx", "my", "r", "a", "x"):
                d = (w.state()[key] - k.state()[key]).abs().double().cpu().numpy()
                if d.max() > 0:
                    idx = np.argwhere(d > 0)
                    rows = sorted(set(int(i[2]) for i in idx))
                    msg.append(f"{key}: {len(idx)} max {d.max():.1e} rows {rows[:10]}")
            print((B, T, ny, nx), env.get("UOT_PROX_WAVE_H", "model"), chunks, "; ".join(msg) if msg else "equal", flush=True)
