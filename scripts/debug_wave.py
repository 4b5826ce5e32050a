# Debug helper: temporally blocked passes vs the one-pass kernel on a BASELINE config.
#   python scripts/debug_wave.py C3 16        (env: UOT_WAVE_H, UOT_PASS_COST, ...)
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem, default_steps

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
full = inputs.generate(name)
fr = torch.from_numpy(np.ascontiguousarray(full)).cuda()
B, T, ny, nx = fr.shape
cfg = inputs.CONFIGS[name]
tau, _ = default_steps(nx, ny, n_frames=T, rho=float("inf"))
res = {}
for temporal in (False, True):
    p = Problem(fr, cfg.alpha, tau1=tau, tau2=tau)
    p.set_temporal(temporal)
    p.step(n)
    torch.cuda.synchronize()
    res[temporal] = {k: v.double().cpu().numpy() for k, v in p.state().items()}
    print("temporal" if temporal else "one-pass", p.kernel_path, flush=True)
for k in res[False]:
    a, b = res[False][k], res[True][k]
    bad = ~np.isfinite(b)
    err = np.abs(np.where(bad, 0, b) - a)
    idx = np.unravel_index(np.argmax(err), err.shape)
    print(k, "nan", int(bad.sum()), "max err", float(err.max()), "at", idx, "scale", float(np.abs(a).max()))
    if bad.any():
        w = np.argwhere(bad)
        print("   first non-finite", w[:5].tolist())

# reductions: solve with checks every 10 (the bench's protocol)
p = Problem(fr, cfg.alpha, tau1=tau, tau2=tau)
for chk in (10,):
    p.reset()
    try:
        rep = p.solve(n, tol=1e-12, check_every=chk)
        print("solve ok", {k: rep[k] for k in ("objective", "primal_res", "dual_res", "iterations")})
    except Exception as ex:
        print("solve failed:", ex)
    st = {k: v.double().cpu().numpy() for k, v in p.state().items()}
    for k, v in st.items():
        print(" ", k, "non-finite", int((~np.isfinite(v)).sum()))
