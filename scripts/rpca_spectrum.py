"""Debug: spectrum of G = M^T M (M = L + D) along an RPCA+UOT-DF run on the C3 video."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import RPCAProblem
Y = torch.from_numpy(inputs.gen_c3()[0]).cuda()
prob = RPCAProblem(Y, 0.05, 0.05 * 256, 0.5, 2.0, 1.0)
tau = 0.05 * 256
for k in range(6):
    rep = prob.solve(1 if k == 0 else 40, 0.0, 1)
    st = prob.state()
    M = (st["L"] + st["D"]).double().cpu().numpy().reshape(64, -1)
    ev = np.sort(np.linalg.eigvalsh(M @ M.T))[::-1]
    print(rep["iterations"], "sweeps", rep["jacobi_sweeps"], "n>tau2", int((ev > tau**2).sum()),
          "n>tau2/2", int((ev > tau**2 / 2).sum()), "top", np.round(ev[:6], 1), "near", np.round(ev[(ev < 2*tau**2) & (ev > tau**2/4)], 1))
