import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1909_00149_b200 import inputs
from paper_1909_00149_b200.uot import Problem, default_steps
cfg = inputs.CONFIGS["C1"]
fr = torch.from_numpy(inputs.gen_c1()).cuda()
tau, _ = default_steps(64, 64, n_frames=2, rho=float("inf"))
p = Problem(fr, cfg.alpha, tau1=tau, tau2=tau)
s = torch.cuda.current_stream()
def timeit(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n): fn()
    e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
def full():
    p.reset(); p.iterate(500, check_every=10, tol=1e-12); p.report()
def noreset():
    p.iterate(500, check_every=10, tol=0.0); p.report()
def reset_only():
    p.reset()
def iter_async():
    p.iterate(500, check_every=10, tol=0.0)
print("full step us", timeit(full))
print("iterate+report (tol 0) us", timeit(noreset))
print("reset only us (async)", timeit(reset_only, 200))
print("iterate async (tol 0) us", timeit(iter_async))
