#!/usr/bin/env python
"""Host enqueue cost of one chain-prox iteration of dist.ShardedChain (interior + boundary
launches through the C-ABI, the Python loop) against its device time, for a C4 shard at
G = 8 ranks (32 pairs of 1024^2).  The NCCL batch_isend_irecv of the boundary duals is not
included (one GPU here); the loop keeps the device busy while host time < device time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1909_00149_b200 import inputs  # noqa: E402
from paper_1909_00149_b200._lib import UOT_PART_BOUNDARY, UOT_PART_INTERIOR  # noqa: E402
from paper_1909_00149_b200.uot import Problem, default_steps  # noqa: E402

fr = torch.from_numpy(inputs.gen_c4_frames(0, 33)).cuda()          # one rank's 32 pairs (+ boundary frame)
tau = default_steps(1024, 1024, n_frames=256, rho=10.0)[0]
p = Problem(fr, 2.0, rho=10.0, tau1=tau, tau2=tau, halos=(True, True))
n = 200
for _ in range(20):
    p.iterate_part(UOT_PART_INTERIOR, False)
    p.iterate_part(UOT_PART_BOUNDARY, False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for k in range(n):
    red = (k + 1) % 10 == 0
    p.iterate_part(UOT_PART_INTERIOR, red)
    p.iterate_part(UOT_PART_BOUNDARY, red)
t_host = time.perf_counter() - t0
e1.record()
torch.cuda.synchronize()
out = {"iterations": n, "host_us_per_iter": 1e6 * t_host / n, "device_us_per_iter": 1e3 * e0.elapsed_time(e1) / n,
       "pairs": p.G, "note": "host = enqueue of the interior + boundary launches (C-ABI via ctypes) in the Python loop"}
print(json.dumps(out))
