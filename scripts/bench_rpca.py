#!/usr/bin/env python
"""Per-stage timing of Algorithm 3 (RPCA+UOT-DF ADMM) on the C3 video (T = 64, 256^2) or, with
a third argument C4, on the C4 video (T = 256 frames of 1024^2: line 10 by the partial SVD of
the T > 128 path).

  python scripts/bench_rpca.py [iters] [inner_iters] [C3|C4]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_00149_b200 import inputs  # noqa: E402
from paper_1909_00149_b200.uot import RPCAProblem  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    inner = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    video = sys.argv[3] if len(sys.argv) > 3 else "C3"
    Y = torch.from_numpy(inputs.gen_c3()[0] if video == "C3" else inputs.gen_c4_frames(0, 256)[0]).cuda()
    T, ny, nx = Y.shape
    prob = RPCAProblem(Y, 0.05, 0.05 * max(Y.shape[1], Y.shape[2]), 0.5, 2.0, 1.0, inner_iters=inner)
    prob.solve(20, 0.0, 10)
    prob.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = prob.solve(iters, 0.0, 10)            # untimed stages: SVT chain overlapped with the prox
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prob.reset()
    prob.set_timing(True)                       # per-stage events serialise the two streams
    prob.solve(iters, 0.0, 10)
    st, n = prob.get_timing()
    out = {"video": video, "T": T, "ny": ny, "nx": nx, "iters": iters, "inner_iters": inner, "ms_total": ms, "us_per_iter": 1e3 * ms / iters,
           "stage_us_per_iter": {k: 1e3 * v / max(n, 1) for k, v in st.items()}, "report": rep}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
