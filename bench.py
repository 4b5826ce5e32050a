#!/usr/bin/env python
"""Benchmark of the fused UOT iteration (Algorithm 1, arXiv 1909.00149) on B200.

Metric (BASELINE.json): pixel-iterations/sec of the UOT prox step, with the
achieved HBM GB/s of the fused iteration kernel vs the measured peak.

A STEP is one full solve of the configured workload on this rank's pairs:
cold start (uot_reset: zero state + f = x_{t+1} - x_t, row a0) followed by the
config's iteration count of the fused kernel (rows a1-a6), residual/objective
reductions every 10 iterations evaluated on the device with the stopping test
(tol 1e-12, never met at these counts), and the report read back.
px-it per step = pairs x N x iterations actually executed.

Default workload: BASELINE configs[3] (C4: T=256 video, 1024^2, 255 pairs,
500 iterations), the HBM-bound configuration that is sharded over 1/2/4/8
GPUs; --config selects another.  Inputs (9.7 GB of state at N=1) exceed the
126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

N>1: launched by torchrun, one process per GPU; contiguous pair ranges per
rank ("strong" scaling: the config's total work is fixed); the shared
boundary frame of each shard comes from the next rank over NCCL.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# DESIGN.md "Algorithmic bytes" (fp32): fixed marginals read Mx,My,r,a,f and write Mx,My,r,a = 36 B per
# pair-pixel-iteration; chain prox adds per frame x,p read + x write = 12 B (and has no f): 32 B/pair + 12 B/frame.
def alg_bytes_per_iter(mode, G, B, T, N):
    return 36 * G * N if mode == "fixed" else (32 * G + 12 * B * T) * N
PROX_RHO = 10.0   # L15: chain-prox runs use rho = 10
METRIC = "pixel-iterations/sec of the UOT prox step; achieved HBM GB/s vs peak"
UNIT = "px-it/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--e2e-chunks", type=int, default=4,
                    help="N=1: pair ranges solved on separate streams in the e2e measurement (1 = one problem)")
    ap.add_argument("--iters", type=int, default=0, help="override the config's iteration count (testing only)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="fixed", choices=["fixed", "prox"],
                    help="fixed marginals (rho=inf) or chain prox (rho=10, per-iteration boundary-dual exchange)")
    ap.add_argument("--check-every", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--prox-shard", default="ghost", choices=["ghost", "halo"],
                    help="chain prox at N > 1: ghost pairs (k_wave_prox passes, boundary pairs' state swapped "
                         "every 3 / 2 iterations; dist.GhostChain) or one boundary dual per iteration "
                         "(k_iter passes; dist.ShardedChain)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N>1 code path with ranks sharing the visible GPUs and host-staged "
                         "exchanges (functional check on a 1-GPU box; not a performance number)")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------ helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def pair_range(n_pairs, world, rank):
    from paper_1909_00149_b200.dist import shard_range
    return shard_range(n_pairs, world, rank)


def make_frames(cfg, f0, f1, rank_chain=None):
    """Frames of chain 0 (or of the batched pairs), indices [f0, f1)."""
    from paper_1909_00149_b200 import inputs
    if cfg.name == "C4":
        return inputs.gen_c4_frames(f0, f1)
    if cfg.name == "C5":
        return inputs.gen_c5(pairs=range(f0, f1))
    full = inputs.generate(cfg.name)
    if cfg.n_chains == 1:
        return full[:, f0:f1]
    return full[f0:f1]


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index):
        self.dev = dev_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------ CPU oracle
def cpu_oracle_rate(cfg, seconds_target=12.0, rho=math.inf):
    """Oracle (oracle/, fp64 C, OpenMP over pairs) on a bounded sample of the workload.
    Returns (px-it/s, cores used, sample description)."""
    import numpy as np
    import oracle
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    n_pairs = min(cfg.n_pairs, max(2, cores))
    if cfg.n_chains == 1:
        fr = np.ascontiguousarray(make_frames(cfg, 0, n_pairs + 1))
    else:
        fr = np.ascontiguousarray(make_frames(cfg, 0, n_pairs))
    pairs = fr.shape[0] * (fr.shape[1] - 1)
    N = cfg.nx * cfg.ny
    t1 = oracle.default_steps(cfg.nx, cfg.ny, prox=math.isfinite(rho), n_frames=cfg.n_frames)[0]
    # calibrate: 2 iterations, then size the sample to ~seconds_target
    t0 = time.perf_counter()
    oracle.iterate(fr, cfg.alpha, rho, t1, t1, 2)
    dt = max(time.perf_counter() - t0, 1e-3)
    its = int(max(2, min(cfg.iters, 2 * seconds_target / dt)))
    t0 = time.perf_counter()
    oracle.iterate(fr, cfg.alpha, rho, t1, t1, its)
    dt = time.perf_counter() - t0
    threads = min(int(os.environ.get("OMP_NUM_THREADS", cores)), pairs)
    mode = "fixed marginals" if not math.isfinite(rho) else f"chain prox rho={rho}"
    sample = f"{cfg.name} ({mode}): {pairs} of {cfg.n_pairs} pairs x {N} px x {its} of {cfg.iters} iterations, fp64"
    return pairs * N * its / dt, threads, sample, dt


def lscpu_info():
    """Host CPU model / sockets / cores (BASELINE.md section 4 protocol)."""
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            k, v = k.strip(), v.strip()
            if k in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)"):
                info[k] = v
    except Exception as ex:
        info["error"] = str(ex)
    return info


def cpu_oracle_rate_1thread(cfg, seconds_target, rho):
    """The same oracle sample with OMP_NUM_THREADS=1 (OpenMP reads it at start-up, so in a
    child process).  Returns (px-it/s, sample) or (None, reason)."""
    code = ("import json, math, sys; sys.path.insert(0, %r); import bench; "
            "from paper_1909_00149_b200 import inputs; "
            "r = bench.cpu_oracle_rate(inputs.CONFIGS[%r], %r, rho=%r); print(json.dumps([r[0], r[2]]))"
            % (ROOT, cfg.name, seconds_target, rho if math.isfinite(rho) else float("inf")))
    code = code.replace("rho=inf", "rho=float('inf')")
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                             timeout=20 * seconds_target + 120)
        v, sample = json.loads(out.stdout.strip().splitlines()[-1])
        return v, sample
    except Exception as ex:
        return None, f"failed: {ex}"


# ------------------------------------------------------------------------------------------ reference arm
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    rates = []
    for k in range(args.warmup + args.steps):
        rate, threads, sample, dt = cpu_oracle_rate(cfg, seconds_target=min(args.cpu_seconds, 8.0),
                                                    rho=PROX_RHO if args.mode == "prox" else math.inf)
        if k >= args.warmup:
            rates.append((rate, dt))
    value = sum(r for r, _ in rates) / len(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(d for _, d in rates) / len(rates),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, paper_1909_00149_b200/inputs.py)",
        "config": config_dict(cfg, args.gpus, args.mode),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg, gpus, mode="fixed"):
    return {"workload": f"{cfg.name}: {cfg.note}", "B": cfg.n_chains, "T": cfg.n_frames, "pairs": cfg.n_pairs,
            "ny": cfg.ny, "nx": cfg.nx, "iterations": cfg.iters, "alpha": cfg.alpha,
            "mode": "fixed marginals (rho=inf)" if mode == "fixed" else f"chain prox (rho={PROX_RHO}, L15/L19)",
            "parallelism": f"frame-range shards x{gpus}" if gpus > 1 else "single GPU",
            "l2": "inputs larger than L2 (no flush needed)" if cfg.n_pairs * cfg.nx * cfg.ny * 36 > 126e6 * 4
            else "L2-resident workload (effective GB/s may exceed HBM peak)"}


# ------------------------------------------------------------------------------------------ main arm
def relaunch_distributed(args):
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and return its exit code; rank 0 prints the JSON line.
    NCCL's communicator-init lines go to stderr (NCCL_DEBUG=INFO, subsystem INIT) so the rank
    count of every communicator is visible in the log."""
    import socket
    import torch
    if args.dist_backend == "nccl" and torch.cuda.device_count() < args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but only {torch.cuda.device_count()} CUDA devices are visible")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    from paper_1909_00149_b200 import inputs
    cfg = inputs.CONFIGS[args.config]
    if args.iters:
        cfg = inputs.Config(**{**cfg.__dict__, "iters": args.iters})
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1909_00149_b200.uot import Problem
    from paper_1909_00149_b200 import dist as udist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and args.dist_backend == "gloo":
        dist.init_process_group("gloo")
    elif world > 1:
        # communicator-init lines (rank counts) on stderr, also when a launcher started us
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)

    # ---- this rank's shard: pairs [p0, p1) -> frames [p0, p1] (last = shared boundary frame)
    p0, p1 = udist.shard_range(cfg.n_pairs, world, rank)
    ghost = args.mode == "prox" and args.prox_shard == "ghost" and world > 1 and cfg.n_chains == 1
    if ghost:
        # chain prox with ghost pairs: frames [q0, q1] of the ghost range, all loaded from the host
        _, _, q0, q1 = udist.ghost_range(cfg.n_pairs, world, rank)
        own = make_frames(cfg, q0, q1 + 1)
        host = torch.from_numpy(np.ascontiguousarray(own))
        shape = tuple(own.shape)
    elif cfg.n_chains == 1:
        own = make_frames(cfg, p0, p1 if rank < world - 1 else p1 + 1)      # owned frames
        host = torch.from_numpy(np.ascontiguousarray(own))
        shape = (1, p1 - p0 + 1, cfg.ny, cfg.nx)
    else:
        own = make_frames(cfg, p0, p1)                                       # batched independent pairs
        host = torch.from_numpy(np.ascontiguousarray(own))
        shape = tuple(own.shape)
    host_pinned = host.pin_memory()
    frames = torch.empty(shape, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def upload(src_pinned):
        """H2D of the owned frames + boundary frame from the next rank (NCCL)."""
        n_own = src_pinned.shape[1] if cfg.n_chains == 1 else src_pinned.shape[0]
        if ghost:
            frames.copy_(src_pinned, non_blocking=True)
        elif cfg.n_chains == 1:
            frames[:, :n_own].copy_(src_pinned, non_blocking=True)
            if world > 1:
                udist.exchange_boundary_frame(frames, rank, world)
        else:
            frames.copy_(src_pinned, non_blocking=True)

    upload(host_pinned)
    torch.cuda.synchronize(dev)
    prox = args.mode == "prox"
    rho = PROX_RHO if prox else math.inf
    from paper_1909_00149_b200.uot import default_steps
    tau, _ = default_steps(cfg.nx, cfg.ny, n_frames=cfg.n_frames, rho=rho)   # global chain length (L12)
    halo = prox and world > 1 and cfg.n_chains == 1 and not ghost
    if ghost:
        os.environ.setdefault("UOT_PROX_WAVE", "2")    # ghost pairs need k_wave_prox whatever the pair-slot rule says
    prob = Problem(frames, cfg.alpha, rho=rho, tau1=tau, tau2=tau, stream=stream,
                   halos=(halo and rank > 0, halo and rank < world - 1))
    driver = udist.GhostChain(prob, cfg.n_pairs, rank, world) if ghost else udist.ShardedChain(prob, rank, world)
    G = (p1 - p0) if ghost else prob.G          # pairs this rank owns (ghost pairs are copies)
    N = cfg.nx * cfg.ny
    bytes_iter = alg_bytes_per_iter(args.mode, G, prob.B, G + 1 if ghost else prob.T, N)

    def step():
        prob.reset()
        # (ghost pairs: fixed iteration counts, tol = 0)
        return driver.run(cfg.iters, check_every=args.check_every, tol=0.0 if ghost else 1e-12)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- warm-up
    for _ in range(args.warmup):
        step()
    barrier()

    # ---- timed region (device-resident inputs)
    launches0 = prob.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters_done = 0
    reps = []
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            rep = step()
            reps.append(rep)
            iters_done += rep["iterations"]
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = prob.launches - launches0
    # per-launch kernel times (CUDA events around every launch on the launching stream) from
    # separate steps: the events serialise launches, so they stay out of the timed region above
    prob.set_timing(True)
    prob.get_timing()
    iters_timed = 0
    for _ in range(min(args.steps, 3)):
        iters_timed += step()["iterations"]
    barrier()
    by_path = prob.get_timing_paths()
    prob.set_timing(False)
    kern_ms = sum(v[0] for v in by_path.values())
    ms_max = max_over_ranks(ms)
    alg_gbs_job = sum_over_ranks(float(bytes_iter) * iters_done) / (ms_max / 1e3) / 1e9
    pxit_total = sum_over_ranks(float(G) * N * iters_done)
    value = pxit_total / (ms_max / 1e3)

    # ---- roofline of the dominant kernel (largest share of the timed launches).  Fixed
    #      marginals: one launch = one HBM pass of the state (k_iter4: four fused iterations,
    #      k_iter2: two, k_iter: one), algorithmic 36 B per pair-pixel per pass.  k_persist:
    #      per iteration.  Chain prox: per iteration (1 launch, or interior + boundary launches);
    #      k_wave_prox: per pass of 3 (2) iterations, algorithmic 44 B per pair-pixel per pass.
    peak, peak_src = load_peaks()
    alg_bytes_launch = bytes_iter
    dom = max(by_path, key=lambda k: by_path[k][0])
    dom_ms, dom_n = by_path[dom]
    if (prox and dom != "k_wave_prox") or dom in ("k_persist", "k_tpersist", "k_single"):
        avg_launch_s = (dom_ms / max(iters_timed, 1)) / 1e3
    else:
        avg_launch_s = (dom_ms / max(dom_n, 1)) / 1e3
    achieved = alg_bytes_launch / avg_launch_s / 1e9
    path = prob.kernel_path
    temporal = path in ("k_iter2", "k_iter4", "k_wave2", "k_wave4", "k_wave3", "k_wave5")
    kernel_name = {"k_wave5": "k_wave<S=5> (five fused Alg.1 iterations per HBM pass, register wavefront)",
                   "k_wave4": "k_wave<S=4> (four fused Alg.1 iterations per HBM pass, register wavefront)",
                   "k_wave3": "k_wave<S=3> (three fused Alg.1 iterations per HBM pass, register wavefront)",
                   "k_wave2": "k_wave<S=2> (two fused Alg.1 iterations per HBM pass, register wavefront)",
                   "k_iter4": "k_iter2<36, S=4> (four fused Alg.1 iterations per HBM pass, SMEM tiles)",
                   "k_iter2": "k_iter2<32, S=2> (two fused Alg.1 iterations per HBM pass, SMEM tiles)",
                   "k_persist": "k_persist (all iterations in one cooperative launch, SMEM-resident)",
                   "k_tpersist": "k_tpersist (all passes of a call in one cooperative launch, SMEM tiles)",
                   "k_single": "k_single (every iteration of a call in ONE CTA, state in registers; "
                               "SMEM/latency-bound on one SM: the HBM fraction is not meaningful)",
                   "k_wave_prox": "k_wave_prox<S=3> (chain prox: three fused Alg.1 iterations per HBM pass, "
                                  "pair groups in clusters exchanging duals by st.async)"}.get(
        dom, f"k_iter<{'prox' if prox else 'fixed'}> (fused Alg.1 iteration)")
    shares = {k: {"ms": v[0], "launches": v[1], "share": v[0] / max(kern_ms, 1e-30)} for k, v in by_path.items()}

    # ---- the one-pass kernel (one iteration per HBM pass) on the same state, for reference
    one_pass = None
    if temporal:
        n1 = 20
        prob.set_temporal(False)
        prob.set_timing(True)
        prob.get_timing()
        barrier()
        o0, o1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        o0.record(stream)
        prob.step(n1)
        o1.record(stream)
        barrier()
        k1_ms, k1_n = prob.get_timing()
        prob.set_timing(False)
        prob.set_temporal(True)
        ms1 = max_over_ranks(o0.elapsed_time(o1))
        a1 = bytes_iter / ((k1_ms / max(k1_n, 1)) / 1e3) / 1e9
        one_pass = {"kernel": "k_iter<fixed> (one Alg.1 iteration per HBM pass)", "achieved": a1, "peak": peak,
                    "unit": "GB/s", "frac": a1 / peak, "px_it_per_s": sum_over_ranks(float(G) * N * n1) / (ms1 / 1e3),
                    "iterations": n1}
    traffic = None
    ncu_dram_gbs = None
    prof_sum = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof_sum):
        try:
            key = cfg.name + (("-k_wave_prox" if dom == "k_wave_prox" else "-prox") if prox
                              else (f"-{dom}" if temporal else ""))
            d = json.load(open(prof_sum)).get(key)
            if d:
                traffic = d.get("dram_bytes_per_launch")
                m = d.get("metrics", {}).get("gpu__time_duration.sum", {})
                ncu_ms = float(m.get("value", "nan")) * {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6}.get(
                    m.get("unit", "ms"), 1.0)
                ncu_dram_gbs = traffic / (ncu_ms / 1e3) / 1e9 if traffic and ncu_ms > 0 else None
        except Exception:
            traffic = None

    # ---- e2e through the public API with HOST buffers
    e2e = None
    if not args.no_e2e:
        h2d = sum_over_ranks(float(host_pinned.numel() * 4))   # owned frames, all ranks
        # the step's result read back: the per-pair objective / certificate rows of the 255
        # evaluated regularisers (uot_objective, 8 doubles per pair) + the solve report
        d2h = sum_over_ranks(float(G * 8 * 8 + 32 * 8))

        # N = 1 or batched pairs, fixed marginals: the pairs are independent given the frames, so the
        # rank's pairs are solved as K pair-range problems on K streams and the H2D copy of
        # one range (uot_load_frames) overlaps the iterations of the others.  Chains: range
        # [q0, q1) owns frames [q0, q1] (the boundary frame is copied twice).  The work per
        # step is the single problem's (same pairs, iterations and checks).
        chunks = []
        K = min(args.e2e_chunks, G)
        # only where the copy is worth hiding: ranges of >= 16 Mpx keep every problem GPU-filling
        if (world == 1 or cfg.n_chains > 1) and not prox and K > 1 and G * N // K >= (1 << 24):
            del driver
            for i in range(K):
                q0, q1 = (G * i) // K, (G * (i + 1)) // K
                hc = (host[:, q0:q1 + 1] if cfg.n_chains == 1 else host[q0:q1]).contiguous().pin_memory()
                st_i = torch.cuda.Stream(dev)
                dfr = torch.empty(tuple(hc.shape), dtype=torch.float32, device=dev)
                dfr.copy_(hc)
                torch.cuda.synchronize(dev)
                chunks.append((Problem(dfr, cfg.alpha, rho=rho, tau1=tau, tau2=tau, stream=st_i), hc, st_i))
            h2d = sum_over_ranks(float(sum(c[1].numel() * 4 for c in chunks)))
            d2h = sum_over_ranks(float(G * 8 * 8 + 32 * 8 * K))

        def e2e_step():
            if chunks:
                for p_i, hc, st_i in chunks:    # all asynchronous: H2D, reset, iterations per range
                    p_i.load_frames_host(hc)
                    p_i.reset()
                    p_i.iterate(cfg.iters, check_every=args.check_every, tol=1e-12)
                its = min(p_i.report()["iterations"] for p_i, _, _ in chunks)
                rows = [p_i.objective(per_pair=True)[1] for p_i, _, _ in chunks]   # D2H of the result
                return {"iterations": its, "rows": sum(r.shape[0] for r in rows)}
            if world == 1:                  # the C-ABI's own H2D (uot_load_frames) from pinned host memory
                prob.load_frames_host(host_pinned)
            else:                           # owned frames + the boundary frame from the next rank (NCCL)
                upload(host_pinned)
            prob.reset()
            rep = driver.run(cfg.iters, check_every=args.check_every, tol=1e-12)
            rows = prob.objective(per_pair=True)[1]                               # D2H of the result
            return {"iterations": rep["iterations"], "rows": rows.shape[0]}

        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _, _, st_i in chunks:
            st_i.wait_event(e0)
        it2 = 0
        for _ in range(args.steps):
            it2 += e2e_step()["iterations"]
        for _, _, st_i in chunks:
            stream.wait_stream(st_i)
        e1.record(stream)
        barrier()
        ms2 = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": sum_over_ranks(float(G) * N * it2) / (ms2 / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "wall_s": time.perf_counter() - t0,
               "pipeline": f"{len(chunks)} pair ranges on {len(chunks)} streams" if chunks else "one problem"}

    # ---- CPU oracle beside it (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            rate, threads, sample, _ = cpu_oracle_rate(cfg, args.cpu_seconds, rho=rho)
            r1, s1 = cpu_oracle_rate_1thread(cfg, max(2.0, args.cpu_seconds / 3), rho)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                   "one_thread": {"value": r1, "unit": UNIT, "cores": 1, "sample": s1},
                   "host": lscpu_info(), "gpu_over_cpu": value / rate if rate else None}
        except Exception as ex:   # the oracle is a reported baseline, not the product
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        last = reps[-1]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generators, paper_1909_00149_b200/inputs.py; no dataset in the paper's bench)",
            "config": config_dict(cfg, world, args.mode),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         # SURVEY 8(d)'s three numbers: px-it/s (value), algorithmic GB/s (achieved), and
                         # ncu DRAM GB/s of the stored capture (cold, serialised launch at ncu's clock)
                         "ncu_dram_gbs": ncu_dram_gbs,
                         "frac_of_spec_8tbs": achieved / 8000.0,
                         "kernel": kernel_name,
                         "alg_bytes_per_launch": alg_bytes_launch, "avg_launch_ms": avg_launch_s * 1e3,
                         "launches_timed": dom_n, "kernels_in_step": shares, "peak_source": peak_src,
                         "traffic_source": "profiles/ncu_summary.json: dram__bytes_read.sum + dram__bytes_write.sum "
                                           "per launch from an ncu --set full capture of this kernel on this config "
                                           "(stored, not measured in this run)" if traffic else None},
            "one_pass_kernel": one_pass,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            # one-pass-equivalent ALGORITHMIC bandwidth of the whole step (36 B per px-it, as if every
            # iteration were its own HBM pass): a rate, not a DRAM measurement -- it exceeds the HBM
            # peak because the passes fuse up to five iterations; see roofline for the DRAM side
            "alg_equiv_gbs_step": alg_gbs_job,
            "dram_bytes_per_step_est": (traffic * dom_n / max(min(args.steps, 3), 1)) if traffic else None,
            "objective": last["objective"], "iterations_per_step": iters_done // args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
