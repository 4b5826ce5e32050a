"""World-2 multi-process runs of the frame-range sharding
on real `Problem` contexts: `dist.ShardedChain.run` end to end in two processes.

The round-end GPU tier has ONE device, so both ranks run on cuda:0 with a gloo group; the
boundary frame, the per-iteration boundary duals (chain prox) and the 8-double stop sums go
through host copies (`dist._staged`) -- the same calls NCCL makes device to device across
GPUs.  No kernel waits on another rank's kernel (the waits are host-side), so sharing one
GPU cannot deadlock.  The sharded run must be BITWISE equal to the unsharded chain (P16):
every pair and frame is computed by the same kernel arithmetic from the same inputs.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

T, NY, NX = 9, 40, 64
ALPHA = 1.3
# the same per-pass kernels on both sides: the persistent kernels are chosen per call (a
# sharded run issues one call per check interval) and the wavefront / SMEM-tile choice
# depends on the pair count, and different kernels need not round identically
PATH_ENV = {"UOT_TPERSIST": "0", "UOT_PERSIST": "0", "UOT_WAVE": "1", "UOT_PROX_WAVE": "0"}
# the persistent SMEM-tile passes (one cooperative launch per call): the same 4 + 4 + 2 pass plan
# per check interval on both sides, so also bitwise
PATH_ENV_TP = {"UOT_TPERSIST": "1", "UOT_PERSIST": "0", "UOT_WAVE": "0", "UOT_SINGLE": "0"}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames():
    from paper_1909_00149_b200 import inputs
    return inputs.gen_random(1, T, NY, NX, seed=77, kind="sparse")


def _tau(prox):
    from paper_1909_00149_b200.uot import default_steps
    return default_steps(NX, NY, n_frames=T, rho=10.0 if prox else math.inf)[0]


def _worker(rank, world, port, mode, n, check, tol, out, env=None):
    import torch.distributed as dist
    from paper_1909_00149_b200 import dist as udist
    from paper_1909_00149_b200.uot import Problem
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.update(env or PATH_ENV)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    prox = mode == "prox"
    full = _frames()
    p0, p1 = udist.shard_range(T - 1, world, rank)
    own_hi = p1 if rank < world - 1 else p1 + 1
    fr = torch.zeros((1, p1 - p0 + 1, NY, NX), dtype=torch.float32, device="cuda")
    fr[:, : own_hi - p0].copy_(torch.from_numpy(full[:, p0:own_hi]))
    udist.exchange_boundary_frame(fr, rank, world)            # frame p1 from the next rank
    tau = _tau(prox)
    prob = Problem(fr, ALPHA, rho=10.0 if prox else math.inf, tau1=tau, tau2=tau,
                   halos=(prox and rank > 0, prox and rank < world - 1))
    rep = udist.ShardedChain(prob, rank, world).run(n, check_every=check, tol=tol)
    st = {k: v.cpu().numpy() for k, v in prob.state().items()}
    out[rank] = (p0, p1, st, rep)
    dist.destroy_process_group()


def _sharded(mode, n, check, tol, world=2, env=None):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), mode, n, check, tol, out, env), nprocs=world, join=True)
    return [out[r] for r in range(world)]


def _unsharded(mode, n, check, tol, env=None):
    from paper_1909_00149_b200.uot import Problem
    prox = mode == "prox"
    tau = _tau(prox)
    env = env or PATH_ENV
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        prob = _make(Problem, prox, tau)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    prob.iterate(n, check_every=check, tol=tol)
    rep = prob.report()
    return {k: v.cpu().numpy() for k, v in prob.state().items()}, rep


def _make(Problem, prox, tau):
    return Problem(torch.from_numpy(_frames()).cuda(), ALPHA, rho=10.0 if prox else math.inf, tau1=tau, tau2=tau)


@pytest.mark.parametrize("mode,n,check,tol,tp", [("fixed", 37, 10, 0.0, False), ("prox", 23, 5, 0.0, False),
                                                 ("fixed", 4000, 10, 1e-3, False), ("fixed", 4000, 10, 1e-3, True)])
def test_sharded_chain_world2_bitwise(mode, n, check, tol, tp):
    env = PATH_ENV_TP if tp else PATH_ENV
    full_st, full_rep = _unsharded(mode, n, check, tol, env)
    shards = _sharded(mode, n, check, tol, env=env)
    if tol > 0:
        assert full_rep["converged"] and full_rep["iterations"] < n
    for p0, p1, st, rep in shards:
        # every rank reports the global sums and the same (global) stop iteration
        assert rep["iterations"] == full_rep["iterations"]
        assert rep["converged"] == full_rep["converged"]
        for key in ("objective", "transport", "growth", "prox_term", "upper_bound", "primal_res", "dual_res",
                    "f_norm"):
            assert rep[key] == pytest.approx(full_rep[key], rel=1e-12, abs=1e-300), key
        for key in ("mx", "my", "r", "a"):
            assert np.array_equal(st[key][:, : p1 - p0], full_st[key][:, p0:p1]), key
        if mode == "prox":
            assert np.array_equal(st["x"], full_st["x"][:, p0:p1 + 1])


# ----------------------------------------------------------------------------- Algorithm 3 shards
def _rpca_video():
    g = np.random.default_rng(4)
    Y = (g.random((9, 16, 16)) * 0.3).astype(np.float32)
    Y[:, 4:8, 3:7] += 1.0
    return Y


RP = dict(lam=0.05, gamma=0.4, kappa=0.3, mu=1.5, rho=2.0)


def _rpca_make(Y, shard=None):
    from paper_1909_00149_b200.uot import RPCAProblem
    import oracle
    t = oracle.default_steps(Y.shape[2], Y.shape[1], prox=True)[0]
    return RPCAProblem(torch.from_numpy(np.ascontiguousarray(Y)).cuda(), RP["lam"], RP["gamma"], RP["kappa"], RP["mu"],
                       RP["rho"], tau1=t, tau2=t, shard=shard)


def _rpca_worker(rank, world, port, n, check, eps, out):
    import torch.distributed as dist
    from paper_1909_00149_b200 import dist as udist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["UOT_PERSIST"] = "0"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    Y = _rpca_video()
    T = Y.shape[0]
    p0, p1 = udist.shard_range(T - 1, world, rank)                 # pairs [p0, p1) -> frames [p0, p1]
    prob = _rpca_make(Y[p0:p1 + 1], shard=(p0, T))
    rep = udist.ShardedRPCA(prob, rank, world).run(n, check_every=check, eps=eps)
    out[rank] = (p0, p1, {k: v.cpu().numpy() for k, v in prob.state().items()}, rep)
    dist.destroy_process_group()


@pytest.mark.parametrize("n,check,eps", [(20, 5, 0.0), (3000, 10, 1e-3)])
def test_sharded_rpca_world2_bitwise(n, check, eps):
    old = os.environ.get("UOT_PERSIST")
    os.environ["UOT_PERSIST"] = "0"
    try:
        full = _rpca_make(_rpca_video())
    finally:
        if old is None:
            os.environ.pop("UOT_PERSIST", None)
        else:
            os.environ["UOT_PERSIST"] = old
    rf = full.solve(n, eps, check)
    fs = {k: v.cpu().numpy() for k, v in full.state().items()}
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.spawn(_rpca_worker, args=(2, _free_port(), n, check, eps, out), nprocs=2, join=True)
    for r in range(2):
        p0, p1, st, rep = out[r]
        assert rep["iterations"] == rf["iterations"] and rep["converged"] == rf["converged"]
        for key in ("objective", "data_term", "l1_term", "nuclear", "transport", "growth", "primal_res", "dual_res"):
            assert rep[key] == pytest.approx(rf[key], rel=1e-12, abs=1e-300), key
        for key in ("S", "L", "X", "Tm", "A", "D"):
            assert np.array_equal(st[key], fs[key][p0:p1 + 1]), key
        for key in ("Z", "W", "Bd", "Cd", "mx", "my", "r", "ain"):
            assert np.array_equal(st[key], fs[key][p0:p1]), key


@pytest.mark.parametrize("mode,shard", [("fixed", "ghost"), ("prox", "ghost"), ("prox", "halo")])
def test_bench_two_ranks_functional(mode, shard):
    """`bench.py --gpus 2` without a launcher re-launches itself as 2 ranks (torch.distributed.run);
    with --dist-backend gloo both share this GPU (functional check of the N > 1 bench path: frame
    shards, boundary-frame exchange, global stop, report all-reduce; chain prox with ghost pairs
    (dist.GhostChain) or per-iteration boundary duals (dist.ShardedChain); not a timing).  The
    job's objective equals the one-rank run's."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = [sys.executable, os.path.join(root, "bench.py"), "--config", "C3", "--iters", "20", "--steps", "1",
            "--warmup", "3", "--no-cpu", "--no-e2e", "--mode", mode, "--prox-shard", shard]
    env = dict(os.environ, UOT_TPERSIST="0", UOT_PERSIST="0")
    one = subprocess.run(base, capture_output=True, text=True, timeout=600, env=env)
    two = subprocess.run(base + ["--gpus", "2", "--dist-backend", "gloo"], capture_output=True, text=True,
                         timeout=600, env=env)
    assert one.returncode == 0, one.stderr[-2000:]
    assert two.returncode == 0, two.stderr[-2000:]
    l1 = json.loads([ln for ln in one.stdout.splitlines() if ln.startswith("{")][-1])
    l2 = json.loads([ln for ln in two.stdout.splitlines() if ln.startswith("{")][-1])
    assert l2["n_gpus"] == 2 and l2["iterations_per_step"] == 20
    # (the shards may select other pass kernels than the whole chain: fp32 rounding order only)
    assert l2["objective"] == pytest.approx(l1["objective"], rel=1e-5)


# ----------------------------------------------------------------------------- ghost pairs (chain prox)
def _ghost_worker(rank, world, port, passes, out):
    import torch.distributed as dist
    from paper_1909_00149_b200 import dist as udist
    from paper_1909_00149_b200.uot import Problem
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.update({"UOT_PROX_WAVE": "2", "UOT_PROX_CL": "2"})
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    full = _frames()
    p0, p1, q0, q1 = udist.ghost_range(T - 1, world, rank)
    tau = _tau(True)
    prob = Problem(torch.from_numpy(full[:, q0:q1 + 1]).cuda(), ALPHA, rho=10.0, tau1=tau, tau2=tau)
    rep = udist.GhostChain(prob, T - 1, rank, world).run(passes, check_every=10)
    st = {k: v.cpu().numpy() for k, v in prob.state().items()}
    out[rank] = (p0, p1, q0, st, rep)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ghost_chain_world_bitwise(world):
    """dist.GhostChain over `world` processes (gloo, one GPU): 3 ghost pairs per shared side,
    k_wave_prox passes of 3 / 2 iterations (20 = 3 + 3 + 2 + 2 per check of 10), the boundary
    pairs' state swapped after every pass -- every own pair and frame equals the unsharded
    chain's (the same passes) bitwise; the report is the global one."""
    n = 20
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.spawn(_ghost_worker, args=(world, _free_port(), n, out), nprocs=world, join=True)
    # the unsharded chain through the same driver (world 1: the same 3 / 2 passes, no exchange)
    from paper_1909_00149_b200 import dist as udist
    from paper_1909_00149_b200.uot import Problem
    env = {"UOT_PROX_WAVE": "2", "UOT_PROX_CL": "2"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        fp = _make(Problem, True, _tau(True))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    full_rep = udist.GhostChain(fp, T - 1, 0, 1).run(n, check_every=10)
    full_st = {k: v.cpu().numpy() for k, v in fp.state().items()}
    for r in range(world):
        p0, p1, q0, st, rep = out[r]
        for key in ("mx", "my", "r", "a"):
            assert np.array_equal(st[key][:, p0 - q0:p1 - q0], full_st[key][:, p0:p1]), (key, r)
        last = p1 + (1 if p1 == T - 1 else 0)
        assert np.array_equal(st["x"][:, p0 - q0:last - q0], full_st["x"][:, p0:last]), ("x", r)
        assert rep["iterations"] == full_rep["iterations"] == n
        for key in ("objective", "transport", "prox_term", "primal_res", "dual_res"):
            assert rep[key] == pytest.approx(full_rep[key], rel=1e-10), key
