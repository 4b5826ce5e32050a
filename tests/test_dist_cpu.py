"""Multi-process (gloo, world_size 2/3, CPU) tests of the frame-range sharding
host logic used by bench.py and the multi-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_00149_b200.dist import (all_reduce_report, exchange_boundary_duals,
                                        exchange_boundary_frame, shard_range)


@pytest.mark.parametrize("n,w", [(255, 1), (255, 2), (255, 4), (255, 8), (63, 8), (8, 8), (64, 8)])
def test_shard_range_partitions(n, w):
    seen = []
    sizes = []
    for r in range(w):
        p0, p1 = shard_range(n, w, r)
        seen.extend(range(p0, p1))
        sizes.append(p1 - p0)
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = torch.arange(T * 3 * 4, dtype=torch.float32).reshape(1, T, 3, 4)
    p0, p1 = shard_range(T - 1, world, rank)
    own_hi = p1 if rank < world - 1 else p1 + 1
    frames = torch.zeros(1, p1 - p0 + 1, 3, 4)
    frames[:, : own_hi - p0] = full[:, p0:own_hi]
    exchange_boundary_frame(frames, rank, world)
    ok_frames = torch.equal(frames, full[:, p0:p1 + 1])
    # dual halo exchange: a_first/a_last tagged by rank
    a_first = torch.full((1, 3, 4), 10.0 * rank + 1)
    a_last = torch.full((1, 3, 4), 10.0 * rank + 2)
    prev = torch.zeros(1, 3, 4)
    nxt = torch.zeros(1, 3, 4)
    exchange_boundary_duals(a_first, a_last, prev, nxt, rank, world)
    ok_prev = rank == 0 or bool(torch.all(prev == 10.0 * (rank - 1) + 2))
    ok_next = rank == world - 1 or bool(torch.all(nxt == 10.0 * (rank + 1) + 1))
    rep = {"objective": 1.0 + rank, "transport": 1.0, "growth": 0.5, "prox_term": 0.0, "upper_bound": 2.0,
           "primal_res": 3.0, "dual_res": 4.0, "f_norm": 1.0}
    tot = all_reduce_report(rep, "cpu")
    ok_rep = abs(tot["objective"] - sum(1.0 + r for r in range(world))) < 1e-12 and \
        abs(tot["primal_res"] - 3.0 * world ** 0.5) < 1e-12
    out[rank] = (ok_frames, ok_prev, ok_next, ok_rep)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 9), (3, 10)])
def test_gloo_boundary_exchange(world, T):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), T, out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == (True, True, True, True), (r, out[r])


class _StubProb:
    """The parts of uot.Problem that dist.GhostChain touches, on CPU tensors: the state of the
    ghost range of a chain whose every value encodes (plane, chain, pair / frame)."""

    def __init__(self, B, q0, q1, ny=2, nx=4):
        P = q1 - q0
        self.P = P
        self.frames = torch.zeros(B, P + 1, ny, nx)
        self.own = None
        idx = torch.arange(q0, q1, dtype=torch.float32).view(1, P, 1, 1)
        b = torch.arange(B, dtype=torch.float32).view(B, 1, 1, 1)
        self.planes = {k: (1000 * (i + 1) + 100 * b + idx).expand(B, P, ny, nx).clone() for i, k in
                       enumerate(("mx", "my", "r", "a"))}
        fidx = torch.arange(q0, q1 + 1, dtype=torch.float32).view(1, P + 1, 1, 1)
        self.planes["x"] = (9000 + 100 * b + fidx).expand(B, P + 1, ny, nx).clone()

    def set_own_pairs(self, lo, hi):
        self.own = (lo, hi)

    def state(self):
        return self.planes


def _ghost_worker(rank, world, port, n_pairs, B, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_00149_b200.dist import GhostChain, ghost_range
    p0, p1, q0, q1 = ghost_range(n_pairs, world, rank)
    prob = _StubProb(B, q0, q1)
    # ghosts start as garbage: the exchange must fill them with the neighbours' own values
    for k, t in prob.planes.items():
        lo, hi = p0 - q0, p1 - q0
        t[:, :lo] = -1.0
        t[:, (hi + 1 if k == "x" else hi):] = -1.0
    gc = GhostChain(prob, n_pairs, rank, world)
    gc.exchange()
    ok = prob.own == ((p0 - q0, p1 - q0) if world > 1 else None)
    exp = _StubProb(B, q0, q1).planes
    for k in prob.planes:
        ok = ok and torch.equal(prob.planes[k], exp[k])
    out[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_pairs,B", [(2, 19, 1), (3, 25, 2)])
def test_gloo_ghost_pair_exchange(world, n_pairs, B):
    """dist.GhostChain.exchange fills every shard's ghost pairs (3 per shared side) and ghost
    frames with the neighbours' own values (world 2 / 3, gloo); own values are untouched."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ghost_worker, args=(world, _free_port(), n_pairs, B, out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] is True, r
