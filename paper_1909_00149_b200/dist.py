"""Frame-range sharding of video chains over torch.distributed.

A chain of T frames has P = T-1 pair terms (eq:RPCA_UOTDF).  Rank g
of G owns the contiguous pair range [p0, p1) and therefore frames [p0, p1];
frame p1 is the first frame of rank g+1 (the shared boundary frame).  With
fixed marginals the pairs are independent given the frames, so the
only exchange is that boundary frame, once per new set of frames: NCCL
send/recv over NVLink (gloo in the CPU tests).  Batched independent pairs
(C5) shard with no exchange at all.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_pairs: int, world: int, rank: int):
    """Contiguous, balanced pair range [p0, p1) of `rank` (sizes differ by <= 1)."""
    if not (0 <= rank < world) or n_pairs < world:
        raise ValueError(f"cannot shard {n_pairs} pairs over {world} ranks (rank {rank})")
    base, extra = divmod(n_pairs, world)
    p0 = rank * base + min(rank, extra)
    p1 = p0 + base + (1 if rank < extra else 0)
    return p0, p1


def exchange_boundary_frame(frames: torch.Tensor, rank: int, world: int, group=None):
    """frames: [1][n][ny][nx] of this rank (frames p0..p1).  Send frame 0 to
    rank-1 (its boundary frame), receive frame n-1 from rank+1.  The last rank
    owns its final frame.  Grouped P2P so neither side blocks the other."""
    if world == 1:
        return
    ops = []
    send_buf = frames[:, 0].contiguous()
    recv_buf = None
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, send_buf, rank - 1, group))
    if rank < world - 1:
        recv_buf = torch.empty_like(frames[:, -1])
        ops.append(dist.P2POp(dist.irecv, recv_buf, rank + 1, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    if recv_buf is not None:
        frames[:, -1].copy_(recv_buf)


def exchange_boundary_duals(a_first: torch.Tensor, a_last: torch.Tensor, prev_halo: torch.Tensor | None,
                            next_halo: torch.Tensor | None, rank: int, world: int, group=None, wait: bool = True):
    """Chain-prox exchange (L19): the dual of this shard's first pair goes to
    rank-1 (its next_halo), the dual of the last pair to rank+1 (its prev_halo).
    wait=False returns the works (the caller waits before the boundary pairs)."""
    if world == 1:
        return []
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, a_first.contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, prev_halo, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, a_last.contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, next_halo, rank + 1, group))
    works = dist.batch_isend_irecv(ops)
    if wait:
        for w in works:
            w.wait()
        return []
    return works


def all_reduce_report(rep: dict, device, keys=("objective", "transport", "growth", "prox_term", "upper_bound")):
    """Sum additive report fields over ranks (residual norms combine as sqrt of summed squares)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return dict(rep)
    v = [rep[k] for k in keys] + [rep["primal_res"] ** 2, (rep["dual_res"]) ** 2, rep["f_norm"] ** 2]
    t = torch.tensor(v, dtype=torch.float64, device=device)
    dist.all_reduce(t)
    out = dict(rep)
    for i, k in enumerate(keys):
        out[k] = float(t[i])
    out["primal_res"] = float(t[len(keys)].sqrt())
    out["dual_res"] = float(t[len(keys) + 1].sqrt())
    out["f_norm"] = float(t[len(keys) + 2].sqrt())
    return out


class ShardedChain:
    """Drive one rank's shard of a chain (or batch) problem (a `uot.Problem`).

    Fixed marginals: iterations have no data-path exchange -- one async
    `uot_iterate` call.  Chain prox with world > 1: every iteration k sends the
    shard's first/last pair duals a^k to the neighbours (NCCL P2P over NVLink)
    while the INTERIOR pairs of iteration k run; the two boundary pairs run
    after the receive completes (`uot_iterate_part`), so the exchange overlaps
    compute.
    """

    def __init__(self, prob, rank: int = 0, world: int = 1, group=None, overlap: bool = True):
        self.prob, self.rank, self.world, self.group, self.overlap = prob, rank, world, group, overlap
        self.exchanging = prob.prox and world > 1
        if self.exchanging and (prob.a_prev_halo is None or prob.a_next_halo is None):
            raise ValueError("chain-prox shards need Problem(..., halos=True)")

    def run(self, n_iters: int, check_every: int = 10, tol: float = 0.0) -> dict:
        from ._lib import UOT_PART_ALL, UOT_PART_BOUNDARY, UOT_PART_INTERIOR
        p = self.prob
        if not self.exchanging:
            p.iterate(n_iters, check_every=check_every, tol=tol)
            return p.report()
        for k in range(n_iters):
            red = (check_every > 0 and (k + 1) % check_every == 0) or k == n_iters - 1
            s = p.slot
            works = exchange_boundary_duals(p.a[s][:, 0], p.a[s][:, -1], p.a_prev_halo, p.a_next_halo,
                                            self.rank, self.world, self.group, wait=not self.overlap)
            if self.overlap:
                p.iterate_part(UOT_PART_INTERIOR, red)
                for w in works:
                    w.wait()
                p.iterate_part(UOT_PART_BOUNDARY, red)
            else:
                p.iterate_part(UOT_PART_ALL, red)
        return p.report()
