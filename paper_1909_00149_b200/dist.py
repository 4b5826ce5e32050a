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
from torch.cuda import nvtx


def shard_range(n_pairs: int, world: int, rank: int):
    """Contiguous, balanced pair range [p0, p1) of `rank` (sizes differ by <= 1)."""
    if not (0 <= rank < world) or n_pairs < world:
        raise ValueError(f"cannot shard {n_pairs} pairs over {world} ranks (rank {rank})")
    base, extra = divmod(n_pairs, world)
    p0 = rank * base + min(rank, extra)
    p1 = p0 + base + (1 if rank < extra else 0)
    return p0, p1


def _staged(t: torch.Tensor, group=None) -> bool:
    """gloo has no CUDA point-to-point: device tensors go through host copies (the CPU
    multi-process tests run two ranks on one device this way).  NCCL moves them directly."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def _p2p(sends, recvs, group=None):
    """Grouped point-to-point: sends = [(tensor, peer)], recvs = [(tensor, peer)] (filled in
    place).  Returns the works; staged (gloo) transfers complete before returning."""
    if not sends and not recvs:
        return []
    probe = (sends or recvs)[0][0]
    if _staged(probe, group):
        ops, fix = [], []
        for t, peer in sends:
            ops.append(dist.P2POp(dist.isend, t.detach().cpu().contiguous(), peer, group))
        for t, peer in recvs:
            h = torch.empty(t.shape, dtype=t.dtype)
            ops.append(dist.P2POp(dist.irecv, h, peer, group))
            fix.append((t, h))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        for t, h in fix:
            t.copy_(h)
        return []
    ops = [dist.P2POp(dist.isend, t.contiguous(), peer, group) for t, peer in sends]
    ops += [dist.P2POp(dist.irecv, t, peer, group) for t, peer in recvs]
    return dist.batch_isend_irecv(ops)


def all_reduce_sum_(t: torch.Tensor, group=None):
    """In-place sum over ranks (NCCL on the current stream; gloo through a host copy)."""
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


def exchange_boundary_frame(frames: torch.Tensor, rank: int, world: int, group=None):
    """frames: [1][n][ny][nx] of this rank (frames p0..p1).  Send frame 0 to
    rank-1 (its boundary frame), receive frame n-1 from rank+1.  The last rank
    owns its final frame.  Grouped P2P so neither side blocks the other."""
    if world == 1:
        return
    recv_buf = torch.empty_like(frames[:, -1]) if rank < world - 1 else None
    works = _p2p([(frames[:, 0].contiguous(), rank - 1)] if rank > 0 else [],
                 [(recv_buf, rank + 1)] if recv_buf is not None else [], group)
    for w in works:
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
    sends, recvs = [], []
    if rank > 0:
        sends.append((a_first, rank - 1))
        recvs.append((prev_halo, rank - 1))
    if rank < world - 1:
        sends.append((a_last, rank + 1))
        recvs.append((next_halo, rank + 1))
    works = _p2p(sends, recvs, group)
    if wait:
        for w in works:
            w.wait()
        return []
    return works


def all_reduce_report(rep: dict, device, keys=("objective", "transport", "growth", "prox_term", "upper_bound"),
                      group=None):
    """Sum additive report fields over ranks (residual norms combine as sqrt of summed squares)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return dict(rep)
    v = [rep[k] for k in keys] + [rep["primal_res"] ** 2, (rep["dual_res"]) ** 2, rep["f_norm"] ** 2]
    t = torch.tensor(v, dtype=torch.float64, device=device)
    all_reduce_sum_(t, group)
    out = dict(rep)
    for i, k in enumerate(keys):
        out[k] = float(t[i])
    out["primal_res"] = float(t[len(keys)].sqrt())
    out["dual_res"] = float(t[len(keys) + 1].sqrt())
    out["f_norm"] = float(t[len(keys) + 2].sqrt())
    return out


class ShardedChain:
    """Drive one rank's shard of a chain (or batch) problem (a `uot.Problem`).

    Fixed marginals: iterations have no data-path exchange.  Chain prox with world > 1:
    every iteration k sends the shard's first/last pair duals a^k to the neighbours (NCCL
    P2P over NVLink) while the INTERIOR pairs of iteration k run; the two boundary pairs run
    after the receive completes (`uot_iterate_part`), so the exchange overlaps compute.

    Stopping (L13) with world > 1 is GLOBAL: the residuals and ||f|| of every shard are
    summed before the test, so all ranks stop at the same checked iteration.  The run arms
    the C-ABI's external stop once, and at every checked iteration packs this shard's sums
    (uot_stop_pack), all-reduces them (8 doubles, on the stream) and applies the test
    (uot_stop_apply) -- no host synchronisation inside the run.  run() returns the report
    summed over ranks (all_reduce_report).  World 1: the device-side test of uot_iterate.
    """

    def __init__(self, prob, rank: int = 0, world: int = 1, group=None, overlap: bool = True):
        self.prob, self.rank, self.world, self.group, self.overlap = prob, rank, world, group, overlap
        self.exchanging = prob.prox and world > 1
        if self.exchanging and ((rank > 0) != (prob.a_prev_halo is not None) or
                                (rank < world - 1) != (prob.a_next_halo is not None)):
            raise ValueError("chain-prox shards need Problem(..., halos=(rank > 0, rank < world - 1))")
        self._sums = None

    def _global_check(self, tol):
        nvtx.range_push("global_stop_check")
        self._global_check_(tol)
        nvtx.range_pop()

    def _global_check_(self, tol):
        p = self.prob
        if self._sums is None:
            self._sums = torch.zeros(8, dtype=torch.float64, device=p.frames.device)
        p.stop_pack(self._sums)
        all_reduce_sum_(self._sums, self.group)
        p.stop_apply(self._sums, tol)

    def run(self, n_iters: int, check_every: int = 10, tol: float = 0.0) -> dict:
        from ._lib import UOT_PART_ALL, UOT_PART_BOUNDARY, UOT_PART_INTERIOR
        p = self.prob
        if self.world == 1:
            p.iterate(n_iters, check_every=check_every, tol=tol)
            return p.report()
        p.stop_external()
        ce = check_every if check_every > 0 else max(n_iters, 1)
        if not self.exchanging:
            k = 0
            while k < n_iters:
                d = min(ce - k % ce, n_iters - k)
                p.iterate(d, check_every=d, tol=0.0)          # reductions on the chunk's last iteration
                k += d
                self._global_check(tol)
        else:
            for k in range(n_iters):
                red = (k + 1) % ce == 0 or k == n_iters - 1
                s = p.slot
                nvtx.range_push("exchange_boundary_duals")
                works = exchange_boundary_duals(p.a[s][:, 0], p.a[s][:, -1], p.a_prev_halo, p.a_next_halo,
                                                self.rank, self.world, self.group, wait=not self.overlap)
                nvtx.range_pop()
                if self.overlap:
                    p.iterate_part(UOT_PART_INTERIOR, red)
                    for w in works:
                        w.wait()
                    p.iterate_part(UOT_PART_BOUNDARY, red)
                else:
                    p.iterate_part(UOT_PART_ALL, red)
                if red:
                    self._global_check(tol)
        return all_reduce_report(p.report(), p.frames.device, group=self.group)


class ShardedRPCA:
    """Drive one rank's frame-range shard of Algorithm 3 (RPCA+UOT-DF; a
    `uot.RPCAProblem(..., shard=(frame0, T_total))`), SURVEY 8(f) NEXT(3).

    Per ADMM iteration (stream-ordered, no host synchronisation; NCCL over NVLink):
      uot_rpca_iterate_pre   lines 5-9, 12 and line 11's centres on this shard's frames
                             (the halo frame too); M = L + D of its OWNED frames into mgather
      all-reduce(mgather)    line 10 needs the Gram matrix of every frame: the shards' disjoint
                             rows sum exactly (Tg x N floats)
      uot_rpca_iterate_post  line 10 (Gram + eigen-decomposition of all Tg frames, redundant per
                             rank; T = M W for this shard's frames), line 11 (T-1 independent pair
                             proxes), lines 13-15
      boundary exchange      (z, b) of the first pair -> previous rank, (w, c) of the last pair ->
                             next rank: the only per-iteration coupling of line 11's pairs
                             (lines 5-7 of the shared frame read both neighbours' pairs)
      at checked iterations  8 partial sums all-reduced, L28 test on the global sums (every rank
                             stops at the same iteration)
    run() returns the report with the additive terms summed over ranks.
    """

    def __init__(self, prob, rank: int = 0, world: int = 1, group=None):
        if (rank > 0) != prob.has_prev or (rank < world - 1) != prob.has_next:
            raise ValueError("RPCAProblem shard does not match the rank's position")
        self.prob, self.rank, self.world, self.group = prob, rank, world, group
        self._sums = None

    def _exchange(self):
        p = self.prob
        first, last = p.boundary_planes()
        sends, recvs = [], []
        chains = len(first)
        if self.rank > 0:
            for c in range(chains):
                sends += [(first[c][0], self.rank - 1), (first[c][1], self.rank - 1)]
                recvs += [(p.halo_prev[c, 0], self.rank - 1), (p.halo_prev[c, 1], self.rank - 1)]
        if self.rank < self.world - 1:
            for c in range(chains):
                sends += [(last[c][0], self.rank + 1), (last[c][1], self.rank + 1)]
                recvs += [(p.halo_next[c, 0], self.rank + 1), (p.halo_next[c, 1], self.rank + 1)]
        for w in _p2p(sends, recvs, self.group):
            w.wait()

    def run(self, n_iters: int, check_every: int = 10, eps: float = 0.0) -> dict:
        p = self.prob
        if self.world == 1 and p.mgather is None:
            return p.solve(n_iters, eps=eps, check_every=check_every)
        if self._sums is None:
            self._sums = torch.zeros(8, dtype=torch.float64, device=p.Y.device)
        p.stop_external()
        ce = max(int(check_every), 1)
        for k in range(n_iters):
            red = (k + 1) % ce == 0 or k == n_iters - 1
            p.iterate_pre(red)
            nvtx.range_push("allreduce_mgather")
            all_reduce_sum_(p.mgather, self.group)
            nvtx.range_pop()
            p.iterate_post(red)
            if self.world > 1:
                nvtx.range_push("exchange_boundary_pairs")
                self._exchange()
                nvtx.range_pop()
            if red:
                p.stop_pack(self._sums)
                all_reduce_sum_(self._sums, self.group)
                p.stop_apply(self._sums, eps)
        rep = p.get_report()
        if self.world > 1:
            keys = ("data_term", "l1_term", "transport", "growth")
            t = torch.tensor([rep[k] for k in keys] + [rep["primal_res"] ** 2, rep["dual_res"] ** 2],
                             dtype=torch.float64, device=p.Y.device)
            all_reduce_sum_(t, self.group)
            for i, k in enumerate(keys):
                rep[k] = float(t[i])
            rep["primal_res"], rep["dual_res"] = float(t[4].sqrt()), float(t[5].sqrt())
            rep["objective"] = rep["data_term"] + rep["l1_term"] + p._p.gamma * rep["nuclear"] + \
                p._p.kappa * (rep["transport"] + rep["growth"])
        return rep


# ----------------------------------------------------------------------------- ghost pairs
def ghost_range(n_pairs: int, world: int, rank: int, S: int = 3):
    """Chain prox with ghost pairs: rank owns pairs [p0, p1) (shard_range) and holds pairs
    [q0, q1) = [p0 - S, p1 + S) clipped to the chain (frames q0 .. q1) in its context."""
    p0, p1 = shard_range(n_pairs, world, rank)
    return p0, p1, max(0, p0 - S), min(n_pairs, p1 + S)


def ghost_planes(prob):
    """The current state planes of a Problem: [mx, my, r, a] ([B][P][ny][nx]) and x ([B][T][ny][nx])."""
    st = prob.state()
    return [st["mx"], st["my"], st["r"], st["a"]], st["x"]


class GhostChain:
    """Chain prox (rho < inf) over frame-range shards with S GHOST pairs per shared side, on the
    temporally blocked kernel (k_wave_prox, DESIGN.md §6/§8).

    Rank r owns pairs [p0, p1) and keeps copies of the S pairs (and S + 1 frames) on each side
    that a pass of S iterations reads (the dependency cone: after S iterations a pair is exact
    iff its S neighbours on both sides were); `uot_set_own_pairs` makes the kernel write and
    reduce only the own pairs.  After every pass the shards swap their S boundary pairs' full
    state (M, r, a and the frames x): 4 S planes + S (+1) frames per side every S iterations,
    instead of one dual plane per iteration (ShardedChain).  NCCL P2P (gloo through host copies
    in the CPU tests); the reports of checked passes are summed over ranks.  tol = 0 only.
    """

    def __init__(self, prob, n_pairs: int, rank: int = 0, world: int = 1, group=None, S: int = 3):
        self.prob, self.rank, self.world, self.group, self.S = prob, rank, world, group, S
        self.p0, self.p1, self.q0, self.q1 = ghost_range(n_pairs, world, rank, S)
        if prob.P != self.q1 - self.q0:
            raise ValueError(f"context holds {prob.P} pairs, the ghost range [{self.q0}, {self.q1}) needs "
                             f"{self.q1 - self.q0}")
        if world > 1:
            prob.set_own_pairs(self.p0 - self.q0, self.p1 - self.q0)

    def exchange(self):
        """Swap the boundary pairs' state with the neighbours (after a pass)."""
        if self.world == 1:
            return
        S, lo, hi = self.S, self.p0 - self.q0, self.p1 - self.q0
        planes, x = ghost_planes(self.prob)
        sends, recvs = [], []
        if self.rank > 0:       # own pairs [lo, lo+S) and frames [lo, lo+S] -> left; ghosts [0, S), frames [0, S) <- left
            for t in planes:
                sends.append((t[:, lo:lo + S].contiguous(), self.rank - 1))
                recvs.append((t[:, 0:S], self.rank - 1))
            sends.append((x[:, lo:lo + S + 1].contiguous(), self.rank - 1))
            recvs.append((x[:, 0:S], self.rank - 1))
        if self.rank < self.world - 1:   # own pairs [hi-S, hi), frames [hi-S, hi) -> right; ghosts, frames [hi, hi+S] <- right
            for t in planes:
                sends.append((t[:, hi - S:hi].contiguous(), self.rank + 1))
                recvs.append((t[:, hi:hi + S], self.rank + 1))
            sends.append((x[:, hi - S:hi].contiguous(), self.rank + 1))
            recvs.append((x[:, hi:hi + S + 1], self.rank + 1))
        bufs = [(torch.empty_like(dst), dst) for dst, _ in recvs]
        works = _p2p(sends, [(b, peer) for (b, _), (_, peer) in zip(bufs, recvs)], self.group)
        for w in works:
            w.wait()
        for b, dst in bufs:
            dst.copy_(b)

    def passes(self, n_iters: int, check_every: int = 0):
        """The pass lengths of a run: each stretch up to a checked iteration split into passes of
        2 and 3 (a one-iteration stretch cannot be run on ghost pairs)."""
        out, k = [], 0
        while k < n_iters:
            d = n_iters - k
            if check_every:
                d = min(d, check_every - k % check_every)
            if d == 1:
                raise ValueError("ghost-pair runs need stretches of >= 2 iterations between checks")
            # passes of 2 with one 3 first when the stretch is odd: the library's own split
            # (uot_api.cu launch_iters, UOT_PROX_PASS default), so world 1 reproduces it exactly
            seg = ([3] if d % 2 else []) + [2] * ((d - 3) // 2 if d % 2 else d // 2)
            out += [(s, i == len(seg) - 1) for i, s in enumerate(seg)]
            k += d
        return out

    def run(self, n_iters: int, check_every: int = 0, tol: float = 0.0):
        """n_iters iterations as passes of 2 / 3 with an exchange after each; reductions on the
        checked passes; returns the last checked pass's report summed over ranks."""
        if tol > 0:
            raise ValueError("GhostChain: tol = 0 only (fixed iteration counts)")
        for s, checked in self.passes(n_iters, check_every):
            if checked:
                self.prob.iterate(s, check_every=s)      # reductions of its last iteration
            else:
                self.prob.step(s)                         # no reductions
            self.exchange()
        rep = self.prob.report()
        if self.world > 1:
            rep = all_reduce_report(rep, self.prob.frames.device, group=self.group)
        return rep
