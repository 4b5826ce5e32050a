"""Python surface of the B200 UOT hot path (thin layer over include/uot.h).

PyTorch is used only for device memory and streams: every buffer the C
library works on is a torch tensor allocated here and passed by pointer; every
arithmetic step of Algorithm 1 runs in the library's
CUDA kernels.  There is no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (Buffers, DfBuffers, DfParams, DfReport, Params, Report, RpcaBuffers, RpcaParams, RpcaReport,
                   check, lib)

__all__ = ["Problem", "DFProblem", "RPCAProblem", "default_steps", "scratch_doubles", "Report"]


def _params(nx, ny, B, T, alpha, rho, tau1, tau2, flags=0) -> Params:
    return Params(int(nx), int(ny), int(B), int(T), float(alpha), float(rho),
                  float(tau1 or 0.0), float(tau2 or 0.0), int(flags))


def default_steps(nx, ny, n_frames=2, rho=math.inf, safety=0.99, fix_first=False):
    """Theorem-1 steps (L11/L12) from the library."""
    t1, t2 = ctypes.c_double(), ctypes.c_double()
    p = _params(nx, ny, 1, n_frames, 1.0, rho, 0, 0, _lib.UOT_FIX_FIRST_FRAME if fix_first else 0)
    check(lib().uot_default_steps(ctypes.byref(p), float(safety), ctypes.byref(t1), ctypes.byref(t2)))
    return t1.value, t2.value


def scratch_doubles(nx, ny, B, T, rho=math.inf) -> int:
    p = _params(nx, ny, B, T, 1.0, rho, 0, 0)
    return int(lib().uot_scratch_doubles(ctypes.byref(p)))


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


@dataclass
class PairCert:
    """uot_objective per-pair rows: see include/uot.h."""
    rows: "object"   # numpy [G][8]: transport, sum|r|, U, <a,f>, max||div*a||, max|a|, L, objective


class Problem:
    """B chains of T frames [B][T][ny][nx] (fp32, CUDA), one UOT term per adjacent pair.

    rho = inf: fixed marginals (evaluation of eq:Unbal_OT_beckman);
    finite rho: prox mode (eq:Prox_UOT, L2/L19).
    """

    def __init__(self, frames: torch.Tensor, alpha: float, rho: float = math.inf,
                 tau1: float | None = None, tau2: float | None = None, *, stream: torch.cuda.Stream | None = None,
                 force_steps: bool = False, reset: bool = True, halos: bool | tuple = False,
                 p_norm: int = 1, fix_first: bool = False):
        if frames.dim() != 4:
            raise ValueError("frames must be [B][T][ny][nx]")
        if not frames.is_cuda or frames.dtype != torch.float32:
            raise ValueError("frames must be a float32 CUDA tensor")
        self.frames = frames.contiguous()
        B, T, ny, nx = self.frames.shape
        self.B, self.T, self.ny, self.nx = B, T, ny, nx
        self.P = T - 1
        self.G = B * self.P
        self.alpha, self.rho = float(alpha), float(rho)
        self.prox = math.isfinite(self.rho)
        dev = self.frames.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        plane = (B, self.P, ny, nx)
        e = lambda shape: torch.empty(shape, dtype=torch.float32, device=dev)
        self.f = e(plane) if not self.prox else None
        self.mx = [e(plane), e(plane)]
        self.my = [e(plane), e(plane)]
        self.r = e(plane)
        # second r buffer for the multi-iteration passes (k_wave / k_iter2; chain prox: k_wave_prox)
        self.r_alt = e(plane)
        self.a = [e(plane), e(plane)]
        self.x = [e(self.frames.shape), e(self.frames.shape)] if self.prox else [None, None]
        # chain-prox shard halos (L19): duals of the pairs just outside this shard, [B][ny][nx]
        # halos = (has_prev, has_next) or a bool for both: a shard with no neighbour on a side
        # passes no halo there (the chain ends; its end frame is reduced by this shard)
        hp, hn = (halos, halos) if isinstance(halos, bool) else (bool(halos[0]), bool(halos[1]))
        self.a_prev_halo = torch.zeros((B, ny, nx), dtype=torch.float32, device=dev) if hp else None
        self.a_next_halo = torch.zeros((B, ny, nx), dtype=torch.float32, device=dev) if hn else None
        flags = (_lib.UOT_FORCE_STEPS if force_steps else 0) | (_lib.UOT_RESIDUAL_L2 if p_norm == 2 else 0) | \
            (_lib.UOT_FIX_FIRST_FRAME if fix_first else 0)
        if p_norm not in (1, 2):
            raise ValueError("p_norm must be 1 or 2")
        self.p_norm, self.fix_first = p_norm, fix_first
        self._params = _params(nx, ny, B, T, alpha, rho, tau1, tau2, flags)
        nsc = int(lib().uot_scratch_doubles(ctypes.byref(self._params)))
        self.scratch = torch.zeros(nsc, dtype=torch.float64, device=dev)
        self._bufs = self._make_buffers()
        ctx = ctypes.c_void_p()
        check(lib().uot_create(ctypes.byref(self._params), ctypes.byref(self._bufs),
                               ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(ctx)))
        self._ctx = ctx
        if tau1 is None or tau2 is None:
            d1, d2 = default_steps(nx, ny, T, rho, fix_first=fix_first)
            self.tau1 = float(tau1) if tau1 is not None else d1
            self.tau2 = float(tau2) if tau2 is not None else d2
        else:
            self.tau1, self.tau2 = float(tau1), float(tau2)
        if reset:
            self.reset()

    def _make_buffers(self) -> Buffers:
        b = Buffers()
        b.frames = self.frames.data_ptr()
        b.f = self.f.data_ptr() if self.f is not None else None
        for k in range(2):
            b.mx[k] = self.mx[k].data_ptr()
            b.my[k] = self.my[k].data_ptr()
            b.a[k] = self.a[k].data_ptr()
            b.x[k] = self.x[k].data_ptr() if self.x[k] is not None else None
        b.r = self.r.data_ptr()
        b.r_alt = self.r_alt.data_ptr() if self.r_alt is not None else None
        b.a_prev_halo = self.a_prev_halo.data_ptr() if self.a_prev_halo is not None else None
        b.a_next_halo = self.a_next_halo.data_ptr() if self.a_next_halo is not None else None
        b.scratch = self.scratch.data_ptr()
        return b

    # ------------------------------------------------------------------ calls
    def reset(self, x_from_p: bool = False):
        check(lib().uot_reset(self._ctx, _lib.UOT_RESET_X_FROM_P if x_from_p else 0), self._ctx)

    def load_frames_host(self, host_frames: torch.Tensor):
        """H2D copy of new frames (pinned host tensor, same shape) + recompute f (warm state kept)."""
        if host_frames.is_cuda or host_frames.dtype != torch.float32 or host_frames.shape != self.frames.shape:
            raise ValueError("host_frames must be a CPU float32 tensor of the frames' shape")
        if not host_frames.is_contiguous():
            raise ValueError("host_frames must be contiguous")
        self._host_keepalive = host_frames
        check(lib().uot_load_frames(self._ctx, ctypes.c_void_p(host_frames.data_ptr())), self._ctx)

    def step(self, n: int = 1, report: bool = False) -> dict | None:
        """n iterations of Alg.1 lines 3-7; report=True syncs and returns the reductions of the last."""
        if report:
            rep = Report()
            check(lib().uot_prox_step(self._ctx, int(n), ctypes.byref(rep)), self._ctx)
            return rep.as_dict()
        check(lib().uot_prox_step(self._ctx, int(n), None), self._ctx)
        return None

    def iterate(self, n: int, check_every: int = 0, tol: float = 0.0):
        """Enqueue n iterations asynchronously (reductions every check_every and on the last)."""
        check(lib().uot_iterate(self._ctx, int(n), int(check_every), float(tol)), self._ctx)

    def iterate_part(self, part: int, reduce: bool = False):
        """One iteration on a part of the pairs (_lib.UOT_PART_INTERIOR / _BOUNDARY / _ALL)."""
        check(lib().uot_iterate_part(self._ctx, int(part), int(bool(reduce))), self._ctx)

    def stop_external(self):
        """Arm the cross-rank stop (uot_stop_external): chunks then run with tol = 0 and the
        L13 test is applied to all-reduced sums by stop_apply."""
        check(lib().uot_stop_external(self._ctx), self._ctx)

    def stop_pack(self, sums8: torch.Tensor):
        """sums8 (8 float64 on the device) <- this shard's sums of the last checked iteration."""
        if not (sums8.is_cuda and sums8.dtype == torch.float64 and sums8.numel() >= 8 and sums8.is_contiguous()):
            raise ValueError("sums8 must be a contiguous CUDA float64 tensor of >= 8 elements")
        check(lib().uot_stop_pack(self._ctx, ctypes.c_void_p(sums8.data_ptr())), self._ctx)

    def stop_apply(self, sums8: torch.Tensor, tol: float):
        """Set the stop flag if the (all-reduced) sums8 pass the L13 test at tol."""
        check(lib().uot_stop_apply(self._ctx, ctypes.c_void_p(sums8.data_ptr()), float(tol)), self._ctx)

    def report(self) -> dict:
        """Sync and return the reductions of the last reducing iteration."""
        rep = Report()
        check(lib().uot_get_report(self._ctx, ctypes.byref(rep)), self._ctx)
        return rep.as_dict()

    def solve(self, max_iters: int, tol: float = 0.0, check_every: int = 10, raise_not_converged=False) -> dict:
        rep = Report()
        allow = () if raise_not_converged else (_lib.UOT_E_NOT_CONVERGED,)
        rc = check(lib().uot_solve(self._ctx, int(max_iters), float(tol), int(check_every), ctypes.byref(rep)),
                   self._ctx, allow=allow)
        d = rep.as_dict()
        d["status"] = rc
        return d

    def objective(self, per_pair: bool = False):
        """Objective + weak-duality certificate of the current state (see include/uot.h)."""
        import numpy as np
        rep = Report()
        rows = np.zeros((self.G, 8), dtype=np.float64) if per_pair else None
        ptr = rows.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if per_pair else None
        check(lib().uot_objective(self._ctx, ptr, ctypes.byref(rep)), self._ctx)
        return (rep.as_dict(), rows) if per_pair else rep.as_dict()

    def set_timing(self, enable: bool = True):
        check(lib().uot_set_timing(self._ctx, int(bool(enable))), self._ctx)

    def get_timing(self):
        """(summed device ms of the timed fused-iteration launches, their count); clears."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        check(lib().uot_get_timing(self._ctx, ctypes.byref(ms), ctypes.byref(n)), self._ctx)
        return ms.value, n.value

    PATH_NAMES = ("k_iter", "k_iter2", "k_persist", "k_iter4", "k_df", "k_wave2", "k_wave4", "k_wave3", "k_tpersist", "k_wave5", "k_single",
                  "k_wave_prox")

    def get_timing_paths(self):
        """{kernel: (summed device ms, launches)} of the timed launches, split by kernel
        (k_iter2 = two-iteration passes, k_iter4 = four-iteration passes); clears."""
        from ._lib import UOT_N_PATHS
        ms = (ctypes.c_double * UOT_N_PATHS)()
        n = (ctypes.c_int64 * UOT_N_PATHS)()
        check(lib().uot_get_timing_paths(self._ctx, ms, n), self._ctx)
        return {self.PATH_NAMES[k]: (ms[k], n[k]) for k in range(UOT_N_PATHS) if n[k]}

    @property
    def slot(self) -> int:
        return int(lib().uot_state_slot(self._ctx))

    @property
    def kernel_path(self) -> str:
        """'k_iter' (one pass per iteration), 'k_iter2' / 'k_iter4' (SMEM tiles, two / four
        iterations per pass), 'k_wave2' / 'k_wave4' (register wavefront) or 'k_persist'."""
        return self.PATH_NAMES[int(lib().uot_kernel_path(self._ctx))]

    @property
    def wave_cols(self) -> int:
        """Strip width of the register-wavefront passes: 128 (k_wave_pk), 64 (k_wave_n, narrow
        strips) or 0 (no wavefront passes); include/uot.h uot_wave_cols."""
        return int(lib().uot_wave_cols(self._ctx))

    def set_own_pairs(self, lo: int, hi: int):
        """Chain prox on k_wave_prox: only pairs [lo, hi) are written and reduced; the others are
        ghost copies of neighbouring shards' pairs, refreshed by the caller after each pass
        (include/uot.h uot_set_own_pairs; dist.GhostChain)."""
        check(lib().uot_set_own_pairs(self._ctx, int(lo), int(hi)), self._ctx)

    def set_temporal(self, enable: bool = True):
        """Fixed marginals: two iterations per HBM pass (k_iter2, default) or one (k_iter)."""
        check(lib().uot_set_temporal(self._ctx, int(bool(enable))), self._ctx)

    @property
    def launches(self) -> int:
        return int(lib().uot_launch_count(self._ctx))

    def state(self) -> dict:
        """Current iterate (views of the ping-pong slot)."""
        s = self.slot
        rs = int(lib().uot_r_slot(self._ctx))
        d = {"mx": self.mx[s], "my": self.my[s], "r": self.r_alt if rs else self.r, "a": self.a[s]}
        if self.prox:
            d["x"] = self.x[s]
        return d

    def state_dict(self) -> dict:
        """Checkpoint: copies of the current state (+ iteration count)."""
        d = {k: v.detach().clone() for k, v in self.state().items()}
        d["iterations"] = self.iterations
        return d

    def load_state_dict(self, d: dict):
        """Resume from a checkpoint (a state_dict of a problem with the same frames, shape and
        parameters): copies the iterate into the current buffers.  Algorithm 1 recomputes K^k
        from the state at the start of every call (L8), so continuing after a load equals
        continuing the original run; the iteration count restarts at this problem's own."""
        cur = self.state()
        for k, v in cur.items():
            if k not in d or tuple(d[k].shape) != tuple(v.shape):
                raise ValueError(f"checkpoint lacks {k} or has the wrong shape")
            v.copy_(d[k])

    @property
    def iterations(self) -> int:
        return int(self.report()["iterations"])

    def close(self):
        if getattr(self, "_ctx", None):
            lib().uot_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DFProblem:
    """UOT-DF ADMM (Algorithm 2) with Phi = I, R = 0 on B problems:
    min_{s >= 0} 1/2 ||y - s||^2 + kappa V_mu(s0, s)   (eq:UOT-DF).

    y, s0: float32 CUDA tensors [B][ny][nx].  inner_iters = 1 runs one
    fused kernel per ADMM iteration.  All steps run in libuot_b200.so."""

    STATE = ("s", "x", "a", "b")

    def __init__(self, y: torch.Tensor, s0: torch.Tensor, mu: float, kappa: float, rho: float = 1.0,
                 tau1: float | None = None, tau2: float | None = None, inner_iters: int = 1, p_norm: int = 1,
                 *, stream: torch.cuda.Stream | None = None, reset: bool = True):
        if y.dim() != 3 or y.shape != s0.shape:
            raise ValueError("y and s0 must be [B][ny][nx] of the same shape")
        if not (y.is_cuda and s0.is_cuda) or y.dtype != torch.float32 or s0.dtype != torch.float32:
            raise ValueError("y, s0 must be float32 CUDA tensors")
        self.y, self.s0 = y.contiguous(), s0.contiguous()
        B, ny, nx = self.y.shape
        self.B, self.ny, self.nx = B, ny, nx
        dev = self.y.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        e = lambda *shape: torch.zeros(shape, dtype=torch.float32, device=dev)
        self.s, self.x, self.a, self.b = e(B, ny, nx), e(B, ny, nx), e(B, ny, nx), e(B, ny, nx)
        self.pf = e(B, 2, ny, nx)
        self.xz = [e(B, 2, ny, nx), e(B, 2, ny, nx)]
        self.mx, self.my, self.ain = [e(B, ny, nx), e(B, ny, nx)], [e(B, ny, nx), e(B, ny, nx)], [e(B, ny, nx), e(B, ny, nx)]
        self.r = e(B, ny, nx)
        self.tmp = [e(B, ny, nx), e(B, ny, nx)] if inner_iters > 1 else [None, None]
        flags = _lib.UOT_RESIDUAL_L2 if p_norm == 2 else 0
        self._p = DfParams(nx, ny, B, float(mu), float(kappa), float(rho), float(tau1 or 0.0), float(tau2 or 0.0),
                           int(inner_iters), flags)
        nsc = int(lib().uot_df_scratch_doubles(ctypes.byref(self._p)))
        self.scratch = torch.zeros(nsc, dtype=torch.float64, device=dev)
        bf = DfBuffers()
        bf.y, bf.s0, bf.s, bf.x = self.y.data_ptr(), self.s0.data_ptr(), self.s.data_ptr(), self.x.data_ptr()
        bf.a, bf.b, bf.pf = self.a.data_ptr(), self.b.data_ptr(), self.pf.data_ptr()
        for k in range(2):
            bf.xz[k] = self.xz[k].data_ptr()
            bf.mx[k] = self.mx[k].data_ptr()
            bf.my[k] = self.my[k].data_ptr()
            bf.ain[k] = self.ain[k].data_ptr()
            bf.tmp[k] = self.tmp[k].data_ptr() if self.tmp[k] is not None else None
        bf.r = self.r.data_ptr()
        bf.scratch = self.scratch.data_ptr()
        self._bufs = bf
        ctx = ctypes.c_void_p()
        check(lib().uot_df_create(ctypes.byref(self._p), ctypes.byref(bf), ctypes.c_void_p(self.stream.cuda_stream),
                                  ctypes.byref(ctx)), None, df=True)
        self._ctx = ctx
        self.iterations = 0
        if reset:
            self.reset()

    def reset(self):
        check(lib().uot_df_reset(self._ctx), self._ctx, df=True)
        self.iterations = 0

    def solve(self, max_iters: int, eps: float = 0.0, check_every: int = 10) -> dict:
        rep = DfReport()
        rc = check(lib().uot_df_solve(self._ctx, int(max_iters), float(eps), int(check_every), ctypes.byref(rep)),
                   self._ctx, allow=(_lib.UOT_E_NOT_CONVERGED,), df=True)
        d = rep.as_dict()
        d["status"] = rc
        self.iterations = d["iterations"]
        return d

    def inner_state(self) -> dict:
        """Inner prox state (M, r, a_in, z) of the current iterate."""
        s = int(self.iterations_inner() & 1)
        return {"mx": self.mx[s], "my": self.my[s], "r": self.r, "ain": self.ain[s], "z": self.xz[s][:, 1]}

    def iterations_inner(self) -> int:
        return self.iterations * int(self._p.inner_iters)

    def set_timing(self, enable=True):
        check(lib().uot_df_set_timing(self._ctx, int(bool(enable))), self._ctx, df=True)

    def get_timing(self):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        check(lib().uot_df_get_timing(self._ctx, ctypes.byref(ms), ctypes.byref(n)), self._ctx, df=True)
        return ms.value, n.value

    @property
    def launches(self) -> int:
        return int(lib().uot_df_launch_count(self._ctx))

    def close(self):
        if getattr(self, "_ctx", None):
            lib().uot_df_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RPCAProblem:
    """RPCA+UOT-DF ADMM (Algorithm 3) on one video Y [T][ny][nx]:
    min_{S, L >= 0} 1/2 sum_t ||y_t - Phi_t(s_t + l_t)||^2 + lambda||S||_1 + gamma||L||_*
                    + kappa sum_t V_mu(s_t, s_{t+1})          (eq:RPCA_UOTDF)
    with diagonal Phi (``phi`` [T][ny][nx] per-pixel weights, None = identity).
    signed=True: the signed split eq:RPCA_UOTDF_PN, S = S+ - S-, with one
    UOT chain per sign (reading L30).

    Every line of Algorithm 3 (including the SVT of line 10) runs in libuot_b200.so;
    this class only allocates the torch buffers and marshals pointers."""

    STATE = ("S", "L", "X", "Tm", "A", "D")

    def __init__(self, Y: torch.Tensor, lam: float, gamma: float, kappa: float, mu: float, rho: float = 1.0,
                 phi: torch.Tensor | None = None, tau1: float | None = None, tau2: float | None = None,
                 inner_iters: int = 1, p_norm: int = 1, signed: bool = False, *,
                 stream: torch.cuda.Stream | None = None, reset: bool = True, shard: tuple | None = None):
        """shard = (frame0, T_total): Y holds frames [frame0, frame0 + T) of a T_total-frame
        video (a frame-range shard; the last frame is the next shard's first when
        frame0 + T < T_total); driven by dist.ShardedRPCA."""
        if Y.dim() != 3:
            raise ValueError("Y must be [T][ny][nx]")
        if not Y.is_cuda or Y.dtype != torch.float32:
            raise ValueError("Y must be a float32 CUDA tensor")
        if phi is not None and (phi.shape != Y.shape or not phi.is_cuda or phi.dtype != torch.float32):
            raise ValueError("phi must be a float32 CUDA tensor shaped like Y")
        self.Y = Y.contiguous()
        self.phi = phi.contiguous() if phi is not None else None
        T, ny, nx = self.Y.shape
        self.T, self.ny, self.nx = T, ny, nx
        self.signed = bool(signed)
        P = T - 1
        Q = 2 * P if self.signed else P
        dev = self.Y.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        e = lambda *shape: torch.zeros(shape, dtype=torch.float32, device=dev)
        for k in self.STATE:
            setattr(self, k, e(T, ny, nx))
        self.Sm = e(T, ny, nx) if self.signed else None
        self.pc, self.bc = e(Q, 2, ny, nx), e(Q, 2, ny, nx)
        self.zw = [e(Q, 2, ny, nx), e(Q, 2, ny, nx)]
        self.zprev = e(Q, 2, ny, nx) if inner_iters > 1 else None
        self.mx, self.my, self.ain = [e(Q, ny, nx), e(Q, ny, nx)], [e(Q, ny, nx), e(Q, ny, nx)], [e(Q, ny, nx), e(Q, ny, nx)]
        self.r = e(Q, ny, nx)
        flags = (_lib.UOT_RESIDUAL_L2 if p_norm == 2 else 0) | (_lib.UOT_RPCA_SIGNED if self.signed else 0)
        f0, Tt = (0, T) if shard is None else (int(shard[0]), int(shard[1]))
        self.frame0, self.T_total = f0, Tt
        self.has_prev, self.has_next = f0 > 0, f0 + T < Tt
        sflags = (_lib.UOT_RPCA_HAS_PREV if self.has_prev else 0) | (_lib.UOT_RPCA_HAS_NEXT if self.has_next else 0)
        chains = 2 if self.signed else 1
        self.mgather = e(Tt, ny, nx) if Tt > T else None
        self.halo_prev = e(chains, 2, ny, nx) if self.has_prev else None     # (w, c) of pair frame0 - 1
        self.halo_next = e(chains, 2, ny, nx) if self.has_next else None     # (z, b) of the pair after the last frame
        self._p = RpcaParams(nx, ny, T, float(lam), float(gamma), float(kappa), float(mu), float(rho),
                             float(tau1 or 0.0), float(tau2 or 0.0), int(inner_iters), flags, f0,
                             Tt if Tt > T else 0, sflags)
        nsc = int(lib().uot_rpca_scratch_doubles(ctypes.byref(self._p)))
        if nsc == 0:
            raise ValueError(f"unsupported shape (2 <= T <= {_lib.UOT_RPCA_MAX_T})")
        self.scratch = torch.zeros(nsc, dtype=torch.float64, device=dev)
        bf = RpcaBuffers()
        bf.y = self.Y.data_ptr()
        bf.phi = self.phi.data_ptr() if self.phi is not None else None
        for k in self.STATE:
            setattr(bf, k, getattr(self, k).data_ptr())
        bf.Sm = self.Sm.data_ptr() if self.Sm is not None else None
        bf.pc, bf.bc = self.pc.data_ptr(), self.bc.data_ptr()
        bf.zprev = self.zprev.data_ptr() if self.zprev is not None else None
        for k in range(2):
            bf.zw[k] = self.zw[k].data_ptr()
            bf.mx[k] = self.mx[k].data_ptr()
            bf.my[k] = self.my[k].data_ptr()
            bf.ain[k] = self.ain[k].data_ptr()
        bf.r = self.r.data_ptr()
        bf.scratch = self.scratch.data_ptr()
        bf.mgather = self.mgather.data_ptr() if self.mgather is not None else None
        bf.halo_prev = self.halo_prev.data_ptr() if self.halo_prev is not None else None
        bf.halo_next = self.halo_next.data_ptr() if self.halo_next is not None else None
        self._bufs = bf
        ctx = ctypes.c_void_p()
        check(lib().uot_rpca_create(ctypes.byref(self._p), ctypes.byref(bf), ctypes.c_void_p(self.stream.cuda_stream),
                                    ctypes.byref(ctx)), None, rpca=True)
        self._ctx = ctx
        self.iterations = 0
        if reset:
            self.reset()

    def reset(self):
        check(lib().uot_rpca_reset(self._ctx), self._ctx, rpca=True)
        self.iterations = 0

    def solve(self, max_iters: int, eps: float = 0.0, check_every: int = 10, report: bool = True):
        """Up to max_iters ADMM iterations (eps <= 0: exactly max_iters).  report=False keeps
        the call asynchronous (no host synchronisation)."""
        if not report:
            check(lib().uot_rpca_solve(self._ctx, int(max_iters), float(eps), int(check_every), None),
                  self._ctx, rpca=True)
            self.iterations += int(max_iters)
            return None
        rep = RpcaReport()
        rc = check(lib().uot_rpca_solve(self._ctx, int(max_iters), float(eps), int(check_every), ctypes.byref(rep)),
                   self._ctx, allow=(_lib.UOT_E_NOT_CONVERGED,), rpca=True)
        d = rep.as_dict()
        d["status"] = rc
        self.iterations = d["iterations"]
        return d

    # ---- sharded iteration (include/uot.h "Sharded ADMM iteration"); see dist.ShardedRPCA
    def iterate_pre(self, reduce: bool = False):
        check(lib().uot_rpca_iterate_pre(self._ctx, int(bool(reduce))), self._ctx, rpca=True)

    def iterate_post(self, reduce: bool = False):
        check(lib().uot_rpca_iterate_post(self._ctx, int(bool(reduce))), self._ctx, rpca=True)
        self.iterations += 1

    def stop_external(self):
        check(lib().uot_rpca_stop_external(self._ctx), self._ctx, rpca=True)

    def stop_pack(self, sums8: torch.Tensor):
        check(lib().uot_rpca_stop_pack(self._ctx, ctypes.c_void_p(sums8.data_ptr())), self._ctx, rpca=True)

    def stop_apply(self, sums8: torch.Tensor, eps: float):
        check(lib().uot_rpca_stop_apply(self._ctx, ctypes.c_void_p(sums8.data_ptr()), float(eps)), self._ctx, rpca=True)

    def get_report(self) -> dict:
        rep = RpcaReport()
        check(lib().uot_rpca_get_report(self._ctx, ctypes.byref(rep)), self._ctx, rpca=True)
        d = rep.as_dict()
        self.iterations = d["iterations"]
        return d

    def boundary_planes(self):
        """Planes this shard sends after an iteration: (z, b) of its first pair (to the previous
        shard's halo_next) and (w, c) of its last pair (to the next shard's halo_prev), one
        [2][ny][nx] pair per sign chain (views; z/w from the current ping-pong slot)."""
        s = int(lib().uot_rpca_state_slot(self._ctx))
        P = self.T - 1
        chains = [0, P] if self.signed else [0]
        first = [(self.zw[s][c0, 0], self.bc[c0, 0]) for c0 in chains]
        last = [(self.zw[s][c0 + P - 1, 1], self.bc[c0 + P - 1, 1]) for c0 in chains]
        return first, last

    def state(self) -> dict:
        """Current iterate: S, L, X, Tm, A, D [T][ny][nx]; Z, W, Bd, Cd [T-1][ny][nx] (z_t, w_{t+1},
        b_t, c_{t+1} at index t, the oracle's layout); inner mx, my, r, ain."""
        s = int(lib().uot_rpca_state_slot(self._ctx))
        d = {k: getattr(self, k) for k in self.STATE}
        d.update(mx=self.mx[s], my=self.my[s], r=self.r, ain=self.ain[s])
        if not self.signed:
            d.update(Z=self.zw[s][:, 0], W=self.zw[s][:, 1], Bd=self.bc[:, 0], Cd=self.bc[:, 1])
            return d
        P = self.T - 1
        d["Sp"] = d.pop("S")
        d.update(Sm=self.Sm, Zp=self.zw[s][:P, 0], Wp=self.zw[s][:P, 1], Zm=self.zw[s][P:, 0], Wm=self.zw[s][P:, 1],
                 Bp=self.bc[:P, 0], Cp=self.bc[:P, 1], Bm=self.bc[P:, 0], Cm=self.bc[P:, 1])
        return d

    def set_timing(self, enable=True):
        check(lib().uot_rpca_set_timing(self._ctx, int(bool(enable))), self._ctx, rpca=True)

    STAGES = ("pre", "gram", "eig", "apply", "prox", "post")

    def get_timing(self):
        """({stage: summed ms}, timed iterations) since set_timing."""
        ms = (ctypes.c_double * 6)()
        n = ctypes.c_int64()
        check(lib().uot_rpca_get_timing(self._ctx, ms, ctypes.byref(n)), self._ctx, rpca=True)
        return dict(zip(self.STAGES, list(ms))), n.value

    @property
    def launches(self) -> int:
        return int(lib().uot_rpca_launch_count(self._ctx))

    def close(self):
        if getattr(self, "_ctx", None):
            lib().uot_rpca_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
