"""Float64 CPU oracle for Algorithm 1 of arXiv 1909.00149.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with the CUDA path (``paper_1909_00149_b200``):
neither imports the other.  The C source is ``oracle/uot_oracle.c``; this
module only compiles it (gcc) and marshals numpy arrays.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(P1..P20, DF1..DF4) and ``tests/test_oracle_residual_pins.py`` (P21..P23, the
stopping-rule reductions), DESIGN.md section "Oracle and its pins"; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "uot_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

REP_FIELDS = ("transport", "growth_l1", "primal_sq", "dual_sq", "ub_l1", "prox_sq", "f_sq", "npix")
CERT_FIELDS = ("transport", "growth_l1", "upper", "a_dot_f", "max_divadj", "max_abs_a", "lower", "objective")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, OpenMP over independent pairs)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("n_chains", ctypes.c_int32),
                ("n_frames", ctypes.c_int32), ("alpha", ctypes.c_double), ("rho", ctypes.c_double),
                ("tau1", ctypes.c_double), ("tau2", ctypes.c_double), ("p_norm", ctypes.c_int32),
                ("fix_first", ctypes.c_int32)]


class _DfParams(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("n_problems", ctypes.c_int32),
                ("mu", ctypes.c_double), ("kappa", ctypes.c_double), ("rho", ctypes.c_double),
                ("tau1", ctypes.c_double), ("tau2", ctypes.c_double), ("inner_iters", ctypes.c_int32),
                ("p_norm", ctypes.c_int32)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        L.uot_ref_div.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.uot_ref_div_adj.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.uot_ref_shrink_l2.argtypes = [ctypes.c_int64, dp, dp, ctypes.c_double, dp, dp]
        L.uot_ref_shrink_l1.argtypes = [ctypes.c_int64, dp, ctypes.c_double, dp]
        L.uot_ref_lambda_max.argtypes = [ctypes.c_int, ctypes.c_int]
        L.uot_ref_lambda_max.restype = ctypes.c_double
        L.uot_ref_iterate.argtypes = [ctypes.POINTER(_Params), dp, dp, dp, dp, dp, dp, ctypes.c_int, dp]
        L.uot_ref_iterate.restype = ctypes.c_int
        L.uot_ref_certificate.argtypes = [ctypes.POINTER(_Params), dp, dp, dp, dp, dp, dp, dp]
        L.uot_ref_certificate.restype = ctypes.c_int
        L.uot_ref_df_admm.argtypes = [ctypes.POINTER(_DfParams), dp, dp] + [dp] * 9 + [ctypes.c_int, dp]
        L.uot_ref_df_admm.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(arr):
    if arr is None:
        return None
    assert arr.dtype == np.float64 and arr.flags.c_contiguous
    return arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# --------------------------------------------------------------------------- grid operators
def div(mx, my):
    """div(M), P:153-158 (zero flux outside; Mx[:, -1], My[-1, :] do not exist)."""
    mx, my = _f64(mx), _f64(my)
    ny, nx = mx.shape
    out = np.empty_like(mx)
    lib().uot_ref_div(nx, ny, _p(mx), _p(my), _p(out))
    return out


def div_adj(a):
    """div^*(a), the adjoint of div."""
    a = _f64(a)
    ny, nx = a.shape
    gx, gy = np.empty_like(a), np.empty_like(a)
    lib().uot_ref_div_adj(nx, ny, _p(a), _p(gx), _p(gy))
    return gx, gy


def shrink_l2(qx, qy, sigma):
    """shrink^{l2}_sigma per 2-vector row."""
    qx, qy = _f64(qx), _f64(qy)
    ox, oy = np.empty_like(qx), np.empty_like(qy)
    lib().uot_ref_shrink_l2(qx.size, _p(qx), _p(qy), float(sigma), _p(ox), _p(oy))
    return ox, oy


def shrink_l1(q, sigma):
    """shrink^{l1}_sigma."""
    q = _f64(q)
    out = np.empty_like(q)
    lib().uot_ref_shrink_l1(q.size, _p(q), float(sigma), _p(out))
    return out


def lambda_max(nx: int, ny: int) -> float:
    """lambda_max(nabla^2) of Theorem 1, closed form."""
    return float(lib().uot_ref_lambda_max(int(nx), int(ny)))


def default_steps(nx: int, ny: int, prox: bool, n_frames: int = 2, safety: float = 0.99, fix_first: bool = False):
    """tau1 = tau2 = sqrt(safety/||K||^2) with ||K||^2 from Theorem 1 (L11/L12):
    lambda_max + 1 (fixed marginals), + 3 (pair prox), + 3 + 2cos(pi/T) (chain prox),
    + 2 (fixed-first-argument pair prox, K = [D, -I, -I])."""
    lam = lambda_max(nx, ny)
    if not prox:
        extra = 1.0
    elif fix_first and n_frames == 2:
        extra = 2.0
    else:
        extra = 1.0 + 2.0 + 2.0 * math.cos(math.pi / n_frames) if n_frames > 2 else 3.0
    t = math.sqrt(safety / (lam + extra))
    return t, t


# --------------------------------------------------------------------------- Algorithm 1
@dataclass
class State:
    mx: np.ndarray
    my: np.ndarray
    r: np.ndarray
    a: np.ndarray
    x: np.ndarray | None


def zero_state(frames, prox: bool, x_from_p: bool = False, fix_first: bool = False) -> State:
    """Cold start (P:532 'initialized to 0'); x0 = 0, or Pi_+(p) with x_from_p (L8);
    with fix_first the first frame of each chain starts (and stays) at p_0."""
    frames = _f64(frames)
    B, T, ny, nx = frames.shape
    z = lambda: np.zeros((B, T - 1, ny, nx))
    x = None
    if prox:
        x = np.maximum(frames, 0.0).copy() if x_from_p else np.zeros_like(frames)
        if fix_first:
            x[:, 0] = frames[:, 0]
    return State(z(), z(), z(), z(), x)


def iterate(frames, alpha, rho, tau1, tau2, n_iters, state: State | None = None, p_norm: int = 1,
            fix_first: bool = False):
    """Run n_iters iterations of Algorithm 1 on frames [B][T][ny][nx].

    Returns (state, rep) where rep[B*(T-1), 8] are the reductions of the last
    iteration (fields REP_FIELDS).  rho = inf -> fixed marginals; alpha = inf ->
    balanced Beckmann; p_norm 2 -> alpha ||r||_2^2; fix_first -> eq:Prox_UOT_specialcase.
    """
    frames = _f64(frames)
    if frames.ndim == 2:
        raise ValueError("frames must be [B][T][ny][nx]")
    B, T, ny, nx = frames.shape
    prox = math.isfinite(rho)
    st = state if state is not None else zero_state(frames, prox, fix_first=fix_first)
    st = State(_f64(st.mx).copy(), _f64(st.my).copy(), _f64(st.r).copy(), _f64(st.a).copy(),
               None if st.x is None else _f64(st.x).copy())
    if prox and st.x is None:
        st.x = np.zeros_like(frames)
    prm = _Params(nx, ny, B, T, float(alpha), float(rho), float(tau1), float(tau2), int(p_norm), int(fix_first))
    rep = np.zeros((B * (T - 1), 8))
    rc = lib().uot_ref_iterate(ctypes.byref(prm), _p(frames), _p(st.mx), _p(st.my), _p(st.r),
                               _p(st.a), _p(st.x) if prox else None, int(n_iters), _p(rep))
    if rc == 2:
        raise ValueError("invalid oracle parameters")
    if rc == 4:
        raise FloatingPointError("oracle produced a non-finite iterate")
    return st, rep


def certificate(frames, state: State, alpha, rho=math.inf, p_norm: int = 1):
    """Objective and weak-duality bounds L <= V <= U per pair (fields CERT_FIELDS)."""
    frames = _f64(frames)
    B, T, ny, nx = frames.shape
    prm = _Params(nx, ny, B, T, float(alpha), float(rho), 0.0, 0.0, int(p_norm), 0)
    cert = np.zeros((B * (T - 1), 8))
    prox = math.isfinite(rho)
    lib().uot_ref_certificate(ctypes.byref(prm), _p(frames), _p(_f64(state.mx)), _p(_f64(state.my)),
                              _p(_f64(state.r)), _p(_f64(state.a)),
                              _p(_f64(state.x)) if prox else None, _p(cert))
    return cert


def evaluate(p, q, alpha, iters=20000, tol=1e-9, tau=None, chunk=2000, p_norm: int = 1):
    """V_alpha(p, q) of eq:Unbal_OT_beckman by Algorithm 1 without the
    x-block, run until the certified gap (U-L)/max(U,1e-12) <= tol or iters.
    Returns (value_upper, value_lower, objective).  alpha = inf: balanced (U is
    then the objective once div M = f holds to rounding, see certificate)."""
    p, q = _f64(p), _f64(q)
    if p.ndim == 1:
        p, q = p[None, :], q[None, :]
    ny, nx = p.shape
    frames = np.stack([p, q])[None]
    t1, t2 = default_steps(nx, ny, prox=False) if tau is None else (tau, tau)
    st = None
    done = 0
    cert = None
    while done < iters:
        n = min(chunk, iters - done)
        st, _ = iterate(frames, alpha, math.inf, t1, t2, n, st, p_norm=p_norm)
        done += n
        cert = certificate(frames, st, alpha, p_norm=p_norm)
        U, L = cert[0, 2], cert[0, 6]
        if not math.isfinite(alpha):     # balanced: U needs exact feasibility; use the objective
            U = cert[0, 7]
        if U - L <= tol * max(abs(U), 1e-12):
            break
    return cert[0, 2], cert[0, 6], cert[0, 7]


# --------------------------------------------------------------------------- Algorithm 2
DF_STATE = ("s", "x", "z", "a", "b", "mx", "my", "r", "ain")


def df_zero_state(B, ny, nx):
    """Alg. 2 line 2: s = x = z = a = b = 0; inner prox state 0."""
    return {k: np.zeros((B, ny, nx)) for k in DF_STATE}


def df_admm(y, s0, mu, kappa, rho, tau1, tau2, n_outer, inner_iters=1, state=None, p_norm=1):
    """Algorithm 2, Phi = I, R = 0, for B problems y, s0 [B][ny][nx].
    Returns (state dict, res[n_outer][2] = primal, dual residuals of P:562-567)."""
    y, s0 = _f64(y), _f64(s0)
    B, ny, nx = y.shape
    st = {k: _f64(v).copy() for k, v in (state or df_zero_state(B, ny, nx)).items()}
    prm = _DfParams(nx, ny, B, float(mu), float(kappa), float(rho), float(tau1), float(tau2),
                    int(inner_iters), int(p_norm))
    res = np.zeros((n_outer, 2))
    rc = lib().uot_ref_df_admm(ctypes.byref(prm), _p(y), _p(s0), *[_p(st[k]) for k in DF_STATE],
                               int(n_outer), _p(res))
    if rc == 4:
        raise FloatingPointError("non-finite iterate")
    return st, res
