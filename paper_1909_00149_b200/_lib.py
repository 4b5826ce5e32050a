"""ctypes binding of the C-ABI in include/uot.h (argument marshalling only).

Loads the IN-TREE library ``paper_1909_00149_b200/libuot_b200.so``.  There is
no fallback of any kind: if the library is missing or cannot be loaded, every
entry point raises.  Every step of the hot path runs in the library's kernels.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libuot_b200.so")

UOT_OK = 0
UOT_E_INVALID = 2
UOT_E_NOT_CONVERGED = 3
UOT_E_NONFINITE = 4
UOT_E_CUDA = 5
UOT_FORCE_STEPS = 1
UOT_FIX_FIRST_FRAME = 2
UOT_RESIDUAL_L2 = 4
UOT_RESET_X_FROM_P = 1
UOT_PART_ALL, UOT_PART_INTERIOR, UOT_PART_BOUNDARY = 0, 1, 2

EXPORTED = ("uot_scratch_doubles", "uot_default_steps", "uot_create", "uot_reset", "uot_load_frames",
            "uot_iterate", "uot_iterate_part", "uot_get_report", "uot_prox_step", "uot_solve", "uot_objective", "uot_set_timing", "uot_get_timing",
            "uot_get_timing_paths",
            "uot_state_slot", "uot_r_slot", "uot_set_temporal", "uot_kernel_path", "uot_wave_cols", "uot_set_own_pairs", "uot_launch_count",
            "uot_stop_external", "uot_stop_pack", "uot_stop_apply",
            "uot_destroy", "uot_last_error",
            "uot_df_scratch_doubles", "uot_df_create", "uot_df_reset", "uot_df_solve", "uot_df_set_timing",
            "uot_df_get_timing", "uot_df_launch_count", "uot_df_destroy", "uot_df_last_error",
            "uot_rpca_scratch_doubles", "uot_rpca_create", "uot_rpca_reset", "uot_rpca_solve",
            "uot_rpca_set_timing", "uot_rpca_get_timing", "uot_rpca_state_slot", "uot_rpca_launch_count",
            "uot_rpca_destroy", "uot_rpca_last_error", "uot_rpca_iterate_pre", "uot_rpca_iterate_post",
            "uot_rpca_stop_external", "uot_rpca_stop_pack", "uot_rpca_stop_apply", "uot_rpca_get_report")
UOT_N_PATHS = 12
UOT_RPCA_MAX_T = 512
UOT_RPCA_SIGNED = 8


class Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("n_chains", ctypes.c_int32),
                ("n_frames", ctypes.c_int32), ("alpha", ctypes.c_double), ("rho", ctypes.c_double),
                ("tau1", ctypes.c_double), ("tau2", ctypes.c_double), ("flags", ctypes.c_uint32)]


_fp = ctypes.c_void_p


class Buffers(ctypes.Structure):
    _fields_ = [("frames", _fp), ("f", _fp), ("mx", _fp * 2), ("my", _fp * 2), ("r", _fp),
                ("a", _fp * 2), ("x", _fp * 2), ("a_prev_halo", _fp), ("a_next_halo", _fp),
                ("scratch", _fp), ("r_alt", _fp)]


class Report(ctypes.Structure):
    _fields_ = [("objective", ctypes.c_double), ("transport", ctypes.c_double), ("growth", ctypes.c_double),
                ("prox_term", ctypes.c_double), ("primal_res", ctypes.c_double), ("dual_res", ctypes.c_double),
                ("upper_bound", ctypes.c_double), ("lower_bound", ctypes.c_double), ("f_norm", ctypes.c_double),
                ("iterations", ctypes.c_int64), ("converged", ctypes.c_int32), ("nonfinite", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class DfParams(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("n_problems", ctypes.c_int32),
                ("mu", ctypes.c_double), ("kappa", ctypes.c_double), ("rho", ctypes.c_double),
                ("tau1", ctypes.c_double), ("tau2", ctypes.c_double), ("inner_iters", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class DfBuffers(ctypes.Structure):
    _fields_ = [("y", _fp), ("s0", _fp), ("s", _fp), ("x", _fp), ("a", _fp), ("b", _fp), ("pf", _fp),
                ("xz", _fp * 2), ("mx", _fp * 2), ("my", _fp * 2), ("r", _fp), ("ain", _fp * 2),
                ("tmp", _fp * 2), ("scratch", _fp)]


class DfReport(ctypes.Structure):
    _fields_ = [("primal_res", ctypes.c_double), ("dual_res", ctypes.c_double), ("data_term", ctypes.c_double),
                ("transport", ctypes.c_double), ("growth", ctypes.c_double), ("objective", ctypes.c_double),
                ("iterations", ctypes.c_int64), ("converged", ctypes.c_int32), ("nonfinite", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class RpcaParams(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("n_frames", ctypes.c_int32),
                ("lam", ctypes.c_double), ("gamma", ctypes.c_double), ("kappa", ctypes.c_double),
                ("mu", ctypes.c_double), ("rho", ctypes.c_double), ("tau1", ctypes.c_double),
                ("tau2", ctypes.c_double), ("inner_iters", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("frame0", ctypes.c_int32), ("n_frames_total", ctypes.c_int32), ("shard_flags", ctypes.c_uint32)]


UOT_RPCA_HAS_PREV, UOT_RPCA_HAS_NEXT = 1, 2


class RpcaBuffers(ctypes.Structure):
    _fields_ = [("y", _fp), ("phi", _fp), ("S", _fp), ("L", _fp), ("X", _fp), ("Tm", _fp), ("A", _fp), ("D", _fp),
                ("Sm", _fp), ("pc", _fp), ("zw", _fp * 2), ("bc", _fp), ("zprev", _fp), ("mx", _fp * 2), ("my", _fp * 2),
                ("r", _fp), ("ain", _fp * 2), ("scratch", _fp), ("mgather", _fp), ("halo_prev", _fp),
                ("halo_next", _fp)]


class RpcaReport(ctypes.Structure):
    _fields_ = [("primal_res", ctypes.c_double), ("dual_res", ctypes.c_double), ("data_term", ctypes.c_double),
                ("l1_term", ctypes.c_double), ("nuclear", ctypes.c_double), ("transport", ctypes.c_double),
                ("growth", ctypes.c_double), ("objective", ctypes.c_double), ("iterations", ctypes.c_int64),
                ("converged", ctypes.c_int32), ("nonfinite", ctypes.c_int32), ("jacobi_sweeps", ctypes.c_int32),
                ("svt_min_ritz", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class UotError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"uot error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libuot_b200.so (raises if it is not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_1909_00149_b200.build` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, B, R = ctypes.POINTER(Params), ctypes.POINTER(Buffers), ctypes.POINTER(Report)
    ctx_pp = ctypes.POINTER(ctypes.c_void_p)
    L.uot_scratch_doubles.argtypes = [P]; L.uot_scratch_doubles.restype = ctypes.c_size_t
    L.uot_default_steps.argtypes = [P, ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    L.uot_default_steps.restype = ctypes.c_int
    L.uot_create.argtypes = [P, B, ctypes.c_void_p, ctx_pp]; L.uot_create.restype = ctypes.c_int
    L.uot_reset.argtypes = [ctypes.c_void_p, ctypes.c_uint32]; L.uot_reset.restype = ctypes.c_int
    L.uot_load_frames.argtypes = [ctypes.c_void_p, ctypes.c_void_p]; L.uot_load_frames.restype = ctypes.c_int
    L.uot_iterate.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_double]
    L.uot_iterate.restype = ctypes.c_int
    L.uot_iterate_part.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
    L.uot_iterate_part.restype = ctypes.c_int
    L.uot_get_report.argtypes = [ctypes.c_void_p, R]; L.uot_get_report.restype = ctypes.c_int
    L.uot_prox_step.argtypes = [ctypes.c_void_p, ctypes.c_int32, R]; L.uot_prox_step.restype = ctypes.c_int
    L.uot_solve.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, R]
    L.uot_solve.restype = ctypes.c_int
    L.uot_objective.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), R]
    L.uot_objective.restype = ctypes.c_int
    L.uot_set_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]; L.uot_set_timing.restype = ctypes.c_int
    L.uot_get_timing.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    L.uot_get_timing.restype = ctypes.c_int
    L.uot_get_timing_paths.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    L.uot_get_timing_paths.restype = ctypes.c_int
    L.uot_state_slot.argtypes = [ctypes.c_void_p]; L.uot_state_slot.restype = ctypes.c_int
    L.uot_r_slot.argtypes = [ctypes.c_void_p]; L.uot_r_slot.restype = ctypes.c_int
    L.uot_set_temporal.argtypes = [ctypes.c_void_p, ctypes.c_int]; L.uot_set_temporal.restype = ctypes.c_int
    L.uot_kernel_path.argtypes = [ctypes.c_void_p]; L.uot_kernel_path.restype = ctypes.c_int
    L.uot_wave_cols.argtypes = [ctypes.c_void_p]; L.uot_wave_cols.restype = ctypes.c_int
    L.uot_set_own_pairs.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
    L.uot_set_own_pairs.restype = ctypes.c_int
    L.uot_launch_count.argtypes = [ctypes.c_void_p]; L.uot_launch_count.restype = ctypes.c_int64
    L.uot_stop_external.argtypes = [ctypes.c_void_p]; L.uot_stop_external.restype = ctypes.c_int
    L.uot_stop_pack.argtypes = [ctypes.c_void_p, ctypes.c_void_p]; L.uot_stop_pack.restype = ctypes.c_int
    L.uot_stop_apply.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double]
    L.uot_stop_apply.restype = ctypes.c_int
    L.uot_destroy.argtypes = [ctypes.c_void_p]; L.uot_destroy.restype = None
    L.uot_last_error.argtypes = [ctypes.c_void_p]; L.uot_last_error.restype = ctypes.c_char_p
    DP, DB, DR = ctypes.POINTER(DfParams), ctypes.POINTER(DfBuffers), ctypes.POINTER(DfReport)
    L.uot_df_scratch_doubles.argtypes = [DP]; L.uot_df_scratch_doubles.restype = ctypes.c_size_t
    L.uot_df_create.argtypes = [DP, DB, ctypes.c_void_p, ctx_pp]; L.uot_df_create.restype = ctypes.c_int
    L.uot_df_reset.argtypes = [ctypes.c_void_p]; L.uot_df_reset.restype = ctypes.c_int
    L.uot_df_solve.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, DR]
    L.uot_df_solve.restype = ctypes.c_int
    L.uot_df_set_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]; L.uot_df_set_timing.restype = ctypes.c_int
    L.uot_df_get_timing.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    L.uot_df_get_timing.restype = ctypes.c_int
    L.uot_df_launch_count.argtypes = [ctypes.c_void_p]; L.uot_df_launch_count.restype = ctypes.c_int64
    L.uot_df_destroy.argtypes = [ctypes.c_void_p]; L.uot_df_destroy.restype = None
    L.uot_df_last_error.argtypes = [ctypes.c_void_p]; L.uot_df_last_error.restype = ctypes.c_char_p
    RP, RB, RR = ctypes.POINTER(RpcaParams), ctypes.POINTER(RpcaBuffers), ctypes.POINTER(RpcaReport)
    L.uot_rpca_scratch_doubles.argtypes = [RP]; L.uot_rpca_scratch_doubles.restype = ctypes.c_size_t
    L.uot_rpca_create.argtypes = [RP, RB, ctypes.c_void_p, ctx_pp]; L.uot_rpca_create.restype = ctypes.c_int
    L.uot_rpca_reset.argtypes = [ctypes.c_void_p]; L.uot_rpca_reset.restype = ctypes.c_int
    L.uot_rpca_solve.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, RR]
    L.uot_rpca_solve.restype = ctypes.c_int
    L.uot_rpca_set_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]; L.uot_rpca_set_timing.restype = ctypes.c_int
    L.uot_rpca_get_timing.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    L.uot_rpca_get_timing.restype = ctypes.c_int
    L.uot_rpca_state_slot.argtypes = [ctypes.c_void_p]; L.uot_rpca_state_slot.restype = ctypes.c_int
    L.uot_rpca_launch_count.argtypes = [ctypes.c_void_p]; L.uot_rpca_launch_count.restype = ctypes.c_int64
    for fn in ("uot_rpca_iterate_pre", "uot_rpca_iterate_post"):
        getattr(L, fn).argtypes = [ctypes.c_void_p, ctypes.c_int32]; getattr(L, fn).restype = ctypes.c_int
    L.uot_rpca_stop_external.argtypes = [ctypes.c_void_p]; L.uot_rpca_stop_external.restype = ctypes.c_int
    L.uot_rpca_stop_pack.argtypes = [ctypes.c_void_p, ctypes.c_void_p]; L.uot_rpca_stop_pack.restype = ctypes.c_int
    L.uot_rpca_stop_apply.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double]
    L.uot_rpca_stop_apply.restype = ctypes.c_int
    L.uot_rpca_get_report.argtypes = [ctypes.c_void_p, RR]; L.uot_rpca_get_report.restype = ctypes.c_int
    L.uot_rpca_destroy.argtypes = [ctypes.c_void_p]; L.uot_rpca_destroy.restype = None
    L.uot_rpca_last_error.argtypes = [ctypes.c_void_p]; L.uot_rpca_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def check(rc, ctx=None, allow=(), df=False, rpca=False):
    if rc == UOT_OK or rc in allow:
        return rc
    fn = lib().uot_rpca_last_error if rpca else (lib().uot_df_last_error if df else lib().uot_last_error)
    msg = fn(ctx)
    raise UotError(rc, msg.decode() if msg else "")
