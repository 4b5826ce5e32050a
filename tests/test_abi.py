"""Host-side checks of the C-ABI library (no GPU needed): it builds, loads,
exports every symbol include/uot.h declares, and its host-only entry points
agree with Theorem 1.  Compute entry points need a GPU and fail
loudly without one (no CPU fallback)."""
import ctypes
import math
import os
import re

import pytest

from paper_1909_00149_b200 import _lib
from paper_1909_00149_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build()
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "uot.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?\s*(uot_[a-z_]+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED), declared ^ set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(L, name), name


def test_struct_sizes_match_header(tmp_path):
    """The ctypes mirrors have the sizes the C compiler gives the structs of include/uot.h."""
    import subprocess
    names = ["uot_params", "uot_buffers", "uot_report", "uot_df_params", "uot_df_buffers", "uot_df_report",
             "uot_rpca_params", "uot_rpca_buffers", "uot_rpca_report"]
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "uot.h"\nint main(void) {\n' +
                   "".join(f'  printf("%zu\\n", sizeof({n}));\n' for n in names) + "  return 0;\n}\n")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    sizes = [int(v) for v in subprocess.check_output([str(exe)], text=True).split()]
    mirrors = [_lib.Params, _lib.Buffers, _lib.Report, _lib.DfParams, _lib.DfBuffers, _lib.DfReport,
               _lib.RpcaParams, _lib.RpcaBuffers, _lib.RpcaReport]
    for n, m, c in zip(names, mirrors, sizes):
        assert ctypes.sizeof(m) == c, (n, ctypes.sizeof(m), c)


@pytest.mark.parametrize("nx,ny,T,rho", [(64, 64, 2, math.inf), (3, 5, 2, 1.0), (6, 6, 4, 2.0), (1, 2, 2, math.inf)])
def test_default_steps_theorem1(L, nx, ny, T, rho):
    import oracle
    p = _lib.Params(nx, ny, 1, T, 1.0, rho, 0.0, 0.0, 0)
    t1, t2 = ctypes.c_double(), ctypes.c_double()
    assert L.uot_default_steps(ctypes.byref(p), 0.9, ctypes.byref(t1), ctypes.byref(t2)) == 0
    o1, o2 = oracle.default_steps(nx, ny, prox=math.isfinite(rho), n_frames=T, safety=0.9)
    assert t1.value == pytest.approx(o1, rel=1e-14) and t2.value == pytest.approx(o2, rel=1e-14)
    assert L.uot_default_steps(ctypes.byref(p), 1.5, ctypes.byref(t1), ctypes.byref(t2)) == _lib.UOT_E_INVALID


def test_scratch_size_positive(L):
    p = _lib.Params(1024, 1024, 1, 256, 2.0, math.inf, 0.0, 0.0, 0)
    n = L.uot_scratch_doubles(ctypes.byref(p))
    assert n > 255 * 8
    bad = _lib.Params(0, 4, 1, 2, 1.0, math.inf, 0, 0, 0)
    assert L.uot_scratch_doubles(ctypes.byref(bad)) == 0


def test_create_validates_and_fails_loudly_without_gpu(L):
    p = _lib.Params(8, 8, 1, 2, -1.0, math.inf, 0.0, 0.0, 0)
    b = _lib.Buffers()
    ctx = ctypes.c_void_p()
    assert L.uot_create(ctypes.byref(p), ctypes.byref(b), None, ctypes.byref(ctx)) == _lib.UOT_E_INVALID
    assert b"alpha" in L.uot_last_error(None)
    p.alpha = 1.0
    p.tau1 = p.tau2 = 0.5                   # 0.25 > 1/(lambda+1): Theorem 1 violated
    assert L.uot_create(ctypes.byref(p), ctypes.byref(b), None, ctypes.byref(ctx)) == _lib.UOT_E_INVALID
    assert b"Theorem 1" in L.uot_last_error(None)
    p.tau1 = p.tau2 = 0.0
    assert L.uot_create(ctypes.byref(p), ctypes.byref(b), None, ctypes.byref(ctx)) == _lib.UOT_E_INVALID  # NULL buffers


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle and has no torch/numpy compute path."""
    pkg = os.path.join(ROOT, "paper_1909_00149_b200")
    for name in os.listdir(pkg):
        if name.endswith(".py"):
            src = open(os.path.join(pkg, name)).read()
            assert "import oracle" not in src and "from oracle" not in src, name
