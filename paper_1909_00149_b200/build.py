"""Build the in-tree CUDA library libuot_b200.so for sm_100a with nvcc.

The library is compiled IN-TREE (paper_1909_00149_b200/libuot_b200.so) so the
built .so travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libuot_b200.so")
SOURCES = [os.path.join(CSRC, "uot_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, n) for n in os.listdir(CSRC) if n.endswith((".cuh", ".h", ".inc"))] + \
    [os.path.join(ROOT, "include", "uot.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2",
    "-shared", "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    extra = os.environ.get("UOT_NVCC_EXTRA", "").split()      # A/B experiments, e.g. -DUOT_PROX_MIN_BLOCKS=3
    cmd = [NVCC, *FLAGS, *extra, "-o", tmp, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libuot_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
        fh.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
