"""B200-native (sm_100a) hot path of arXiv 1909.00149: the fused Chambolle-Pock
iteration (Algorithm 1) of the unbalanced Beckmann OT regulariser.

Layout: ``csrc/`` CUDA kernels + C-ABI (include/uot.h) built into the in-tree
``libuot_b200.so``; ``_lib`` ctypes binding; ``uot`` Problem API; ``dist``
frame-range sharding over torch.distributed; ``inputs`` seeded generators.
"""
__version__ = "0.1.0"


def build(force: bool = False) -> str:
    from .build import build as _b
    return _b(force=force)
