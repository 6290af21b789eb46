"""B200-native FilterGS per-frame renderer (arXiv 2603.23891 hot path).

Public surface: ``paper_2603_23891_b200.lodgs`` (the reference API mirror) over
the C ABI in ``include/lodgs_gpu.h``.
"""
from . import lodgs  # noqa: F401

__all__ = ["lodgs"]
