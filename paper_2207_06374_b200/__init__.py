"""B200-native TRST-MI hot path (arXiv 2207.06374).

Kernels: paper_2207_06374_b200/csrc (CUDA, sm_100a) behind the C ABI in
include/trstmi_b200.h.  Python binding: api.py (ctypes).  Layouts: abi.py.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
