"""paper_2011_12984_b200 — B200-native N_Vector kernels, batched block-diagonal
LU and the advection–reaction Newton driver of arXiv 2011.12984 (SUNDIALS on
GPUs), behind the C ABI in include/sunbw.h.

The compute path is libsunbw.so (hand-written sm_100a CUDA); ``sunbw`` is its
ctypes binding.  Build with ``__graft_entry__.build()`` or
``python -m paper_2011_12984_b200._build``.
"""
from . import sunbw  # noqa: F401
from .sunbw import lib  # noqa: F401

__all__ = ["sunbw", "lib"]
