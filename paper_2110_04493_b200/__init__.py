"""paper_2110_04493_b200 — B200-native filtered PIM matrix exponential (arXiv 2110.04493).

The product path is libsexpm.so (include/sexpm.h: hand-written sm_100a CUDA kernels and a
C++ host driver) reached through `binding` (ctypes).  There is no CPU fallback.
"""
from . import binding  # noqa: F401
from .binding import Plan, expm, expm_host  # noqa: F401
