"""B200-native gSmart hot path (arXiv 2106.14038): C-ABI library libgsmart.so
(sm_100a CUDA kernels) + this thin ctypes binding.  See include/gsmart.h and
DESIGN.md.  Importing fails loudly when libgsmart.so is missing: there is no
CPU fallback.
"""
from .gsmart import *  # noqa: F401,F403
from .gsmart import Engine, Plan, GsmartError, LIB_PATH  # noqa: F401
