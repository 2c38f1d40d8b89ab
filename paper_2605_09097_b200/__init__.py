"""B200-native (sm_100a) OS-MPM hot path (arXiv 2605.09097): see DESIGN.md.

The product is libosmpm.so (csrc/, C ABI in include/osmpm.h); `osmpm` is its
ctypes binding.  There is no CPU fallback.
"""
from . import osmpm  # noqa: F401
