"""B200-native multi-stixel estimation hot path (arXiv 1610.04124).

The compute lives in `libstixels.so` (hand-written sm_100a CUDA behind the C ABI
of include/stixels.h); `stixels` is the thin ctypes binding.
"""
from .build import LIB, build as build_library  # noqa: F401
