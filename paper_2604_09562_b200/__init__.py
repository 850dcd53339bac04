"""B200-native speculative-verify hot path of StreamServe (arXiv 2604.09562).

The product is libsv.so (CUDA kernels for sm_100a + C++ host runtime behind the
C ABI in include/sv.h); `sv` is its thin ctypes binding. No CPU fallback.
"""
from .sv import Lane, SvError, load, GREEDY, SAMPLE  # noqa: F401
