"""B200-native escape-time Mandelbrot (hot path of arXiv 2007.00745).

``libmandel.so`` (built from ``csrc/`` for sm_100a) is the product; ``mandel``
is its ctypes binding with the C ABI's names (include/mandel.h).
"""
from . import mandel  # noqa: F401

__all__ = ["mandel"]
