"""B200-native differentiable forward projector of arXiv 2404.19075 (DINR).

The product is libdinr.so (C ABI in include/dinr.h, CUDA kernels for sm_100a in csrc/);
``paper_2404_19075_b200._lib`` is its thin ctypes binding and ``synth`` the seeded input
generators shared with the tests.  Importing this package does not load the library; the
first binding call does, and fails loudly if it is missing.
"""
from . import synth  # noqa: F401

__all__ = ["synth", "lib"]


def lib():
    from . import _lib

    return _lib
