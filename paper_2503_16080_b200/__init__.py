"""B200-native ciphertext × plaintext matrix multiplication (arXiv 2503.16080, Algorithm 6).

The product is ``libctpt.so`` (C ABI in include/ctpt.h, CUDA for sm_100a in csrc/);
``ctpt`` is its ctypes binding and ``engine`` manages the caller-owned device buffers.
"""
from . import ctpt  # noqa: F401  (raises ImportError if the native library is missing)

__all__ = ["ctpt"]
