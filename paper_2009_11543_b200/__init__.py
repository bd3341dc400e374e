"""B200-native compressed key sort (arXiv 2009.11543): the hot path of index
reconstruction -- distinction-bit mask, bit-gather compression, LSD radix sort of
(compressed key, row id), bottom-up bulk load -- as CUDA kernels for sm_100a behind
the C ABI in include/cks.h. `cks` is the ctypes binding."""
from . import cks  # noqa: F401

__all__ = ["cks"]
