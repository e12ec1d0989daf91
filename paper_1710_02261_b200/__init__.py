"""B200-native P-Tucker (arXiv 1710.02261) row-wise ALS hot path.

The product is the C-ABI library libptucker.so (include/ptucker.h) built from
csrc/ for sm_100a; `ptucker` is its thin ctypes binding.
"""
from . import ptucker  # noqa: F401
