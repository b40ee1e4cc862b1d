"""B200-native adaptive speculative verification (DSD, arXiv 2511.11733).

The product is libdsdv.so (sm_100a kernels behind the C-ABI in
include/dsdv/dsdv.h) and libdsd_b200.so (the reference's `dsd::` C++ API over
it). `dsdv` is the Python binding used by the tests and bench.
"""
from . import dsdv  # noqa: F401  (fails loudly if libdsdv.so is missing)

__all__ = ["dsdv"]
