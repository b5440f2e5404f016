"""B200-native block-sparse FP64 multiply (arXiv 1910.13555 / DBCSR hot path).

The compute lives in libbtcuda.so (sm_100a CUDA, C-ABI in include/btcuda.h);
this package is the Python mirror of the reference's C++ API over it.
"""
from .store import Context, LocalStore, multiply_local, unique_id  # noqa: F401
from ._lib import (BlockTensorError, DeadlockError, GridError, InvalidArgument,  # noqa: F401
                   LayoutError, OwnershipError)

__version__ = "0.1.0"
