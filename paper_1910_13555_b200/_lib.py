"""ctypes binding of libbtcuda.so (the C-ABI in include/btcuda.h).

The product path: every call goes to the sm_100a library; there is no CPU
fallback.  Loading fails loudly when the library is missing or cannot find a
B200.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbtcuda.so")

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


# ---- exceptions: errors.hpp:14-53 ----------------------------------------
class BlockTensorError(RuntimeError):
    """blocktensor::error (errors.hpp:14-17)."""


class InvalidArgument(BlockTensorError, ValueError):
    """blocktensor::invalid_argument (errors.hpp:20-23)."""


class OwnershipError(BlockTensorError):
    """blocktensor::ownership_error (errors.hpp:26-29)."""


class GridError(BlockTensorError):
    """blocktensor::grid_error (errors.hpp:32-35)."""


class LayoutError(BlockTensorError):
    """blocktensor::layout_error (errors.hpp:39-47); carries the dimension name."""

    def __init__(self, dimension: str, what: str):
        super().__init__(what)
        self.dimension = dimension


class DeadlockError(BlockTensorError):
    """blocktensor::deadlock_error (errors.hpp:50-53)."""


class DeviceError(BlockTensorError):
    """CUDA / NCCL / device-allocation failure."""


_CODES = {1: InvalidArgument, 2: OwnershipError, 3: GridError, 5: DeadlockError,
          10: DeviceError, 11: DeviceError, 12: DeviceError, 13: BlockTensorError}


class BtStats(C.Structure):
    _fields_ = [("candidates", C.c_int64), ("products", C.c_int64), ("flops", C.c_double),
                ("c_blocks_in", C.c_int64), ("c_blocks_out", C.c_int64),
                ("elements_sent", C.c_int64), ("elements_received", C.c_int64),
                ("meta_sent", C.c_int64), ("meta_received", C.c_int64),
                ("kernels", C.c_int32), ("reserved", C.c_int32),
                ("ms_numeric", C.c_double), ("ms_total", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


# name -> (restype, argtypes); every symbol include/btcuda.h declares
SIGNATURES = {
    "bt_last_error": (C.c_char_p, []),
    "bt_version": (C.c_int, []),
    "bt_get_unique_id": (C.c_int, [C.c_void_p]),
    "bt_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "bt_ctx_destroy": (C.c_int, [C.c_void_p]),
    "bt_ctx_split": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "bt_ctx_sync": (C.c_int, [C.c_void_p]),
    "bt_ctx_rank": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "bt_ctx_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "bt_ctx_kernel_count": (C.c_int, [C.c_void_p, _i64p]),
    "bt_ctx_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "bt_ctx_last_timing": (C.c_int, [C.c_void_p, _f64p, _f64p]),
    "bt_mat_create": (C.c_int, [C.c_void_p, C.c_int64, _i32p, C.c_int64, _i32p,
                                C.POINTER(C.c_void_p)]),
    "bt_mat_destroy": (C.c_int, [C.c_void_p]),
    "bt_mat_clear": (C.c_int, [C.c_void_p]),
    "bt_mat_copy": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bt_mat_put_blocks": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _i64p, _f64p, C.c_int]),
    "bt_mat_info": (C.c_int, [C.c_void_p, _i64p, _i64p]),
    "bt_mat_export": (C.c_int, [C.c_void_p, _i64p, _i64p, _f64p]),
    "bt_mat_export_async": (C.c_int, [C.c_void_p, _i64p, _i64p, _f64p]),
    "bt_mat_get_block": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, _f64p,
                                   C.POINTER(C.c_int)]),
    "bt_mat_norms": (C.c_int, [C.c_void_p, _f64p]),
    "bt_multiply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                              C.POINTER(BtStats)]),
    "bt_filter": (C.c_int, [C.c_void_p, C.c_double]),
    "bt_filter_report": (C.c_int, [C.c_void_p, C.c_double, C.c_double, _i64p, _i64p]),
    "bt_grid_create": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "bt_grid_destroy": (C.c_int, [C.c_void_p]),
    "bt_grid_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int)]),
    "bt_grid_ledger": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_int, _i64p]),
    "bt_grid_reset_ledger": (C.c_int, [C.c_void_p]),
    "bt_grid_sum": (C.c_int, [C.c_void_p, _i64p, C.c_int]),
    "bt_dmat_create": (C.c_int, [C.c_void_p, C.c_int64, _i32p, C.c_int64, _i32p, C.c_int,
                                 C.c_int, _i32p, _i32p, C.POINTER(C.c_void_p)]),
    "bt_dmat_destroy": (C.c_int, [C.c_void_p]),
    "bt_dmat_local": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "bt_dmat_owner": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_int)]),
    "bt_dmat_put_blocks": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _i64p, _f64p, C.c_int]),
    "bt_redistribute": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_char_p]),
    "bt_multiply_cannon": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                     C.POINTER(BtStats)]),
    "bt_multiply_case1": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                    C.POINTER(BtStats)]),
    "bt_multiply_case2": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                    C.c_double, C.POINTER(BtStats)]),
    "bt_tensor_remap": (C.c_int, [C.c_void_p, C.c_int, _i64p, C.POINTER(_i32p), C.c_int,
                                  C.POINTER(C.c_int), C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                  C.c_void_p]),
}

_lib = None


def load(path: str | None = None) -> C.CDLL:
    """Loads libbtcuda.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("BT_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(f"{p} not built: run `make -C paper_1910_13555_b200/csrc` "
                          "(or __graft_entry__.build())")
    lib = C.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = load().bt_last_error().decode(errors="replace")
    cls = _CODES.get(rc, BlockTensorError)
    raise cls(f"{what}: {msg}" if what else msg)


def ptr(a, t):
    return a.ctypes.data_as(t)
