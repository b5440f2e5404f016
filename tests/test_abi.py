"""The C-ABI boundary (include/btcuda.h): library loads, every declared symbol
is exported and bound, status codes mirror the reference exceptions.  No
compute calls (runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "btcuda.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bt_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1910_13555_b200 import _lib
    lib = _lib.load()
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "python binding out of sync with btcuda.h"
    assert lib.bt_version() >= 1


def test_status_codes_map_reference_exceptions():
    from paper_1910_13555_b200 import _lib
    src = open(HEADER).read()
    codes = dict((k, int(v)) for k, v in re.findall(r"#define (BT_\w+) (\d+)", src))
    assert _lib._CODES[codes["BT_ERR_INVALID_ARGUMENT"]] is _lib.InvalidArgument
    assert _lib._CODES[codes["BT_ERR_OWNERSHIP"]] is _lib.OwnershipError
    assert _lib._CODES[codes["BT_ERR_GRID"]] is _lib.GridError
    assert _lib._CODES[codes["BT_ERR_DEADLOCK"]] is _lib.DeadlockError


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1910_13555_b200.store import Context
    from paper_1910_13555_b200._lib import BlockTensorError
    with pytest.raises(BlockTensorError):
        Context(0)


def test_sm100a_cubin_only():
    so = os.path.join(ROOT, "paper_1910_13555_b200", "libbtcuda.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data
