"""Device context and one-rank block-CSR store over the C-ABI.

``Context``     -- bt_ctx: one GPU (and, for nranks > 1, one NCCL rank).
``LocalStore``  -- bt_mat: a device-resident block-CSR tile with global block
                   indices (reference LocalStore, matrix.hpp:137-275).
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from ._lib import BtStats, check, ptr

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


def unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    check(_lib.load().bt_get_unique_id(buf), "bt_get_unique_id")
    return buf.raw


class Context:
    """One GPU; optionally rank `rank` of an `nranks` NCCL world."""

    def __init__(self, device: int = 0, nranks: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None):
        self.lib = _lib.load()
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        check(self.lib.bt_ctx_create(device, nranks, rank, idbuf, C.byref(h)), "bt_ctx_create")
        self.h = h
        self.device, self.nranks, self.rank = device, nranks, rank
        self._stores = weakref.WeakSet()

    def close(self):
        """Destroys the context; matrices still alive are released first (the
        C-ABI requires every bt_mat to go before its bt_ctx)."""
        if self.h:
            for s in list(self._stores):
                s.close()
            check(self.lib.bt_ctx_destroy(self.h), "bt_ctx_destroy")
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(self.lib.bt_ctx_sync(self.h), "bt_ctx_sync")

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        check(self.lib.bt_ctx_stream(self.h, C.byref(s)), "bt_ctx_stream")
        return s.value or 0

    def set_timing(self, on=True):
        """True / 1: multiplies report device times in their stats (and wait);
        2: events only, read with last_timing() (multiplies do not wait)."""
        check(self.lib.bt_ctx_set_timing(self.h, int(on)), "bt_ctx_set_timing")

    def last_timing(self):
        """(ms_numeric, ms_total) of the last multiply (timing mode 1 or 2)."""
        a, b = C.c_double(), C.c_double()
        check(self.lib.bt_ctx_last_timing(self.h, C.byref(a), C.byref(b)), "bt_ctx_last_timing")
        return a.value, b.value

    @property
    def kernel_count(self) -> int:
        n = C.c_int64()
        check(self.lib.bt_ctx_kernel_count(self.h, C.byref(n)), "bt_ctx_kernel_count")
        return n.value


class LocalStore:
    """A device block-CSR tile (one rank's LocalStore) with the full blockings."""

    def __init__(self, ctx: Context, row_sizes, col_sizes):
        self.ctx = ctx
        self.lib = ctx.lib
        self.rsz = np.ascontiguousarray(row_sizes, dtype=np.int32)
        self.csz = np.ascontiguousarray(col_sizes, dtype=np.int32)
        h = C.c_void_p()
        check(self.lib.bt_mat_create(ctx.h, len(self.rsz), ptr(self.rsz, _i32p), len(self.csz),
                                     ptr(self.csz, _i32p), C.byref(h)), "new_matrix")
        self.h = h
        self.owned = True
        ctx._stores.add(self)

    @classmethod
    def borrow(cls, ctx: Context, handle, row_sizes, col_sizes) -> "LocalStore":
        """Non-owning view of a store owned by a distributed matrix."""
        s = cls.__new__(cls)
        s.ctx, s.lib, s.h, s.owned = ctx, ctx.lib, handle, False
        s.rsz = np.ascontiguousarray(row_sizes, dtype=np.int32)
        s.csz = np.ascontiguousarray(col_sizes, dtype=np.int32)
        return s

    def close(self):
        if getattr(self, "h", None) and getattr(self, "owned", False) and self.ctx.h:
            self.lib.bt_mat_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- content
    def put_blocks(self, bi, bj, vals, accumulate: bool = False):
        """Batched put_block (matrix.hpp:305-309); vals compact in listed order."""
        bi = np.ascontiguousarray(bi, np.int64)
        bj = np.ascontiguousarray(bj, np.int64)
        if isinstance(vals, np.ndarray):
            v = np.ascontiguousarray(vals, np.float64)
            vp = ptr(v, _f64p)
        else:  # pinned torch tensor or raw pointer
            v = vals
            vp = C.cast(C.c_void_p(vals.data_ptr()), _f64p)
        check(self.lib.bt_mat_put_blocks(self.h, len(bi), ptr(bi, _i64p), ptr(bj, _i64p), vp,
                                         int(bool(accumulate))), "put_block")

    def put_block(self, i: int, j: int, block, accumulate: bool = False):
        b = np.ascontiguousarray(block, np.float64)
        if b.shape != (int(self.rsz[i]), int(self.csz[j])):
            from ._lib import InvalidArgument
            raise InvalidArgument(
                f"put_block: block is {b.shape[0]}x{b.shape[1] if b.ndim > 1 else 1} but slot "
                f"({i},{j}) requires {self.rsz[i]}x{self.csz[j]}")
        self.put_blocks([i], [j], b.ravel(), accumulate)

    def info(self):
        nb, ne = C.c_int64(), C.c_int64()
        check(self.lib.bt_mat_info(self.h, C.byref(nb), C.byref(ne)), "bt_mat_info")
        return nb.value, ne.value

    @property
    def nblk(self) -> int:
        return self.info()[0]

    def export(self, vals_out=None, asynchronous: bool = False):
        """Canonical (bi, bj, vals) -- vals may be a preallocated (pinned) buffer.
        asynchronous=True (bt_mat_export_async): returns once bi/bj are filled;
        the values land in `vals` by the next Context.sync()."""
        nb, ne = self.info()
        bi = np.zeros(nb, np.int64)
        bj = np.zeros(nb, np.int64)
        if vals_out is None:
            vals = np.zeros(ne, np.float64)
            vp = ptr(vals, _f64p)
        elif isinstance(vals_out, np.ndarray):
            if vals_out.dtype != np.float64 or not vals_out.flags.c_contiguous or vals_out.size < ne:
                from ._lib import InvalidArgument
                raise InvalidArgument("export: output must be a contiguous float64 array of "
                                      f"at least {ne} elements")
            vals = vals_out
            vp = ptr(vals_out, _f64p)
        else:  # torch tensor (e.g. pinned)
            vals = vals_out
            vp = C.cast(C.c_void_p(vals_out.data_ptr()), _f64p)
        fn = self.lib.bt_mat_export_async if asynchronous else self.lib.bt_mat_export
        check(fn(self.h, ptr(bi, _i64p), ptr(bj, _i64p), vp), "export")
        return bi, bj, vals

    def get_block(self, i: int, j: int):
        out = np.zeros((int(self.rsz[i]), int(self.csz[j])))
        found = C.c_int()
        check(self.lib.bt_mat_get_block(self.h, i, j, ptr(out, _f64p), C.byref(found)),
              "get_block")
        return out if found.value else None

    def norms(self):
        nb, _ = self.info()
        out = np.zeros(nb)
        check(self.lib.bt_mat_norms(self.h, ptr(out, _f64p)), "norms")
        return out

    def clear(self):
        check(self.lib.bt_mat_clear(self.h), "clear")

    def copy_from(self, other: "LocalStore"):
        check(self.lib.bt_mat_copy(other.h, self.h), "copy")

    def filter(self, eps: float, band: float = 1e-12) -> dict:
        """Post-filter: drops blocks with ||C_ij||_F < eps.  Returns
        {"dropped": n, "borderline": n} -- borderline blocks have
        | ||C_ij|| - eps | <= band * eps."""
        d, b = C.c_int64(), C.c_int64()
        check(self.lib.bt_filter_report(self.h, eps, band, C.byref(d), C.byref(b)), "filter")
        return {"dropped": d.value, "borderline": b.value}


def multiply_local(ctx: Context, a: LocalStore, b: LocalStore, c: LocalStore,
                   eps: float = 0.0) -> dict:
    """C += A*B on one device (multiply_tiles_into, multiply_cannon.hpp:24-44)."""
    st = BtStats()
    check(ctx.lib.bt_multiply(ctx.h, a.h, b.h, c.h, eps, C.byref(st)), "multiply")
    return st.as_dict()
