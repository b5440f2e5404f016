"""ctypes front-end for the test-only oracles.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package.

* ``Oracle``    -> oracle/liboracle.so, the C restatement (bt_oracle.c).
* ``Reference`` -> oracle/_ref/libbtref.so, the unmodified reference headers
  compiled through ref_shim.cpp (built here from /root/reference; the built .so
  travels to the GPU box, the reference tree does not).

Matrices cross this boundary as ``Blocks`` -- canonical (i, j)-sorted block
lists with compact row-major values, the same form libbtcuda's bt_mat_export
produces, so comparisons are plain array equality.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Blocks:
    """Canonical block list: blockings + sorted (bi, bj) + concatenated values."""

    rsz: np.ndarray  # int32 [nbr]
    csz: np.ndarray  # int32 [nbc]
    bi: np.ndarray  # int64 [nblk]
    bj: np.ndarray  # int64 [nblk]
    vals: np.ndarray  # float64 [sum of block sizes]

    @property
    def nblk(self) -> int:
        return int(self.bi.shape[0])

    def offsets(self) -> np.ndarray:
        sz = self.rsz[self.bi].astype(np.int64) * self.csz[self.bj].astype(np.int64)
        off = np.zeros(self.nblk + 1, dtype=np.int64)
        np.cumsum(sz, out=off[1:])
        return off

    def block(self, t: int) -> np.ndarray:
        off = self.offsets()
        m, n = int(self.rsz[self.bi[t]]), int(self.csz[self.bj[t]])
        return self.vals[off[t]:off[t + 1]].reshape(m, n)

    def to_dense(self) -> np.ndarray:
        ro = np.concatenate([[0], np.cumsum(self.rsz)]).astype(np.int64)
        co = np.concatenate([[0], np.cumsum(self.csz)]).astype(np.int64)
        out = np.zeros((ro[-1], co[-1]))
        off = self.offsets()
        for t in range(self.nblk):
            i, j = int(self.bi[t]), int(self.bj[t])
            m, n = int(self.rsz[i]), int(self.csz[j])
            out[ro[i]:ro[i] + m, co[j]:co[j] + n] = self.vals[off[t]:off[t + 1]].reshape(m, n)
        return out

    @staticmethod
    def empty(rsz, csz) -> "Blocks":
        return Blocks(np.asarray(rsz, np.int32), np.asarray(csz, np.int32),
                      np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))


class _BtoMat(C.Structure):
    _fields_ = [("nbr", C.c_int64), ("nbc", C.c_int64), ("rsz", _i32p), ("csz", _i32p),
                ("nblk", C.c_int64), ("row_ptr", _i64p), ("col", _i64p), ("off", _i64p),
                ("vals", _f64p), ("nvals", C.c_int64)]


class Oracle:
    """The C restatement of the reference path (oracle/bt_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.bto_mat_free.argtypes = [C.POINTER(_BtoMat)]
        L.bto_mat_from_blocks.argtypes = [C.POINTER(_BtoMat), C.c_int64, _i32p, C.c_int64, _i32p,
                                          C.c_int64, _i64p, _i64p, _f64p]
        L.bto_mat_empty.argtypes = [C.POINTER(_BtoMat), C.c_int64, _i32p, C.c_int64, _i32p]
        L.bto_random_matrix.argtypes = [C.POINTER(_BtoMat), C.c_uint64, C.c_int64, _i32p,
                                        C.c_int64, _i32p, C.c_double, C.c_double]
        L.bto_multiply.argtypes = [C.POINTER(_BtoMat), C.POINTER(_BtoMat), C.POINTER(_BtoMat),
                                   C.c_double, _i64p, _f64p]
        L.bto_filter.argtypes = [C.POINTER(_BtoMat), C.c_double]
        L.bto_block_norm.argtypes = [_f64p, C.c_int, C.c_int]
        L.bto_block_norm.restype = C.c_double
        L.bto_block_gemm_acc.argtypes = [_f64p, _f64p, _f64p, C.c_int, C.c_int, C.c_int]
        L.bto_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.bto_rng_next.argtypes = [C.c_void_p]
        L.bto_rng_next.restype = C.c_uint64
        L.bto_rng_normal.argtypes = [C.c_void_p]
        L.bto_rng_normal.restype = C.c_double
        L.bto_rng_uniform_int.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.bto_rng_uniform_int.restype = C.c_int64
        L.bto_random_blocking.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, _i32p,
                                          C.c_int64]
        L.bto_random_blocking.restype = C.c_int64
        L.bto_mixed_radix.argtypes = [_i64p, _i64p, C.c_int]
        L.bto_mixed_radix.restype = C.c_int64
        L.bto_mixed_radix_inv.argtypes = [C.c_int64, _i64p, C.c_int, _i64p]

    # -- conversion helpers
    def _from(self, m: _BtoMat) -> Blocks:
        nbr, nbc, nblk = m.nbr, m.nbc, m.nblk
        rsz = np.ctypeslib.as_array(m.rsz, (nbr,)).copy() if nbr else np.zeros(0, np.int32)
        csz = np.ctypeslib.as_array(m.csz, (nbc,)).copy() if nbc else np.zeros(0, np.int32)
        rp = np.ctypeslib.as_array(m.row_ptr, (nbr + 1,)).copy()
        bj = np.ctypeslib.as_array(m.col, (nblk,)).copy() if nblk else np.zeros(0, np.int64)
        bi = np.repeat(np.arange(nbr, dtype=np.int64), np.diff(rp))
        vals = np.ctypeslib.as_array(m.vals, (m.nvals,)).copy() if m.nvals else np.zeros(0)
        return Blocks(rsz, csz, bi, bj, vals)

    def _to(self, b: Blocks) -> _BtoMat:
        m = _BtoMat()
        rsz = np.ascontiguousarray(b.rsz, np.int32)
        csz = np.ascontiguousarray(b.csz, np.int32)
        bi = np.ascontiguousarray(b.bi, np.int64)
        bj = np.ascontiguousarray(b.bj, np.int64)
        v = np.ascontiguousarray(b.vals, np.float64)
        rc = self.lib.bto_mat_from_blocks(C.byref(m), len(rsz), _p(rsz, _i32p), len(csz),
                                          _p(csz, _i32p), len(bi), _p(bi, _i64p),
                                          _p(bj, _i64p), _p(v, _f64p))
        if rc:
            raise ValueError(f"bto_mat_from_blocks failed ({rc})")
        return m

    # -- API
    def random_matrix(self, seed, rsz, csz, occ, scale_exp=0.0) -> Blocks:
        rsz = np.ascontiguousarray(rsz, np.int32)
        csz = np.ascontiguousarray(csz, np.int32)
        m = _BtoMat()
        rc = self.lib.bto_random_matrix(C.byref(m), seed, len(rsz), _p(rsz, _i32p), len(csz),
                                        _p(csz, _i32p), occ, scale_exp)
        if rc:
            raise ValueError(f"bto_random_matrix failed ({rc})")
        out = self._from(m)
        self.lib.bto_mat_free(C.byref(m))
        return out

    def multiply(self, a: Blocks, b: Blocks, c: Blocks, eps: float = 0.0):
        """Returns (C_out, executed products, useful flops)."""
        ma, mb, mc = self._to(a), self._to(b), self._to(c)
        npd = C.c_int64(0)
        fl = C.c_double(0)
        rc = self.lib.bto_multiply(C.byref(ma), C.byref(mb), C.byref(mc), eps, C.byref(npd),
                                   C.byref(fl))
        try:
            if rc:
                raise ValueError(f"bto_multiply: nonconformal operands ({rc})")
            return self._from(mc), npd.value, fl.value
        finally:
            for m in (ma, mb, mc):
                self.lib.bto_mat_free(C.byref(m))

    def filter(self, c: Blocks, eps: float) -> Blocks:
        mc = self._to(c)
        self.lib.bto_filter(C.byref(mc), eps)
        out = self._from(mc)
        self.lib.bto_mat_free(C.byref(mc))
        return out

    def norms(self, c: Blocks) -> np.ndarray:
        """Block Frobenius norms in canonical order (bto_block_norm: sequential,
        unfused row sums -- the filter's definition)."""
        off = c.offsets()
        v = np.ascontiguousarray(c.vals, np.float64)
        out = np.zeros(c.nblk)
        for t in range(c.nblk):
            m, n = int(c.rsz[c.bi[t]]), int(c.csz[c.bj[t]])
            out[t] = self.lib.bto_block_norm(v[off[t]:].ctypes.data_as(_f64p), m, n)
        return out

    def block_gemm_acc(self, c, a, b):
        c = np.ascontiguousarray(c, np.float64).copy()
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        m, k = a.shape
        n = b.shape[1]
        self.lib.bto_block_gemm_acc(_p(c, _f64p), _p(a, _f64p), _p(b, _f64p), m, n, k)
        return c

    def rng(self, seed):
        buf = C.create_string_buffer(312 * 8 + 16)
        self.lib.bto_rng_seed(buf, seed)
        return buf

    def random_blocking(self, seed, total, bmin, bmax):
        out = np.zeros(total + 1, np.int32)
        n = self.lib.bto_random_blocking(seed, total, bmin, bmax, _p(out, _i32p), len(out))
        return out[:n].copy()

    def mixed_radix(self, coords, extents) -> int:
        c = np.ascontiguousarray(coords, np.int64)
        e = np.ascontiguousarray(extents, np.int64)
        return int(self.lib.bto_mixed_radix(_p(c, _i64p), _p(e, _i64p), len(e)))

    def mixed_radix_inv(self, idx, extents):
        e = np.ascontiguousarray(extents, np.int64)
        out = np.zeros(len(e), np.int64)
        self.lib.bto_mixed_radix_inv(idx, _p(e, _i64p), len(e), _p(out, _i64p))
        return out


class Reference:
    """The unmodified reference compiled from /root/reference (oracle/_ref/libbtref.so)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libbtref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_block_gemm_acc.argtypes = [_f64p, _f64p, _f64p, C.c_int, C.c_int, C.c_int]
        L.ref_random_matrix.argtypes = [C.c_uint64, C.c_int64, _i32p, C.c_int64, _i32p,
                                        C.c_double]
        L.ref_random_matrix.restype = C.c_void_p
        L.ref_multiply.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int64, _i32p, C.c_int64, _i32p, C.c_int64, _i32p,
                                   C.c_int64, _i64p, _i64p, _f64p,
                                   C.c_int64, _i64p, _i64p, _f64p,
                                   C.c_int64, _i64p, _i64p, _f64p]
        L.ref_multiply.restype = C.c_void_p
        for f in ("ref_res_nblk", "ref_res_nvals"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_int64
        L.ref_res_seconds.argtypes = [C.c_void_p]
        L.ref_res_seconds.restype = C.c_double
        L.ref_res_nranks.argtypes = [C.c_void_p]
        L.ref_res_copy.argtypes = [C.c_void_p, _i64p, _i64p, _f64p]
        L.ref_res_ledger.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int]
        L.ref_res_ledger.restype = C.c_int64
        L.ref_res_free.argtypes = [C.c_void_p]
        L.ref_cost.argtypes = [C.c_int] + [C.c_double] * 7
        L.ref_cost.restype = C.c_double
        L.ref_io_write.argtypes = [C.c_char_p, C.c_int, C.c_int64, _i32p, C.c_int64, _i32p,
                                   C.c_int64, _i64p, _i64p, _f64p]
        L.ref_io_read.argtypes = [C.c_char_p, C.c_int]
        L.ref_io_read.restype = C.c_void_p

    def _err(self):
        return self.lib.ref_last_error().decode()

    def _take(self, h, rsz, csz) -> Blocks:
        if not h:
            raise RuntimeError(self._err())
        n = self.lib.ref_res_nblk(h)
        nv = self.lib.ref_res_nvals(h)
        bi = np.zeros(n, np.int64)
        bj = np.zeros(n, np.int64)
        v = np.zeros(nv)
        self.lib.ref_res_copy(h, _p(bi, _i64p), _p(bj, _i64p), _p(v, _f64p))
        return Blocks(np.asarray(rsz, np.int32), np.asarray(csz, np.int32), bi, bj, v)

    def block_gemm_acc(self, c, a, b):
        c = np.ascontiguousarray(c, np.float64).copy()
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        m, k = a.shape
        n = b.shape[1]
        if self.lib.ref_block_gemm_acc(_p(c, _f64p), _p(a, _f64p), _p(b, _f64p), m, n, k):
            raise ValueError(self._err())
        return c

    def random_matrix(self, seed, rsz, csz, occ) -> Blocks:
        rsz = np.ascontiguousarray(rsz, np.int32)
        csz = np.ascontiguousarray(csz, np.int32)
        h = self.lib.ref_random_matrix(seed, len(rsz), _p(rsz, _i32p), len(csz), _p(csz, _i32p),
                                       occ)
        try:
            return self._take(h, rsz, csz)
        finally:
            if h:
                self.lib.ref_res_free(h)

    ALGOS = {"cannon": 0, "case1": 1, "case2": 2}

    def multiply(self, a: Blocks, b: Blocks, c: Blocks, algo="cannon", grid_q=1, nprocs=1,
                 sequential=False):
        """Runs the reference multiply_dispatch; returns (C_out, seconds, ledger dict)."""
        args = []
        m_sz = np.ascontiguousarray(a.rsz, np.int32)
        k_sz = np.ascontiguousarray(a.csz, np.int32)
        n_sz = np.ascontiguousarray(b.csz, np.int32)
        keep = []
        for x in (a, b, c):
            bi = np.ascontiguousarray(x.bi, np.int64)
            bj = np.ascontiguousarray(x.bj, np.int64)
            v = np.ascontiguousarray(x.vals, np.float64)
            keep += [bi, bj, v]
            args += [len(bi), _p(bi, _i64p), _p(bj, _i64p), _p(v, _f64p)]
        h = self.lib.ref_multiply(self.ALGOS[algo], grid_q, nprocs, int(sequential),
                                  len(m_sz), _p(m_sz, _i32p), len(k_sz), _p(k_sz, _i32p),
                                  len(n_sz), _p(n_sz, _i32p), *args)
        if not h:
            raise RuntimeError(self._err())
        try:
            out = self._take(h, m_sz, n_sz)
            secs = self.lib.ref_res_seconds(h)
            nr = self.lib.ref_res_nranks(h)
            ledger = {}
            for r in range(nr):
                ledger[r] = {w: self.lib.ref_res_ledger(h, r, None, i)
                             for i, w in enumerate(("sent", "received", "meta_sent",
                                                    "meta_received"))}
                for ph in ("cannon", "multiply", "reduce", "collect", "ring", "redistribute"):
                    s = self.lib.ref_res_ledger(h, r, ph.encode(), 0)
                    if s:
                        ledger[r]["sent:" + ph] = s
            return out, secs, ledger
        finally:
            self.lib.ref_res_free(h)

    def cost(self, which, m, n, k, oa, ob, oc, p) -> float:
        return self.lib.ref_cost(which, m, n, k, oa, ob, oc, p)

    # -- fixture I/O with the reference's own io.hpp (fmt "text" | "binary")
    def write_matrix_file(self, path: str, b: Blocks, fmt: str = "binary"):
        rsz = np.ascontiguousarray(b.rsz, np.int32)
        csz = np.ascontiguousarray(b.csz, np.int32)
        bi = np.ascontiguousarray(b.bi, np.int64)
        bj = np.ascontiguousarray(b.bj, np.int64)
        v = np.ascontiguousarray(b.vals, np.float64)
        if self.lib.ref_io_write(path.encode(), int(fmt == "binary"), len(rsz), _p(rsz, _i32p),
                                 len(csz), _p(csz, _i32p), len(bi), _p(bi, _i64p),
                                 _p(bj, _i64p), _p(v, _f64p)):
            raise RuntimeError(self._err())

    def read_matrix_file(self, path: str, fmt: str = "binary") -> Blocks:
        h = self.lib.ref_io_read(path.encode(), int(fmt == "binary"))
        if not h:
            raise RuntimeError(self._err())
        try:
            # blockings from the file header (the reader validated them)
            rsz, csz = _file_blockings(path, fmt)
            return self._take(h, rsz, csz)
        finally:
            self.lib.ref_res_free(h)


def _file_blockings(path, fmt):
    if fmt == "binary":
        raw = open(path, "rb").read(32)
        nbr, nbc = np.frombuffer(raw, "<i8")[2:4]
        data = np.fromfile(path, "<i8", count=4 + int(nbr) + int(nbc))
        return data[4:4 + nbr].astype(np.int32), data[4 + nbr:].astype(np.int32)
    with open(path) as f:
        nbr, nbc = [int(x) for x in f.readline().split()][2:4]
        rs = np.array(f.readline().split(), np.int32) if nbr else np.zeros(0, np.int32)
        cs = np.array(f.readline().split(), np.int32) if nbc else np.zeros(0, np.int32)
    return rs, cs
