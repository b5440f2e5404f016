"""Block-sparse tensors and contraction (the reference has no
tensor code, so this module follows the spec text).

A rank-n tensor (2 <= n <= 4) is stored as a device matrix (``LocalStore``)
under a matricization map (row-group dims, col-group dims); block and element
indices are mixed radix with later-listed dimensions fastest (SPEC.md:505-513,
533).  ``contract`` brings the operands into contraction-compatible maps with
the device index-remap kernel (``bt_tensor_remap``), runs the block-sparse
multiply, and remaps C back if needed -- all on the GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import InvalidArgument, check, ptr
from .store import Context, LocalStore, multiply_local

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


def mixed_radix(coords, extents) -> int:
    """later dimensions vary fastest."""
    idx = 0
    for c, e in zip(coords, extents):
        if c < 0 or c >= e:
            raise InvalidArgument("tensor index out of range")
        idx = idx * e + c
    return idx


def mixed_radix_inv(idx, extents):
    out = [0] * len(extents)
    for d in range(len(extents) - 1, -1, -1):
        out[d] = idx % extents[d]
        idx //= extents[d]
    return out


def _group_sizes(dim_sizes, dims):
    """block sizes of a matricized dimension group, in mixed-radix order"""
    out = np.ones(1, dtype=np.int64)
    for d in dims:
        out = np.multiply.outer(out, dim_sizes[d]).ravel()
    return out.astype(np.int32)


class SparseTensor:
    """SPEC.md:487-493 on one GPU: per-dimension blockings + matricization map."""

    def __init__(self, ctx: Context, blockings, row_dims, col_dims):
        self.ctx = ctx
        self.sizes = [np.ascontiguousarray(b, np.int32) for b in blockings]
        n = len(self.sizes)
        if not 2 <= n <= 4:
            raise InvalidArgument("tensor: rank must be in [2, 4]")
        row_dims, col_dims = list(row_dims), list(col_dims)
        if (sorted(row_dims + col_dims) != list(range(n)) or not row_dims or not col_dims):
            raise InvalidArgument("tensor: map is not a partition of the dimensions into two "
                                  "non-empty groups")
        self.row_dims, self.col_dims = row_dims, col_dims
        self.nb = [len(s) for s in self.sizes]
        self.store = LocalStore(ctx, _group_sizes(self.sizes, row_dims),
                                _group_sizes(self.sizes, col_dims))

    @property
    def rank(self):
        return len(self.sizes)

    def to_matrix_index(self, coords):
        """tensor_to_matrix_index."""
        r = mixed_radix([coords[d] for d in self.row_dims], [self.nb[d] for d in self.row_dims])
        c = mixed_radix([coords[d] for d in self.col_dims], [self.nb[d] for d in self.col_dims])
        return r, c

    def from_matrix_index(self, row, col):
        out = [0] * self.rank
        for d, v in zip(self.row_dims, mixed_radix_inv(row, [self.nb[d] for d in self.row_dims])):
            out[d] = v
        for d, v in zip(self.col_dims, mixed_radix_inv(col, [self.nb[d] for d in self.col_dims])):
            out[d] = v
        return out

    def block_shape(self, coords):
        return tuple(int(self.sizes[d][coords[d]]) for d in range(self.rank))

    def _to_mat_block(self, block):
        R = int(np.prod([block.shape[d] for d in self.row_dims]))
        return np.transpose(block, self.row_dims + self.col_dims).reshape(R, -1)

    def put_blocks(self, items, accumulate=False):
        """items: iterable of (coords, tensor-shaped block)."""
        bi, bj, vals = [], [], []
        for coords, blk in items:
            blk = np.asarray(blk, np.float64)
            if blk.shape != self.block_shape(coords):
                raise InvalidArgument(f"put_block: block shape {blk.shape} != "
                                      f"{self.block_shape(coords)}")
            r, c = self.to_matrix_index(coords)
            bi.append(r)
            bj.append(c)
            vals.append(self._to_mat_block(blk).ravel())
        if bi:
            self.store.put_blocks(np.array(bi), np.array(bj), np.concatenate(vals), accumulate)

    def put_block(self, coords, block, accumulate=False):
        self.put_blocks([(coords, block)], accumulate)

    def get_block(self, coords):
        r, c = self.to_matrix_index(coords)
        m = self.store.get_block(r, c)
        if m is None:
            return None
        shape = self.block_shape(coords)
        perm = self.row_dims + self.col_dims
        t = m.reshape([shape[d] for d in perm])
        return np.transpose(t, np.argsort(perm))

    def blocks(self):
        bi, bj, vals = self.store.export()
        off = 0
        for r, c in zip(bi, bj):
            coords = self.from_matrix_index(int(r), int(c))
            shape = self.block_shape(coords)
            n = int(np.prod(shape))
            perm = self.row_dims + self.col_dims
            t = vals[off:off + n].reshape([shape[d] for d in perm])
            off += n
            yield coords, np.transpose(t, np.argsort(perm))

    def to_dense(self):
        offs = [np.concatenate([[0], np.cumsum(s)]) for s in self.sizes]
        out = np.zeros([int(o[-1]) for o in offs])
        for coords, blk in self.blocks():
            sl = tuple(slice(offs[d][c], offs[d][c] + blk.shape[d]) for d, c in enumerate(coords))
            out[sl] = blk
        return out

    def remap_into_store(self, out: "SparseTensor"):
        """out := this tensor under out's map (device remap kernel)."""
        _remap_store(self.ctx, self.sizes, self.nb, self.store, self.row_dims, self.col_dims,
                     out.store, out.row_dims, out.col_dims)

    def remap(self, row_dims, col_dims) -> "SparseTensor":
        """The same tensor under another map, via the device remap kernel."""
        out = SparseTensor(self.ctx, self.sizes, row_dims, col_dims)
        nb = np.ascontiguousarray(self.nb, np.int64)
        arrs = (_i32p * self.rank)(*[ptr(s, _i32p) for s in self.sizes])
        src = (C.c_int * self.rank)(*(self.row_dims + self.col_dims))
        dst = (C.c_int * self.rank)(*(list(row_dims) + list(col_dims)))
        check(self.ctx.lib.bt_tensor_remap(self.ctx.h, self.rank, ptr(nb, _i64p), arrs,
                                           len(self.row_dims), src, self.store.h,
                                           len(row_dims), dst, out.store.h), "tensor_remap")
        return out


def contract(a: SparseTensor, b: SparseTensor, contract_a, contract_b, c: SparseTensor,
             eps: float = 0.0) -> dict:
    """C += sum over (A dims contract_a) == (B dims contract_b) of A*B.

    C's dimensions are A's retained dimensions (ascending) followed by B's.
    Operands already in compatible maps are used as they are ("the
    redistribution step can be skipped"); otherwise they are
    remapped on the device first, and C is remapped back to its own map."""
    contract_a, contract_b = list(contract_a), list(contract_b)
    if len(contract_a) != len(contract_b) or not contract_a:
        raise InvalidArgument("contract: contracted index lists must be non-empty and equal "
                              "in length")
    for da, db in zip(contract_a, contract_b):
        if not np.array_equal(a.sizes[da], b.sizes[db]):
            raise InvalidArgument("contract: blockings of contracted indices differ")
    ra = [d for d in range(a.rank) if d not in contract_a]
    rb = [d for d in range(b.rank) if d not in contract_b]
    if c.rank != len(ra) + len(rb):
        raise InvalidArgument("contract: C rank does not match the retained indices")
    for q, (t, d) in enumerate([(a, d) for d in ra] + [(b, d) for d in rb]):
        if not np.array_equal(c.sizes[q], t.sizes[d]):
            raise InvalidArgument("contract: C blockings do not match the retained indices")
    am = a if (a.row_dims == ra and a.col_dims == contract_a) else a.remap(ra, contract_a)
    bm = b if (b.row_dims == contract_b and b.col_dims == rb) else b.remap(contract_b, rb)
    crow, ccol = list(range(len(ra))), list(range(len(ra), c.rank))
    compatible = c.row_dims == crow and c.col_dims == ccol
    cm = c if compatible else c.remap(crow, ccol)
    st = multiply_local(a.ctx, am.store, bm.store, cm.store, eps)
    if not compatible:
        back = cm.remap(c.row_dims, c.col_dims)
        c.store.copy_from(back.store)
    return st


# --------------------------------------------------------------------------
# Distributed tensors: the backing matrix is a DistMatrix over the process
# group.  The spec's n-dimensional tensor grid is folded onto
# the 2-D grid of the backing matrix: a tensor block is owned by the owner of
# its matricized (row, col) block under round-robin row/column distributions
# (DESIGN.md 3).  Remaps between matricization maps are a local device remap
# of every rank's store followed by a redistribution to the new owners, whose
# volume is charged to the ledger under phase "tensor_remap".

def _remap_store(ctx, sizes, nb, src_store, src_rows, src_cols, dst_store, dst_rows, dst_cols):
    n = len(sizes)
    nbv = np.ascontiguousarray(nb, np.int64)
    arrs = (_i32p * n)(*[ptr(s, _i32p) for s in sizes])
    src = (C.c_int * n)(*(list(src_rows) + list(src_cols)))
    dst = (C.c_int * n)(*(list(dst_rows) + list(dst_cols)))
    check(ctx.lib.bt_tensor_remap(ctx.h, n, ptr(nbv, _i64p), arrs, len(src_rows), src,
                                  src_store.h, len(dst_rows), dst, dst_store.h), "tensor_remap")


class DistTensor:
    """A block-sparse tensor (rank 2..4) distributed over a SimComm's ranks."""

    def __init__(self, comm, blockings, row_dims, col_dims, grid=None):
        from . import dist as dd
        self.comm = comm
        self.sizes = [np.ascontiguousarray(b, np.int32) for b in blockings]
        n = len(self.sizes)
        if not 2 <= n <= 4:
            raise InvalidArgument("tensor: rank must be in [2, 4]")
        row_dims, col_dims = list(row_dims), list(col_dims)
        if sorted(row_dims + col_dims) != list(range(n)) or not row_dims or not col_dims:
            raise InvalidArgument("tensor: map is not a partition of the dimensions into two "
                                  "non-empty groups")
        self.row_dims, self.col_dims = row_dims, col_dims
        self.nb = [len(s) for s in self.sizes]
        self.grid = grid or comm.grid()
        if self.grid.ndims() != 2:
            raise InvalidArgument("DistTensor: the backing matrix grid must be 2-dimensional")
        self.mat = dd.new_matrix_round_robin(
            dd.Blocking(_group_sizes(self.sizes, row_dims)),
            dd.Blocking(_group_sizes(self.sizes, col_dims)), self.grid, comm)

    @property
    def rank(self):
        return len(self.sizes)

    def _like(self, row_dims, col_dims) -> "DistTensor":
        return DistTensor(self.comm, self.sizes, row_dims, col_dims, self.grid)

    def to_matrix_index(self, coords):
        r = mixed_radix([coords[d] for d in self.row_dims], [self.nb[d] for d in self.row_dims])
        c = mixed_radix([coords[d] for d in self.col_dims], [self.nb[d] for d in self.col_dims])
        return r, c

    def from_matrix_index(self, row, col):
        out = [0] * self.rank
        for d, v in zip(self.row_dims, mixed_radix_inv(row, [self.nb[d] for d in self.row_dims])):
            out[d] = v
        for d, v in zip(self.col_dims, mixed_radix_inv(col, [self.nb[d] for d in self.col_dims])):
            out[d] = v
        return out

    def block_shape(self, coords):
        return tuple(int(self.sizes[d][coords[d]]) for d in range(self.rank))

    def owner_rank(self, coords):
        return self.mat.owner_rank(*self.to_matrix_index(coords))

    def put_blocks(self, items, owned_only: bool = True, accumulate: bool = False):
        """items: (coords, tensor-shaped block); with owned_only the blocks owned
        by another process are skipped (each process puts its own share)."""
        local = set(self.comm.local_ranks())
        bi, bj, vals = [], [], []
        perm = self.row_dims + self.col_dims
        for coords, blk in items:
            blk = np.asarray(blk, np.float64)
            if blk.shape != self.block_shape(coords):
                raise InvalidArgument(f"put_block: block shape {blk.shape} != "
                                      f"{self.block_shape(coords)}")
            r, c = self.to_matrix_index(coords)
            if owned_only and self.mat.owner_rank(r, c) not in local:
                continue
            bi.append(r)
            bj.append(c)
            R = int(np.prod([blk.shape[d] for d in self.row_dims]))
            vals.append(np.transpose(blk, perm).reshape(R, -1).ravel())
        if bi:
            self.mat.put_blocks(np.array(bi), np.array(bj), np.concatenate(vals), accumulate)

    def blocks(self):
        """(coords, block) of every block held by this process's ranks."""
        bi, bj, vals = self.mat.blocks()
        perm = self.row_dims + self.col_dims
        off = 0
        for r, c in zip(bi, bj):
            coords = self.from_matrix_index(int(r), int(c))
            shape = self.block_shape(coords)
            n = int(np.prod(shape))
            t = vals[off:off + n].reshape([shape[d] for d in perm])
            off += n
            yield coords, np.transpose(t, np.argsort(perm))

    def to_dense(self):
        """The blocks held by this process's ranks as a dense array (zeros elsewhere)."""
        offs = [np.concatenate([[0], np.cumsum(s)]) for s in self.sizes]
        out = np.zeros([int(o[-1]) for o in offs])
        for coords, blk in self.blocks():
            sl = tuple(slice(offs[d][c], offs[d][c] + blk.shape[d]) for d, c in enumerate(coords))
            out[sl] = blk
        return out

    def remap_into(self, dst: "DistTensor", phase: str = "tensor_remap"):
        """dst := this tensor under dst's map: device remap of every local store,
        then redistribution to dst's owners (volume charged to `phase`)."""
        from . import dist as dd
        if dst.comm is not self.comm or any(not np.array_equal(a, b)
                                            for a, b in zip(self.sizes, dst.sizes)):
            raise InvalidArgument("tensor remap: different group or blockings")
        tmp = dd.new_matrix_round_robin(dst.mat.rows(), dst.mat.cols(), dst.grid, self.comm)
        for r in self.comm.local_ranks():
            if r < self.mat.nranks():
                _remap_store(self.comm.ctx, self.sizes, self.nb, self.mat.local(r),
                             self.row_dims, self.col_dims, tmp.local(r), dst.row_dims,
                             dst.col_dims)
        check(self.comm.lib.bt_redistribute(tmp.h, dst.mat.h, 0, 0, phase.encode()),
              "tensor_remap")
        tmp._close()

    def remap(self, row_dims, col_dims, phase: str = "tensor_remap") -> "DistTensor":
        out = self._like(row_dims, col_dims)
        self.remap_into(out, phase)
        return out


def contract_dist(a: DistTensor, b: DistTensor, contract_a, contract_b, c: DistTensor,
                  eps: float = 0.0) -> dict:
    """contract() over the process group: C += A.B with the
    contracted indices summed.  Operands in contraction-compatible maps are
    used as they are (no redistribution, zero "tensor_remap" ledger);
    otherwise they are remapped and redistributed first, and C is brought back
    to its own map afterwards, the volume charged to the ledger.  The
    matricized multiply is Cannon on square grids, else case 2."""
    from . import dist as dd
    contract_a, contract_b = list(contract_a), list(contract_b)
    if len(contract_a) != len(contract_b) or not contract_a:
        raise InvalidArgument("contract: contracted index lists must be non-empty and equal "
                              "in length")
    for da, db in zip(contract_a, contract_b):
        if not np.array_equal(a.sizes[da], b.sizes[db]):
            raise InvalidArgument("contract: blockings of contracted indices differ")
    ra = [d for d in range(a.rank) if d not in contract_a]
    rb = [d for d in range(b.rank) if d not in contract_b]
    if c.rank != len(ra) + len(rb):
        raise InvalidArgument("contract: C rank does not match the retained indices")
    for q, (t, d) in enumerate([(a, d) for d in ra] + [(b, d) for d in rb]):
        if not np.array_equal(c.sizes[q], t.sizes[d]):
            raise InvalidArgument("contract: C blockings do not match the retained indices")
    temps = []
    am = a if (a.row_dims == ra and a.col_dims == contract_a) else a.remap(ra, contract_a)
    bm = b if (b.row_dims == contract_b and b.col_dims == rb) else b.remap(contract_b, rb)
    crow, ccol = list(range(len(ra))), list(range(len(ra), c.rank))
    compatible = c.row_dims == crow and c.col_dims == ccol
    cm = c if compatible else c.remap(crow, ccol)
    temps += [t for t in (am, bm, cm) if t not in (a, b, c)]
    g = a.grid
    P = g.size()
    if g.dim(0) == g.dim(1):
        st = dd.multiply_cannon(a.comm, am.mat, bm.mat, cm.mat, eps)
    else:
        st = dd.multiply_virtual_case2(a.comm, am.mat, bm.mat, cm.mat, P, eps)
    if not compatible:
        cm.remap_into(c)
    for t in temps:
        t.mat._close()
    return st
