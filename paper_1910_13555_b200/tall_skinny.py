"""Tall-and-skinny layer over the B200 multiply.

The reference has this module only in its spec (no code in proj/); it is the
SURVEY 8(f)-1 "next" row.  A tall-and-skinny matrix is split along its long
dimension into ``f`` approximately square submatrices; index data along that
dimension comes from function objects (``IndexFuncs``, the spec's form of
``Axis::functional``, matrix.hpp:50-58), so no rank ever holds a block-size or
distribution array as long as the full split dimension -- each submatrix's
blocking covers only its own block range.

B200 placement: every submatrix is an ordinary device ``DistMatrix`` on the
full communicator (distributed by ``dist_fn`` over the grid), not on a rank
subgroup: with NVSwitch every GPU reaches every peer at full bandwidth, so the
sub-multiplications simply run one after another on all GPUs instead of
concurrently on disjoint subgroups (the spec allows either: "Sequential
schedule must be result-identical").  Partial C contributions of a split
contraction dimension need no separate reduction: every multiply accumulates
(C += A_s * B_s).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from ._lib import InvalidArgument, LayoutError
from .dist import (Algorithm, Blocking, DistMatrix, ProcessGrid, SimComm, measured_spec,
                   multiply_dispatch, new_matrix, select_algorithm)


@dataclass
class IndexFuncs:
    """block-index -> block size, block-index -> grid coordinate."""
    n_blocks: int
    block_size_fn: Callable[[int], int]
    dist_fn: Callable[[int], int]

    def size(self, b: int) -> int:
        if not 0 <= b < self.n_blocks:
            raise InvalidArgument(f"IndexFuncs: block {b} out of range [0,{self.n_blocks})")
        s = int(self.block_size_fn(b))
        if s < 1:
            raise InvalidArgument(f"IndexFuncs: block size of {b} must be >= 1, got {s}")
        return s

    def dist(self, b: int) -> int:
        return int(self.dist_fn(b))

    def total_elements(self) -> int:
        return sum(self.size(b) for b in range(self.n_blocks))


def ceil_partition(n: int, f: int):
    """SPEC.md 'Design decisions': the first submatrices get ceil(n/f) block
    indices, the last the remainder -- e.g. n=10, f=3 -> [0,4), [4,8), [8,10)."""
    if f < 1:
        raise InvalidArgument("ceil_partition: factor must be >= 1")
    w = -(-n // f) if n else 0
    return [(min(n, s * w), min(n, (s + 1) * w)) for s in range(f)]


def choose_split_factor(long_dim_elements: float, short_dim_elements: float, nprocs: int) -> int:
    """argmin over f in 1..P of |long/f - short| (approximately
    square submatrices, in element units); ties toward the smaller f."""
    if long_dim_elements <= 0 or short_dim_elements <= 0 or nprocs < 1:
        raise InvalidArgument("choose_split_factor: inputs must be positive")
    best, bd = 1, abs(long_dim_elements - short_dim_elements)
    for f in range(2, nprocs + 1):
        d = abs(long_dim_elements / f - short_dim_elements)
        if d < bd:
            best, bd = f, d
    return best


class TallSkinnyMatrix:
    """f submatrices along ``split_dim`` ("rows" or "cols")."""

    def __init__(self, rows: IndexFuncs, cols: IndexFuncs, grid: ProcessGrid, split_dim: str,
                 factor: int, comm: SimComm | None = None):
        if split_dim not in ("rows", "cols"):
            raise InvalidArgument("create_tall_skinny: split_dim must be 'rows' or 'cols'")
        if grid.ndims() != 2:
            raise InvalidArgument("create_tall_skinny: grid must be 2-dimensional")
        gdim = 0 if split_dim == "rows" else 1
        if factor < 1 or factor > grid.dim(gdim):
            raise InvalidArgument(f"create_tall_skinny: factor {factor} must be in "
                                  f"[1,{grid.dim(gdim)}] (grid extent of the split dimension)")
        self.rows_funcs, self.cols_funcs = rows, cols
        self.grid, self.split_dim, self.factor = grid, split_dim, factor
        self.comm = comm or SimComm.current()
        n_split = rows.n_blocks if split_dim == "rows" else cols.n_blocks
        self.ranges = ceil_partition(n_split, factor)
        self.subs = []
        # index arrays resident on the host, per submatrix (for the no-long-index property)
        self.index_lengths = []
        for (b0, b1) in self.ranges:
            if split_dim == "rows":
                rb = Blocking([rows.size(b) for b in range(b0, b1)])
                rd = np.array([rows.dist(b) % grid.dim(0) for b in range(b0, b1)], np.int32)
                cb = Blocking([cols.size(b) for b in range(cols.n_blocks)])
                cd = np.array([cols.dist(b) % grid.dim(1) for b in range(cols.n_blocks)],
                              np.int32)
            else:
                rb = Blocking([rows.size(b) for b in range(rows.n_blocks)])
                rd = np.array([rows.dist(b) % grid.dim(0) for b in range(rows.n_blocks)],
                              np.int32)
                cb = Blocking([cols.size(b) for b in range(b0, b1)])
                cd = np.array([cols.dist(b) % grid.dim(1) for b in range(b0, b1)], np.int32)
            self.subs.append(new_matrix(rb, cb, grid, rd, cd, self.comm))
            self.index_lengths.append(b1 - b0)

    # -- index mapping (bijection global <-> (submatrix, local))
    def locate(self, b: int):
        """Global split-dimension block index -> (submatrix id, local block index)."""
        n = self.ranges[-1][1] if self.ranges else 0
        if not 0 <= b < n:
            raise InvalidArgument(f"TallSkinnyMatrix: block {b} out of range [0,{n})")
        w = self.ranges[0][1] - self.ranges[0][0]
        s = b // w
        return s, b - self.ranges[s][0]

    def global_index(self, s: int, local: int) -> int:
        b0, b1 = self.ranges[s]
        if not 0 <= local < b1 - b0:
            raise InvalidArgument("TallSkinnyMatrix: local block index out of range")
        return b0 + local

    # -- content
    def put_block(self, i: int, j: int, block, accumulate: bool = False):
        if self.split_dim == "rows":
            s, li = self.locate(i)
            self.subs[s].put_block(li, j, block, accumulate)
        else:
            s, lj = self.locate(j)
            self.subs[s].put_block(i, lj, block, accumulate)

    def put_blocks(self, bi, bj, vals, accumulate: bool = False):
        bi = np.asarray(bi, np.int64)
        bj = np.asarray(bj, np.int64)
        split = bi if self.split_dim == "rows" else bj
        w = self.ranges[0][1] - self.ranges[0][0]
        sub = split // w
        rsz = np.array([self.rows_funcs.size(int(b)) for b in bi], np.int64)
        csz = np.array([self.cols_funcs.size(int(b)) for b in bj], np.int64)
        off = np.concatenate([[0], np.cumsum(rsz * csz)])
        vals = np.asarray(vals, np.float64)
        for s in np.unique(sub):
            sel = np.nonzero(sub == s)[0]
            v = np.concatenate([vals[off[t]:off[t + 1]] for t in sel]) if len(sel) else vals[:0]
            b0 = self.ranges[int(s)][0]
            if self.split_dim == "rows":
                self.subs[int(s)].put_blocks(bi[sel] - b0, bj[sel], v, accumulate)
            else:
                self.subs[int(s)].put_blocks(bi[sel], bj[sel] - b0, v, accumulate)

    def blocks(self):
        """Canonical global (bi, bj, vals)."""
        parts = []
        for s, m in enumerate(self.subs):
            bi, bj, v = m.blocks()
            b0 = self.ranges[s][0]
            if self.split_dim == "rows":
                bi = bi + b0
            else:
                bj = bj + b0
            rs = np.array([self.rows_funcs.size(int(b)) for b in bi], np.int64)
            cs = np.array([self.cols_funcs.size(int(b)) for b in bj], np.int64)
            parts.append((bi, bj, v, rs * cs))
        bi = np.concatenate([p[0] for p in parts])
        bj = np.concatenate([p[1] for p in parts])
        sz = np.concatenate([p[3] for p in parts])
        vals = np.concatenate([p[2] for p in parts])
        order = np.lexsort((bj, bi))
        off = np.concatenate([[0], np.cumsum(sz)])
        out = np.concatenate([vals[off[t]:off[t + 1]] for t in order]) if len(order) else vals
        return bi[order], bj[order], out

    def max_resident_index_length(self) -> int:
        """Longest host index array along the split dimension (one submatrix)."""
        return max(self.index_lengths) if self.index_lengths else 0


def create_tall_skinny(rows_funcs: IndexFuncs, cols_funcs: IndexFuncs, grid: ProcessGrid,
                       split_dim: str, split_factor: int, comm=None) -> TallSkinnyMatrix:
    """SPEC.md:432-436."""
    return TallSkinnyMatrix(rows_funcs, cols_funcs, grid, split_dim, split_factor, comm)


def _same_funcs(x: IndexFuncs, y: IndexFuncs) -> bool:
    return x.n_blocks == y.n_blocks and all(x.size(b) == y.size(b) for b in range(x.n_blocks))


def multiply_tall_skinny(a: TallSkinnyMatrix, b: TallSkinnyMatrix, c, nprocs: int | None = None,
                         eps: float = 0.0, select=select_algorithm) -> dict:
    """C += A * B by submatrix multiplications, each through
    the distributed drivers with the algorithm ``select`` picks (the
    reference's volume argmin by default, or dist.select_algorithm_b200).

    Supported split layouts (others raise LayoutError naming the dimension):
      * K split: A split on cols, B split on rows with the same factor and
        index functions; C is a plain DistMatrix (or unsplit): C += sum_s A_s B_s;
      * M split: A split on rows, C a TallSkinnyMatrix split the same way,
        B plain: C_s += A_s B;
      * N split: B split on cols, C split the same way, A plain: C_s += A B_s.
    """
    comm = (a.comm if isinstance(a, TallSkinnyMatrix) else b.comm)
    p = nprocs or comm.nranks()
    totals = {"products": 0, "flops": 0.0, "multiplies": 0}

    def run(x: DistMatrix, y: DistMatrix, z: DistMatrix):
        occ_c = 1.0
        algo = select(*_dims(x, y), x.occupancy(), y.occupancy(), occ_c, p)
        if algo == Algorithm.cannon and int(round(math.sqrt(p))) ** 2 != p:
            algo = Algorithm.case2
        if algo == Algorithm.cannon and x.grid().dim(0) != x.grid().dim(1):
            algo = Algorithm.case2
        st = multiply_dispatch(comm, algo, x, y, z, p, eps)
        totals["products"] += st["products"]
        totals["flops"] += st["flops"]
        totals["multiplies"] += 1

    a_ts, b_ts, c_ts = (isinstance(m, TallSkinnyMatrix) for m in (a, b, c))
    if a_ts and b_ts and a.split_dim == "cols" and b.split_dim == "rows":
        if a.factor != b.factor or not _same_funcs(a.cols_funcs, b.rows_funcs):
            raise LayoutError("k", "multiply_tall_skinny: contracted dimension splits differ")
        target = c.subs[0] if c_ts and c.factor == 1 else c
        if isinstance(target, TallSkinnyMatrix):
            raise LayoutError("k", "multiply_tall_skinny: C must not be split when K is split")
        for s in range(a.factor):
            run(a.subs[s], b.subs[s], target)
    elif a_ts and a.split_dim == "rows" and c_ts and c.split_dim == "rows" and not b_ts:
        if a.factor != c.factor or not _same_funcs(a.rows_funcs, c.rows_funcs):
            raise LayoutError("m", "multiply_tall_skinny: A and C row splits differ")
        for s in range(a.factor):
            run(a.subs[s], b, c.subs[s])
    elif b_ts and b.split_dim == "cols" and c_ts and c.split_dim == "cols" and not a_ts:
        if b.factor != c.factor or not _same_funcs(b.cols_funcs, c.cols_funcs):
            raise LayoutError("n", "multiply_tall_skinny: B and C column splits differ")
        for s in range(b.factor):
            run(a, b.subs[s], c.subs[s])
    else:
        raise LayoutError("k", "multiply_tall_skinny: unsupported split layout")
    return totals


def _dims(x: DistMatrix, y: DistMatrix):
    return x.rows().total(), y.cols().total(), x.cols().total()
