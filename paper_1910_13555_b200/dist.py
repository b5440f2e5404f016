"""Python mirror of the reference's distributed API over libbtcuda.

Same names, argument meaning and error classes as the reference headers
(grid.hpp, comm.hpp, matrix.hpp, multiply_cannon.hpp, multiply_rect.hpp,
cost_model.hpp, partition.hpp), so the parity tests read like the reference's
own tests:

    grid = ProcessGrid([2, 2]); comm = SimComm(grid)          # 4 ranks
    a = new_matrix_round_robin(Blocking.uniform(8, 23), ..., grid)
    a.put_block(i, j, block); multiply_cannon(comm, a, b, c)

``SimComm(grid)`` places every rank of the grid on this process's GPU
("virtual ranks": messages are device copies, the ledger counts them exactly
like the reference's); ``SimComm.nccl(ctx)`` is the one-process-per-GPU form
over NCCL (torchrun).  All compute runs in libbtcuda on the B200 -- there is no
CPU path here.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (BlockTensorError, BtStats, DeadlockError, GridError, InvalidArgument,
                   LayoutError, OwnershipError, check, ptr)
from .store import Context, LocalStore

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)

__all__ = [
    "Algorithm", "Blocking", "ChunkPartition", "DistMatrix", "Ledger", "MultiplySpec",
    "ProcessGrid", "SimComm", "TrafficCounters", "algorithm_name", "cannon_volume",
    "case1_volume", "case2_volume", "estimate_result_occupancy", "filter", "measured_spec",
    "multiply_cannon", "multiply_dispatch", "multiply_reduce_case1",
    "multiply_virtual_case2", "new_matrix", "new_matrix_round_robin",
    "occupancy_limit_case1", "occupancy_ratio_bound", "predicted_volume", "redistribute",
    "redistribute_add", "select_algorithm", "split_grid", "Subgroup",
    "BlockTensorError", "InvalidArgument", "OwnershipError", "GridError", "LayoutError",
    "DeadlockError",
]


# --------------------------------------------------------------- blocking
class Blocking:
    """block.hpp:70-97: block sizes along one dimension plus prefix sums."""

    def __init__(self, sizes):
        self._sizes = np.asarray(list(sizes), dtype=np.int32)
        if np.any(self._sizes < 1):
            raise InvalidArgument("Blocking: block sizes must be positive")
        self._off = np.concatenate([[0], np.cumsum(self._sizes, dtype=np.int64)])

    @staticmethod
    def uniform(n_blocks: int, block_size: int) -> "Blocking":
        return Blocking([block_size] * n_blocks)

    def n_blocks(self) -> int:
        return int(self._sizes.shape[0])

    def size(self, b: int) -> int:
        return int(self._sizes[b])

    def offset(self, b: int) -> int:
        return int(self._off[b])

    def total(self) -> int:
        return int(self._off[-1])

    def sizes(self) -> np.ndarray:
        return self._sizes

    def __eq__(self, other):
        return isinstance(other, Blocking) and np.array_equal(self._sizes, other._sizes)


class ChunkPartition:
    """partition.hpp:17-41: contiguous ceil(n/parts) slabs."""

    def __init__(self, n: int, parts: int):
        if n < 0 or parts < 1:
            raise InvalidArgument("ChunkPartition: bad arguments")
        self._n, self._parts = n, parts
        self._chunk = (n + parts - 1) // parts

    def begin(self, p):
        return min(self._n, self._chunk * p)

    def end(self, p):
        return min(self._n, self._chunk * (p + 1))

    def size(self, p):
        return self.end(p) - self.begin(p)

    def part_of(self, i):
        if i < 0 or i >= self._n:
            raise InvalidArgument("ChunkPartition: index out of range")
        return 0 if self._chunk == 0 else i // self._chunk

    def n(self):
        return self._n

    def parts(self):
        return self._parts


# ------------------------------------------------------------------- grid
class ProcessGrid:
    """grid.hpp:17-69: row-major rank <-> coordinates."""

    def __init__(self, dims=(1,)):
        dims = list(dims)
        if not dims:
            raise InvalidArgument("ProcessGrid: dims must be non-empty")
        if any(d < 1 for d in dims):
            raise InvalidArgument("ProcessGrid: every grid extent must be >= 1")
        self._dims = dims
        self._size = int(np.prod(dims))

    def ndims(self):
        return len(self._dims)

    def dim(self, i):
        return self._dims[i]

    def dims(self):
        return list(self._dims)

    def size(self):
        return self._size

    def coords_of(self, rank):
        if rank < 0 or rank >= self._size:
            raise InvalidArgument(f"coords_of: rank {rank} out of range [0,{self._size})")
        out = [0] * len(self._dims)
        for d in range(len(self._dims) - 1, -1, -1):
            out[d] = rank % self._dims[d]
            rank //= self._dims[d]
        return out

    def rank_of(self, coords):
        if len(coords) != len(self._dims):
            raise InvalidArgument(f"rank_of: expected {len(self._dims)} coordinates, "
                                  f"got {len(coords)}")
        r = 0
        for d, c in enumerate(coords):
            if c < 0 or c >= self._dims[d]:
                raise InvalidArgument(f"rank_of: coordinate {c} out of range for dimension {d}")
            r = r * self._dims[d] + c
        return r

    def __eq__(self, o):
        return isinstance(o, ProcessGrid) and self._dims == o._dims


@dataclass
class Subgroup:
    """grid.hpp:74-97."""
    parent: ProcessGrid
    split_dim: int
    factor: int
    coord_begin: int
    coord_end: int
    members: list
    local_grid: ProcessGrid

    def local_rank_of(self, parent_rank):
        c = self.parent.coords_of(parent_rank)
        if not (self.coord_begin <= c[self.split_dim] < self.coord_end):
            raise InvalidArgument("local_rank_of: rank not in subgroup")
        c[self.split_dim] -= self.coord_begin
        return self.local_grid.rank_of(c)

    def parent_rank_of(self, local_rank):
        c = self.local_grid.coords_of(local_rank)
        c[self.split_dim] += self.coord_begin
        return self.parent.rank_of(c)


def split_grid(grid: ProcessGrid, dim: int, factor: int):
    """grid.hpp:102-135: remainder goes to the lowest-indexed subgroups."""
    if dim < 0 or dim >= grid.ndims():
        raise InvalidArgument("split_grid: dimension index out of range")
    extent = grid.dim(dim)
    if factor < 1 or factor > extent:
        raise InvalidArgument(f"split_grid: factor {factor} must be in [1,{extent}]")
    base, rem = divmod(extent, factor)
    groups, begin = [], 0
    for s in range(factor):
        width = base + (1 if s < rem else 0)
        dims = grid.dims()
        dims[dim] = width
        members = [r for r in range(grid.size())
                   if begin <= grid.coords_of(r)[dim] < begin + width]
        groups.append(Subgroup(grid, dim, factor, begin, begin + width, members,
                               ProcessGrid(dims)))
        begin += width
    return groups


# ------------------------------------------------------------ comm/ledger
@dataclass
class TrafficCounters:
    """comm.hpp:41-58."""
    elements_sent: int = 0
    elements_received: int = 0
    meta_sent: int = 0
    meta_received: int = 0


class Ledger:
    """comm.hpp:60-150, read from the device group's counters."""

    def __init__(self, comm: "SimComm"):
        self._comm = comm

    def nranks(self):
        return self._comm.nranks()

    def _get(self, rank, phase, what):
        out = C.c_int64()
        check(self._comm.lib.bt_grid_ledger(self._comm.g, rank,
                                            phase.encode() if phase else None, what,
                                            C.byref(out)), "ledger")
        return out.value

    def rank_total(self, rank) -> TrafficCounters:
        return TrafficCounters(*[self._get(rank, None, w) for w in range(4)])

    def rank_phase(self, rank, phase) -> TrafficCounters:
        return TrafficCounters(*[self._get(rank, phase, w) for w in range(4)])

    def total_elements_sent(self):
        return sum(self._get(r, None, 0) for r in range(self.nranks()))

    def total_elements_received(self):
        return sum(self._get(r, None, 1) for r in range(self.nranks()))

    def mean_elements_sent(self):
        n = self.nranks()
        return self.total_elements_sent() / n if n else 0.0

    def max_elements_sent(self):
        return max((self._get(r, None, 0) for r in range(self.nranks())), default=0)

    def phase_elements_sent(self, phase):
        return sum(self._get(r, phase, 0) for r in range(self.nranks()))


class SimComm:
    """The device group replacing SimComm (comm.hpp:152-397).

    ``SimComm(grid)``: every rank of ``grid`` is a virtual rank on one GPU of
    this process.  ``SimComm.nccl(ctx)``: one rank per process over NCCL."""

    def __init__(self, grid: ProcessGrid, ctx: Context | None = None, device: int = 0):
        self.lib = _lib.load()
        self._grid = grid
        self.ctx = ctx if ctx is not None else Context(device)
        h = C.c_void_p()
        check(self.lib.bt_grid_create(self.ctx.h, grid.size(), C.byref(h)), "SimComm")
        self.g = h
        self._matrices = []
        SimComm._current = self

    _current = None

    @staticmethod
    def nccl(ctx: Context) -> "SimComm":
        return SimComm(ProcessGrid([ctx.nranks]), ctx=ctx)

    @staticmethod
    def current() -> "SimComm":
        if SimComm._current is None:
            raise InvalidArgument("no SimComm created yet")
        return SimComm._current

    def grid(self):
        return self._grid

    def nranks(self):
        n = C.c_int()
        check(self.lib.bt_grid_info(self.g, C.byref(n), None, None), "grid_info")
        return n.value

    def local_ranks(self):
        n, f, nl = C.c_int(), C.c_int(), C.c_int()
        check(self.lib.bt_grid_info(self.g, C.byref(n), C.byref(f), C.byref(nl)), "grid_info")
        return list(range(f.value, f.value + nl.value))

    def ledger(self) -> Ledger:
        return Ledger(self)

    def reset_ledger(self):
        check(self.lib.bt_grid_reset_ledger(self.g), "reset_ledger")

    def close(self):
        if getattr(self, "g", None):
            for m in self._matrices:
                m._close()
            self.lib.bt_grid_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- matrix
class DistMatrix:
    """matrix.hpp:279-401 over one device store per local rank."""

    def __init__(self, rows: Blocking, cols: Blocking, grid: ProcessGrid, row_dist, col_dist,
                 comm: SimComm | None = None):
        if grid.ndims() != 2:
            raise InvalidArgument("DistMatrix: grid must be 2-dimensional")
        self.comm = comm or SimComm.current()
        self._rows, self._cols, self._grid = rows, cols, grid
        rd = np.ascontiguousarray(row_dist, np.int32)
        cd = np.ascontiguousarray(col_dist, np.int32)
        if len(rd) != rows.n_blocks() or len(cd) != cols.n_blocks():
            raise InvalidArgument("Axis: distribution length does not match block count")
        self._rd, self._cd = rd, cd
        rs, cs = rows.sizes(), cols.sizes()
        h = C.c_void_p()
        check(self.comm.lib.bt_dmat_create(self.comm.g, len(rs), ptr(rs, _i32p), len(cs),
                                           ptr(cs, _i32p), grid.dim(0), grid.dim(1),
                                           ptr(rd, _i32p), ptr(cd, _i32p), C.byref(h)),
              "new_matrix")
        self.h = h
        self.comm._matrices.append(self)

    def _close(self):
        if getattr(self, "h", None):
            self.comm.lib.bt_dmat_destroy(self.h)
            self.h = None

    # -- layout
    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def grid(self):
        return self._grid

    def row_dist(self):
        return self._rd

    def col_dist(self):
        return self._cd

    def n_block_rows(self):
        return self._rows.n_blocks()

    def n_block_cols(self):
        return self._cols.n_blocks()

    def owner_rank(self, i, j):
        return self._grid.rank_of([int(self._rd[i]), int(self._cd[j])])

    def nranks(self):
        return self._grid.size()

    def local(self, rank) -> LocalStore:
        s = C.c_void_p()
        check(self.comm.lib.bt_dmat_local(self.h, rank, C.byref(s)), "local")
        return LocalStore.borrow(self.comm.ctx, s, self._rows.sizes(), self._cols.sizes())

    # -- content
    def put_block(self, i, j, block, accumulate=False):
        b = np.ascontiguousarray(block, np.float64)
        if b.shape != (self._rows.size(i), self._cols.size(j)):
            raise InvalidArgument(
                f"put_block: block is {b.shape[0]}x{b.shape[1] if b.ndim > 1 else 1} but slot "
                f"({i},{j}) requires {self._rows.size(i)}x{self._cols.size(j)}")
        self.put_blocks([i], [j], b.ravel(), accumulate)

    def put_blocks(self, bi, bj, vals, accumulate=False):
        bi = np.ascontiguousarray(bi, np.int64)
        bj = np.ascontiguousarray(bj, np.int64)
        v = np.ascontiguousarray(vals, np.float64)
        check(self.comm.lib.bt_dmat_put_blocks(self.h, len(bi), ptr(bi, _i64p), ptr(bj, _i64p),
                                               ptr(v, _f64p), int(bool(accumulate))),
              "put_block")

    def get_block(self, i, j):
        return self.local(self.owner_rank(i, j)).get_block(i, j)

    def blocks(self):
        """Canonical (bi, bj, vals) of every block held by this process's ranks."""
        parts = [self.local(r).export() for r in self.comm.local_ranks() if r < self.nranks()]
        if not parts:
            return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)
        bi = np.concatenate([p[0] for p in parts])
        bj = np.concatenate([p[1] for p in parts])
        sz = self._rows.sizes()[bi].astype(np.int64) * self._cols.sizes()[bj]
        vals = np.concatenate([p[2] for p in parts])
        order = np.lexsort((bj, bi))
        off = np.concatenate([[0], np.cumsum(sz)])
        out = np.concatenate([vals[off[t]:off[t + 1]] for t in order]) if len(order) else vals
        return bi[order], bj[order], out

    def _global_counts(self):
        """(blocks, elements) stored over ALL ranks (matrix.hpp stored_* are
        global); with one process per GPU this is a collective over the group
        (bt_grid_sum) -- every process must call it."""
        v = np.zeros(2, np.int64)
        for r in self.comm.local_ranks():
            if r < self.nranks():
                v += np.array(self.local(r).info(), np.int64)
        check(self.comm.lib.bt_grid_sum(self.comm.g, ptr(v, _i64p), 2), "grid_sum")
        return int(v[0]), int(v[1])

    def stored_blocks(self):
        return self._global_counts()[0]

    def stored_elements(self):
        return self._global_counts()[1]

    def occupancy(self):
        dense = self._rows.total() * self._cols.total()
        return 0.0 if dense == 0 else self.stored_elements() / dense


def new_matrix(row_blocking, col_blocking, grid, row_dist, col_dist, comm=None):
    """matrix.hpp:404-410."""
    if grid.ndims() != 2:
        raise InvalidArgument("new_matrix: grid must be 2-dimensional")
    return DistMatrix(row_blocking, col_blocking, grid, row_dist, col_dist, comm)


def new_matrix_round_robin(row_blocking, col_blocking, grid, comm=None):
    """matrix.hpp:413-418: block index mod grid extent."""
    if grid.ndims() != 2:
        raise InvalidArgument("new_matrix: grid must be 2-dimensional")
    rd = np.arange(row_blocking.n_blocks()) % grid.dim(0)
    cd = np.arange(col_blocking.n_blocks()) % grid.dim(1)
    return DistMatrix(row_blocking, col_blocking, grid, rd, cd, comm)


def redistribute(comm, src: DistMatrix, new_rows, new_cols, new_grid, transpose=False,
                 phase="redistribute", row_dist=None, col_dist=None) -> DistMatrix:
    """matrix.hpp:567-600; new_rows/new_cols are Blockings, distributions given
    explicitly (row_dist/col_dist) or round robin."""
    rd = row_dist if row_dist is not None else np.arange(new_rows.n_blocks()) % new_grid.dim(0)
    cd = col_dist if col_dist is not None else np.arange(new_cols.n_blocks()) % new_grid.dim(1)
    dst = DistMatrix(new_rows, new_cols, new_grid, rd, cd, comm)
    check(comm.lib.bt_redistribute(src.h, dst.h, int(transpose), 0, phase.encode()),
          "redistribute")
    return dst


def redistribute_add(comm, src: DistMatrix, dst: DistMatrix, phase="redistribute"):
    """matrix.hpp:604-622."""
    check(comm.lib.bt_redistribute(src.h, dst.h, 0, 1, phase.encode()), "redistribute_add")


def filter(m: DistMatrix, eps: float):
    """Drop stored blocks with Frobenius norm < eps."""
    for r in m.comm.local_ranks():
        if r < m.nranks():
            m.local(r).filter(eps)


# -------------------------------------------------------------- multiply
def _stats(st: BtStats) -> dict:
    return st.as_dict()


def multiply_cannon(comm, a, b, c, eps=0.0) -> dict:
    """multiply_cannon.hpp:62-118."""
    st = BtStats()
    check(comm.lib.bt_multiply_cannon(a.h, b.h, c.h, eps, C.byref(st)), "multiply_cannon")
    return _stats(st)


def multiply_reduce_case1(comm, a, b, c, nprocs, eps=0.0) -> dict:
    """multiply_rect.hpp:123-192."""
    st = BtStats()
    check(comm.lib.bt_multiply_case1(a.h, b.h, c.h, nprocs, eps, C.byref(st)),
          "multiply_reduce_case1")
    return _stats(st)


def multiply_virtual_case2(comm, a, b, c, nprocs, eps=0.0, gather=False) -> dict:
    """multiply_rect.hpp:199-238 (gather=True: one-step NVLink gather of B)."""
    st = BtStats()
    check(comm.lib.bt_multiply_case2(a.h, b.h, c.h, nprocs, int(gather), eps, C.byref(st)),
          "multiply_virtual_case2")
    return _stats(st)


class Algorithm:
    cannon, case1, case2, auto = 0, 1, 2, 3


def algorithm_name(a):
    return {0: "cannon", 1: "case1", 2: "case2", 3: "auto"}.get(a, "?")


def cannon_ready(a, b, c, nprocs) -> bool:
    """Cannon's layout preconditions (multiply_cannon.hpp:65-78): a square grid
    of nprocs ranks, C distributed as A's rows x B's columns."""
    g = a.grid()
    q = g.dim(0)
    return (g.dim(0) == g.dim(1) and q * q == nprocs and b.grid() == g and c.grid() == g
            and np.array_equal(c.row_dist(), a.row_dist())
            and np.array_equal(c.col_dist(), b.col_dist())
            and np.array_equal(a.col_dist(), b.row_dist()))


def select_for(a, b, c, nprocs, machine=None):
    """The B200 selection for these operands: measured occupancies (a
    collective with one process per GPU), C's occupancy estimated from them
    (multiply_rect.hpp:84-88), argmin of predicted_time_b200 over the
    algorithms whose preconditions hold."""
    s = measured_spec(a, b, 0.0, nprocs)
    s.occ_c = estimate_result_occupancy(s.occ_a, s.occ_b, a.n_block_cols())
    machine = machine or B200Machine()
    cands = ([Algorithm.cannon] if cannon_ready(a, b, c, nprocs) else []) + \
        [Algorithm.case1, Algorithm.case2]
    times = {al: predicted_time_b200(al, s, machine) for al in cands}
    return min(cands, key=lambda al: (times[al], al)), times


def multiply_dispatch(comm, algo, a, b, c, nprocs, eps=0.0) -> dict:
    """multiply_rect.hpp:242-250; Algorithm.auto picks the algorithm with the
    NVLink-aware time model (select_for) and runs case 2 in its
    one-step NVLink gather form."""
    if algo == Algorithm.auto:
        algo, _ = select_for(a, b, c, nprocs)
        if algo == Algorithm.case2:
            st = multiply_virtual_case2(comm, a, b, c, nprocs, eps, gather=True)
            st["algorithm"] = "case2"
            return st
        st = multiply_dispatch(comm, algo, a, b, c, nprocs, eps)
        st["algorithm"] = algorithm_name(algo)
        return st
    if algo == Algorithm.cannon:
        return multiply_cannon(comm, a, b, c, eps)
    if algo == Algorithm.case1:
        return multiply_reduce_case1(comm, a, b, c, nprocs, eps)
    if algo == Algorithm.case2:
        return multiply_virtual_case2(comm, a, b, c, nprocs, eps)
    raise InvalidArgument("multiply_dispatch: unknown algorithm")


# ------------------------------------------------------------ cost model
@dataclass
class MultiplySpec:
    """cost_model.hpp:19-39 (volumes in matrix elements per process)."""
    m: float = 0
    n: float = 0
    k: float = 0
    occ_a: float = 1.0
    occ_b: float = 1.0
    occ_c: float = 1.0
    nprocs: float = 1

    def stored_a(self):
        return self.occ_a * self.m * self.k

    def stored_b(self):
        return self.occ_b * self.k * self.n

    def stored_c(self):
        return self.occ_c * self.m * self.n

    def validate(self):
        if self.m < 1 or self.n < 1 or self.k < 1:
            raise InvalidArgument("MultiplySpec: dims must be >= 1")
        if self.nprocs < 1:
            raise InvalidArgument("MultiplySpec: process count must be >= 1")
        for o in (self.occ_a, self.occ_b, self.occ_c):
            if o < 0.0 or o > 1.0:
                raise InvalidArgument("MultiplySpec: occupancies must be in [0,1]")


def cannon_volume(s):  # Eq. 1, cost_model.hpp:43-46
    s.validate()
    return (s.stored_a() + s.stored_b()) / math.sqrt(s.nprocs)


def case1_volume(s):  # Eq. 2, :50-53
    s.validate()
    return (s.stored_a() + s.stored_b()) / s.nprocs + s.stored_c()


def case2_volume(s):  # Eq. 5, :57-60
    s.validate()
    return (s.stored_a() + s.stored_b() + s.stored_c()) / s.nprocs + s.stored_b()


def occupancy_limit_case1(s):  # Eq. 3, :64-69
    s.validate()
    tw = cannon_volume(s)
    raw = (tw - (s.stored_a() + s.stored_b()) / s.nprocs) / (s.m * s.n)
    return min(max(raw, 0.0), 1.0)


def occupancy_ratio_bound(m, n, k, nprocs):  # Eq. 4, :74-78
    if m < 1 or n < 1 or k < 1 or nprocs < 1:
        raise InvalidArgument("occupancy_ratio_bound: arguments must be >= 1")
    return k * (m + n) / (m * n * math.sqrt(nprocs))


def estimate_result_occupancy(occ_a, occ_b, n_blocks_k):  # :84-88
    if n_blocks_k < 0:
        raise InvalidArgument("estimate_result_occupancy: negative block count")
    p = min(max(occ_a * occ_b, 0.0), 1.0)
    return min(max(1.0 - (1.0 - p) ** n_blocks_k, 0.0), 1.0)


def predicted_volume(algo, s):  # multiply_rect.hpp:34-41
    return {0: cannon_volume, 1: case1_volume, 2: case2_volume}[algo](s)


def select_algorithm(m, n, k, occ_a, occ_b, occ_c_estimate, nprocs):
    """multiply_rect.hpp:45-63: argmin volume, ties cannon > case1 > case2."""
    s = MultiplySpec(m, n, k, occ_a, occ_b, occ_c_estimate, nprocs)
    best, bv = Algorithm.cannon, cannon_volume(s)
    if case1_volume(s) < bv:
        best, bv = Algorithm.case1, case1_volume(s)
    if case2_volume(s) < bv:
        best = Algorithm.case2
    return best


@dataclass
class B200Machine:
    """Rates of the B200 time model, FITTED (least squares on log time) to the
    measured multiply times of tests/golden/algo_times_b200.jsonl
    (tools/algo_sweep.py: square / tall-skinny / dense / wide-C workloads on 2
    and 4 B200s, every algorithm, inputs in a round-robin layout).  Effective
    rates of this implementation, not hardware peaks: they fold in the host
    planning of redistributions and the gather assembly."""
    fp64_flops: float = 25.6e12    # local multiply, useful FP64
    hbm_bytes: float = 6.55e12     # C written once (MEASURED_PEAKS.json copy rate)
    cannon_bytes: float = 237e9    # Cannon panel shifts
    redist_bytes: float = 126e9    # input/output layout changes of case 1 / case 2
    reduce_bytes: float = 265e9    # case 1: partial-C reduction to the owners
    gather_bytes: float = 33.1e9   # case 2: B gather incl. assembly
    cannon_overhead: float = 0.86e-3
    case1_overhead: float = 2.92e-3
    case2_overhead: float = 0.0


def predicted_time_b200(algo, s: MultiplySpec, machine: B200Machine = B200Machine()):
    """Extension (not in the reference): seconds per multiply on
    s.nprocs B200s joined by NVSwitch, from the paper's stored sizes S_A, S_B,
    S_C (cost_model.hpp:19-39) and the fitted rates of B200Machine:
      * compute = useful flops / (P * F) + C written once per rank (S_C / P);
      * Cannon (square P only): max(compute, Eq.-1 panel traffic) -- the
        shifts are posted before each local multiply;
      * case 1: every rank writes a full partial C (S_C), the K-slab
        redistribution of A and B, then the partial-C reduction
        S_C (P-1)/P (not hidden);
      * case 2: max(compute, B gather S_B (P-1)/P) -- the gather runs under
        the symbolic passes and the multiply -- plus the row-slab
        redistribution of A and C.
    Fit quality and the selection check: tests/test_host_logic.py."""
    s.validate()
    p = s.nprocs
    flops = 2.0 * s.m * s.n * s.k * s.occ_a * s.occ_b
    sa, sb, sc = s.stored_a(), s.stored_b(), s.stored_c()
    hw = machine
    compute = flops / (p * hw.fp64_flops) + 8.0 * sc / p / hw.hbm_bytes
    if algo == Algorithm.cannon:
        q = round(math.sqrt(p))
        if q * q != p:
            return math.inf
        if p == 1:
            return compute
        return max(compute, 8.0 * cannon_volume(s) / hw.cannon_bytes) + hw.cannon_overhead
    if p == 1 and algo in (Algorithm.case1, Algorithm.case2):
        return compute
    if algo == Algorithm.case1:
        return (flops / (p * hw.fp64_flops) + 8.0 * sc / hw.hbm_bytes
                + 8.0 * (sa + sb) / p / hw.redist_bytes
                + 8.0 * sc * (p - 1) / p / hw.reduce_bytes + hw.case1_overhead)
    if algo == Algorithm.case2:
        return (max(compute, 8.0 * sb * (p - 1) / p / hw.gather_bytes)
                + 8.0 * (sa + sc) / p / hw.redist_bytes + hw.case2_overhead)
    raise InvalidArgument("predicted_time_b200: unknown algorithm")


def select_algorithm_b200(m, n, k, occ_a, occ_b, occ_c_estimate, nprocs,
                          machine: B200Machine = B200Machine()):
    """argmin of predicted_time_b200, ties cannon > case1 > case2 (the
    reference's tie order, multiply_rect.hpp:45-63)."""
    s = MultiplySpec(m, n, k, occ_a, occ_b, occ_c_estimate, nprocs)
    best, bt = Algorithm.cannon, predicted_time_b200(Algorithm.cannon, s, machine)
    for algo in (Algorithm.case1, Algorithm.case2):
        t = predicted_time_b200(algo, s, machine)
        if t < bt:
            best, bt = algo, t
    return best


def measured_spec(a: DistMatrix, b: DistMatrix, occ_c, nprocs):
    """multiply_rect.hpp:254-265."""
    return MultiplySpec(a.rows().total(), b.cols().total(), a.cols().total(), a.occupancy(),
                        b.occupancy(), occ_c, nprocs)
