"""Distributed drivers on one B200 with virtual ranks, against the oracle and
the compiled reference (values, pattern AND per-rank ledgers).

The reference's SimComm runs P ranks in one process; SimComm(grid) here runs
the same P ranks as virtual ranks on one GPU (device-copy transport), so
Cannon, case 1 and case 2 can be checked rank by rank on a single GPU.  The
NCCL transport (one process per GPU) is exercised by tests/test_nccl_gpu.py.
"""
import json
import os

import numpy as np
import pytest

from helpers import assert_parity
from oracle.oracle import Blocks

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _dm(d, grid, comm, blocks: Blocks):
    m = d.new_matrix_round_robin(d.Blocking(blocks.rsz), d.Blocking(blocks.csz), grid, comm)
    if blocks.nblk:
        m.put_blocks(blocks.bi, blocks.bj, blocks.vals)
    return m


def _got(m):
    bi, bj, v = m.blocks()
    return Blocks(m.rows().sizes(), m.cols().sizes(), bi, bj, v)


def _inputs(oracle, seed, rs, ks, ns, oa=0.4, ob=0.4, oc=0.15):
    A = oracle.random_matrix(seed, rs, ks, oa)
    B = oracle.random_matrix(seed + 1, ks, ns, ob)
    Cin = oracle.random_matrix(seed + 2, rs, ns, oc)
    return A, B, Cin


def _run(ctx, algo, q, nprocs, A, B, Cin, gather=False):
    from paper_1910_13555_b200 import dist as d
    world = max(q * q, nprocs)
    grid = d.ProcessGrid([q, q])
    comm = d.SimComm(d.ProcessGrid([world]), ctx=ctx)
    a, b, c = _dm(d, grid, comm, A), _dm(d, grid, comm, B), _dm(d, grid, comm, Cin)
    if algo == "cannon":
        st = d.multiply_cannon(comm, a, b, c)
    elif algo == "case1":
        st = d.multiply_reduce_case1(comm, a, b, c, nprocs)
    else:
        st = d.multiply_virtual_case2(comm, a, b, c, nprocs, gather=gather)
    out = _got(c)
    led = comm.ledger()
    ledger = {r: led.rank_total(r) for r in range(world)}
    phases = {r: {p: led.rank_phase(r, p).elements_sent
                  for p in ("cannon", "redistribute", "ring", "collect", "reduce")}
              for r in range(world)}
    comm.close()
    return out, st, ledger, phases


MIXED = dict(rs=[3, 5, 2, 7, 1, 4, 6, 2, 5], ks=[2, 6, 3, 5, 4, 1, 7], ns=[4, 1, 3, 6, 2, 8])


@pytest.mark.parametrize("q", [1, 2, 3])
def test_cannon_matches_oracle_and_reference_ledger(oracle, reference, ctx, q):
    A, B, Cin = _inputs(oracle, 40 + q, **MIXED)
    want, _, _ = oracle.multiply(A, B, Cin)
    got, st, ledger, _ = _run(ctx, "cannon", q, q * q, A, B, Cin)
    assert_parity(got, want)
    _, _, rled = reference.multiply(A, B, Cin, "cannon", q, q * q)
    for r in range(q * q):
        assert ledger[r].elements_sent == rled[r]["sent"], r
        assert ledger[r].elements_received == rled[r]["received"], r
        assert ledger[r].meta_sent == rled[r]["meta_sent"], r
        assert ledger[r].meta_received == rled[r]["meta_received"], r
    if q == 1:
        assert st["elements_sent"] == 0


def test_cannon_dense_ledger_is_eq1_exact(oracle, ctx):
    """SPEC acceptance 2: dense uniform Cannon, mean per-rank = (MK+KN)/sqrt(P)."""
    from paper_1910_13555_b200 import dist as d
    n, bs, q = 6, 4, 3
    A, B, Cin = _inputs(oracle, 7, [bs] * n, [bs] * n, [bs] * n, 1.0, 1.0, 0.0)
    got, _, ledger, _ = _run(ctx, "cannon", q, q * q, A, B, Cin)
    mean = sum(ledger[r].elements_sent for r in range(q * q)) / (q * q)
    M = K = N = n * bs
    assert mean == (M * K + K * N) / q
    want, _, _ = oracle.multiply(A, B, Cin)
    assert_parity(got, want)
    del d


@pytest.mark.parametrize("nprocs", [1, 2, 4])
def test_case2_ring_matches_oracle_and_reference_ledger(oracle, reference, ctx, nprocs):
    rs = [5] * 24
    A, B, Cin = _inputs(oracle, 60 + nprocs, rs, [5] * 6, [5] * 5, 0.35, 0.5, 0.2)
    want, _, _ = oracle.multiply(A, B, Cin)
    got, _, ledger, phases = _run(ctx, "case2", 1, nprocs, A, B, Cin)
    assert_parity(got, want)
    _, _, rled = reference.multiply(A, B, Cin, "case2", 1, nprocs)
    for r in range(nprocs):
        assert ledger[r].elements_sent == rled[r]["sent"], (r, ledger[r], rled[r])
        assert ledger[r].elements_received == rled[r]["received"], r
        assert ledger[r].meta_sent == rled[r]["meta_sent"], r
        for p in ("ring", "redistribute", "collect"):
            assert phases[r][p] == rled[r].get("sent:" + p, 0), (r, p)


@pytest.mark.parametrize("nprocs", [2, 4])
def test_case2_gather_matches_oracle(oracle, ctx, nprocs):
    A, B, Cin = _inputs(oracle, 70 + nprocs, [7] * 20, [3] * 8, [6] * 5, 0.4, 0.4, 0.1)
    want, _, _ = oracle.multiply(A, B, Cin)
    got, _, _, _ = _run(ctx, "case2", 1, nprocs, A, B, Cin, gather=True)
    assert_parity(got, want)


@pytest.mark.parametrize("nprocs,q", [(1, 1), (4, 1), (3, 2), (5, 2)])
def test_case1_matches_oracle(oracle, reference, ctx, nprocs, q):
    A, B, Cin = _inputs(oracle, 80 + nprocs, [6] * 4, [4] * 30, [5] * 3, 0.4, 0.4, 0.3)
    want, _, _ = oracle.multiply(A, B, Cin)
    got, _, ledger, phases = _run(ctx, "case1", q, nprocs, A, B, Cin)
    assert_parity(got, want)
    # A and B move to the same K-slab owners as in the reference: same
    # redistribution traffic per rank
    _, _, rled = reference.multiply(A, B, Cin, "case1", q, nprocs)
    for r in range(max(q * q, nprocs)):
        assert phases[r]["redistribute"] == rled[r].get("sent:redistribute", 0), r


def _golden():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_golden().keys()))
def test_drivers_reproduce_golden(oracle, ctx, name):
    meta = _golden()[name]
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    sa, sb, sc = meta["seeds"]
    oa, ob, oc = meta["occ"]
    A = oracle.random_matrix(sa, z["rsz"], z["ksz"], oa)
    B = oracle.random_matrix(sb, z["ksz"], z["nsz"], ob)
    Cin = oracle.random_matrix(sc, z["rsz"], z["nsz"], oc)
    got, _, ledger, _ = _run(ctx, meta["algo"], meta["grid_q"], meta["nprocs"], A, B, Cin)
    gold = Blocks(z["rsz"], z["nsz"], z["c_bi"], z["c_bj"], z["c_vals"])
    assert_parity(got, gold)
    if meta["algo"] in ("cannon",):
        for r, led in meta["ledger"].items():
            assert ledger[int(r)].elements_sent == led["sent"]


def test_errors_match_reference_classes(oracle, ctx):
    from paper_1910_13555_b200 import dist as d
    comm = d.SimComm(d.ProcessGrid([2]), ctx=ctx)
    g12 = d.ProcessGrid([1, 2])
    bl = d.Blocking([2, 2])
    a = d.new_matrix_round_robin(bl, bl, g12, comm)
    with pytest.raises(d.GridError):
        d.multiply_cannon(comm, a, a, a)
    g11 = d.ProcessGrid([1, 1])
    a1 = d.new_matrix_round_robin(bl, bl, g11, comm)
    b1 = d.new_matrix_round_robin(d.Blocking([3]), bl, g11, comm)
    with pytest.raises(d.InvalidArgument):
        d.multiply_cannon(comm, a1, b1, a1)
    with pytest.raises(d.InvalidArgument):
        a1.put_block(0, 0, np.zeros((3, 2)))
    comm.close()


def test_redistribute_roundtrip_and_transpose(oracle, ctx):
    from paper_1910_13555_b200 import dist as d
    A = oracle.random_matrix(5, [3, 4, 2, 5, 1], [2, 6, 3, 4], 0.6)
    comm = d.SimComm(d.ProcessGrid([4]), ctx=ctx)
    g22 = d.ProcessGrid([2, 2])
    a = _dm(d, g22, comm, A)
    lin = d.redistribute(comm, a, a.rows(), a.cols(), d.ProcessGrid([4, 1]))
    assert_parity(_got(lin), A, tol=0.0)
    led = comm.ledger()
    moved = sum(led.rank_total(r).elements_sent for r in range(4))
    assert moved > 0
    t = d.redistribute(comm, a, a.cols(), a.rows(), g22, transpose=True)
    dense = _got(t).to_dense()
    assert np.array_equal(dense, A.to_dense().T)
    # identical layout moves nothing (test_matrix.cpp:202-208)
    comm.reset_ledger()
    same = d.redistribute(comm, a, a.rows(), a.cols(), g22)
    assert sum(comm.ledger().rank_total(r).elements_sent for r in range(4)) == 0
    assert_parity(_got(same), A, tol=0.0)
    comm.close()


@pytest.mark.parametrize("gdims,nprocs", [([2, 2], 4), ([2, 1], 2)])
def test_dispatch_auto(oracle, ctx, gdims, nprocs):
    """multiply_dispatch(Algorithm.auto): the fitted B200 model's choice among
    the algorithms whose layout preconditions hold (Cannon on the square
    round-robin grid), results equal to the oracle."""
    from paper_1910_13555_b200 import dist as dd
    grid = dd.ProcessGrid(gdims)
    comm = dd.SimComm(grid, ctx=ctx)
    sz = np.full(24, 23, np.int32)
    A = oracle.random_matrix(71, sz, sz, 0.3)
    B = oracle.random_matrix(72, sz, sz, 0.3)
    bl = dd.Blocking(sz)
    a = dd.new_matrix_round_robin(bl, bl, grid, comm)
    b = dd.new_matrix_round_robin(bl, bl, grid, comm)
    c = dd.new_matrix_round_robin(bl, bl, grid, comm)
    a.put_blocks(A.bi, A.bj, A.vals)
    b.put_blocks(B.bi, B.bj, B.vals)
    choice, times = dd.select_for(a, b, c, nprocs)
    if gdims == [2, 2]:
        assert dd.Algorithm.cannon in times
    else:
        assert dd.Algorithm.cannon not in times
    st = dd.multiply_dispatch(comm, dd.Algorithm.auto, a, b, c, nprocs)
    assert st["algorithm"] == dd.algorithm_name(choice)
    want, _, _ = oracle.multiply(A, B, Blocks.empty(sz, sz))
    bi, bj, v = c.blocks()
    assert_parity(Blocks(sz, sz, bi, bj, v), want)
    comm.close()
