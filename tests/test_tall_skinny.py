"""Tall-and-skinny layer: the spec's examples for
the partition rule and the split factor (CPU), and submatrix multiplies on one
B200 with virtual ranks against the oracle (GPU)."""
import numpy as np
import pytest

from helpers import assert_parity
from oracle.oracle import Blocks
from paper_1910_13555_b200 import tall_skinny as ts
from paper_1910_13555_b200._lib import InvalidArgument, LayoutError


def test_ceil_partition_spec_examples():
    assert ts.ceil_partition(12, 3) == [(0, 4), (4, 8), (8, 12)]
    assert ts.ceil_partition(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert ts.ceil_partition(5, 1) == [(0, 5)]


def test_choose_split_factor_spec_examples():
    assert ts.choose_split_factor(1000, 1000, 8) == 1
    assert ts.choose_split_factor(100 * 7, 7, 10) == 10
    assert ts.choose_split_factor(4 * 9, 9, 16) == 4
    with pytest.raises(InvalidArgument):
        ts.choose_split_factor(0, 1, 4)


def test_index_funcs_validation():
    f = ts.IndexFuncs(10, lambda b: 13 if b % 2 else 23, lambda b: b % 2)
    assert f.size(3) == 13 and f.dist(3) == 1 and f.total_elements() == 5 * 13 + 5 * 23
    with pytest.raises(InvalidArgument):
        f.size(10)
    with pytest.raises(InvalidArgument):
        ts.IndexFuncs(2, lambda b: 0, lambda b: 0).size(0)


def _funcs(n, sizes=(5, 13, 23), extent=2):
    return ts.IndexFuncs(n, lambda b: sizes[(7 * b) % len(sizes)], lambda b: b % extent)


def _blocks_for(oracle, seed, rf, cf, occ):
    rs = np.array([rf.size(b) for b in range(rf.n_blocks)], np.int32)
    cs = np.array([cf.size(b) for b in range(cf.n_blocks)], np.int32)
    return oracle.random_matrix(seed, rs, cs, occ)


@pytest.mark.gpu
def test_k_split_matches_oracle(oracle, ctx):
    """A 8x128 split f=4 on K, B 128x8 split f=4 -> C equals the oracle."""
    from paper_1910_13555_b200 import dist as d
    grid = d.ProcessGrid([2, 2])
    comm = d.SimComm(d.ProcessGrid([4]), ctx=ctx)
    fm, fk, fn = _funcs(8), _funcs(128), _funcs(8)
    A = _blocks_for(oracle, 61, fm, fk, 0.3)
    B = _blocks_for(oracle, 62, fk, fn, 0.3)
    a = ts.create_tall_skinny(fm, fk, grid, "cols", 2, comm)
    b = ts.create_tall_skinny(fk, fn, grid, "rows", 2, comm)
    a.put_blocks(A.bi, A.bj, A.vals)
    b.put_blocks(B.bi, B.bj, B.vals)
    # no rank-side index array along K longer than one submatrix's range
    assert a.max_resident_index_length() == 64 and b.max_resident_index_length() == 64
    rs = np.array([fm.size(i) for i in range(8)], np.int32)
    ns = np.array([fn.size(j) for j in range(8)], np.int32)
    c = d.new_matrix(d.Blocking(rs), d.Blocking(ns), grid, np.arange(8) % 2, np.arange(8) % 2,
                     comm)
    st = ts.multiply_tall_skinny(a, b, c, 4)
    want, nprod, _ = oracle.multiply(A, B, Blocks.empty(rs, ns))
    assert st["products"] == nprod and st["multiplies"] == 2
    bi, bj, v = c.blocks()
    assert_parity(Blocks(rs, ns, bi, bj, v), want)
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("factor", [1, 2])
def test_m_split_and_degenerate(oracle, ctx, factor):
    """M split (A and C split on rows the same way); f=1 is a plain multiply."""
    from paper_1910_13555_b200 import dist as d
    grid = d.ProcessGrid([2, 2])
    comm = d.SimComm(d.ProcessGrid([4]), ctx=ctx)
    fm, fk, fn = _funcs(40), _funcs(6), _funcs(5)
    A = _blocks_for(oracle, 71, fm, fk, 0.4)
    B = _blocks_for(oracle, 72, fk, fn, 0.4)
    a = ts.create_tall_skinny(fm, fk, grid, "rows", factor, comm)
    a.put_blocks(A.bi, A.bj, A.vals)
    ks = np.array([fk.size(k) for k in range(6)], np.int32)
    ns = np.array([fn.size(j) for j in range(5)], np.int32)
    b = d.new_matrix(d.Blocking(ks), d.Blocking(ns), grid, np.arange(6) % 2, np.arange(5) % 2,
                     comm)
    b.put_blocks(B.bi, B.bj, B.vals)
    c = ts.create_tall_skinny(fm, fn, grid, "rows", factor, comm)
    # bijection global <-> (submatrix, local)
    for i in range(40):
        s, li = c.locate(i)
        assert c.global_index(s, li) == i
    st = ts.multiply_tall_skinny(a, b, c, 4, select=d.select_algorithm_b200)
    rs = np.array([fm.size(i) for i in range(40)], np.int32)
    want, nprod, _ = oracle.multiply(A, B, Blocks.empty(rs, ns))
    assert st["products"] == nprod and st["multiplies"] == factor
    bi, bj, v = c.blocks()
    assert_parity(Blocks(rs, ns, bi, bj, v), want)
    comm.close()


@pytest.mark.gpu
def test_incompatible_split_raises(ctx):
    from paper_1910_13555_b200 import dist as d
    grid = d.ProcessGrid([2, 2])
    comm = d.SimComm(d.ProcessGrid([4]), ctx=ctx)
    a = ts.create_tall_skinny(_funcs(4), _funcs(16), grid, "cols", 2, comm)
    b = ts.create_tall_skinny(_funcs(16), _funcs(4), grid, "rows", 1, comm)
    c = ts.create_tall_skinny(_funcs(4), _funcs(4), grid, "rows", 1, comm)
    with pytest.raises(LayoutError):
        ts.multiply_tall_skinny(a, b, c.subs[0], 4)
    with pytest.raises(InvalidArgument):
        ts.create_tall_skinny(_funcs(4), _funcs(16), grid, "cols", 3, comm)
    comm.close()
