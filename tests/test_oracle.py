"""Pins the CPU oracle (oracle/bt_oracle.c) before it is trusted as the checker.

1. The reference's own known-answer tests for the hot path
   (proj/tests/test_blocks.cpp:33-76).
2. The compiled reference itself (oracle/_ref/libbtref.so) on seeded inputs:
   Rng stream, random_matrix and the full multiply, bit for bit.
3. The committed golden fixtures (tests/golden/, made by make_golden.py from
   the compiled reference) -- these travel without /root/reference.
"""
import json
import os

import numpy as np
import pytest

from helpers import assert_parity
from oracle.oracle import Blocks

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def naive(c, a, b):
    """test_blocks.cpp:15-23: plain i-j-k loop, k innermost, unfused."""
    c = c.copy()
    for i in range(c.shape[0]):
        for j in range(c.shape[1]):
            acc = float(c[i, j])
            for k in range(a.shape[1]):
                acc += float(a[i, k]) * float(b[k, j])
            c[i, j] = acc
    return c


def test_kat_identity(oracle):
    # test_blocks.cpp:34-40
    c = oracle.block_gemm_acc(np.zeros((2, 2)), np.eye(2), np.array([[1., 2.], [3., 4.]]))
    assert c.tolist() == [[1, 2], [3, 4]]


def test_kat_accumulate_16(oracle):
    # test_blocks.cpp:41-47: 5 + 1*3 + 2*4 = 16
    c = oracle.block_gemm_acc(np.array([[5.0]]), np.array([[1., 2.]]), np.array([[3.], [4.]]))
    assert c.tolist() == [[16.0]]


def _rblock(oracle, rng, m, n):
    return np.array([oracle.lib.bto_rng_normal(rng) for _ in range(m * n)]).reshape(m, n)


def test_kat_bit_identical_to_naive(oracle, reference):
    # test_blocks.cpp:54-76 with Rng(7): 3x4*4x2, then m,k,n in {1,4,7}
    rng = oracle.rng(7)
    shapes = [(3, 4, 2)] + [(m, k, n) for m in (1, 4, 7) for k in (1, 4, 7) for n in (1, 4, 7)]
    for m, k, n in shapes:
        a = _rblock(oracle, rng, m, k)
        b = _rblock(oracle, rng, k, n)
        c = _rblock(oracle, rng, m, n)
        want = naive(c, a, b)
        assert np.array_equal(oracle.block_gemm_acc(c, a, b), want)
        assert np.array_equal(reference.block_gemm_acc(c, a, b), want)


@pytest.mark.parametrize("seed,occ", [(1, 0.1), (42, 0.5), (7, 1.0), (3, 0.0)])
def test_random_matrix_matches_reference(oracle, reference, seed, occ):
    rs = np.array([3, 5, 2, 7, 1, 4, 9, 2], np.int32)
    cs = np.array([2, 6, 3, 5, 4], np.int32)
    a = oracle.random_matrix(seed, rs, cs, occ)
    b = reference.random_matrix(seed, rs, cs, occ)
    assert np.array_equal(a.bi, b.bi) and np.array_equal(a.bj, b.bj)
    assert np.array_equal(a.vals, b.vals)


def test_random_blocking_rule(oracle):
    # oracles.hpp:60-70: sizes in [bmin, bmax] summing to total
    s = oracle.random_blocking(5, 100, 1, 9)
    assert s.sum() == 100 and s.min() >= 1 and s.max() <= 9


@pytest.mark.parametrize("seed", range(8))
def test_multiply_bit_exact_vs_reference_cannon_1x1(oracle, reference, seed):
    rng = np.random.default_rng(seed)
    rs = rng.integers(1, 10, 7).astype(np.int32)
    ks = rng.integers(1, 10, 6).astype(np.int32)
    ns = rng.integers(1, 10, 5).astype(np.int32)
    A = oracle.random_matrix(seed, rs, ks, 0.4)
    B = oracle.random_matrix(seed + 50, ks, ns, 0.4)
    C = oracle.random_matrix(seed + 99, rs, ns, 0.2)
    mine, _, _ = oracle.multiply(A, B, C)
    ref, _, _ = reference.multiply(A, B, C, "cannon", 1)
    assert np.array_equal(mine.bi, ref.bi) and np.array_equal(mine.bj, ref.bj)
    assert np.array_equal(mine.vals, ref.vals)  # bit-identical


@pytest.mark.parametrize("algo,q,p", [("cannon", 2, 4), ("cannon", 3, 9), ("case1", 1, 4),
                                      ("case2", 1, 3), ("case1", 2, 5)])
def test_pattern_independent_of_algorithm(oracle, reference, algo, q, p):
    rs = np.array([4, 3, 5, 2, 6, 1, 3], np.int32)
    A = oracle.random_matrix(3, rs, rs, 0.4)
    B = oracle.random_matrix(4, rs, rs, 0.4)
    C = oracle.random_matrix(5, rs, rs, 0.1)
    mine, _, _ = oracle.multiply(A, B, C)
    ref, _, _ = reference.multiply(A, B, C, algo, q, p)
    assert_parity(ref, mine, tol=1e-14)


def test_eps_zero_equals_unfiltered(oracle):
    rs = np.array([5, 13, 23, 5], np.int32)
    A = oracle.random_matrix(1, rs, rs, 0.6, 12.0)
    B = oracle.random_matrix(2, rs, rs, 0.6, 12.0)
    C = Blocks.empty(rs, rs)
    a, n0, _ = oracle.multiply(A, B, C, 0.0)
    b, n1, _ = oracle.multiply(A, B, C, 1e-300)
    assert n0 == n1 and np.array_equal(a.vals, b.vals)
    c, n2, _ = oracle.multiply(A, B, C, 1e-8)
    assert n2 < n0  # scaled values: the filter removes products


def _golden():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_golden().keys()))
def test_oracle_reproduces_golden(oracle, name):
    meta = _golden()[name]
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    sa, sb, sc = meta["seeds"]
    oa, ob, oc = meta["occ"]
    A = oracle.random_matrix(sa, z["rsz"], z["ksz"], oa)
    B = oracle.random_matrix(sb, z["ksz"], z["nsz"], ob)
    C = oracle.random_matrix(sc, z["rsz"], z["nsz"], oc)
    mine, _, _ = oracle.multiply(A, B, C)
    gold = Blocks(z["rsz"], z["nsz"], z["c_bi"], z["c_bj"], z["c_vals"])
    if meta["algo"] == "cannon" and meta["grid_q"] == 1:
        assert np.array_equal(mine.vals, gold.vals) and np.array_equal(mine.bj, gold.bj)
    assert_parity(mine, gold, tol=1e-14)


def test_mixed_radix_roundtrip(oracle):
    # dims (3,4 | 5), coords (2,3,4) -> (2*4+3, 4) = (11, 4)
    assert oracle.mixed_radix([2, 3], [3, 4]) == 11
    ext = [2, 3, 2]
    seen = set()
    for idx in range(12):
        c = oracle.mixed_radix_inv(idx, ext)
        assert oracle.mixed_radix(c, ext) == idx
        seen.add(tuple(c))
    assert len(seen) == 12
