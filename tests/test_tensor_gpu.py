"""Tensor contraction on the GPU vs a nested-loop dense
oracle.  No reference code exists for tensors: parity is pinned to the spec's
canonical test and its layout-independence property
(SPEC.md:528-531), at tolerance 1e-12."""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand_tensor(ctx, rng, sizes, row_dims, col_dims, occ):
    from paper_1910_13555_b200.tensor import SparseTensor
    t = SparseTensor(ctx, sizes, row_dims, col_dims)
    items = []
    for coords in itertools.product(*[range(len(s)) for s in sizes]):
        if rng.random() < occ:
            items.append((list(coords), rng.standard_normal(t.block_shape(coords))))
    t.put_blocks(items)
    return t


def _rel(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / max(np.sum(b * b), 1e-300)))


def test_spec_canonical_contraction(ctx):
    """C_mn = sum_kl A_mkl B_kln, dims 6,4,4,6, blocks of 2."""
    from paper_1910_13555_b200.tensor import SparseTensor, contract
    rng = np.random.default_rng(1)
    two = lambda n: np.full(n // 2, 2, np.int32)  # noqa: E731
    A = _rand_tensor(ctx, rng, [two(6), two(4), two(4)], [0], [1, 2], 0.7)
    B = _rand_tensor(ctx, rng, [two(4), two(4), two(6)], [0, 1], [2], 0.7)
    Cm = SparseTensor(ctx, [two(6), two(6)], [0], [1])
    contract(A, B, [1, 2], [0, 1], Cm)
    want = np.zeros((6, 6))
    Ad, Bd = A.to_dense(), B.to_dense()
    for m, n, k, l in itertools.product(range(6), range(6), range(4), range(4)):
        want[m, n] += Ad[m, k, l] * Bd[k, l, n]
    assert _rel(Cm.to_dense(), want) <= 1e-12


@pytest.mark.parametrize("amap", [([0], [1, 2]), ([1, 2], [0]), ([2, 0], [1]), ([1], [0, 2])])
def test_every_legal_map_gives_the_same_values(ctx, amap):
    """rank-3 x rank-3 over 2 indices; layout independence."""
    from paper_1910_13555_b200.tensor import SparseTensor, contract
    rng = np.random.default_rng(7)
    s = [np.array([3, 2, 4], np.int32), np.array([2, 3], np.int32), np.array([4, 1, 2], np.int32)]
    A = _rand_tensor(ctx, rng, s, *amap, 0.6)
    B = _rand_tensor(ctx, rng, [s[1], s[2], s[0]], [2], [0, 1], 0.6)
    Cm = SparseTensor(ctx, [s[0], s[0]], [1], [0])  # incompatible C map on purpose
    contract(A, B, [1, 2], [0, 1], Cm)
    want = np.einsum("mkl,kln->mn", A.to_dense(), B.to_dense())
    assert _rel(Cm.to_dense(), want) <= 1e-12


def test_remap_roundtrip_is_exact(ctx):
    rng = np.random.default_rng(3)
    s = [np.array([2, 3], np.int32), np.array([1, 4, 2], np.int32), np.array([3, 3], np.int32),
         np.array([2, 5], np.int32)]
    T = _rand_tensor(ctx, rng, s, [0, 2], [3, 1], 0.5)
    U = T.remap([3], [1, 0, 2]).remap([0, 2], [3, 1])
    assert np.array_equal(T.to_dense(), U.to_dense())
    assert np.array_equal(T.to_dense(), T.remap([1, 2, 3], [0]).to_dense())


def test_rpa_like_3c_contraction_tall_blocks(ctx):
    """config-4 shape at small scale: R_(ab)Q = sum_P T_(ab)P M_PQ, AO blocks 13/23
    -> matricized rows of 169/299/529 (tall DMMA tiles)."""
    from paper_1910_13555_b200.tensor import SparseTensor, contract
    rng = np.random.default_rng(11)
    ao = np.array([13, 23, 13], np.int32)
    aux = np.array([23, 13, 23, 13], np.int32)
    T = _rand_tensor(ctx, rng, [ao, ao, aux], [0, 1], [2], 0.4)
    M = _rand_tensor(ctx, rng, [aux, aux], [0], [1], 0.6)
    R = SparseTensor(ctx, [ao, ao, aux], [0, 1], [2])
    st = contract(T, M, [2], [0], R)
    want = np.einsum("abp,pq->abq", T.to_dense(), M.to_dense())
    assert _rel(R.to_dense(), want) <= 1e-12
    assert st["products"] > 0


def test_map_errors(ctx):
    from paper_1910_13555_b200 import InvalidArgument
    from paper_1910_13555_b200.tensor import SparseTensor
    s = np.array([2, 2], np.int32)
    with pytest.raises(InvalidArgument):
        SparseTensor(ctx, [s, s, s], [0, 1], [1])
    with pytest.raises(InvalidArgument):
        SparseTensor(ctx, [s, s, s], [0, 1, 2], [])
