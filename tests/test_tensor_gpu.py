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


def _rand_items(rng, sizes, occ):
    items = []
    for coords in itertools.product(*[range(len(s)) for s in sizes]):
        if rng.random() < occ:
            items.append((list(coords), rng.standard_normal([int(s[c]) for s, c in
                                                             zip(sizes, coords)])))
    return items


def _dense_of(sizes, items):
    offs = [np.concatenate([[0], np.cumsum(s)]) for s in sizes]
    out = np.zeros([int(o[-1]) for o in offs])
    for coords, blk in items:
        out[tuple(slice(offs[d][c], offs[d][c] + blk.shape[d]) for d, c in enumerate(coords))] = blk
    return out


def test_rank4_contraction_with_remaps(ctx):
    """Rank-4 x rank-4 over two indices, every operand (and C) in a map that
    needs a remap: C_ijmn = sum_kl A_ikjl B_lkmn."""
    from paper_1910_13555_b200.tensor import SparseTensor, contract
    rng = np.random.default_rng(44)
    s = [np.array([3, 5], np.int32), np.array([4, 2, 3], np.int32),
         np.array([2, 6], np.int32), np.array([5, 1, 3], np.int32),
         np.array([2, 3], np.int32), np.array([4, 4], np.int32)]
    i, k, j, l, m, n = s
    A = _rand_tensor(ctx, rng, [i, k, j, l], [0], [1, 2, 3], 0.5)
    B = _rand_tensor(ctx, rng, [l, k, m, n], [2, 0], [1, 3], 0.5)
    Cm = SparseTensor(ctx, [i, j, m, n], [0, 2], [1, 3])
    contract(A, B, [1, 3], [1, 0], Cm)
    want = np.einsum("ikjl,lkmn->ijmn", A.to_dense(), B.to_dense())
    assert _rel(Cm.to_dense(), want) <= 1e-12


@pytest.mark.parametrize("gdims", [[2, 2], [2, 1], [1, 3]])
def test_dist_contraction_virtual_ranks_and_ledger(gdims):
    """contract_dist on virtual ranks: the canonical rank-3 contraction and a
    rank-4 one.  Compatible maps: no remap traffic ("tensor_remap" ledger 0,
    SPEC.md 'compatibility fast path'); incompatible maps: identical values
    (<= 1e-12) and a strictly larger ledger."""
    from paper_1910_13555_b200 import dist as dd
    from paper_1910_13555_b200.tensor import DistTensor, contract_dist
    grid = dd.ProcessGrid(gdims)
    comm = dd.SimComm(grid)
    rng = np.random.default_rng(sum(gdims))
    two = lambda q: np.full(q // 2, 2, np.int32)  # noqa: E731
    sa = [two(6), two(4), two(4)]
    sb = [two(4), two(4), two(6)]
    ia, ib = _rand_items(rng, sa, 0.7), _rand_items(rng, sb, 0.7)
    want = np.einsum("mkl,kln->mn", _dense_of(sa, ia), _dense_of(sb, ib))
    results = {}
    for mode in ("compatible", "remapped"):
        comm.reset_ledger()
        amap = ([0], [1, 2]) if mode == "compatible" else ([2], [0, 1])
        bmap = ([0, 1], [2]) if mode == "compatible" else ([1], [2, 0])
        cmap = ([0], [1]) if mode == "compatible" else ([1], [0])
        A = DistTensor(comm, sa, *amap)
        A.put_blocks(ia)
        B = DistTensor(comm, sb, *bmap)
        B.put_blocks(ib)
        Cm = DistTensor(comm, [two(6), two(6)], *cmap)
        contract_dist(A, B, [1, 2], [0, 1], Cm)
        got = Cm.to_dense()
        assert _rel(got, want) <= 1e-12
        led = comm.ledger()
        results[mode] = (got, sum(led.rank_phase(r, "tensor_remap").elements_sent
                                  for r in range(grid.size())), led.total_elements_sent())
    assert results["compatible"][1] == 0
    if grid.size() > 1:
        assert results["remapped"][1] > 0
        assert results["remapped"][2] > results["compatible"][2]
    assert _rel(results["remapped"][0], results["compatible"][0]) <= 1e-12
    # rank 4 on the same group
    s4 = [np.array([3, 5], np.int32), np.array([4, 2], np.int32), np.array([2, 6], np.int32),
          np.array([5, 1], np.int32)]
    i, k, j, l = s4
    ia4 = _rand_items(rng, [i, k, j, l], 0.6)
    ib4 = _rand_items(rng, [l, k, j, i], 0.6)
    A = DistTensor(comm, [i, k, j, l], [0, 2], [1, 3])
    A.put_blocks(ia4)
    B = DistTensor(comm, [l, k, j, i], [1], [0, 2, 3])
    B.put_blocks(ib4)
    Cm = DistTensor(comm, [i, j, j, i], [0, 1], [2, 3])
    contract_dist(A, B, [1, 3], [1, 0], Cm)
    want4 = np.einsum("ikjl,lkmn->ijmn", _dense_of([i, k, j, l], ia4),
                      _dense_of([l, k, j, i], ib4))
    assert _rel(Cm.to_dense(), want4) <= 1e-12
    comm.close()
