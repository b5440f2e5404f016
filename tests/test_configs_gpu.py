"""BASELINE configs 2-4 at full size on one B200 against the oracle (C
restatement): C pattern bit-exact, values <= 1e-12 Frobenius-relative, the
product count (after the eps filter) identical.  Inputs: tools/run_config.py."""
import os
import sys

import numpy as np
import pytest

from helpers import assert_parity
from oracle.oracle import Blocks

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tools"))


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_config_full_size(oracle, ctx, name):
    import run_config
    from paper_1910_13555_b200.store import LocalStore, multiply_local
    rsz, ksz, nsz, A, B, eps, _ = run_config.config(name, np.random.default_rng(2024))
    a = LocalStore(ctx, rsz, ksz)
    a.put_blocks(*A)
    b = LocalStore(ctx, ksz, nsz)
    b.put_blocks(*B)
    c = LocalStore(ctx, rsz, nsz)
    st = multiply_local(ctx, a, b, c, eps)
    want, nprod, flops = oracle.multiply(Blocks(rsz, ksz, *A), Blocks(ksz, nsz, *B),
                                         Blocks.empty(rsz, nsz), eps)
    assert st["products"] == nprod
    assert st["flops"] == flops
    bi, bj, v = c.export()
    assert_parity(Blocks(rsz, nsz, bi, bj, v), want)
    for s in (a, b, c):
        s.close()


def test_c4_through_contract_full_size(oracle, ctx):
    """BASELINE config 4 through the tensor API at full size (tools/run_c4_contract.py's
    workload): R_(ab)Q = sum_P T_(ab)P M_PQ with contract(), T given both in the
    compatible layout ((a,b),(P)) and stored as ((a),(b,P)) so that contract()
    remaps it on the device first.  Both results against the oracle's multiply
    of the matricized operands (pattern bit-exact, values <= 1e-12), and
    bit-identical to each other (the remap is an exact permutation)."""
    import run_config
    from paper_1910_13555_b200.tensor import SparseTensor, contract
    rows, aux, _, T, M, eps, _ = run_config.config("c4", np.random.default_rng(2024))
    ao = np.tile(np.array([13, 23], np.int32), 100)
    t = SparseTensor(ctx, [ao, ao, aux], [0, 1], [2])
    t.store.put_blocks(*T)
    m = SparseTensor(ctx, [aux, aux], [0], [1])
    m.store.put_blocks(*M)
    t_alt = t.remap([0], [1, 2])
    want, nprod, flops = oracle.multiply(Blocks(rows, aux, *T), Blocks(aux, aux, *M),
                                         Blocks.empty(rows, aux), eps)
    got = {}
    for name, src in (("compatible", t), ("remapped", t_alt)):
        r = SparseTensor(ctx, [ao, ao, aux], [0, 1], [2])
        st = contract(src, m, [2], [0], r)
        assert st["products"] == nprod and st["flops"] == flops
        bi, bj, v = r.store.export()
        got[name] = Blocks(rows, aux, bi, bj, v)
        assert_parity(got[name], want)
        r.store.close()
    assert np.array_equal(got["compatible"].vals, got["remapped"].vals)
