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
