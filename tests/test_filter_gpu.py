"""Block norms and the eps post-filter (bt_mat_norms / bt_filter_report) against
the oracle's restatement (bto_block_norm / bto_filter, oracle/bt_oracle.c).

The reference fixes eps = 0, so the filter is build-defined
(DESIGN.md 3): norm = sqrt of the row-ordered sum of unfused row sums of
squares; bt_filter drops blocks with ||C_ij||_F < eps.  Norms of stored
(put) blocks are bit-identical to the oracle's.  After a multiply the GPU's C
values differ from the oracle's by ULPs (fused DMMA, another summation
order), so a post-filter decision can only differ for blocks within
1e-12 * eps of eps: those are reported as borderline and the
patterns must agree on every other block.
"""
import numpy as np
import pytest

from helpers import assert_parity, from_store, to_store
from oracle.oracle import Blocks

pytestmark = pytest.mark.gpu

BAND = 1e-12


def _mixed(oracle, seed, sizes, occ, scale=0.0):
    sz = np.asarray(sizes, np.int32)
    return oracle.random_matrix(seed, sz, sz, occ, scale)


@pytest.mark.parametrize("sizes", [[5, 13, 23] * 6, [1, 4, 7, 8, 9, 16, 31, 32],
                                   [37, 40, 5, 64, 33]])
def test_put_store_norms_bit_identical(oracle, ctx, sizes):
    A = _mixed(oracle, 7, sizes, 0.5, 6.0)
    a = to_store(ctx, A)
    got = a.norms()
    want = oracle.norms(A)
    assert got.shape == want.shape
    assert np.array_equal(got, want), np.max(np.abs(got - want) / want)


@pytest.mark.parametrize("eps_q", [0.1, 0.5, 0.9])
def test_filter_put_store_matches_oracle(oracle, ctx, eps_q):
    A = _mixed(oracle, 11, [5, 13, 23] * 8, 0.4, 8.0)
    nrm = oracle.norms(A)
    eps = float(np.quantile(nrm, eps_q))
    want = oracle.filter(A, eps)
    a = to_store(ctx, A)
    rep = a.filter(eps, BAND)
    got = from_store(a)
    assert rep["dropped"] == A.nblk - want.nblk
    # put-store norms are bit-identical, so the only borderline blocks are those
    # the oracle itself sees within the band
    assert rep["borderline"] == int(np.sum(np.abs(nrm - eps) <= BAND * eps))
    assert np.array_equal(got.bi, want.bi) and np.array_equal(got.bj, want.bj)
    assert np.array_equal(got.vals, want.vals)  # a filter moves values, never changes them
    # the cached norms follow the filtered store
    assert np.array_equal(a.norms(), oracle.norms(want))


def test_filter_after_multiply_reports_borderline(oracle, ctx):
    """Post-filter of a multiply's C: identical decisions except borderline blocks.
    The threshold is put exactly on one block's (oracle) norm so the borderline
    report is exercised with a real straddling block."""
    from paper_1910_13555_b200.store import multiply_local
    sz = np.array([5, 13, 23] * 6, np.int32)
    A = oracle.random_matrix(21, sz, sz, 0.3, 4.0)
    B = oracle.random_matrix(22, sz, sz, 0.3, 4.0)
    want_c, _, _ = oracle.multiply(A, B, Blocks.empty(sz, sz))
    cn = oracle.norms(want_c)
    eps = float(np.sort(cn)[len(cn) // 2])      # a block sits exactly on eps
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Blocks.empty(sz, sz))
    multiply_local(ctx, a, b, c)
    gpu_c = from_store(c)
    gn = c.norms()
    # norms of ULP-different values: within a few ULPs of the oracle's
    assert np.max(np.abs(gn - cn) / cn) <= 1e-13
    rep = c.filter(eps, BAND)
    border_oracle = np.abs(cn - eps) <= BAND * eps
    assert border_oracle.sum() >= 1
    border_gpu = np.abs(gn - eps) <= BAND * eps
    assert rep["borderline"] == int(border_gpu.sum())
    kept_gpu = gn >= eps
    kept_oracle = cn >= eps
    differ = kept_gpu != kept_oracle
    # every differing decision is a reported borderline block
    assert np.all(border_gpu[differ] | border_oracle[differ])
    want = oracle.filter(want_c, eps)
    got = from_store(c)
    sel = ~(border_gpu | border_oracle)
    key = lambda bi, bj: set(zip(bi.tolist(), bj.tolist()))
    gk = key(got.bi, got.bj)
    wk = key(want.bi, want.bj)
    allk = list(zip(gpu_c.bi.tolist(), gpu_c.bj.tolist()))
    for t, k in enumerate(allk):
        if sel[t]:
            assert (k in gk) == (k in wk), k
    assert rep["dropped"] == gpu_c.nblk - got.nblk


def test_generic_blocks_zero_padding(oracle, ctx):
    """n > 32 blocks go to the generic kernel; its output slot padding must be
    zero: the norms of C (which read the column padding) and C used
    as the A operand of a DMMA multiply (which reads the k padding) must match
    the oracle.  The pool is first dirtied with NaN so stale padding shows."""
    from paper_1910_13555_b200.store import multiply_local
    sz = np.array([37, 40, 13, 5, 40, 37], np.int32)
    A = oracle.random_matrix(31, sz, sz, 0.6)
    B = oracle.random_matrix(32, sz, sz, 0.6)
    C1, _, _ = oracle.multiply(A, B, Blocks.empty(sz, sz))
    a, b = to_store(ctx, A), to_store(ctx, B)
    full = oracle.random_matrix(33, sz, sz, 1.0)
    for _ in range(3):
        junk = to_store(ctx, Blocks(full.rsz, full.csz, full.bi, full.bj,
                                    np.full_like(full.vals, np.nan)))
        junk.close()
    c = to_store(ctx, Blocks.empty(sz, sz))
    multiply_local(ctx, a, b, c)
    assert_parity(from_store(c), C1)
    cn = oracle.norms(C1)
    assert np.max(np.abs(c.norms() - cn) / cn) <= 1e-13
    # C as the A operand; D's narrow columns make DMMA read C's k padding
    nsz = np.array([13, 5, 8], np.int32)
    D = oracle.random_matrix(34, sz, nsz, 0.7)
    want2, _, _ = oracle.multiply(C1, D, Blocks.empty(sz, nsz))
    d = to_store(ctx, D)
    e = to_store(ctx, Blocks.empty(sz, nsz))
    multiply_local(ctx, c, d, e)
    got2 = from_store(e)
    assert np.all(np.isfinite(got2.vals))
    assert_parity(got2, want2)


def test_eps_multiply_uses_cached_norms(oracle, ctx):
    """The eps product filter reads the cached norms; after a put changes A the
    cache is recomputed (a stale cache would keep the old decisions)."""
    from paper_1910_13555_b200.store import multiply_local
    sz = np.array([5, 13, 23] * 5, np.int32)
    A = oracle.random_matrix(41, sz, sz, 0.3, 12.0)
    B = oracle.random_matrix(42, sz, sz, 0.3, 12.0)
    eps = 1e-8
    a, b = to_store(ctx, A), to_store(ctx, B)
    for _ in range(2):   # second call: norms from the cache
        c = to_store(ctx, Blocks.empty(sz, sz))
        st = multiply_local(ctx, a, b, c, eps)
        want, nprod, _ = oracle.multiply(A, B, Blocks.empty(sz, sz), eps)
        assert st["products"] == nprod
        assert_parity(from_store(c), want)
    # scale every block of A up: more products survive; the cache must follow
    A2 = Blocks(A.rsz, A.csz, A.bi, A.bj, A.vals * 1e6)
    a.put_blocks(A2.bi, A2.bj, A2.vals)      # replace
    c = to_store(ctx, Blocks.empty(sz, sz))
    st = multiply_local(ctx, a, b, c, eps)
    want, nprod, _ = oracle.multiply(A2, B, Blocks.empty(sz, sz), eps)
    assert st["products"] == nprod
    assert_parity(from_store(c), want)
