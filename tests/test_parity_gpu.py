"""GPU parity: libbtcuda (through the C-ABI) vs the oracle on seeded inputs.

Pattern and block index bit-exact; values within 1e-12 Frobenius-relative
(north_star tolerance, FP64), globally and per block.
"""
import numpy as np
import pytest

from helpers import assert_parity, from_store, to_store

pytestmark = pytest.mark.gpu


def _case(oracle, seed, rsz, ksz, nsz, occ_a, occ_b, occ_c, scale=0.0):
    A = oracle.random_matrix(seed, rsz, ksz, occ_a, scale)
    B = oracle.random_matrix(seed + 1, ksz, nsz, occ_b, scale)
    Cin = oracle.random_matrix(seed + 2, rsz, nsz, occ_c, scale)
    return A, B, Cin


@pytest.mark.parametrize("bs", [1, 4, 5, 7, 8, 13, 16, 20, 23, 24, 32])
def test_uniform_blocks(oracle, ctx, bs):
    n = 12
    A, B, Cin = _case(oracle, 100 + bs, [bs] * n, [bs] * n, [bs] * n, 0.3, 0.3, 0.1)
    want, nprod, flops = oracle.multiply(A, B, Cin)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    from paper_1910_13555_b200.store import multiply_local
    st = multiply_local(ctx, a, b, c)
    assert st["products"] == nprod
    assert st["flops"] == flops
    assert_parity(from_store(c), want)


@pytest.mark.parametrize("seed", range(6))
def test_mixed_blocks(oracle, ctx, seed):
    rng = np.random.default_rng(seed)
    rsz = rng.integers(1, 10, 9).astype(np.int32)
    ksz = rng.integers(1, 10, 7).astype(np.int32)
    nsz = rng.integers(1, 10, 8).astype(np.int32)
    A, B, Cin = _case(oracle, 10 * seed, rsz, ksz, nsz, 0.4, 0.4, 0.2)
    want, nprod, _ = oracle.multiply(A, B, Cin)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    from paper_1910_13555_b200.store import multiply_local
    st = multiply_local(ctx, a, b, c)
    assert st["products"] == nprod
    assert_parity(from_store(c), want)


def test_h2o_sizes_with_filter(oracle, ctx):
    rng = np.random.default_rng(5)
    sizes = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 40)]
    A, B, Cin = _case(oracle, 77, sizes, sizes, sizes, 0.2, 0.2, 0.0, scale=12.0)
    for eps in (0.0, 1e-8):
        want, nprod, flops = oracle.multiply(A, B, Cin, eps)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        from paper_1910_13555_b200.store import multiply_local
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod
        assert st["flops"] == flops
        assert_parity(from_store(c), want)


def test_tall_blocks(oracle, ctx):
    rsz = np.array([169, 299, 529, 40], np.int32)
    ksz = np.array([13, 23, 13, 23, 13], np.int32)
    nsz = np.array([23, 13, 23], np.int32)
    A, B, Cin = _case(oracle, 5, rsz, ksz, nsz, 0.6, 0.6, 0.3)
    want, nprod, _ = oracle.multiply(A, B, Cin)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    from paper_1910_13555_b200.store import multiply_local
    multiply_local(ctx, a, b, c)
    assert_parity(from_store(c), want)


def test_generic_large_blocks(oracle, ctx):
    A, B, Cin = _case(oracle, 9, [40, 70], [33, 80, 20], [48, 65], 0.8, 0.8, 0.5)
    want, _, _ = oracle.multiply(A, B, Cin)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    from paper_1910_13555_b200.store import multiply_local
    multiply_local(ctx, a, b, c)
    assert_parity(from_store(c), want)


def test_config1_pattern_and_values(oracle, ctx):
    """BASELINE config 1 (400^2 blocks of 23, 10 %), pinned seeds 1001/1002."""
    sz = np.full(400, 23, np.int32)
    A = oracle.random_matrix(1001, sz, sz, 0.10)
    B = oracle.random_matrix(1002, sz, sz, 0.10)
    Cin = oracle.random_matrix(1003, sz, sz, 0.0)
    want, nprod, flops = oracle.multiply(A, B, Cin)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    from paper_1910_13555_b200.store import multiply_local
    st = multiply_local(ctx, a, b, c)
    assert st["products"] == nprod and st["flops"] == flops
    assert_parity(from_store(c), want)


@pytest.mark.parametrize("npanels", [2, 3, 7])
def test_k_panels(oracle, ctx, monkeypatch, npanels):
    """K-panel L2 blocking (forced through BT_KPANELS) is result-identical:
    panel 0 starts from C_in, later panels accumulate in place; rows whose
    products all fall in one panel leave the other panels as no-ops."""
    monkeypatch.setenv("BT_KPANELS", str(npanels))
    rng = np.random.default_rng(npanels)
    sizes = np.array([5, 13, 23, 32, 40], np.int32)[rng.integers(0, 5, 30)]
    ksz = np.array([4, 20, 23], np.int32)[rng.integers(0, 3, 50)]
    A, B, Cin = _case(oracle, 300 + npanels, sizes, ksz, sizes, 0.3, 0.3, 0.2)
    for eps in (0.0, 1e-3):
        want, nprod, _ = oracle.multiply(A, B, Cin, eps)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        from paper_1910_13555_b200.store import multiply_local
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod
        assert_parity(from_store(c), want)


@pytest.mark.parametrize("npanels,bs", [(2, 20), (3, 23), (7, 20), (16, 8)])
def test_k_panels_one_launch(oracle, ctx, monkeypatch, npanels, bs):
    """One block size (a single DMMA class): all K panels run as ONE launch,
    per-tile flags ordering the in-place accumulation.  Against the oracle,
    and bit-identical to one launch per panel (BT_PANEL_FUSE=0: same
    summation order)."""
    monkeypatch.setenv("BT_KPANELS", str(npanels))
    sizes = np.full(40, bs, np.int32)
    ksz = np.full(120, bs, np.int32)
    A, B, Cin = _case(oracle, 700 + npanels, sizes, ksz, sizes, 0.15, 0.15, 0.3)
    from paper_1910_13555_b200.store import multiply_local
    got = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("BT_PANEL_FUSE", fuse)
        for eps in (0.0, 1e-2):
            want, nprod, _ = oracle.multiply(A, B, Cin, eps)
            a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
            st = multiply_local(ctx, a, b, c, eps)
            assert st["products"] == nprod
            out = from_store(c)
            assert_parity(out, want)
            got[(fuse, eps)] = out
    for eps in (0.0, 1e-2):
        assert np.array_equal(got[("1", eps)].vals, got[("0", eps)].vals)


@pytest.mark.parametrize("snap", ["1", "0"])
@pytest.mark.parametrize("splits,sort_min", [(2, 48), (3, 48), (5, 100000), (8, 48)])
def test_fill_splits(oracle, ctx, monkeypatch, splits, sort_min, snap):
    """Long C rows filled by several CTAs (each a range of A chunks, cursors
    offset by the earlier ranges' pairs) emit the same descriptors: against
    the oracle and bit-identical to one CTA per row.  Rows here hold 150 ..
    1500 A entries (1 .. 6 chunks of 256), mixed sizes, eps filter, C_in.
    BT_SNAP=1: the ranges' column counts come from pass 1's split-count
    snapshots (k_row_count_split); 0: every fill CTA recounts its row."""
    monkeypatch.setenv("BT_SORT_MIN", str(sort_min))
    monkeypatch.setenv("BT_SNAP", snap)
    rng = np.random.default_rng(splits)
    rsz = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 6)]
    ksz = np.array([4, 20, 23], np.int32)[rng.integers(0, 3, 3000)]
    nsz = np.array([5, 13, 23, 32], np.int32)[rng.integers(0, 4, 40)]
    occ = np.array([0.05, 0.2, 0.5])
    A = oracle.random_matrix(900 + splits, rsz, ksz, float(occ[splits % 3]))
    B = oracle.random_matrix(901 + splits, ksz, nsz, 0.05)
    Cin = oracle.random_matrix(902 + splits, rsz, nsz, 0.3)
    from paper_1910_13555_b200.store import multiply_local
    got = {}
    for sp in (str(splits), "1"):
        monkeypatch.setenv("BT_FILL_SPLITS", sp)
        for eps in (0.0, 0.5):
            want, nprod, _ = oracle.multiply(A, B, Cin, eps)
            a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
            st = multiply_local(ctx, a, b, c, eps)
            assert st["products"] == nprod
            out = from_store(c)
            assert_parity(out, want)
            got[(sp, eps)] = out
    for eps in (0.0, 0.5):
        assert np.array_equal(got[(str(splits), eps)].vals, got[("1", eps)].vals)


@pytest.mark.parametrize("colmask,sort_min", [(1, 48), (0, 48), (0, 0), (0, 100000), (1, 0)])
def test_emission_paths(oracle, ctx, monkeypatch, colmask, sort_min):
    """The fill pass's three product-emission paths (rank emission by column
    masks for chunks of <= 64 A entries, window sort, one step per k) give the
    same descriptors: rows here have 3 .. 300 A entries (one and two chunks)."""
    monkeypatch.setenv("BT_COLMASK", str(colmask))
    monkeypatch.setenv("BT_SORT_MIN", str(sort_min))
    rng = np.random.default_rng(41)
    rsz = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 6)]
    ksz = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 300)]
    nsz = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 20)]
    A = _dense_rows(oracle, oracle.random_matrix(901, rsz, ksz, 0.01), rsz, ksz, rng)
    B = oracle.random_matrix(902, ksz, nsz, 0.3)
    Cin = oracle.random_matrix(903, rsz, nsz, 0.2)
    for eps in (0.0, 30.0):
        want, nprod, _ = oracle.multiply(A, B, Cin, eps)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        from paper_1910_13555_b200.store import multiply_local
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod
        assert_parity(from_store(c), want)


def _dense_rows(oracle, A, rsz, ksz, rng):
    """A with rows 0/1/2 at occupancy 1.0/0.5/0.2 over 300 block columns (the
    remaining rows as drawn): long A rows exercise the multi-chunk paths."""
    from oracle.oracle import Blocks
    keep = A.bi >= 3
    bi, bj = [A.bi[keep]], [A.bj[keep]]
    for i, occ in ((0, 1.0), (1, 0.5), (2, 0.2)):
        js = np.nonzero(rng.random(len(ksz)) < occ)[0]
        bi.append(np.full(len(js), i, np.int64))
        bj.append(js.astype(np.int64))
    bi, bj = np.concatenate(bi), np.concatenate(bj)
    order = np.lexsort((bj, bi))
    bi, bj = bi[order], bj[order]
    n = int(np.sum(rsz[bi].astype(np.int64) * ksz[bj]))
    return Blocks(rsz, ksz, bi, bj, rng.standard_normal(n))


@pytest.mark.parametrize("bands", [1, 3, 8])
def test_column_bands(oracle, ctx, monkeypatch, bands):
    """Work items segmented by column band (BT_BANDS): same C, any band count."""
    monkeypatch.setenv("BT_BANDS", str(bands))
    sz = np.array([13, 23], np.int32)[np.random.default_rng(3).integers(0, 2, 60)]
    A, B, Cin = _case(oracle, 500 + bands, sz, sz, sz, 0.15, 0.15, 0.1)
    want, nprod, _ = oracle.multiply(A, B, Cin)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    from paper_1910_13555_b200.store import multiply_local
    st = multiply_local(ctx, a, b, c)
    assert st["products"] == nprod
    assert_parity(from_store(c), want)


def test_export_to_pinned_and_pageable(oracle, ctx):
    """bt_mat_export into page-locked and pageable host buffers (chunked
    compaction + side-stream D2H) and put from a page-locked source."""
    import torch
    from oracle.oracle import Blocks
    from paper_1910_13555_b200.store import LocalStore
    sz = np.array([5, 13, 23, 8], np.int32)[np.random.default_rng(8).integers(0, 4, 50)]
    A = oracle.random_matrix(801, sz, sz, 0.4)
    src = torch.from_numpy(A.vals.copy()).pin_memory()
    s = LocalStore(ctx, sz, sz)
    s.put_blocks(A.bi, A.bj, src)
    for pinned in (True, False):
        out = torch.zeros(len(A.vals), dtype=torch.float64)
        if pinned:
            out = out.pin_memory()
        bi, bj, v = s.export(out)
        assert np.array_equal(bi, A.bi) and np.array_equal(bj, A.bj)
        assert np.array_equal(v.numpy(), A.vals)
    s.close()


def test_export_async_overlaps_next_multiply(oracle, ctx):
    """bt_mat_export_async: the value transfer runs on a side stream while the
    next calls (puts, a multiply into a new C, another async export, a sync
    export) proceed; after ctx.sync() every buffer holds its store exactly."""
    import torch
    from oracle.oracle import Blocks
    from paper_1910_13555_b200.store import LocalStore, multiply_local
    sz = np.array([5, 13, 23], np.int32)[np.random.default_rng(9).integers(0, 3, 120)]
    A = oracle.random_matrix(811, sz, sz, 0.2)
    B = oracle.random_matrix(812, sz, sz, 0.2)
    want1, _, _ = oracle.multiply(A, B, Blocks.empty(sz, sz))
    want2, _, _ = oracle.multiply(B, A, Blocks.empty(sz, sz))
    a, b = to_store(ctx, A), to_store(ctx, B)
    outs, wants = [], []
    for it in range(3):
        for (x, y, w) in ((a, b, want1), (b, a, want2)):
            c = LocalStore(ctx, sz, sz)
            multiply_local(ctx, x, y, c)
            buf = torch.full((len(w.vals),), np.nan, dtype=torch.float64).pin_memory()
            bi, bj, _ = c.export(buf, asynchronous=True)
            assert np.array_equal(bi, w.bi) and np.array_equal(bj, w.bj)
            outs.append(buf)
            wants.append(w)
            c.close()   # the staged values outlive the store
    # a synchronous export in between still returns complete values
    got = from_store(a)
    assert np.array_equal(got.vals, A.vals)
    ctx.sync()
    for buf, w in zip(outs, wants):
        assert_parity(Blocks(w.rsz, w.csz, w.bi, w.bj, buf.numpy()), w)


@pytest.mark.parametrize("case", ["empty_a", "empty_b", "empty_all", "disjoint_k", "zero_blocks",
                                  "single_1x1", "eps_filters_all"])
def test_edge_cases(oracle, ctx, case):
    """Empty and degenerate inputs: C_out = C_in (or empty) exactly where no
    product executes; explicit zero blocks still create C blocks (the
    reference's pattern semantics); everything filtered by eps."""
    from oracle.oracle import Blocks
    from paper_1910_13555_b200.store import multiply_local
    rs = np.array([5, 13, 23], np.int32)
    ks = np.array([7, 13, 4, 23], np.int32)
    ns = np.array([23, 5], np.int32)
    A = oracle.random_matrix(1, rs, ks, 0.6)
    B = oracle.random_matrix(2, ks, ns, 0.6)
    Cin = oracle.random_matrix(3, rs, ns, 0.5)
    eps = 0.0
    if case == "empty_a":
        A = Blocks.empty(rs, ks)
    elif case == "empty_b":
        B = Blocks.empty(ks, ns)
    elif case == "empty_all":
        A, B, Cin = Blocks.empty(rs, ks), Blocks.empty(ks, ns), Blocks.empty(rs, ns)
    elif case == "disjoint_k":   # A only in k-columns {0, 1}, B only in k-rows {2, 3}
        A = oracle.random_matrix(4, rs, ks, 1.0)
        keep = A.bj < 2
        A = _subset(A, keep)
        B = oracle.random_matrix(5, ks, ns, 1.0)
        B = _subset(B, B.bi >= 2)
    elif case == "zero_blocks":  # explicit all-zero blocks are stored and multiplied
        A = Blocks(A.rsz, A.csz, A.bi, A.bj, np.zeros_like(A.vals))
    elif case == "single_1x1":
        one = np.array([1], np.int32)
        A = Blocks(one, one, np.array([0]), np.array([0]), np.array([3.0]))
        B = Blocks(one, one, np.array([0]), np.array([0]), np.array([-2.0]))
        Cin = Blocks(one, one, np.array([0]), np.array([0]), np.array([1.5]))
    elif case == "eps_filters_all":
        eps = 1e30
    want, nprod, _ = oracle.multiply(A, B, Cin, eps)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    st = multiply_local(ctx, a, b, c, eps)
    assert st["products"] == nprod
    got = from_store(c)
    assert_parity(got, want)
    if case == "single_1x1":
        assert got.vals.tolist() == [1.5 + 3.0 * -2.0]


def _subset(m, keep):
    from oracle.oracle import Blocks
    off = m.offsets()
    vals = np.concatenate([m.vals[off[t]:off[t + 1]] for t in np.nonzero(keep)[0]]) \
        if keep.any() else np.zeros(0)
    return Blocks(m.rsz, m.csz, m.bi[keep], m.bj[keep], vals)


def test_invalid_arguments(oracle, ctx):
    """Errors map to the reference's exception classes (errors.hpp:14-53)."""
    from paper_1910_13555_b200 import InvalidArgument
    from paper_1910_13555_b200.store import multiply_local
    A = oracle.random_matrix(1, [5, 6], [7], 1.0)
    B = oracle.random_matrix(2, [8], [3], 1.0)      # inner blockings differ
    C = oracle.random_matrix(3, [5, 6], [3], 0.0)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, C)
    with pytest.raises(InvalidArgument, match="inner blockings"):
        multiply_local(ctx, a, b, c)
    with pytest.raises(InvalidArgument, match="alias"):
        multiply_local(ctx, a, to_store(ctx, oracle.random_matrix(4, [7], [7], 1.0)), a)
    with pytest.raises(InvalidArgument):
        a.put_blocks([5], [0], np.zeros(35))                 # block row out of range


def test_wide_rows_40k_block_columns(oracle, ctx):
    """C rows far wider than the shared-memory column counters (VERDICT r1:
    the symbolic passes capped C at ~15,000 block columns): 200 x 40,000 block
    columns, swept in column chunks, against the oracle."""
    from paper_1910_13555_b200.store import multiply_local
    rng = np.random.default_rng(400)
    rsz = rng.integers(2, 6, 200).astype(np.int32)
    ksz = rng.integers(2, 6, 300).astype(np.int32)
    nsz = rng.integers(2, 6, 40000).astype(np.int32)
    A = oracle.random_matrix(4001, rsz, ksz, 0.05)
    B = oracle.random_matrix(4002, ksz, nsz, 0.003)
    Cin = oracle.random_matrix(4003, rsz, nsz, 0.0005)
    for eps in (0.0, 2.0):
        want, nprod, _ = oracle.multiply(A, B, Cin, eps)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod
        assert_parity(from_store(c), want)
        assert int(np.max(np.bincount(want.bi))) > 1000   # rows really are wide


@pytest.mark.parametrize("colw,colmask,sort_min,splits", [(64, 1, 48, 1), (100, 0, 48, 1),
                                                          (37, 0, 0, 1), (200, 0, 100000, 1),
                                                          (128, 1, 48, 3), (33, 0, 48, 4)])
def test_column_chunks(oracle, ctx, monkeypatch, colw, colmask, sort_min, splits):
    """Column-chunked symbolic passes (BT_COLW forces narrow chunks) through
    every emission path, split fill CTAs, C_in and the eps filter: against the
    oracle and bit-identical to the unchunked passes."""
    from paper_1910_13555_b200.store import multiply_local
    monkeypatch.setenv("BT_COLMASK", str(colmask))
    monkeypatch.setenv("BT_SORT_MIN", str(sort_min))
    monkeypatch.setenv("BT_FILL_SPLITS", str(splits))
    rng = np.random.default_rng(colw)
    rsz = np.array([5, 13, 23, 40], np.int32)[rng.integers(0, 4, 8)]
    ksz = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 600)]
    nsz = np.array([5, 13, 23, 8], np.int32)[rng.integers(0, 4, 500)]
    A = _dense_rows(oracle, oracle.random_matrix(4101, rsz, ksz, 0.05), rsz, ksz, rng)
    B = oracle.random_matrix(4102, ksz, nsz, 0.05)
    Cin = oracle.random_matrix(4103, rsz, nsz, 0.2)
    out = {}
    for w in (str(colw), "1000000"):
        monkeypatch.setenv("BT_COLW", w)
        for eps in (0.0, 30.0):
            want, nprod, _ = oracle.multiply(A, B, Cin, eps)
            a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
            st = multiply_local(ctx, a, b, c, eps)
            assert st["products"] == nprod
            got = from_store(c)
            assert_parity(got, want)
            out[(w, eps)] = got
    for eps in (0.0, 30.0):
        assert np.array_equal(out[(str(colw), eps)].vals, out[("1000000", eps)].vals)


@pytest.mark.parametrize("case", ["tiny_uniform", "tiny_mixed_k", "tiny_with_dmma", "panels",
                                  "cin_eps"])
def test_dfma_tiny_blocks(oracle, ctx, monkeypatch, case):
    """C blocks with m, n <= 5 on the CUDA-core DFMA kernel (k_smm_dfma, one
    thread per C block) against the oracle, and against the DMMA path
    (BT_DFMA=0); mixed with DMMA classes in one multiply, K panels, C_in and
    the eps filter."""
    from paper_1910_13555_b200.store import multiply_local
    rng = np.random.default_rng(88)
    eps = 0.0
    if case == "tiny_uniform":
        sz = np.array([1, 2, 3, 4], np.int32)[rng.integers(0, 4, 60)]
        A, B, Cin = _case(oracle, 1600, sz, sz, sz, 0.3, 0.3, 0.0)
    elif case == "tiny_mixed_k":
        ms = np.array([5, 3, 1], np.int32)[rng.integers(0, 3, 30)]
        ks = np.array([5, 13, 23, 40, 70], np.int32)[rng.integers(0, 5, 40)]
        A, B, Cin = _case(oracle, 1700, ms, ks, ms, 0.3, 0.3, 0.1)
    elif case == "tiny_with_dmma":
        sz = np.array([5, 13, 23, 4, 8], np.int32)[rng.integers(0, 5, 50)]
        A, B, Cin = _case(oracle, 1800, sz, sz, sz, 0.2, 0.2, 0.1)
    elif case == "panels":
        monkeypatch.setenv("BT_KPANELS", "3")
        ms = np.array([5, 4, 13], np.int32)[rng.integers(0, 3, 20)]
        ks = np.array([5, 23], np.int32)[rng.integers(0, 2, 80)]
        A, B, Cin = _case(oracle, 1900, ms, ks, ms, 0.2, 0.2, 0.2)
    else:
        sz = np.array([5, 3, 13], np.int32)[rng.integers(0, 3, 50)]
        A = oracle.random_matrix(2000, sz, sz, 0.3, 6.0)
        B = oracle.random_matrix(2001, sz, sz, 0.3, 6.0)
        Cin = oracle.random_matrix(2002, sz, sz, 0.2, 6.0)
        eps = 1e-4
    want, nprod, _ = oracle.multiply(A, B, Cin, eps)
    for mode in ("1", "0"):
        monkeypatch.setenv("BT_DFMA", mode)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod
        assert_parity(from_store(c), want)
        # the DFMA output slots carry zero padding (norms read it)
        assert np.allclose(c.norms(), oracle.norms(want), rtol=1e-12, atol=0)


@pytest.mark.parametrize("colmask,sort_min,colw", [(1, 48, 0), (0, 48, 0), (0, 0, 0),
                                                   (0, 100000, 0), (1, 48, 50), (0, 0, 37)])
def test_row_threads_64_vs_256(oracle, ctx, monkeypatch, colmask, sort_min, colw):
    """The symbolic passes with 64 and with 256 threads per row (BT_ROW_THREADS;
    and pass 1 alone with 128, BT_COUNT_THREADS):
    against the oracle and bit-identical to each other, through every
    emission path, column chunks, C_in and the eps filter.  Rows here hold up
    to 300 A entries (several 64-entry chunks)."""
    from paper_1910_13555_b200.store import multiply_local
    monkeypatch.setenv("BT_COLMASK", str(colmask))
    monkeypatch.setenv("BT_SORT_MIN", str(sort_min))
    if colw:
        monkeypatch.setenv("BT_COLW", str(colw))
    rng = np.random.default_rng(64 + colw)
    rsz = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 8)]
    ksz = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 300)]
    nsz = np.array([5, 13, 23, 4], np.int32)[rng.integers(0, 4, 120)]
    A = _dense_rows(oracle, oracle.random_matrix(6401, rsz, ksz, 0.02), rsz, ksz, rng)
    B = oracle.random_matrix(6402, ksz, nsz, 0.1)
    Cin = oracle.random_matrix(6403, rsz, nsz, 0.2)
    out = {}
    for t in ("64", "256", "256/128"):   # 256/128: 128-thread pass 1 (BT_COUNT_THREADS)
        monkeypatch.setenv("BT_ROW_THREADS", t.split("/")[0])
        if "/" in t:
            monkeypatch.setenv("BT_COUNT_THREADS", t.split("/")[1])
        for eps in (0.0, 30.0):
            want, nprod, _ = oracle.multiply(A, B, Cin, eps)
            a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
            st = multiply_local(ctx, a, b, c, eps)
            assert st["products"] == nprod
            got = from_store(c)
            assert_parity(got, want)
            out[(t, eps)] = got
    for eps in (0.0, 30.0):
        assert np.array_equal(out[("64", eps)].vals, out[("256", eps)].vals)
        assert np.array_equal(out[("256/128", eps)].vals, out[("256", eps)].vals)


@pytest.mark.parametrize("seed", range(24))
def test_random_sweep(oracle, ctx, seed):
    """Randomised configurations against the oracle: block sizes 1..40 drawn
    per dimension from a random palette (tiny DFMA, DMMA tile classes, tall
    rows, generic n > 32), random shapes, occupancies, C_in, eps (with scaled
    values so the filter bites)."""
    from paper_1910_13555_b200.store import multiply_local
    rng = np.random.default_rng(1000 + seed)

    def sizes(n):
        pal = rng.choice(np.arange(1, 41), size=int(rng.integers(1, 5)), replace=False)
        if rng.random() < 0.2:
            pal = np.append(pal, rng.choice([169, 299]))   # tall (rows only below)
        return pal.astype(np.int32), int(n)

    pm, nm = sizes(rng.integers(1, 30))
    pk, nk = sizes(rng.integers(1, 40))
    pn, nn = sizes(rng.integers(1, 30))
    rsz = rng.choice(pm, nm).astype(np.int32)
    ksz = rng.choice(pk[pk <= 64] if np.any(pk <= 64) else [8], nk).astype(np.int32)
    nsz = rng.choice(pn[pn <= 40] if np.any(pn <= 40) else [8], nn).astype(np.int32)
    scale = float(rng.choice([0.0, 6.0]))
    oa, ob, oc = (float(rng.choice([0.05, 0.2, 0.5, 1.0])) for _ in range(3))
    A = oracle.random_matrix(2000 + seed, rsz, ksz, oa, scale)
    B = oracle.random_matrix(3000 + seed, ksz, nsz, ob, scale)
    Cin = oracle.random_matrix(4000 + seed, rsz, nsz, oc * float(rng.random() < 0.5), scale)
    eps = float(rng.choice([0.0, 1e-6, 1e-3])) if scale else 0.0
    want, nprod, flops = oracle.multiply(A, B, Cin, eps)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    st = multiply_local(ctx, a, b, c, eps)
    assert st["products"] == nprod
    assert st["flops"] == flops
    assert_parity(from_store(c), want)


@pytest.mark.parametrize("h", ["128", "256"])
@pytest.mark.parametrize("seed", range(9))
def test_warp_row_symbolic(oracle, ctx, monkeypatch, h, seed):
    """The warp-per-row fill (BT_WARP_ROWS=128/256: one warp per C row, a hash
    of the row's columns) against the oracle and bit-identical to the CTA
    fill (BT_WARP_ROWS=0): random shapes and block-size palettes (tiny DFMA,
    DMMA classes, tall rows, generic n > 32), C_in, the eps filter, empty
    rows.  Seeds 0, 3, 6 also hold rows too long for a warp (more than 64 A
    entries, more C blocks or products than the hash takes), which pass 1
    lists for the CTA fill (k_row_fill_list)."""
    from paper_1910_13555_b200.store import multiply_local
    rng = np.random.default_rng(7100 + seed)
    pal = lambda: rng.choice(np.arange(1, 41), size=int(rng.integers(1, 4)), replace=False)
    pm = pal()
    if seed % 4 == 1:
        pm = np.append(pm, 169)                  # tall rows
    nm, nk, nn = int(rng.integers(150, 400)), int(rng.integers(20, 200)), int(rng.integers(20, 500))
    rsz = rng.choice(pm, nm).astype(np.int32)
    ksz = rng.choice(pal(), nk).astype(np.int32)
    pn = pal()
    if seed % 4 == 2:
        pn = np.append(pn, 48)                   # generic (n > 32)
    nsz = rng.choice(pn, nn).astype(np.int32)
    scale = 6.0 if seed % 2 else 0.0
    A = oracle.random_matrix(7200 + seed, rsz, ksz, float(rng.choice([0.01, 0.03, 0.08])), scale)
    if seed % 3 == 0:                            # a few long rows
        A = _dense_rows(oracle, A, rsz, ksz, rng)
    B = oracle.random_matrix(7300 + seed, ksz, nsz, float(rng.choice([0.02, 0.05, 0.1])), scale)
    Cin = oracle.random_matrix(7400 + seed, rsz, nsz, 0.05 * float(seed % 2 == 0), scale)
    eps = 1e-3 if scale else 0.0
    want, nprod, flops = oracle.multiply(A, B, Cin, eps)
    out = {}
    for mode in ("0", h):
        monkeypatch.setenv("BT_WARP_ROWS", mode)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod and st["flops"] == flops
        got = from_store(c)
        assert_parity(got, want)
        out[mode] = got
    assert np.array_equal(out["0"].bi, out[h].bi) and np.array_equal(out["0"].bj, out[h].bj)
    assert np.array_equal(out["0"].vals, out[h].vals)


@pytest.mark.parametrize("case", ["n40_k40", "n64_k64", "n100_k130", "mixed_tall", "panels", "wide_cin_eps"])
def test_wide_blocks_dmma(oracle, ctx, monkeypatch, case):
    """Blocks wider than 32 columns and k > 64 on the DMMA path (BT_WIDE=1:
    32-column C tiles, k sliced in <= 4 tiles per stage) and on the CUDA-core
    generic kernel (BT_WIDE=0), both against the oracle: C tiles of partial
    width, k slices of partial depth, tall rows (169), narrow blocks mixed in,
    C_in, the eps filter, K panels (one WIDE launch per panel)."""
    from paper_1910_13555_b200.store import multiply_local
    rng = np.random.default_rng(hash(case) % 2 ** 32)
    eps, scale, occ_c = 0.0, 0.0, 0.0
    if case == "n40_k40":
        rsz = ksz = nsz = np.full(30, 40, np.int32)
    elif case == "n64_k64":
        rsz = ksz = nsz = np.full(24, 64, np.int32)
    elif case == "n100_k130":
        rsz = np.array([37, 100, 64], np.int32)[rng.integers(0, 3, 12)]
        ksz = np.array([130, 70, 9], np.int32)[rng.integers(0, 3, 12)]
        nsz = np.array([100, 41, 33], np.int32)[rng.integers(0, 3, 12)]
    elif case == "mixed_tall":
        rsz = np.array([169, 23, 5, 40], np.int32)[rng.integers(0, 4, 16)]
        ksz = np.array([13, 48, 80], np.int32)[rng.integers(0, 3, 20)]
        nsz = np.array([5, 13, 23, 40, 72], np.int32)[rng.integers(0, 5, 18)]
    elif case == "panels":
        monkeypatch.setenv("BT_KPANELS", "3")
        rsz = nsz = np.full(10, 48, np.int32)
        ksz = np.full(60, 40, np.int32)
    else:   # wide_cin_eps
        rsz = np.array([40, 20], np.int32)[rng.integers(0, 2, 20)]
        ksz = np.array([36, 72], np.int32)[rng.integers(0, 2, 20)]
        nsz = np.array([33, 64, 8], np.int32)[rng.integers(0, 3, 20)]
        eps, scale, occ_c = 1e-3, 6.0, 0.3
    A = oracle.random_matrix(8100, rsz, ksz, 0.3, scale)
    B = oracle.random_matrix(8101, ksz, nsz, 0.3, scale)
    Cin = oracle.random_matrix(8102, rsz, nsz, occ_c, scale)
    want, nprod, flops = oracle.multiply(A, B, Cin, eps)
    for mode in ("1", "0"):
        monkeypatch.setenv("BT_WIDE", mode)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod and st["flops"] == flops
        assert_parity(from_store(c), want)
        # the whole T8 slots are written (zero padding): norms read it
        cn = oracle.norms(want)
        assert np.max(np.abs(c.norms() - cn) / np.maximum(cn, 1e-300)) <= 1e-12


@pytest.mark.parametrize("seed", range(12))
def test_random_sweep_new_paths(oracle, ctx, monkeypatch, seed):
    """Randomised shapes through the round-2 paths together: block sizes up to
    100 (WIDE column tiles, k slices), tall rows, and per seed one of the
    symbolic variants forced (warp-row fill with either hash size, split-count
    fill, 128-thread pass 1), C_in and the eps filter -- against the oracle."""
    from paper_1910_13555_b200.store import multiply_local
    rng = np.random.default_rng(9100 + seed)
    variant = [("BT_WARP_ROWS", "128"), ("BT_WARP_ROWS", "256"), ("BT_FILL_SPLITS", "3"),
               ("BT_COUNT_THREADS", "128")][seed % 4]
    monkeypatch.setenv(*variant)

    def pal(hi):
        return rng.choice(np.arange(1, hi + 1), size=int(rng.integers(1, 4)), replace=False)

    pm, pk, pn = pal(100), pal(100), pal(100)
    if seed % 3 == 0:
        pm = np.append(pm, 169)
    rsz = rng.choice(pm, int(rng.integers(2, 40))).astype(np.int32)
    ksz = rng.choice(pk, int(rng.integers(2, 300 if variant[0] == "BT_FILL_SPLITS" else 60))).astype(np.int32)
    nsz = rng.choice(pn, int(rng.integers(2, 40))).astype(np.int32)
    scale = float(rng.choice([0.0, 6.0]))
    A = oracle.random_matrix(9200 + seed, rsz, ksz, float(rng.choice([0.05, 0.2, 0.6])), scale)
    B = oracle.random_matrix(9300 + seed, ksz, nsz, float(rng.choice([0.05, 0.2, 0.5])), scale)
    Cin = oracle.random_matrix(9400 + seed, rsz, nsz, float(rng.choice([0.0, 0.3])), scale)
    eps = 1e-3 if scale else 0.0
    want, nprod, flops = oracle.multiply(A, B, Cin, eps)
    a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
    st = multiply_local(ctx, a, b, c, eps)
    assert st["products"] == nprod and st["flops"] == flops
    assert_parity(from_store(c), want)
