"""Host-side logic of the Python mirror (no GPU): grid/partition/cost model vs
the compiled reference, mixed radix vs the oracle restatement."""
import numpy as np
import pytest

from paper_1910_13555_b200 import dist as d
from paper_1910_13555_b200 import tensor as t


def test_process_grid_matches_reference_rules():
    g = d.ProcessGrid([3, 4])
    assert g.rank_of([2, 1]) == 9           # SPEC.md grid example
    assert d.ProcessGrid([2, 3]).coords_of(5) == [1, 2]
    assert d.ProcessGrid([2, 2, 2]).coords_of(6) == [1, 1, 0]
    for r in range(12):
        assert g.rank_of(g.coords_of(r)) == r
    with pytest.raises(d.InvalidArgument):
        d.ProcessGrid([0, 2])


def test_split_grid_remainder_rule():
    groups = d.split_grid(d.ProcessGrid([6, 2]), 0, 4)
    assert [gr.local_grid.dim(0) for gr in groups] == [2, 2, 1, 1]
    members = sorted(m for gr in groups for m in gr.members)
    assert members == list(range(12))


def test_chunk_partition():
    p = d.ChunkPartition(10, 3)
    assert [(p.begin(i), p.end(i)) for i in range(3)] == [(0, 4), (4, 8), (8, 10)]
    assert p.part_of(9) == 2


@pytest.mark.parametrize("args", [(1e3, 1e3, 1e6, 0.5, 0.5, 0.5, 100), (800, 800, 800, 1, 1, 1, 4),
                                  (2000, 2000, 4e5, .1, .1, .9, 8), (400, 20, 20, .5, .5, .5, 4)])
def test_cost_model_matches_reference(reference, args):
    m, n, k, oa, ob, oc, p = args
    s = d.MultiplySpec(m, n, k, oa, ob, oc, p)
    assert d.cannon_volume(s) == pytest.approx(reference.cost(0, *args), rel=1e-15)
    assert d.case1_volume(s) == pytest.approx(reference.cost(1, *args), rel=1e-15)
    assert d.case2_volume(s) == pytest.approx(reference.cost(2, *args), rel=1e-15)
    assert d.occupancy_limit_case1(s) == pytest.approx(reference.cost(3, *args), rel=1e-15)
    assert d.select_algorithm(*args) == int(reference.cost(5, *args))


def test_eq4_paper_value():
    assert d.occupancy_ratio_bound(1e3, 1e3, 1e6, 100) == 200.0


def test_mixed_radix_matches_oracle(oracle):
    ext = [3, 4, 5]
    for idx in range(60):
        c = t.mixed_radix_inv(idx, ext)
        assert t.mixed_radix(c, ext) == idx == oracle.mixed_radix(c, ext)
    assert t.mixed_radix([2, 3], [3, 4]) == 11   # SPEC.md:510 example


@pytest.mark.parametrize("shape,p,want", [
    # c5: dense-ish 65 536^3 at 50 %, square grid -> Cannon (shifts hidden)
    ((65536, 65536, 65536, 0.5, 0.5, 1.0), 4, d.Algorithm.cannon),
    # c5 on 8 GPUs: no square grid -> a rectangular algorithm
    ((65536, 65536, 65536, 0.5, 0.5, 1.0), 8, d.Algorithm.case2),
    # c3: C 2000^2 from K = 400 000 (S_C << S_A, S_B) -> case 1
    ((2000, 2000, 400000, 0.1, 0.1, 1.0), 4, d.Algorithm.case1),
    # c1 weak-scaling shape on 2 GPUs (non-square) -> case 2
    ((9200 * 2, 9200, 9200, 0.1, 0.1, 0.98), 2, d.Algorithm.case2),
])
def test_b200_time_model_selection(shape, p, want):
    """Extension: NVLink-aware selection picks the algorithm the
    measurements favour for the BASELINE shapes."""
    assert d.select_algorithm_b200(*shape, p) == want
    s = d.MultiplySpec(*shape, p)
    times = [d.predicted_time_b200(a, s) for a in (0, 1, 2)]
    assert min(times) == d.predicted_time_b200(want, s)
