"""Host-side logic of the Python mirror (no GPU): grid/partition/cost model vs
the compiled reference, mixed radix vs the oracle restatement."""
import math
import os

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


def _measured_points():
    import json
    from collections import defaultdict
    bs = {"tall_skinny": 20, "square": 23, "dense": 32, "wide_c": 13}
    rows = [json.loads(x) for x in open(os.path.join(os.path.dirname(__file__), "golden",
                                                     "algo_times_b200.jsonl"))]
    pts = defaultdict(dict)
    for r in rows:
        if r["gpus"] < 2:
            continue
        occ_c = d.estimate_result_occupancy(r["occ_a"], r["occ_b"], r["k"] / bs[r["workload"]])
        spec = d.MultiplySpec(r["m"], r["n"], r["k"], r["occ_a"], r["occ_b"], occ_c, r["gpus"])
        algo = {"cannon": 0, "case1": 1, "case2": 2}[r["algo"]]
        pts[(r["workload"], r["gpus"])][algo] = (r["ms"] * 1e-3, spec)
    return pts


def test_b200_time_model_fits_measurements():
    """Extension: predicted_time_b200 against the measured times
    of every algorithm on 2 and 4 B200s (tests/golden/algo_times_b200.jsonl,
    tools/algo_sweep.py): within a factor 2 everywhere, rms log error < 0.3."""
    errs = []
    for (w, p), algos in _measured_points().items():
        for algo, (t, spec) in algos.items():
            e = math.log(d.predicted_time_b200(algo, spec) / t)
            assert abs(e) < math.log(2.0), (w, p, algo, t)
            errs.append(e)
    assert len(errs) == 20
    assert math.sqrt(sum(e * e for e in errs) / len(errs)) < 0.3


def test_b200_selection_picks_measured_fastest():
    """The model's argmin is the measured-fastest algorithm in 7 of the 8
    (workload, GPU count) cases -- every 4-GPU case (Cannon) and the 2-GPU
    square (case 2), tall-skinny (case 1) and dense (case 2) cases.  The miss:
    wide-C on 2 GPUs (C 19 500^2 from K = 780), measured case 2 11.2 ms vs
    case 1 14.5 ms, predicted the other way round."""
    hits, misses = 0, []
    for (w, p), algos in _measured_points().items():
        best = min(algos, key=lambda a: algos[a][0])
        spec = next(iter(algos.values()))[1]
        choice = d.select_algorithm_b200(spec.m, spec.n, spec.k, spec.occ_a, spec.occ_b,
                                         spec.occ_c, p)
        if choice == best:
            hits += 1
        else:
            misses.append((w, p))
    assert hits >= 7 and misses in ([], [("wide_c", 2)]), misses
