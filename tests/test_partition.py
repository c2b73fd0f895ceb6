"""Partition planning and accounting against the reference's own outputs.

tests/golden/partition_plans.json is written by make_partition_golden.py from
the real vpfv.partition (plan reports, segment lists, box grids, formulas,
combine logs); every number here must match exactly.  The reference's own
tests of these functions: /root/reference/pkg/tests/test_partition.py.
"""

import json
import os

import numpy as np
import pytest

from paper_2410_12155_b200 import partition as P
from paper_2410_12155_b200.grid import make_grid

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "partition_plans.json")))


def _grid(d, v, N):
    return make_grid(d, v, N, [0.0] * d + [-6.0] * v, [4 * np.pi] * d + [6.0] * v,
                     periodic=tuple([True] * d + [False] * v))


def _plan(name):
    c = GOLD[name]
    grids = [_grid(*g) for g in c["grids"]]
    n = c["n"] if isinstance(c["n"][0], int) else [tuple(x) for x in c["n"]]
    return P.plan_partitions(grids, n, r=c["r"], strategy=c["strategy"]), c


def _jsonable(x):
    return json.loads(json.dumps(x))


@pytest.mark.parametrize("name", [k for k in GOLD if not k.startswith("_")])
def test_plan_report_segments_and_box_grids_match_reference(name):
    plan, c = _plan(name)
    assert _jsonable(plan.to_report()) == c["report"]
    rows = [[list(s.src_box), list(s.dst_box), s.src_rank, s.dst_rank, s.kind, list(s.dims),
             [list(w) for w in s.src_window], [list(w) for w in s.dst_window], s.count] for s in plan.segments]
    assert rows == c["segments"]
    assert [[list(k[0]), list(k[1]), len(v)] for k, v in plan.directed_pairs()] == c["directed_pairs"]
    for bg in c["box_grids"]:
        g = plan.box_grid(bg["species"], bg["lex"])
        assert list(g.N) == bg["N"] and list(g.periodic) == bg["periodic"]
        assert np.allclose(g.lo, bg["lo"], rtol=0, atol=0) and np.allclose(g.hi, bg["hi"], rtol=0, atol=0)
        b = plan.box(bg["species"], bg["lex"])
        assert b.rank == bg["rank"] and list(b.index) == bg["index"]


def test_counting_and_formulas_match_reference():
    m = GOLD["_misc"]
    for k, want in m["neighbor_pairs"].items():
        assert P.neighbor_pairs(*map(int, k.split(","))) == want
    for k, want in m["edge_pairs"].items():
        assert sorted(map(list, P.correction_edge_pairs(*map(int, k.split(","))))) == want
    for k, want in m["ghost_fraction"].items():
        N, d, v, s = k.split(",")
        assert P.ghost_fraction(int(N), int(d), int(v), s) == want
    f = m["formulas"]
    assert [P.reduce_volume_formula((64, 64, 128, 128), (2, 2, 2, 4), 2, 2, 1),
            P.reduce_volume_formula((64, 64, 128, 128), (2, 2, 1, 1), 2, 3, 1),
            P.reduce_volume_formula((128, 256), (4, 2), 1, 2, 2)] == f["reduce"]
    assert [P.phi_volume_formula((64, 64, 128, 128), (2, 2, 2, 4), (1, 1, 0, 0), 2, 2, 1),
            P.phi_volume_formula((128, 256), (4, 2), (1, 0), 1, 2, 2)] == f["phi"]
    assert [P.ghost_volume_formula((64, 64, 128, 128), (2, 2, 2, 4), (1, 1, 0, 0), 2),
            P.ghost_volume_formula((128, 256), (4, 2), (1, 0), 1)] == f["ghost"]
    assert [P.reduction_rounds(k) for k in range(1, 18)] == m["reduction_rounds"]
    log = P.TrafficLog()
    tot = P.combine_partials([np.arange(4.0) + 10 * k for k in range(5)], ranks=[3, 1, 4, 1, 5], log=log,
                             stage=7, cell_count=4)
    assert tot.tolist() == m["combine"]["sum"]
    assert [list(x) for x in log.to_csv_rows()][1:] == m["combine"]["rows"]


def test_plan_errors_follow_reference():
    g = _grid(1, 1, (32, 32))
    with pytest.raises(ValueError, match="does not divide"):
        P.plan_partitions(g, (3, 1))
    with pytest.raises(ValueError, match="below the stencil"):
        P.plan_partitions(g, (8, 1))
    with pytest.raises(ValueError, match="rank-count mismatch"):
        P.plan_partitions(g, (2, 1), ranks=3)
    with pytest.raises(ValueError, match="unknown ghost strategy"):
        P.plan_partitions(g, (2, 1), strategy="nope")
    with pytest.raises(ValueError, match="must divide species count"):
        P.plan_partitions([g, g], (2, 1), r=3)
    with pytest.raises(ValueError, match="need d >= 1"):
        P.neighbor_pairs(0, 1)


def test_host_exchange_fills_ghosts_like_a_global_fill():
    """Scatter a ghost-filled global array, poison the boxes' exchanged ghost
    cells, run the host Exchanger: every box equals its window of the global
    array wherever a segment lands (the reference's exchange property)."""
    g = _grid(2, 2, (16, 16, 16, 16))
    plan = P.plan_partitions(g, (2, 2, 2, 1), strategy="fvm")
    rng = np.random.default_rng(3)
    glob = rng.random(g.padded_shape)
    # periodic physical wraps of the global ghost shell (velocity ghosts arbitrary, frozen)
    for k in range(2):
        a = np.moveaxis(glob, k, 0)
        a[:3] = a[-6:-3]
        a[-3:] = a[3:6]
    boxes = P.scatter_field(plan, 0, glob)
    want = {k: v.copy() for k, v in boxes.items()}
    for seg in plan.segments:
        w = tuple(slice(a, z) for a, z in seg.dst_window)
        boxes[seg.dst_box][w] = np.nan
    log = P.simulate_exchange(plan, boxes)
    for seg in plan.segments:
        w = tuple(slice(a, z) for a, z in seg.dst_window)
        assert np.array_equal(boxes[seg.dst_box][w], want[seg.dst_box][w])
    assert log.total("ghost") == sum(s.count for s in plan.segments)
    assert np.array_equal(P.gather_field(plan, 0, boxes), glob[g.interior_slices()])
