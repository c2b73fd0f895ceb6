"""Golden fixtures of the reference's partition planning and simulated cluster.

Run in the build container only (imports the REAL reference from
/root/reference, needs numba):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_partition_golden.py

partition_plans.json  plan reports, segment lists, box grids, counting and
                      volume formulas of vpfv.partition for a set of plans
                      (partition.py:47-600), plus combine_partials logs.
cluster_*.npz         vpfv.runner.SimulatedCluster (runner.py:259-496) after
                      two fixed-dt RK4 steps on small set-ups: the gathered
                      state per species and the TrafficLog totals per kind.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from vpfv import partition as P  # noqa: E402
from vpfv.grid import make_grid  # noqa: E402
from vpfv.problems import ProblemSpec, landau_spec, make_problem  # noqa: E402
from vpfv.runner import SimulatedCluster, Simulation  # noqa: E402


def grid(d, v, N, periodic_v=False):
    lo = [0.0] * d + [-6.0] * v
    hi = [4 * np.pi] * d + [6.0] * v
    return make_grid(d, v, N, lo, hi, periodic=tuple([True] * d + [periodic_v] * v))


def seg_rows(plan):
    return [[list(s.src_box), list(s.dst_box), s.src_rank, s.dst_rank, s.kind, list(s.dims),
             [list(w) for w in s.src_window], [list(w) for w in s.dst_window], s.count] for s in plan.segments]


PLANS = [
    # (name, grids, n, r, strategy)
    ("1d1v_x2", [((1, 1, (32, 32)))], (2, 1), 1, "vp"),
    ("1d1v_x2v2_fvm", [((1, 1, (32, 32)))], (2, 2), 1, "fvm"),
    ("1d2v_v2_vp", [((1, 2, (16, 16, 16)))], (1, 2, 2), 1, "vp"),
    ("1d2v_all", [((1, 2, (16, 16, 16)))], (2, 1, 2), 1, "all"),
    ("2d2v_xy", [((2, 2, (16, 16, 16, 16)))], (2, 2, 1, 1), 1, "vp"),
    ("2d2v_vv", [((2, 2, (16, 16, 16, 16)))], (1, 1, 2, 2), 1, "vp"),
    ("2d2v_xv_fvm", [((2, 2, (16, 16, 16, 16)))], (2, 1, 2, 1), 1, "fvm"),
    ("2d2v_all4", [((2, 2, (16, 16, 16, 16)))], (2, 2, 2, 2), 1, "vp"),
    ("2d2v_2sp_r1", [((2, 2, (16, 16, 16, 16))), ((2, 2, (16, 16, 32, 32)))], (2, 1, 1, 2), 1, "vp"),
    ("2d2v_2sp_r2", [((2, 2, (16, 16, 16, 16))), ((2, 2, (16, 16, 16, 16)))], (2, 2, 1, 1), 2, "vp"),
    ("2d2v_2sp_per", [((2, 2, (16, 16, 16, 16))), ((2, 2, (16, 16, 32, 16)))],
     [(2, 1, 1, 1), (2, 1, 2, 1)], 1, "vp"),
]


def plans():
    out = {}
    for name, gspec, n, r, strat in PLANS:
        grids = [grid(*x) for x in gspec]
        plan = P.plan_partitions(grids, n, r=r, strategy=strat)
        rep = plan.to_report()
        bg = []
        for s in range(plan.S):
            for b in plan.boxes[s]:
                lg = plan.box_grid(s, b.lex)
                bg.append({"species": s, "lex": b.lex, "N": list(lg.N), "lo": list(lg.lo), "hi": list(lg.hi),
                           "periodic": list(lg.periodic), "rank": b.rank, "index": list(b.index)})
        pairs = [[list(k[0]), list(k[1]), len(v)] for k, v in plan.directed_pairs()]
        out[name] = {"n": n if isinstance(n[0], int) else [list(x) for x in n], "r": r, "strategy": strat,
                     "grids": [list(x) for x in gspec], "report": rep, "segments": seg_rows(plan),
                     "box_grids": bg, "directed_pairs": pairs}
    misc = {
        "neighbor_pairs": {f"{d},{v}": P.neighbor_pairs(d, v) for d, v in ((1, 1), (1, 2), (2, 2), (1, 3), (3, 3))},
        "edge_pairs": {f"{d},{v}": sorted(map(list, P.correction_edge_pairs(d, v)))
                       for d, v in ((1, 1), (1, 2), (2, 2), (2, 3))},
        "ghost_fraction": {f"{N},{d},{v},{s}": P.ghost_fraction(N, d, v, s)
                           for N in (8, 16, 64) for d, v in ((1, 1), (1, 2), (2, 2)) for s in ("fvm", "vp", "all")},
        "formulas": {
            "reduce": [P.reduce_volume_formula((64, 64, 128, 128), (2, 2, 2, 4), 2, 2, 1),
                       P.reduce_volume_formula((64, 64, 128, 128), (2, 2, 1, 1), 2, 3, 1),
                       P.reduce_volume_formula((128, 256), (4, 2), 1, 2, 2)],
            "phi": [P.phi_volume_formula((64, 64, 128, 128), (2, 2, 2, 4), (1, 1, 0, 0), 2, 2, 1),
                    P.phi_volume_formula((128, 256), (4, 2), (1, 0), 1, 2, 2)],
            "ghost": [P.ghost_volume_formula((64, 64, 128, 128), (2, 2, 2, 4), (1, 1, 0, 0), 2),
                      P.ghost_volume_formula((128, 256), (4, 2), (1, 0), 1)],
        },
        "reduction_rounds": [P.reduction_rounds(m) for m in range(1, 18)],
    }
    log = P.TrafficLog()
    parts = [np.arange(4.0) + 10 * k for k in range(5)]
    tot = P.combine_partials(parts, ranks=[3, 1, 4, 1, 5], log=log, stage=7, cell_count=4)
    misc["combine"] = {"sum": tot.tolist(), "rows": [list(x) for x in log.to_csv_rows()][1:]}
    out["_misc"] = misc
    with open(os.path.join(HERE, "partition_plans.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


def clusters():
    cases = {
        "landau2d_xy": (lambda: make_problem(landau_spec(), 16, 16), (2, 2, 1, 1), 1),
        "landau2d_vv": (lambda: make_problem(landau_spec(), 16, 16), (1, 1, 2, 2), 1),
        "landau2d_xv": (lambda: make_problem(landau_spec(), 16, 16), (2, 1, 1, 2), 1),
        "lhdi_x_r2": (lambda: make_problem(ProblemSpec("lhdi"), 16, 16), (2, 1, 1), 2),
        "lhdi_vv": (lambda: make_problem(ProblemSpec("lhdi"), 16, 16), (1, 2, 2), 1),
    }
    for name, (mk, n, r) in cases.items():
        setup = mk()
        dt = 0.002 if name.startswith("lhdi") else 0.05
        cl = SimulatedCluster(setup, n, species_per_rank=r, dt=dt)
        for _ in range(2):
            cl.advance(dt)
        states = [cl.gather(s) for s in range(len(setup.species))]
        sim = Simulation(mk(), dt=dt)
        for _ in range(2):
            sim.advance(dt)
        single = [sim.ctx.f0[s][setup.dists[s].grid.interior_slices()] for s in range(len(setup.species))]
        tot = {k: cl.log.total(k) for k in ("ghost", "reduce", "field")}
        np.savez_compressed(os.path.join(HERE, f"cluster_{name}.npz"),
                            meta=json.dumps({"n": list(n), "r": r, "dt": dt, "steps": 2, "totals": tot,
                                             "bitwise_single": all(np.array_equal(a, b)
                                                                   for a, b in zip(states, single))}),
                            **{f"f{s}": a for s, a in enumerate(states)})


if __name__ == "__main__":
    plans()
    clusters()
