"""Loading the golden fixtures and regenerating their seeded inputs.

The generator (tests/golden/make_golden.py) ran the real reference; the input
recipe below mirrors its ``stage_inputs`` and the stored SHA-256 digests prove
the regenerated arrays are the bytes the reference consumed.  Ghost filling
uses the oracle restatement of grid.py:227-277 (tests may use the oracle).
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle import vpfv_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def load(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    return meta, arrays


def grid_of(m):
    return O.Grid(m["d"], m["v"], tuple(m["N"]), tuple(float(x) for x in m["lo"]),
                  tuple(float(x) for x in m["hi"]), tuple(m["periodic"]))


def species_of(m):
    return O.Species(m["name"], m["q"], m["m"], m["kappa2"], m["kappa_c"], m["Bz"], tuple(m["G"]))


def stage_inputs(g, seed, frozen_velocity):
    rng = np.random.default_rng(seed)
    src = np.zeros(g.padded_shape)
    src[g.inner()] = 1.0 + 0.3 * rng.random(g.N)
    if frozen_velocity:
        ghost = 1.0 + 0.3 * rng.random(g.padded_shape)
        mask = np.ones(g.padded_shape, bool)
        mask[g.inner()] = False
        src[mask] = ghost[mask]
        O.fill_ghosts(src, g, O.capture_frozen(src, g))
    else:
        O.fill_ghosts(src, g, None)
    A = rng.random(g.padded_shape)
    B = rng.random(g.padded_shape)
    dest = rng.random(g.padded_shape)
    return src, A, B, dest


def stage_case(name):
    meta, arr = load(name + ".npz")
    g = grid_of(meta["grid"])
    sp = species_of(meta["species"])
    src, A, B, dest = stage_inputs(g, meta["seed"], meta["frozen"])
    for k, a in (("src", src), ("A", A), ("B", B), ("dest", dest)):
        assert sha(a) == meta["sha"][k], f"{name}: regenerated {k} differs from the reference input"
    E = {k: arr[k] for k in ("Ex", "Ey") if k in arr}
    return dict(grid=g, species=sp, src=src, A=A, B=B, dest=dest, E=E,
                coefs=[tuple(c) for c in meta["coefs"]], out=arr["out"], rhs=arr["rhs"],
                meta=meta, arrays=arr)


STAGE_NAMES = ["stage_1d1v_periodic", "stage_1d1v_frozen", "stage_1d2v_periodic",
               "stage_1d2v_frozen", "stage_2d2v_periodic", "stage_2d2v_frozen"]
MOMENT_NAMES = ["moment_1d1v", "moment_1d2v", "moment_2d2v", "moment_2d2v_pow2"]
POISSON_NAMES = ["poisson_1d_64", "poisson_1d_odd", "poisson_2d_16", "poisson_2d_odd"]
STEP_NAMES = ["landau1d", "twostream", "dgh", "lhdi", "bimax1d2v", "landau2d"]


def moment_case(name):
    meta, arr = load(name)
    g = grid_of(meta["grid"])
    data = np.random.default_rng(meta["seed"]).random(g.padded_shape)
    assert sha(data) == meta["sha"]
    return g, data, arr["n"]


def poisson_case(name):
    meta, arr = load(name)
    return grid_of(meta["grid"]), arr


def step_case(name):
    meta, init = load(f"init_{name}.npz")
    _, out = load(f"step_{name}.npz")
    grids = [grid_of(m) for m in meta["grids"]]
    species = [species_of(m) for m in meta["species"]]
    datas = [init[f"f{s}"] for s in range(len(grids))]
    return dict(meta=meta, grids=grids, species=species, init=datas, out=out, dt=meta["dt"])
