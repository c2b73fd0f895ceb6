"""Generate the golden fixtures by running the REAL reference (vpfv).

Run in the build container only (needs /root/reference and numba):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Everything it writes is small (< 2 MB total).  Large random inputs are not
stored: they are regenerated in the tests from ``np.random.default_rng(seed)``
(PCG64, stable across platforms) and the SHA-256 of every regenerated input
array is stored so a test can prove it fed the reference's exact bytes.

Fixtures
--------
stage_*.npz   one fused stage through the reference ``fused_stage``
              (_kernels.py:320-373) -- output interior, tables, E.
rhs_*.npz     the reference numpy operator ``vlasov_rhs`` (fvm.py:240-263).
moment_*.npz  ``zeroth_moment`` fold tree (fields.py:86-111).
poisson_*.npz ``poisson_solve`` (fields.py:172-213).
init_*.npz / step_*.npz   reference problem set-ups (problems.py) and the
              production ``Simulation`` (runner.py:126-227) after 1 and 3
              fixed-dt RK4 steps.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from vpfv._kernels import fused_stage  # noqa: E402
from vpfv.fields import poisson_solve, zeroth_moment  # noqa: E402
from vpfv.fvm import SpeciesConfig, correction_coeffs, vlasov_rhs  # noqa: E402
from vpfv.grid import DistField, fill_local_ghosts, make_grid  # noqa: E402
from vpfv.problems import (  # noqa: E402
    ProblemSpec,
    landau_spec,
    make_landau_1d,
    make_problem,
)
from vpfv.runner import SimulatedCluster, Simulation  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def grid_meta(g):
    return dict(d=g.d, v=g.v, N=list(g.N), lo=list(g.lo), hi=list(g.hi),
                periodic=list(g.periodic))


def sp_meta(s):
    return dict(name=s.name, q=s.q, m=s.m, kappa2=s.kappa2, kappa_c=s.kappa_c,
                Bz=s.Bz, G=list(s.G))


def save(name, meta, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, meta=np.array(json.dumps(meta)), **arrays)
    print("wrote", name, os.path.getsize(path), "bytes")


def stage_inputs(g, seed, frozen_velocity):
    """The test-side recipe (mirrored in tests/golden_io.py)."""
    rng = np.random.default_rng(seed)
    src = np.zeros(g.padded_shape)
    src[g.interior_slices()] = 1.0 + 0.3 * rng.random(g.shape)
    if frozen_velocity:
        # velocity ghosts: arbitrary but fixed values, then the fill
        ghost = 1.0 + 0.3 * rng.random(g.padded_shape)
        mask = np.ones(g.padded_shape, bool)
        mask[g.interior_slices()] = False
        src[mask] = ghost[mask]
        from vpfv.grid import FrozenGhosts
        fill_local_ghosts(DistField(g, data=src), FrozenGhosts.capture(DistField(g, data=src)))
    else:
        fill_local_ghosts(DistField(g, data=src), None)
    A = rng.random(g.padded_shape)
    B = rng.random(g.padded_shape)
    dest = rng.random(g.padded_shape)
    return src, A, B, dest


def smooth_E(g):
    if g.d == 1:
        return {"Ex": 0.5 * np.sin(g.centers(0)) + 0.1 * np.cos(3 * g.centers(0))}
    cx, cy = g.centers(0), g.centers(1)
    return {"Ex": 0.4 * np.outer(np.sin(cx), np.cos(cy)) + 0.05,
            "Ey": 0.4 * np.outer(np.cos(cx), np.sin(cy)) - 0.03}


STAGE_CASES = [
    # name, grid args, species, frozen velocity ghosts, seed
    ("stage_1d1v_periodic", (1, 1, [16, 16], [0, -1], [2 * np.pi, 1], (True, True)),
     SpeciesConfig(q=-1.0, G=(0.05,)), False, 10),
    ("stage_1d1v_frozen", (1, 1, [16, 12], [0, -6], [2 * np.pi, 6], None),
     SpeciesConfig(q=-1.0, m=0.5, kappa2=1.2, G=(0.02,)), True, 11),
    ("stage_1d2v_periodic", (1, 2, [12, 10, 14], [0, -1, -1.5], [2 * np.pi, 1, 1.5],
                             (True, True, True)),
     SpeciesConfig(q=-1.0, kappa2=1.1, kappa_c=0.4, Bz=1.0, G=(0.0, 0.1)), False, 12),
    ("stage_1d2v_frozen", (1, 2, [9, 8, 11], [0, -4, -8], [2 * np.pi, 4, 8], None),
     SpeciesConfig(q=1.0, m=2.0, kappa2=1.0, kappa_c=0.05, Bz=1.0, G=(0.01, -0.02)), True, 13),
    ("stage_2d2v_periodic", (2, 2, [8, 9, 10, 8], [0, 0, -1, -1.5],
                             [2 * np.pi, 2 * np.pi, 1, 1.5], (True, True, True, True)),
     SpeciesConfig(q=-1.0, kappa2=1.3, kappa_c=0.4, Bz=1.0), False, 14),
    ("stage_2d2v_frozen", (2, 2, [8, 8, 9, 10], [0, 0, -5, -6], [4 * np.pi, 4 * np.pi, 5, 6],
                           None),
     SpeciesConfig(q=-1.0, m=1.0 / 1836.0, kappa2=1.0, kappa_c=0.02, Bz=1.0, G=(0.0, 0.01)),
     True, 15),
]

# (ca, cb, cd, cL) of a generic stage and of the four RK4 stages
COEFS = [(0.4, -1.1, 2.0, 0.37), (1.0, 0.0, 0.0, 0.01), (2.0, -1.0, 0.0, 0.03),
         (-1.0, 0.0, 2.0, 0.03), (-0.125, 0.375, 0.75, 0.00375)]


def make_stage_fixtures():
    for name, gargs, sp, frozen, seed in STAGE_CASES:
        d, v, N, lo, hi, per = gargs
        g = make_grid(d, v, N, lo, hi, periodic=per)
        E = smooth_E(g)
        src, A, B, dest = stage_inputs(g, seed, frozen)
        outs = []
        for ca, cb, cd, cL in COEFS:
            dd = dest.copy()
            fused_stage(dd, A, B, src, ca, cb, cd, cL, g, sp, E)
            outs.append(dd[g.interior_slices()])
        rhs = vlasov_rhs(DistField(g, data=src), sp, E)
        meta = dict(grid=grid_meta(g), species=sp_meta(sp), seed=seed, frozen=frozen,
                    coefs=COEFS,
                    sha=dict(src=sha(src), A=sha(A), B=sha(B), dest=sha(dest)))
        cc = correction_coeffs(g, sp, E)
        save(name + ".npz", meta, out=np.stack(outs), rhs=rhs,
             **{k: np.asarray(a) for k, a in E.items()},
             **{"coef_" + k: np.asarray(a) for k, a in cc.items()})


def make_moment_fixtures():
    for name, gargs, seed in [
        ("moment_1d1v", (1, 1, [9, 13], [0, -2], [1, 2]), 20),
        ("moment_1d2v", (1, 2, [9, 12, 10], [0, -2, -2], [1, 2, 2]), 21),
        ("moment_2d2v", (2, 2, [9, 8, 10, 9], [0, 0, -2, -2], [1, 1, 2, 2]), 22),
        ("moment_2d2v_pow2", (2, 2, [8, 8, 16, 32], [0, 0, -3, -3], [1, 1, 3, 3]), 23),
    ]:
        d, v, N, lo, hi = gargs
        g = make_grid(d, v, N, lo, hi)
        rng = np.random.default_rng(seed)
        f = DistField(g)
        f.data[...] = rng.random(g.padded_shape)
        n = zeroth_moment(f)
        save(name + ".npz", dict(grid=grid_meta(g), seed=seed, sha=sha(f.data)), n=n)


def make_poisson_fixtures():
    for name, gargs, seed in [
        ("poisson_1d_64", (1, 1, [64, 8], [0, -1], [2 * np.pi / 0.5, 1]), 30),
        ("poisson_1d_odd", (1, 1, [15, 8], [0, -1], [3.0, 1]), 31),
        ("poisson_2d_16", (2, 2, [16, 16, 8, 8], [0, 0, -1, -1], [4 * np.pi, 4 * np.pi, 1, 1]), 32),
        ("poisson_2d_odd", (2, 2, [12, 9, 8, 8], [0, 0, -1, -1], [2.0, 3.0, 1, 1]), 33),
    ]:
        d, v, N, lo, hi = gargs
        g = make_grid(d, v, N, lo, hi)
        rng = np.random.default_rng(seed)
        rho = rng.standard_normal(tuple(N[:d]))
        rho -= rho.mean()
        phi, E = poisson_solve(rho, g)
        save(name + ".npz", dict(grid=grid_meta(g), seed=seed), rho=rho, phi=phi,
             **{k: np.asarray(a) for k, a in E.items()})


def bimaxwellian_1d2v(N, Nvx, Nvy):
    """Config-3 synthetic set-up: anisotropic bi-Maxwellian."""
    from vpfv.problems import ProblemSetup, line_averages
    k = 0.5
    g = make_grid(1, 2, (N, Nvx, Nvy), (0.0, -8.0, -16.0), (2 * np.pi / k, 8.0, 16.0))
    mx = line_averages(lambda v: np.exp(-0.5 * v * v) / np.sqrt(2 * np.pi), g, 1)
    my = line_averages(lambda v: np.exp(-0.5 * v * v / 4.0) / np.sqrt(2 * np.pi * 4.0), g, 2)
    px = 1.0 + 1e-3 * line_averages(lambda x: np.sin(k * x), g, 0)
    data = px[:, None, None] * mx[None, :, None] * my[None, None, :]
    sp = SpeciesConfig(name="e", q=-1.0, m=1.0, kappa2=1.0, kappa_c=0.05, Bz=1.0, G=(0.0, 0.0))
    return ProblemSetup(ProblemSpec("dgh"), (sp,), [DistField(g, "e", data)])


def make_step_fixtures():
    cases = [
        ("landau1d", lambda: make_landau_1d(landau_spec(alpha=0.01), 16, 16), 0.05),
        ("twostream", lambda: make_problem(ProblemSpec("two-stream"), 16, 16), 0.05),
        ("dgh", lambda: make_problem(ProblemSpec("dgh"), 8, 8), 0.05),
        ("lhdi", lambda: make_problem(ProblemSpec("lhdi"), 8, 8), 0.002),
        ("bimax1d2v", lambda: bimaxwellian_1d2v(8, 8, 10), 0.02),
        ("landau2d", lambda: make_problem(landau_spec(), 8, 8), 0.05),
    ]
    for name, mk, dt in cases:
        setup = mk()
        init = {f"f{s}": f.data.copy() for s, f in enumerate(setup.dists)}
        meta = dict(grids=[grid_meta(f.grid) for f in setup.dists],
                    species=[sp_meta(s) for s in setup.species],
                    problem=setup.spec.problem, params={k: v for k, v in setup.spec.params.items()},
                    dt=dt)
        save(f"init_{name}.npz", meta, **init)
        sim = Simulation(mk(), dt=dt)
        out = {}
        for k in range(3):
            sim.advance(dt)
            if k in (0, 2):
                for s, a in enumerate(sim.interiors()):
                    out[f"step{k + 1}_f{s}"] = a
        st = sim.state()
        for comp, a in st.E.items():
            out[f"E3_{comp}"] = a
        save(f"step_{name}.npz", meta, **out)


def make_cluster_fixture():
    """SimulatedCluster (partitioned) equals single-rank bitwise (runner.py:14-18)."""
    spec = ProblemSpec("two-stream")
    a = Simulation(make_problem(spec, 16, 16), dt=1e-3)
    b = SimulatedCluster(make_problem(spec, 16, 16), (2, 2), dt=1e-3)
    for _ in range(2):
        a.advance(1e-3)
        b.advance(1e-3)
    assert np.array_equal(a.interiors()[0], b.gather(0))


def make_diagnostics_fixtures():
    """Reference diagnostics (diagnostics.py:85-180, fields.py:50-161):
    conserved-quantity rows, higher moments and both moment schedules of the
    3-step states of the step fixtures, ``rows_to_csv`` text, growth-rate fits
    (a synthetic series and a real 1D-1V Landau run) and Richardson errors."""
    from vpfv.diagnostics import fit_growth_rate, richardson_error, rows_to_csv
    from vpfv.fields import higher_moments

    cases = [
        ("landau1d", lambda: make_landau_1d(landau_spec(alpha=0.01), 16, 16), 0.05),
        ("twostream", lambda: make_problem(ProblemSpec("two-stream"), 16, 16), 0.05),
        ("dgh", lambda: make_problem(ProblemSpec("dgh"), 8, 8), 0.05),
        ("lhdi", lambda: make_problem(ProblemSpec("lhdi"), 8, 8), 0.002),
        ("bimax1d2v", lambda: bimaxwellian_1d2v(8, 8, 10), 0.02),
        ("landau2d", lambda: make_problem(landau_spec(), 8, 8), 0.05),
    ]
    for name, mk, dt in cases:
        sim = Simulation(mk(), dt=dt)
        rows = [sim.diagnostics_row(0.0)]
        for _ in range(3):
            sim.advance(dt)
        rows.append(sim.diagnostics_row(dt))
        dists = sim._wrap(sim.ctx.f0)
        out = {"row0": np.array(rows[0].values()), "row3": np.array(rows[1].values())}
        for s, f in enumerate(dists):
            mom, kin = higher_moments(f)
            for k, m in enumerate(mom):
                out[f"mom{k}_f{s}"] = np.asarray(m)
            out[f"kin_f{s}"] = np.asarray(kin)
            out[f"nvm_f{s}"] = zeroth_moment(f, "velocity-major")
            out[f"npm_f{s}"] = zeroth_moment(f, "position-major")
        names = [sp.name for sp in sim.species]
        meta = dict(species_names=names, csv=rows_to_csv(rows, names), dt=dt)
        save(f"diag_{name}.npz", meta, **out)

    # growth-rate fits: a synthetic series and a real reference run
    t = np.linspace(0.0, 30.0, 301)
    amp = 1e-3 * np.exp(0.29 * t) * (1.0 + 0.01 * np.sin(3.0 * t))
    g1 = fit_growth_rate(t, amp, (10.0, 25.0))
    sim = Simulation(make_landau_1d(landau_spec(alpha=0.01), 32, 32))
    rows = sim.run(6.0, cadence=1)
    tr = np.array([r.t for r in rows])
    ar = np.array([r.field_amplitude for r in rows])
    g2 = fit_growth_rate(tr, ar, (0.0, 6.0))
    errors = {}
    for bad in [((0.0, 0.5),), ((0.0, 30.0),)]:
        try:
            fit_growth_rate(t, amp if bad[0][1] < 1 else -amp, bad[0])
        except ValueError as e:
            errors[str(bad[0])] = str(e)
    rng = np.random.default_rng(40)
    a, b = rng.random((4, 6)), rng.random((8, 12))
    a3, b3 = rng.random((3, 4, 5)), rng.random((6, 8, 10))
    rich = [richardson_error(a, b), richardson_error(a3, b3)]
    save("fits.npz", dict(fit_synthetic=list(g1), fit_landau=list(g2), errors=errors, seed=40,
                          richardson=rich),
         t=t, amp=amp, t_landau=tr, amp_landau=ar)


if __name__ == "__main__":
    import sys as _sys

    if "--diagnostics" in _sys.argv:
        make_diagnostics_fixtures()
        raise SystemExit(0)
    make_stage_fixtures()
    make_moment_fixtures()
    make_poisson_fixtures()
    make_step_fixtures()
    make_cluster_fixture()
    make_diagnostics_fixtures()
