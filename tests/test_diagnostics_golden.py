"""Diagnostics pinned to the reference (tests/golden/diag_*.npz, fits.npz,
written by tests/golden/make_golden.py from the real vpfv package).

* host: ``conserved_quantities`` (diagnostics.py:85-122), ``rows_to_csv``
  (:125-130), ``fit_growth_rate`` (:133-160, values, stderr and error text),
  ``richardson_error`` (:163-180) -- bitwise; the oracle's
  ``position-major`` moment (fields.py:50-83) -- bitwise;
* GPU: the device diagnostics row and ``higher_moments`` against the
  reference rows (mass bitwise: fold tree; the other sums within 1e-13
  relative: different summation order), ``vpfv_moment_seq`` bitwise the
  reference's sequential moment, and ``Simulation(schedule="position-major")``
  steps against the oracle.
"""

import numpy as np
import pytest

import golden_io as G
from oracle import vpfv_oracle as O
from paper_2410_12155_b200 import diagnostics as D
from paper_2410_12155_b200.grid import make_grid

DIAG = ["landau1d", "twostream", "dgh", "lhdi", "bimax1d2v", "landau2d"]


def pgrid(g):
    return make_grid(g.d, g.v, g.N, g.lo, g.hi, periodic=g.periodic)


def _states(name):
    """(t=0 arrays, 3-step arrays, E of each, case) with synchronised ghosts; the
    oracle steps are bitwise the reference's (tests/test_oracle.py)."""
    c = G.step_case(name)
    sim = O.OracleSimulation(c["grids"], c["species"], c["init"], dt=c["dt"])
    a0 = [np.array(a) for a in sim.ctx.f0]
    _, _, E0 = sim._solve(a0)
    for _ in range(3):
        sim.advance(c["dt"])
    a3 = [np.array(a) for a in sim.ctx.f0]
    _, _, E3 = sim._solve(a3)
    return a0, E0, a3, E3, sim.ctx.t, c


@pytest.mark.parametrize("name", DIAG)
def test_conserved_quantities_rows_bitwise(name):
    meta, ref = G.load(f"diag_{name}.npz")
    a0, E0, a3, E3, t3, c = _states(name)
    grids = [pgrid(g) for g in c["grids"]]
    r0 = D.conserved_quantities_arrays(a0, grids, c["species"], E0, 0.0, 0.0)
    r3 = D.conserved_quantities_arrays(a3, grids, c["species"], E3, t3, c["dt"])
    assert np.array_equal(np.array(r0.values()), ref["row0"])
    assert np.array_equal(np.array(r3.values()), ref["row3"])
    assert D.rows_to_csv([r0, r3], meta["species_names"]) == meta["csv"]
    # the DistField / FieldState signature of the reference
    from paper_2410_12155_b200.fields import FieldState
    from paper_2410_12155_b200.grid import DistField

    dists = [DistField(g, n, a) for g, n, a in zip(grids, meta["species_names"], a3)]
    state = FieldState(n={}, rho=None, phi=None, E=E3)
    r = D.conserved_quantities(dists, c["species"], state, t3, c["dt"])
    assert np.array_equal(np.array(r.values()), ref["row3"])


@pytest.mark.parametrize("name", DIAG)
def test_oracle_position_major_moment_bitwise(name):
    _, ref = G.load(f"diag_{name}.npz")
    _, _, a3, _, _, c = _states(name)
    for s, (a, g) in enumerate(zip(a3, c["grids"])):
        assert np.array_equal(O.zeroth_moment(a, g, "position-major"), ref[f"npm_f{s}"])
        assert np.array_equal(O.zeroth_moment(a, g, "velocity-major"), ref[f"nvm_f{s}"])


def test_fit_growth_rate_bitwise():
    meta, ref = G.load("fits.npz")
    g1 = D.fit_growth_rate(ref["t"], ref["amp"], (10.0, 25.0))
    assert list(g1) == meta["fit_synthetic"]
    g2 = D.fit_growth_rate(ref["t_landau"], ref["amp_landau"], (0.0, 6.0))
    assert list(g2) == meta["fit_landau"]
    with pytest.raises(ValueError) as e:
        D.fit_growth_rate(ref["t"], ref["amp"], (0.0, 0.5))
    assert str(e.value) == meta["errors"][str((0.0, 0.5))]
    with pytest.raises(ValueError) as e:
        D.fit_growth_rate(ref["t"], -ref["amp"], (0.0, 30.0))
    assert str(e.value) == meta["errors"][str((0.0, 30.0))]


def test_richardson_error_bitwise():
    meta, _ = G.load("fits.npz")
    rng = np.random.default_rng(meta["seed"])
    a, b = rng.random((4, 6)), rng.random((8, 12))
    a3, b3 = rng.random((3, 4, 5)), rng.random((6, 8, 10))
    assert [D.richardson_error(a, b), D.richardson_error(a3, b3)] == meta["richardson"]
    with pytest.raises(ValueError):
        D.richardson_error(a, b3)


def test_fit_peak_rate_on_damped_series():
    t = np.linspace(0.0, 20.0, 2001)
    amp = np.exp(-0.153 * t) * np.abs(np.cos(1.4156 * t)) + 1e-12
    gamma, err = D.fit_peak_rate(t, amp, (0.0, 20.0))
    assert abs(gamma + 0.153) < 2e-3 and err < 1e-3


# ---------------------------------------------------------------------------
# device


@pytest.mark.gpu
@pytest.mark.parametrize("name", DIAG)
def test_device_diagnostics_and_moments_vs_reference(name):
    import torch

    from paper_2410_12155_b200 import fields as F
    from paper_2410_12155_b200.fields import FieldState
    from paper_2410_12155_b200.grid import DistField

    meta, ref = G.load(f"diag_{name}.npz")
    _, _, a3, E3, t3, c = _states(name)
    grids = [pgrid(g) for g in c["grids"]]
    dev = [DistField(g, n, torch.from_numpy(a).cuda()) for g, n, a in zip(grids, meta["species_names"], a3)]
    row = D.conserved_quantities(dev, c["species"], FieldState(n={}, rho=None, phi=None, E=E3), t3, c["dt"])
    got, want = np.array(row.values()), ref["row3"]
    S = len(grids)
    assert np.array_equal(got[:2 + S], want[:2 + S])  # t, dt, masses: fold tree, bitwise
    assert np.allclose(got[2 + S:], want[2 + S:], rtol=1e-13, atol=1e-15 * np.abs(want).max())
    for s, f in enumerate(dev):
        n_pm = F.zeroth_moment(f, "position-major").cpu().numpy()
        assert np.array_equal(n_pm, ref[f"npm_f{s}"])
        assert np.array_equal(F.zeroth_moment(f, "velocity-major").cpu().numpy(), ref[f"nvm_f{s}"])
        mom, kin = F.higher_moments(f)
        # momentum is a cancelling sum (two-stream: +-v0 beams give 2e-5 out of
        # terms of order n v0 ~ 1): the absolute bar is set by the summed
        # magnitudes, bounded by sqrt(2 n kin), not by the result
        mscale = np.sqrt(2.0 * np.abs(ref[f"kin_f{s}"]).max() * np.abs(ref[f"nvm_f{s}"]).max())
        for k, m in enumerate(mom):
            w = ref[f"mom{k}_f{s}"]
            assert np.allclose(m.cpu().numpy(), w, rtol=1e-12, atol=1e-13 * mscale)
        w = ref[f"kin_f{s}"]
        assert np.allclose(kin.cpu().numpy(), w, rtol=1e-12, atol=1e-14 * np.abs(w).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["twostream", "lhdi", "landau2d"])
def test_position_major_simulation_vs_oracle(name):
    from paper_2410_12155_b200 import runner as R
    from paper_2410_12155_b200.problems import ProblemSetup  # noqa: F401

    c = G.step_case(name)
    grids = [pgrid(g) for g in c["grids"]]
    from paper_2410_12155_b200.grid import DistField

    class _Setup:
        pass

    setup = _Setup()
    setup.species = tuple(c["species"])
    setup.dists = [DistField(g, f"s{s}", np.array(a)) for s, (g, a) in enumerate(zip(grids, c["init"]))]
    sim = R.Simulation(setup, dt=c["dt"], schedule="position-major")
    assert not sim.fuse_moment
    ref = O.OracleSimulation(c["grids"], c["species"], c["init"], dt=c["dt"], schedule="position-major")
    for _ in range(3):
        sim.advance(c["dt"])
        ref.advance(c["dt"])
        for a, b in zip(sim.interiors(), ref.interiors()):
            assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-12
