"""CPU-side tests: the C ABI library, host API mirror and set-ups (no GPU)."""

import math
import os
import re

import numpy as np
import pytest

import golden_io as G
from paper_2410_12155_b200 import _lib, grid as GR, problems as P, timestepping as TS
from paper_2410_12155_b200.fvm import SpeciesConfig, correction_coeffs
from paper_2410_12155_b200.grid import DistField, FrozenGhosts, fill_local_ghosts, make_grid


def header_symbols():
    import os

    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "vpfv.h")).read()
    return sorted(set(re.findall(r"\b(vpfv_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert lib.vpfv_version() >= 100


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(8|9)\d", out)


@pytest.mark.parametrize("name", G.STEP_NAMES)
def test_problem_setups_bitwise_vs_reference(name):
    c = G.step_case(name)
    mk = {
        "landau1d": lambda: P.make_landau_1d(P.landau_spec(alpha=0.01), 16, 16),
        "twostream": lambda: P.make_problem(P.ProblemSpec("two-stream"), 16, 16),
        "dgh": lambda: P.make_problem(P.ProblemSpec("dgh"), 8, 8),
        "lhdi": lambda: P.make_problem(P.ProblemSpec("lhdi"), 8, 8),
        "bimax1d2v": lambda: P.make_bimaxwellian_1d2v(8, 8, 10),
        "landau2d": lambda: P.make_problem(P.landau_spec(), 8, 8),
    }[name]
    setup = mk()
    assert len(setup.dists) == len(c["init"])
    for f, want, gm, sm in zip(setup.dists, c["init"], c["meta"]["grids"], c["meta"]["species"]):
        assert np.array_equal(f.data, want)
        assert f.grid.N == tuple(gm["N"]) and f.grid.lo == tuple(gm["lo"]) and f.grid.hi == tuple(gm["hi"])
    for sp, sm in zip(setup.species, c["meta"]["species"]):
        assert (sp.q, sp.m, sp.kappa2, sp.kappa_c, sp.Bz) == (sm["q"], sm["m"], sm["kappa2"], sm["kappa_c"], sm["Bz"])


@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_host_correction_coeffs_bitwise(name):
    c = G.stage_case(name)
    g = c["grid"]
    pg = make_grid(g.d, g.v, g.N, g.lo, g.hi, periodic=g.periodic)
    s = c["species"]
    sp = SpeciesConfig(s.name, s.q, s.m, s.kappa2, s.kappa_c, s.Bz, s.G)
    for k, v in correction_coeffs(pg, sp, c["E"]).items():
        assert np.array_equal(np.asarray(v), c["arrays"]["coef_" + k])


class TestGrid:
    def test_validation(self):
        with pytest.raises(ValueError):
            make_grid(2, 1, [8] * 3, [0] * 3, [1] * 3)
        with pytest.raises(ValueError):
            make_grid(1, 1, [7, 8], [0, 0], [1, 1])
        with pytest.raises(ValueError):
            make_grid(1, 1, [8, 8], [0, 1], [1, 1])

    def test_flat_index_round_trip(self):
        g = make_grid(1, 2, [8, 9, 10], [0, -1, -1], [1, 1, 1])
        for mi in [(-3, -3, -3), (0, 0, 0), (7, 8, 9), (10, 11, 12), (3, -1, 4)]:
            assert GR.unflatten(g, GR.flat_index(g, mi)) == mi

    def test_ghost_fill_matches_oracle(self):
        from oracle import vpfv_oracle as O

        g = make_grid(1, 2, [8, 9, 10], [0, -1, -1], [1, 1, 1])
        rng = np.random.default_rng(3)
        a = rng.random(g.padded_shape)
        b = a.copy()
        fr = FrozenGhosts.capture(DistField(g, data=a))
        fill_local_ghosts(DistField(g, data=a), fr)
        og = O.grid_from(g)
        O.fill_ghosts(b, og, O.capture_frozen(b, og))
        assert np.array_equal(a, b)

    def test_float64_enforced(self):
        g = make_grid(1, 1, [8, 8], [0, -1], [1, 1])
        with pytest.raises(TypeError):
            DistField(g, data=np.zeros(g.padded_shape, dtype=np.float32))


class TestStageProtocol:
    @pytest.mark.parametrize("z", [-0.5, -2.0, 0.3, -1.0 + 1.2j, 2.5j])
    def test_low_storage_quartic(self, z):
        dt = 0.7
        lam = z / dt

        def stage(dest, A, B, src, ca, cb, cd, cL, t):
            dest[...] = ca * A + cb * B + cd * dest + cL * (lam * src)

        ctx = TS.StepContext(f0=np.asarray(1.0 + 0j), f1=np.zeros((), complex), fout=np.zeros((), complex))
        TS.rk4_38_low_storage_step(ctx, dt, stage)
        R = 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24
        assert abs(ctx.fout - R) <= 1e-13 * abs(R)

    def test_stage_table_matches_reference_calls(self):
        calls = []
        ctx = TS.StepContext(f0="a", f1="b", fout="c", t=1.0)
        TS.rk4_38_low_storage_step(ctx, 0.3, lambda *a: calls.append(a))
        assert [c[:8] for c in calls] == [
            ("b", "a", "a", "a", 1.0, 0.0, 0.0, 0.3 / 3.0),
            ("c", "a", "b", "b", 2.0, -1.0, 0.0, 0.3),
            ("b", "c", "c", "c", -1.0, 0.0, 2.0, 0.3),
            ("c", "a", "b", "b", -0.125, 0.375, 0.75, 0.3 / 8.0),
        ]
        assert [c[8] for c in calls] == [1.0, 1.0 + 0.3 / 3.0, 1.0 + 2.0 * 0.3 / 3.0, 1.0 + 0.3]
        assert ctx.t == 1.3

    def test_butcher_form_equals_low_storage(self):
        """The tableau form and the three-buffer protocol through
        array_stage agree on a nonlinear, time-dependent RHS (the reference's
        dual run, test_timestepping.py:208-232, on a small system)."""
        rng = np.random.default_rng(3)
        M = rng.standard_normal((6, 6)) * 0.5

        def L(y, t):
            return M @ y - 0.3 * y ** 3 + np.cos(t)

        u0 = rng.standard_normal(6)
        ctx = TS.StepContext(f0=u0.copy(), f1=np.full(6, np.nan), fout=np.full(6, np.nan), t=0.2)
        ub = u0.copy()
        for _ in range(20):
            ub = TS.rk4_butcher_step(ub, 0.05, L, ctx.t)
            TS.rk4_38_low_storage_step(ctx, 0.05, TS.array_stage(L))
            ctx.rotate()
        np.testing.assert_allclose(ctx.f0, ub, rtol=1e-12, atol=1e-13)
        assert ctx.step == 20 and ctx.t == pytest.approx(1.2)

    def test_max_stable_dt(self):
        assert TS.max_stable_dt([[1.0, 1.0]], [1.0, 1.0], sigma=1.73) == pytest.approx(0.865)
        # minimum over species; a species at rest does not limit dt
        assert TS.max_stable_dt([[1.0, 0.0], [0.0, 0.0], [2.0, 2.0]], [0.5, 1.0], safety=0.9) == \
            0.9 * (TS.DEFAULT_SIGMA / (2.0 / 0.5 + 2.0 / 1.0))
        assert TS.max_stable_dt([[0.0, 0.0]], [1.0, 1.0]) == math.inf
        with pytest.raises(ValueError):
            TS.max_stable_dt([[1.0]], [1.0, 1.0])


def test_synthetic_setups_shapes():
    s3 = P.make_bimaxwellian_1d2v(8, 8, 8)
    g = s3.dists[0].grid
    assert (g.d, g.v) == (1, 2) and g.h[1] != g.h[2]
    c = correction_coeffs(g, s3.species[0], {"Ex": np.zeros(8)})
    assert c["c2"] != 0.0
    s5 = P.make_electron_proton_2d2v(8, 8)
    assert [sp.name for sp in s5.species] == ["i", "e"]
    assert s5.species[1].m == pytest.approx(1 / 1836.0)
    assert s5.dists[0].grid.N[:2] == s5.dists[1].grid.N[:2]


def test_snapshot_matches_reference_writer_bytes_and_round_trip(tmp_path):
    """write_snapshot / read_snapshot against a file the reference wrote
    (tests/golden/make_snapshot_golden.py; diagnostics.py:187-234)."""
    import numpy as np

    from paper_2410_12155_b200 import snapshot as S
    from paper_2410_12155_b200.grid import DistField, make_grid

    ref = os.path.join(os.path.dirname(__file__), "golden", "snapshot_ref.vpfv")
    f, t = S.read_snapshot(ref)
    N = (8, 8, 16)
    assert t == 1.25 and f.species == "e-" and tuple(f.grid.N) == N and (f.grid.d, f.grid.v) == (1, 2)
    want = 1.0 + 0.3 * np.random.default_rng(2024).random(N)
    assert np.array_equal(f.data[f.grid.interior_slices()], want)
    g = make_grid(1, 2, N, (0.0, -4.0, -5.0), (2 * np.pi, 4.0, 5.0))
    mine = DistField(g, species="e-")
    mine.data[g.interior_slices()] = want
    out = tmp_path / "mine.vpfv"
    S.write_snapshot(str(out), mine, 1.25)
    assert out.read_bytes() == open(ref, "rb").read()
    with pytest.raises(ValueError):
        bad = tmp_path / "bad.vpfv"
        bad.write_bytes(b"XXXX" + out.read_bytes()[4:])
        S.read_snapshot(str(bad))


def test_richardson_error_mirror():
    """The host mirror against the reference's own cases (test_diagnostics.py:134-154)."""
    import numpy as np

    from paper_2410_12155_b200.diagnostics import richardson_error

    a = np.arange(16.0).reshape(4, 4)
    fine = np.repeat(np.repeat(a, 2, axis=0), 2, axis=1)
    assert richardson_error(a, fine) == 0.0
    assert richardson_error(a + 2.0, fine) == 2.0
    with pytest.raises(ValueError):
        richardson_error(np.zeros((8, 8)), np.zeros((8, 16)))


@pytest.mark.parametrize("which", ["landau2d", "lhdi", "ep", "weibel"])
def test_max_speed_per_dim_equals_broadcast_max(which):
    """The CFL speeds from the field extremes equal the maxima over the full
    broadcast speed arrays (fvm.py:125-127), with and without magnetic field."""
    from paper_2410_12155_b200 import problems as P
    from paper_2410_12155_b200.fvm import advection_speeds, max_speed_per_dim

    setup = {"landau2d": lambda: P.make_problem(P.landau_spec(), 16, 16),
             "lhdi": lambda: P.make_problem(P.ProblemSpec("lhdi"), 16, 32),
             "ep": lambda: P.make_electron_proton_2d2v(16, 32),
             "weibel": lambda: P.make_problem(P.ProblemSpec("weibel"), 16, 32)}[which]()
    rng = np.random.default_rng(7)
    for f, sp in zip(setup.dists, setup.species):
        g = f.grid
        shape = tuple(g.N[:g.d])
        E = {"Ex": 0.3 * rng.standard_normal(shape)}
        if g.d == 2:
            E["Ey"] = 0.3 * rng.standard_normal(shape)
        assert max_speed_per_dim(g, sp, E) == [float(np.max(np.abs(a))) for a in advection_speeds(g, sp, E)]


def test_bench_workloads_and_weak_scaling():
    """bench.py's workloads: config 5 grows its x extent with the rank count
    (weak scaling, 64^4 per species per GPU); the L2 note tells resident
    buffers from streamed ones; the JSON keys the contract needs exist."""
    import bench

    s1, s4 = bench.make_setup("ep2d2v-64"), bench.make_setup("ep2d2v-64", 4)
    assert [f.grid.N for f in s1.dists] == [(64, 64, 64, 64)] * 2
    assert [f.grid.N for f in s4.dists] == [(256, 64, 64, 64)] * 2
    assert "ep2d2v-64" in bench.WEAK and "landau2d-128" not in bench.WEAK
    assert bench.l2_note(bench.make_setup("landau1d-128")).startswith("inputs smaller than L2")
    assert bench.l2_note(bench.make_setup("ep2d2v-64")).startswith("inputs larger than L2")
    assert set(bench.KERNEL_OF) == set(bench.WORKLOADS)
